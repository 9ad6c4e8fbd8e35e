"""The numpy oracle against the reference's own outputs (tests/golden) and its
known-answer tests (reference tests/test_chunked.py, test_attention_forms.py)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import power_oracle as O


@pytest.mark.parametrize("name", golden_names("chunked_"))
def test_chunked_forward_matches_reference(name):
    g = load_golden(name)
    y, r = O.chunked_forward(g["q"], g["k"], g["v"], g.get("gates"), int(g["p"]), int(g["c"]),
                             normalize=bool(g["normalize"]))
    assert O.max_rel_error(y, g["y"]) < 1e-12
    assert O.max_rel_error(r, g["rowsum"]) < 1e-12


@pytest.mark.parametrize("name", golden_names("chunked_"))
def test_chunked_backward_matches_reference(name):
    g = load_golden(name)
    dq, dk, dv, dg = O.chunked_backward(g["q"], g["k"], g["v"], g.get("gates"), int(g["p"]),
                                        int(g["c"]), g["dy"], normalize=bool(g["normalize"]))
    for a, ref in ((dq, g["dq"]), (dk, g["dk"]), (dv, g["dv"])):
        assert O.max_rel_error(a, ref) < 1e-10
    if "dgates" in g:
        assert O.max_rel_error(dg, g["dgates"]) < 1e-10


def test_config1_fp32():
    g = load_golden("config1")
    y, r = O.chunked_forward(g["q"], g["k"], g["v"], g["gates"], 2, 128)
    assert y.dtype == np.float32
    assert O.max_rel_error(y, g["y"]) < 1e-5
    dq, dk, dv, dg = O.chunked_backward(g["q"], g["k"], g["v"], g["gates"], 2, 128, g["dy"])
    for a, ref in ((dq, g["dq"]), (dk, g["dk"]), (dv, g["dv"]), (dg, g["dgates"])):
        assert O.max_rel_error(a, ref) < 1e-5


@pytest.mark.parametrize("name", golden_names("kernels_"))
def test_state_kernels_match_reference(name):
    g = load_golden(name)
    p = int(g["p"])
    st, ks = O.update_state(g["k"], g["v"], g["w"], p)
    np.testing.assert_allclose(st, g["state"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(ks, g["key_sum"], rtol=1e-12, atol=1e-13)
    y, den = O.query_state(g["q"], g["state"], g["key_sum"], p)
    np.testing.assert_allclose(y, g["y"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(den, g["denom"], rtol=1e-12, atol=1e-12)


def test_discumsum_bit_exact():
    g = load_golden("discumsum")
    assert (O.discumsum(g["values"], g["lams"]) == g["out"]).all()
    # hand recurrence (reference test_chunked.py:116-118)
    assert O.discumsum(np.array([1.0, 2.0, 3.0]), np.array([0.5, 0.5])).tolist() == [1.0, 2.5, 4.25]


def test_dimension_table():
    for p, d, D in load_golden("dims")["table"]:
        assert O.feature_dim(int(p), int(d)) == D
        if D < 100000:
            assert O.ndmi_table(int(p), int(d))[0].shape == (D, p)


def test_worked_examples():
    # update_state worked example (reference test_chunked.py:64-69)
    st, ks = O.update_state(np.array([[[1.0, 0.0]]]), np.array([[[5.0]]]), np.array([[1.0]]), 2)
    assert st[0].tolist() == [[5.0], [0.0], [0.0]] and ks[0].tolist() == [1.0, 0.0, 0.0]
    # power worked example y=[10,360], zeta=[1,20] (test_attention_forms.py:107-113)
    q = np.array([1.0, 2.0]).reshape(1, 2, 1, 1)
    v = np.array([10.0, 20.0]).reshape(1, 2, 1, 1)
    y, r = O.attention_forward(q, q, v, None, 2, scale=1.0)
    assert np.allclose(y.ravel(), [10, 360]) and np.allclose(r.ravel(), [1, 20])
    # chunked prefix-sum example [1,3,6,10] (test_chunked.py:251-257)
    ones = np.ones((1, 4, 1, 1))
    vv = np.arange(1.0, 5.0).reshape(1, 4, 1, 1)
    y, _ = O.chunked_forward(ones, ones, vv, None, 2, 2, scale=1.0)
    assert np.allclose(y.ravel(), [1, 3, 6, 10])


def test_log_gate_surface():
    q, k, v, g = O.generate_inputs(1, 12, 2, 4, 3, seed=5, gating=True)
    y1 = O.power_full(q, k, v, np.log(g), p=2, chunk_size=5)
    y2, _ = O.chunked_forward(q, k, v, g, 2, 5)
    assert O.max_rel_error(y1, y2) < 1e-14
    dy = np.ones_like(y1)
    _, _, _, dlg = O.power_full_vjp(q, k, v, np.log(g), dy, p=2, chunk_size=5)
    _, _, _, dg = O.chunked_backward(q, k, v, g, 2, 5, dy)
    assert O.max_rel_error(dlg, dg * g) < 1e-14


@pytest.mark.parametrize("name", golden_names("kinds_"))
def test_expansion_kinds_match_reference(name):
    """TPOW / TSPOW / SPOW tables and the table-driven update/query restatements
    against reference-generated fixtures (make_golden_kinds.py)."""
    g = load_golden(name)
    kind, p, d, dt = str(g["kind"]), int(g["p"]), int(g["d"]), int(g["d_tile"]) or None
    idx, w = O.expansion_table(kind, p, d, dt)
    assert (idx == g["idx"]).all() and idx.shape[0] == int(g["D"])
    np.testing.assert_allclose(w, g["w"], rtol=1e-15)
    st, ks = O.table_update_state(g["k"], g["v"], g["decay"], idx, w)
    np.testing.assert_allclose(st, g["state"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(ks, g["key_sum"], rtol=1e-12, atol=1e-13)
    y, den = O.table_query_state(g["q"], g["state"], g["key_sum"], idx, w)
    np.testing.assert_allclose(y, g["y"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(den, g["denom"], rtol=1e-12, atol=1e-12)
