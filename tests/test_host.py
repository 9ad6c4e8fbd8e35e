"""Host-side helpers (no GPU): synthetic inputs and the error metric."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2507_04239_b200.checks import max_abs_error, max_rel_error
from paper_2507_04239_b200.inputs import generate_batch

# (b, t, h, d, e, gated, seed) of tests/golden/make_golden.py's chunked grid
GRID = {
    0: (1, 9, 2, 4, 3, True, 7),
    1: (2, 16, 2, 4, 3, True, 11),
    4: (1, 17, 2, 4, 3, False, 14),
    6: (1, 24, 1, 4, 3, True, 16),
    9: (1, 130, 1, 8, 8, True, 19),
}


@pytest.mark.parametrize("case", sorted(GRID))
def test_generate_batch_matches_reference_inputs(case):
    """inputs.py:20-35: same Philox draws as the reference, bit for bit."""
    b, t, h, d, e, gated, seed = GRID[case]
    g = load_golden(f"chunked_{case}")
    batch = generate_batch(b, t, h, d, e, seed=seed, gating=gated)
    for name in ("q", "k", "v"):
        assert np.array_equal(getattr(batch, name), g[name])
    if gated:
        assert np.array_equal(batch.gates, g["gates"])
    else:
        assert batch.gates is None


def test_generate_batch_config1_fp32():
    g = load_golden("config1")
    batch = generate_batch(1, 1024, 2, 32, 32, seed=0, dtype=np.float32, gating=True)
    assert batch.q.dtype == np.float32
    for name in ("q", "k", "v", "gates"):
        assert np.array_equal(getattr(batch, name), g[name])


def test_error_metrics():
    """checks.py:26-37 (tests/conftest.py:7-11 of the reference)."""
    assert max_rel_error([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert max_rel_error([0.5], [0.25]) == 0.25          # denominator floors at 1
    assert max_rel_error([10.0], [11.0]) == pytest.approx(1 / 11)
    assert max_abs_error([10.0], [11.0]) == 1.0
    assert max_rel_error([], []) == 0.0


def test_flop_counts_match_reference():
    """flops.py:142-174; expected values printed by the reference's own
    count_flops_chunked / count_flops_attention in this container."""
    from paper_2507_04239_b200.chunked import ChunkPlan
    from paper_2507_04239_b200.expansions import ExpansionSpec
    from paper_2507_04239_b200.flops import count_flops_attention, count_flops_chunked

    assert count_flops_chunked(ChunkPlan(65536, 1024), ExpansionSpec.spow(2, 64), 64) == {
        "intra_attention": 4332748800, "expansion": 545259520, "update_state": 8860467200,
        "discumsum": 8652800, "query_state": 8860467200, "total": 22607595520}
    assert count_flops_chunked(ChunkPlan(130, 64), ExpansionSpec.spow(4, 6), 5) == {
        "intra_attention": 58282, "expansion": 131040, "update_state": 98280, "discumsum": 2268,
        "query_state": 98280, "total": 388150}
    assert count_flops_attention(1000, 32, 16, 4) == {
        "scores": 16016000, "power": 1501500, "score_value": 8008000, "total": 25525500}


def test_cli_dim_matches_reference(capsys):
    """`dim --format json --d 4,64` lines as the reference CLI prints them."""
    import json

    from paper_2507_04239_b200.cli import main

    assert main(["dim", "--format", "json", "--d", "4,64"]) == 0
    rows = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert len(rows) == 10
    assert rows[0] == {"d": 4, "p": 2, "tpow": 16, "spow": 10, "savings": "37%"}
    assert rows[5] == {"d": 64, "p": 2, "tpow": 4096, "spow": 2080, "savings": "49%"}
    assert rows[9] == {"d": 64, "p": 6, "tpow": 68719476736, "spow": 119877472, "savings": "99.8%"}


def test_cli_usage_errors_exit_2():
    from paper_2507_04239_b200.cli import int_list, main

    assert int_list("1024,2..4,1e3") == [1024, 2, 3, 4, 1000]
    assert main(["bench", "--p", "2,4"]) == 2          # bench takes a single --p
    assert main(["check", "--t", "0"]) == 2            # non-positive sizes
    assert main(["check", "--p", "3", "--normalize"]) == 2   # odd degree cannot normalize
