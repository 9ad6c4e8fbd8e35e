"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its host logic (tables, validation, workspace sizing)
agrees with the oracle.  No kernel is launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden
from oracle import power_oracle as O

P = pytest.importorskip("paper_2507_04239_b200")
from paper_2507_04239_b200 import _lib  # noqa: E402

HEADER = os.path.join(ROOT, "include", "power_attention_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(pa_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib.EXPORTED)


@pytest.mark.parametrize("p,d", [(1, 7), (2, 4), (2, 64), (3, 5), (4, 6), (4, 32)])
def test_feature_table_matches_reference_order(p, d):
    spec = P.ExpansionSpec.spow(p, d)
    idx, w = P.monomial_table(spec)
    ridx, rw = O.ndmi_table(p, d)
    assert (idx == ridx).all()
    np.testing.assert_allclose(w, rw, rtol=1e-15)
    assert _lib.load().pa_feature_dim(p, d) == O.feature_dim(p, d)


def _problem(**kw):
    base = dict(b=1, t=64, h=2, d=16, e=16, p=2, chunk=16, normalize=0, dtype=0, gated=1, has_scale=0, flags=0,
                scale=0.0)
    base.update(kw)
    return _lib.PaProblem(**base)


def test_workspace_sizes_and_validation():
    lib = _lib.load()
    pr = _problem()
    assert lib.pa_fwd_workspace_bytes(ctypes.byref(pr)) > 0
    assert lib.pa_bwd_workspace_bytes(ctypes.byref(pr)) > 0
    bad = _problem(p=3, normalize=1)
    assert lib.pa_fwd_workspace_bytes(ctypes.byref(bad)) == 0
    rc = lib.pa_power_full_fwd(ctypes.byref(bad), None, None, None, None, None, None, None, 0, None)
    assert rc == 6 and b"even" in lib.pa_last_error()
    rc = lib.pa_power_full_fwd(ctypes.byref(_problem(chunk=0)), None, None, None, None, None, None, None, 0, None)
    assert rc == 1
    with pytest.raises(P.OddPowerWithNormalize):
        _lib.check(6, "x")


def test_reference_surface_names():
    for name in ("power_full", "attention", "update_state", "query_state", "discumsum",
                 "chunked_power_attention", "power_attention", "vjp_chunked", "stream_chunk",
                 "available_backends", "resolve_backend"):
        assert hasattr(P, name), name
    assert P.available_backends() == ("cuda",)
    assert P.resolve_backend(None) == "cuda"
    with pytest.raises(P.InvalidSpec):
        P.resolve_backend("gpu")


def test_cpu_inputs_fail_loudly():
    import torch
    q = torch.zeros(1, 4, 1, 2)
    with pytest.raises(P.InvalidSpec):
        P.power_full(q, q, q)


def test_logspace_entry_validates_before_launch():
    """pa_power_logspace_fwd (attention.py:289-305) rejects bad problems with
    the reference's error classes before touching the device."""
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    args = [dummy] * 6 + [None]
    rc = lib.pa_power_logspace_fwd(ctypes.byref(_problem(p=3)), 1e-12, *args)
    assert rc == 1 and b"even p" in lib.pa_last_error()          # InvalidSpec
    rc = lib.pa_power_logspace_fwd(ctypes.byref(_problem()), 0.0, *args)
    assert rc == 1 and b"epsilon" in lib.pa_last_error()
    rc = lib.pa_power_logspace_fwd(ctypes.byref(_problem()), 1e-12, None, *args[1:])
    assert rc == 2                                               # ShapeMismatch
    rc = lib.pa_power_logspace_fwd(ctypes.byref(_problem(dtype=1)), 1e-12, *args)
    assert rc == 4 and b"f32 or f64" in lib.pa_last_error()      # bf16 unsupported here


@pytest.mark.parametrize("name", golden_names("kinds_"))
def test_library_expansion_tables_match_reference(name):
    """pa_expansion_table / pa_expansion_dim (host-side, no GPU) against the
    reference's monomial_table for SPOW, TPOW and TSPOW."""
    g = load_golden(name)
    spec = P.ExpansionSpec(str(g["kind"]), int(g["p"]), int(g["d"]), int(g["d_tile"]) or None)
    idx, w = P.monomial_table(spec)
    assert P.expansion_dim(spec) == int(g["D"]) == idx.shape[0]
    assert (idx == g["idx"]).all()
    np.testing.assert_allclose(w, g["w"], rtol=1e-15)
    assert _lib.load().pa_expansion_dim(spec.code, spec.p, spec.d, spec.d_tile or 0) == int(g["D"])


def test_route_and_strict_flag():
    """pa_uses_tensor_cores: tcgen05 for the north-star shape, fp32 kernels
    otherwise; PA_FLAG_STRICT_TC makes a 16-bit problem outside the tensor-core
    shapes an error; invalid problems report make_geo's own error code."""
    lib = _lib.load()
    tc = _problem(t=2048, d=64, e=64, chunk=1024, dtype=1)
    assert lib.pa_uses_tensor_cores(ctypes.byref(tc)) == 1
    # a partial last chunk runs on a zero-padded copy on the tensor cores
    assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(t=1000, d=64, e=64, chunk=256, dtype=1))) == 1
    assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(t=700, d=64, e=64, chunk=4096, dtype=1))) == 1
    # any chunk size (an internal chunk) and fp16 inputs (staged as bf16)
    for ch in (2048, 64, 200):
        assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(t=4096, d=64, e=64, chunk=ch, dtype=1))) == 1
    assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(t=2048, d=64, e=64, chunk=1024, dtype=2))) == 1
    # fp16 stages its inputs: the workspace grows by the staged copies
    f16 = lib.pa_fwd_workspace_bytes(ctypes.byref(_problem(t=2048, d=64, e=64, chunk=1024, dtype=2)))
    assert f16 > lib.pa_fwd_workspace_bytes(ctypes.byref(tc))
    off = _problem(t=1024, d=32, e=32, chunk=256, dtype=1)
    assert lib.pa_uses_tensor_cores(ctypes.byref(off)) == 0
    off.flags = _lib.PA_FLAG_STRICT_TC
    assert lib.pa_uses_tensor_cores(ctypes.byref(off)) == -4
    assert lib.pa_fwd_workspace_bytes(ctypes.byref(off)) == 0
    assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(dtype=0, flags=_lib.PA_FLAG_STRICT_TC))) == 0
    assert lib.pa_uses_tensor_cores(ctypes.byref(_problem(p=3, normalize=1))) == -6
