"""Log-space attention form on the GPU (pa_power_logspace_fwd) against the
reference's own outputs (tests/golden/logspace_*.npz, made by
tests/golden/make_golden_logspace.py from attention.py:289-305)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import power_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(p, d, normalize, **kw):
    from paper_2507_04239_b200 import AttentionConfig, ExpansionSpec

    return AttentionConfig.power(ExpansionSpec.spow(p, d), normalize=normalize, use_log_space=True, **kw)


@pytest.mark.parametrize("name", golden_names("logspace_"))
def test_logspace_matches_reference_f64(name):
    """f64 host inputs run the f64 kernel: the reference's 1e-8 f64 bar (checks.py:22)."""
    from paper_2507_04239_b200 import SequenceBatch, power_attention_form
    from paper_2507_04239_b200.checks import max_rel_error

    g = load_golden(name)
    batch = SequenceBatch(g["q"], g["k"], g["v"], g.get("gates"))
    out = power_attention_form(batch, _cfg(int(g["p"]), g["q"].shape[-1], bool(g["normalize"])))
    assert out.y.dtype == np.float64
    assert max_rel_error(out.y, g["y"]) <= 1e-8
    # rowsum can be ~1e14 at the large-score case: compare relative to its scale
    assert np.max(np.abs(out.rowsum - g["rowsum"]) / np.maximum(1.0, np.abs(g["rowsum"]))) <= 1e-8


@pytest.mark.parametrize("name", golden_names("logspace_"))
def test_logspace_matches_reference_f32(name):
    """f32 inputs run the f32 kernel: the reference's f32 bar 5e-3 (checks.py:22)."""
    from paper_2507_04239_b200 import SequenceBatch, power_attention_form

    g = load_golden(name)
    f = lambda x: None if x is None else x.astype(np.float32)
    batch = SequenceBatch(f(g["q"]), f(g["k"]), f(g["v"]), f(g.get("gates")))
    out = power_attention_form(batch, _cfg(int(g["p"]), g["q"].shape[-1], bool(g["normalize"])))
    y = out.y.astype(np.float64)
    assert np.max(np.abs(y - g["y"]) / np.maximum(1.0, np.abs(g["y"]))) <= 5e-3


def test_logspace_agrees_with_direct_form():
    """test_attention_forms.py:147-166: well-separated scores, the stabilised
    and direct forms agree (f32 device direct path vs f64 log-space)."""
    from paper_2507_04239_b200 import AttentionConfig, ExpansionSpec, SequenceBatch, power_attention_form
    from paper_2507_04239_b200.checks import max_rel_error

    rng = np.random.default_rng(11)
    q = rng.uniform(0.5, 1.5, (1, 8, 2, 4))
    k = rng.uniform(0.5, 1.5, (1, 8, 2, 4))
    v = rng.uniform(-1, 1, (1, 8, 2, 3))
    g = rng.uniform(0.9, 1.0, (1, 8, 2))
    for normalize in (False, True):
        for gates in (None, g):
            batch = SequenceBatch(q, k, v, gates)
            direct = power_attention_form(batch, AttentionConfig.power(ExpansionSpec.spow(2, 4),
                                                                       normalize=normalize))
            stable = power_attention_form(batch, _cfg(2, 4, normalize))
            assert max_rel_error(direct.y, stable.y) < 1e-5   # direct runs in f32 on the device


def test_logspace_f32_survives_overflowing_scores():
    """Scores ~1e10 at p = 4: s^p overflows f32, the normalized log-space form
    stays finite and matches the f64 kernel."""
    import torch

    from paper_2507_04239_b200.power import power_logspace_forward

    gen = torch.Generator().manual_seed(3)
    q = (torch.rand(1, 96, 2, 8, generator=gen, dtype=torch.float64) + 0.5) * 1e5
    k = (torch.rand(1, 96, 2, 8, generator=gen, dtype=torch.float64) + 0.5) * 1e5
    v = torch.rand(1, 96, 2, 16, generator=gen, dtype=torch.float64) * 2 - 1
    lg = torch.log(torch.rand(1, 96, 2, generator=gen, dtype=torch.float64) * 0.1 + 0.9)
    y64, _ = power_logspace_forward(q.cuda(), k.cuda(), v.cuda(), lg.cuda(), p=4, normalize=True)
    y32, _ = power_logspace_forward(q.float().cuda(), k.float().cuda(), v.float().cuda(),
                                    lg.float().cuda(), p=4, normalize=True)
    assert torch.isfinite(y32).all()
    assert (y32.double() - y64).abs().max().item() <= 1e-4


def test_logspace_errors():
    import torch

    from paper_2507_04239_b200 import InvalidSpec
    from paper_2507_04239_b200.power import power_logspace_forward

    x = torch.zeros(1, 4, 1, 4, device="cuda")
    with pytest.raises(InvalidSpec):
        power_logspace_forward(x, x, x, p=3)
    with pytest.raises(InvalidSpec):
        power_logspace_forward(x.half(), x.half(), x.half(), p=2)


def test_logspace_chunked_and_dispatch():
    """test_chunked.py:318-330 and power_attention(form="attention") routing."""
    from paper_2507_04239_b200 import (AttentionConfig, ChunkPlan, ExpansionSpec, SequenceBatch,
                                       chunked_power_attention, power_attention)
    from paper_2507_04239_b200.checks import max_rel_error

    rng = np.random.default_rng(8)
    q = rng.uniform(0.5, 1.5, (1, 12, 1, 4))
    k = rng.uniform(0.5, 1.5, (1, 12, 1, 4))
    v = rng.uniform(-1, 1, (1, 12, 1, 3))
    batch = SequenceBatch(q, k, v)
    plain = AttentionConfig.power(ExpansionSpec.spow(2, 4), normalize=True)
    stable = _cfg(2, 4, True)
    a = chunked_power_attention(batch, plain, ChunkPlan(12, 5))
    b = chunked_power_attention(batch, stable, ChunkPlan(12, 5))
    assert max_rel_error(a.y, b.y) < 1e-6
    att = power_attention(batch, stable, form="attention")
    assert att.y.dtype == np.float64                      # the f64 log-space kernel ran
    assert max_rel_error(att.y, a.y) < 1e-5


def test_log_space_intra_chunk_in_the_chunked_pipeline():
    import paper_2507_04239_b200 as P

    """Reference test_chunked.py:318-330: the chunked form with the log-space
    intra-chunk config equals the plain one within 1e-6 (f64 inputs)."""
    rng = np.random.default_rng(8)
    q = rng.uniform(0.5, 1.5, (1, 12, 1, 4))
    k = rng.uniform(0.5, 1.5, (1, 12, 1, 4))
    v = rng.uniform(-1, 1, (1, 12, 1, 3))
    batch = P.SequenceBatch(q, k, v)
    plain = P.AttentionConfig.power(P.ExpansionSpec.spow(2, 4), normalize=True)
    stable = P.AttentionConfig.power(P.ExpansionSpec.spow(2, 4), normalize=True, use_log_space=True)
    a = P.chunked_power_attention(batch, plain, P.ChunkPlan(12, 5))
    b = P.chunked_power_attention(batch, stable, P.ChunkPlan(12, 5))
    assert O.max_rel_error(a.y, b.y) < 1e-6


@pytest.mark.parametrize("normalize", [False, True])
def test_log_space_chunked_pipeline_with_gates_vs_oracle(normalize):
    """Gated, several streams, a partial last chunk: the log-space chunked
    pipeline against the oracle's chunked form (f64)."""
    import paper_2507_04239_b200 as P

    q, k, v, g = O.generate_inputs(2, 70, 3, 8, 5, seed=17, gating=True)
    batch = P.SequenceBatch(q, k, v, g)
    cfg = P.AttentionConfig.power(P.ExpansionSpec.spow(2, 8), normalize=normalize, use_log_space=True)
    out = P.chunked_power_attention(batch, cfg, P.ChunkPlan(70, 16))
    y_ref, rs_ref = O.chunked_forward(q, k, v, g, 2, 16, normalize=normalize)
    assert O.max_rel_error(out.y, y_ref) < 1e-6
    assert O.max_rel_error(out.rowsum, rs_ref) < 1e-6
