"""Counted MACs of the power-attention pipeline (reference flops.py:142-174).

Only the per-stream counters the bench records need; the weight/state ratio
(WSFR) tables of the reference's `flops` subcommand are model accounting,
outside the hot path.  One MAC = 2 FLOPs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .chunked import ChunkPlan
from .expansions import ExpansionSpec, expansion_dim

MAC = 2


@dataclass
class FlopReport:
    """flops.py:69-90: per-token weight/state FLOPs, ratio, breakdown."""

    weight_flops_per_token: float
    state_flops_per_token: float
    wsfr: tuple[float, float]
    breakdown: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {"weight_flops_per_token": self.weight_flops_per_token,
                "state_flops_per_token": self.state_flops_per_token,
                "wsfr": list(self.wsfr), "breakdown": dict(self.breakdown)}


def count_flops_chunked(plan: ChunkPlan, spec: ExpansionSpec, v_dim: int) -> dict[str, int]:
    """flops.py:142-162: exact per-stream MACs per chunked-pipeline stage."""
    dim = expansion_dim(spec)
    p, d, t = spec.p, spec.d, plan.t
    pairs = sum(ck * (ck + 1) // 2 for ck in (e - s for s, e in plan.bounds()))
    counts = {
        "intra_attention": pairs * (d + (p - 1) + v_dim),
        "expansion": 2 * t * dim * p,
        "update_state": t * dim * (v_dim + 1),
        "discumsum": plan.n_chunks * dim * (v_dim + 1),
        "query_state": t * dim * (v_dim + 1),
    }
    counts["total"] = sum(counts.values())
    return counts


def count_flops_attention(t: int, d: int, v_dim: int, p: int = 1) -> dict[str, int]:
    """flops.py:165-174: exact per-stream MACs of the quadratic form."""
    pairs = t * (t + 1) // 2
    counts = {"scores": pairs * d, "power": pairs * (p - 1), "score_value": pairs * v_dim}
    counts["total"] = sum(counts.values())
    return counts


def bench_flop_report(form: str, t: int, h: int, v_dim: int, spec: ExpansionSpec,
                      plan: ChunkPlan) -> FlopReport:
    """cli.py:170-178: counted FLOPs of one bench config (weight side 0)."""
    if form == "attention":
        macs = count_flops_attention(t, spec.d, v_dim, spec.p)
    else:
        macs = count_flops_chunked(plan if form == "chunked" else ChunkPlan(t, 1), spec, v_dim)
    per_token = {k: float(MAC * v * h / t) for k, v in macs.items() if k != "total"}
    return FlopReport(0.0, float(MAC * macs["total"] * h / t), (0.0, 1.0), per_token)
