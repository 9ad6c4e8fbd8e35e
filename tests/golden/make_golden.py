"""Generate golden fixtures by running the REFERENCE package (read-only at
/root/reference) in this container.  The fixtures travel with the repo; the
reference does not.  Re-run with:

    python tests/golden/make_golden.py

Every case stores its inputs and the reference outputs so tests can check both
the numpy oracle (CPU) and the CUDA path (GPU) against the reference itself.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import power_attention as pa
    from power_attention.inputs import generate_batch
    from power_attention.kernels import query_state_kernel, update_state_kernel

    # ---- chunked forward / backward grid (float64) ----------------------
    cases = {}
    grid = [
        # (b, t, h, d, e, p, c, gated, normalize, seed)
        (1, 9, 2, 4, 3, 2, 3, True, True, 7),
        (2, 16, 2, 4, 3, 2, 5, True, False, 11),
        (1, 33, 1, 8, 4, 2, 7, True, True, 12),
        (1, 20, 2, 4, 4, 2, 20, True, True, 13),   # single chunk == attention
        (1, 17, 2, 4, 3, 2, 1, False, True, 14),   # c=1 == recurrent
        (1, 40, 2, 6, 5, 2, 16, False, False, 15),
        (1, 24, 1, 4, 3, 4, 8, True, True, 16),    # p=4
        (1, 19, 2, 5, 2, 3, 6, True, False, 17),   # odd p, unnormalized
        (1, 64, 2, 16, 16, 2, 16, True, True, 18),
        (1, 130, 1, 8, 8, 2, 64, True, False, 19),  # partial last chunk
    ]
    for i, (b, t, h, d, e, p, c, gated, norm, seed) in enumerate(grid):
        batch = generate_batch(b, t, h, d, e, seed=seed, gating=gated)
        cfg = pa.AttentionConfig.power(pa.ExpansionSpec.spow(p, d), normalize=norm)
        plan = pa.ChunkPlan(t, c)
        out = pa.chunked_power_attention(batch, cfg, plan)
        dy = np.random.default_rng(seed + 1000).uniform(-1, 1, out.y.shape)
        gr = pa.vjp_chunked(batch, cfg, plan, dy)
        rec = dict(q=batch.q, k=batch.k, v=batch.v, p=p, c=c, normalize=int(norm),
                   y=out.y, rowsum=out.rowsum, dy=dy, dq=gr.dq, dk=gr.dk, dv=gr.dv)
        if gated:
            rec["gates"] = batch.gates
            rec["dgates"] = gr.dgates
        cases[f"chunked_{i}"] = rec

    # ---- config 1 (fp32 inputs, BASELINE configs[0]) --------------------
    batch = generate_batch(1, 1024, 2, 32, 32, seed=0, dtype=np.float32, gating=True)
    cfg = pa.AttentionConfig.power(pa.ExpansionSpec.spow(2, 32), normalize=False)
    plan = pa.ChunkPlan(1024, 128)
    out = pa.chunked_power_attention(batch, cfg, plan)
    dy = np.random.default_rng(1).uniform(-1, 1, out.y.shape).astype(np.float32)
    gr = pa.vjp_chunked(batch, cfg, plan, dy)
    cases["config1"] = dict(q=batch.q, k=batch.k, v=batch.v, gates=batch.gates, p=2, c=128,
                            normalize=0, y=out.y, rowsum=out.rowsum, dy=dy,
                            dq=gr.dq.astype(np.float32), dk=gr.dk.astype(np.float32),
                            dv=gr.dv.astype(np.float32), dgates=gr.dgates.astype(np.float32))

    # ---- operator-level kernels (kernels.py:55-110) ---------------------
    rng = np.random.default_rng(1234)
    for p, d, e, n, c in [(2, 4, 3, 3, 5), (2, 8, 4, 2, 130), (3, 5, 4, 2, 9), (4, 6, 3, 2, 7),
                          (1, 7, 4, 2, 6), (2, 64, 64, 2, 64)]:
        spec = pa.ExpansionSpec.spow(p, d)
        kk = rng.uniform(-1, 1, (n, c, d))
        vv = rng.uniform(-1, 1, (n, c, e))
        w = rng.uniform(0.2, 1.0, (n, c))
        st, ks = update_state_kernel(kk, vv, w, spec, backend="python")
        qq = rng.uniform(-1, 1, (n, c, d))
        ys, den = query_state_kernel(qq, st, ks, spec, backend="python")
        cases[f"kernels_p{p}_d{d}_c{c}"] = dict(k=kk, v=vv, w=w, state=st, key_sum=ks,
                                                 q=qq, y=ys, denom=den, p=p)

    # ---- discumsum (chunked.py:156-176) ----------------------------------
    vals = rng.normal(size=(6, 4, 3))
    lams = rng.uniform(0, 1, 5)
    lams[2] = 0.0
    cases["discumsum"] = dict(values=vals, lams=lams, out=pa.discumsum(vals, lams))

    # ---- dimension table (expansions.py:87-99) ---------------------------
    dims = np.array([[p, d, pa.expansion_dim(pa.ExpansionSpec.spow(p, d))]
                     for p, d in [(2, 64), (2, 32), (4, 32), (3, 64), (4, 64), (2, 128)]])
    cases["dims"] = dict(table=dims)

    for name, rec in cases.items():
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(f"wrote {len(cases)} fixtures to {OUT}")


if __name__ == "__main__":
    main()
