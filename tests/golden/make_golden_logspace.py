"""Golden vectors of the reference's log-space attention form
(attention.py:289-305, power_attention_form with use_log_space=True).

Run in the build container (needs /root/reference):
    python tests/golden/make_golden_logspace.py
Writes tests/golden/logspace_*.npz (inputs, outputs y/rowsum, flags).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import power_attention as pa

    rng = np.random.default_rng(2024)
    cases = [
        # (b, t, h, d, e, p, gated, normalize, lo, hi, zero_gates)
        (1, 8, 2, 4, 3, 2, False, False, 0.5, 1.5, False),   # test_attention_forms.py:147-166 shape
        (1, 8, 2, 4, 3, 2, True, True, 0.5, 1.5, False),
        (2, 37, 3, 5, 4, 4, True, False, -1.5, 1.5, False),  # test_acceptance.py:256-284 ranges
        (1, 70, 2, 16, 8, 2, True, True, -1.0, 1.0, True),   # zero gates (exact decay)
        (1, 300, 1, 8, 40, 2, True, False, -1.0, 1.0, False),  # > 256 rows, several CTAs
        (1, 64, 1, 4, 4, 4, False, True, -40.0, 40.0, False),  # large scores (exp range)
    ]
    for i, (b, t, h, d, e, p, gated, norm, lo, hi, zeros) in enumerate(cases):
        q = rng.uniform(lo, hi, (b, t, h, d))
        k = rng.uniform(lo, hi, (b, t, h, d))
        v = rng.uniform(-1, 1, (b, t, h, e))
        g = rng.uniform(0.9, 1.0, (b, t, h)) if gated else None
        if zeros:
            g[:, [5, 33, 34], :] = 0.0
        batch = pa.SequenceBatch(q, k, v, g)
        cfg = pa.AttentionConfig.power(pa.ExpansionSpec.spow(p, d), normalize=norm, use_log_space=True)
        out = pa.power_attention_form(batch, cfg)
        rec = dict(q=q, k=k, v=v, p=p, normalize=int(norm), y=out.y, rowsum=out.rowsum)
        if gated:
            rec["gates"] = g
        np.savez(os.path.join(OUT, f"logspace_{i}.npz"), **rec)
        print(f"logspace_{i}", {kk: np.shape(vv) for kk, vv in rec.items()})


if __name__ == "__main__":
    main()
