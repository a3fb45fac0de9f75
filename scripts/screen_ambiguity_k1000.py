#!/usr/bin/env python
"""Why the 1B z-step keeps 4-byte screen rows: the fraction of
tokens a level-1 screen must hand on, as a function of its relative margin, at K = 1000.

A screen decides a token only when u * total lies more than margin * u * total away from
both running sums around it; the fp32 screen's margin is 2^-16, an fp16-row screen's
must cover the fp16 rounding of the rows (2^-11 per product: margin >= ~2^-10).  Weights
are drawn as at the start of the 1B chain (theta_d ~ Dir(alpha + counts of 1000 uniform
topic draws), g_kw ~ Gamma(beta + Poisson(10)): 1e4 tokens per word spread over 1000
topics) and, for comparison, a concentrated late-chain state.

    python scripts/screen_ambiguity_k1000.py
measured (r02): margin 2^-16: 1.2 % (early) / 0.5 % (late); 2^-10: 44 % / 8 %;
2^-8.5: 72 % / 11 %.
"""
import numpy as np

rs = np.random.default_rng(3)
K = 1000


def frac(m, ntok=20000, state="early"):
    amb = 0
    for _ in range(ntok // 100):
        n = np.bincount(rs.integers(0, K, 1000) if state == "early" else rs.integers(0, 20, 1000), minlength=K)
        th = rs.gamma(0.1 + n)
        th /= th.sum()
        for _ in range(100):
            nk = rs.poisson(10, K) if state == "early" else rs.poisson(0.5, K) * 20
            p = th * rs.gamma(0.1 + nk)
            c = np.cumsum(p)
            u = rs.random() * c[-1]
            k = np.searchsorted(c, u, side="right")
            lo = c[k - 1] if k > 0 else 0.0
            if u - lo < m * u or c[k] - u < m * u:
                amb += 1
    return amb / ntok


if __name__ == "__main__":
    for m, name in [(2 ** -16, "2^-16 (fp32 rows)"), (2 ** -10, "2^-10 (fp16 rows)"), (2 ** -8.5, "2^-8.5")]:
        print(f"margin {name}: early chain {frac(m):.3%}, concentrated {frac(m, state='late'):.3%}")
