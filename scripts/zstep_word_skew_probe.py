"""z-step time vs word-frequency skew at the NIPS shape (next-round lead):
the bench's gen_lda corpus vs uniformly random word ids (no hot phi rows)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1312_3613_b200 as g
from bench import gen_lda_corpus

docs, V, K, L = 1500, 12419, 100, 1267
for name in ("gen_lda", "uniform"):
    w = gen_lda_corpus(docs, V, K, L, 7) if name == "gen_lda" else np.random.default_rng(7).integers(0, V, docs * L)
    counts = np.bincount(np.asarray(w), minlength=V)
    top = np.sort(counts)[::-1]
    e = g.Engine("lda", {"K": K, "V": V, "M": docs, "N": [L] * docs}, g.RunConfig(seed=7))
    s = e.allocate()
    s["w"] = w
    e.prior_init(s, 7)
    e.sweep(s, 0)
    ph = {}
    for it in range(1, 21):
        for k, t in e.sweep_phases(it):
            ph.setdefault(k, []).append(t)
    print(name, "top-100 words hold %.1f%% of tokens;" % (100 * top[:100].sum() / top.sum()),
          {k: round(float(np.mean(v)) * 1e3, 1) for k, v in ph.items()}, "us")
    e.close()
