import time, sys, numpy as np
sys.path.insert(0, '.')
import paper_1312_3613_b200 as g
from bench import gen_lda_corpus
docs, V, K, L = 1500, 12419, 100, 1267
for thin in (1, 5):
    e = g.Engine("lda", {"K": K, "V": V, "M": docs, "N": [L] * docs}, g.RunConfig(seed=1, thin=thin))
    s = e.allocate(); s["w"] = gen_lda_corpus(docs, V, K, L, 1); e.prior_init(s, 1)
    e.run(s, 10)
    t0 = time.perf_counter(); tr = e.run(s, 50); t1 = time.perf_counter()
    print("thin", thin, "run(50) ms per sweep %.3f" % ((t1 - t0) / 50 * 1e3), "samples", len(tr["samples"]))
    e.close()
