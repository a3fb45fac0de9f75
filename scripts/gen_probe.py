"""Wall time of lda_generate (+ its prior_init) and of prior_init alone at the 1B shape
(K=1000, V=1e5, M=1e6 documents of 1000 tokens) or a given document count."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1312_3613_b200 as g  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
K, V, L = 1000, 100000, 1000
e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=3))
torch.cuda.synchronize()
t = time.perf_counter()
e.lda_generate(3)
torch.cuda.synchronize()
t_gen = time.perf_counter() - t
t = time.perf_counter()
e.prior_init_device(4)
torch.cuda.synchronize()
t_prior = time.perf_counter() - t
print(json.dumps({"docs": M, "generate_plus_prior_s": round(t_gen, 3), "prior_init_s": round(t_prior, 3)}))
