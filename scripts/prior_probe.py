"""Times prior_init / lda_generate on the device, thread-per-row vs segmented rows
(BNMC_PRIOR_SERIAL), at the NIPS shape and the 1B phi shape (K=1000, V=1e5, few docs)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1312_3613_b200 as g  # noqa: E402

for name, K, V, M, L in [("nips", 100, 12419, 1500, 1267), ("1b-phi", 1000, 100000, 64, 1000)]:
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    for serial in ("1", "0"):
        os.environ["BNMC_PRIOR_SERIAL"] = serial
        e = g.Engine("lda", hyper, g.RunConfig(seed=3))
        e.lda_generate(3)
        torch.cuda.synchronize()
        t = time.perf_counter()
        e.prior_init_device(4)
        torch.cuda.synchronize()
        t_prior = time.perf_counter() - t
        t = time.perf_counter()
        e.lda_generate(5)
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t
        s = e.allocate()
        e.download(s)
        print(json.dumps({"shape": name, "serial": serial, "prior_init_ms": round(t_prior * 1e3, 3),
                          "generate_plus_prior_ms": round(t_gen * 1e3, 3),
                          "phi_checksum": float(np.sum(s["phi"][:4096]))}), flush=True)
        e.close()
