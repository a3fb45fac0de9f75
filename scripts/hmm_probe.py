"""HMM sweep time, chunked s-scan vs the site-by-site scan (BNMC_HMM_SERIAL=1)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1312_3613_b200 as g  # noqa: E402

for N, S in [(100000, 3), (1000000, 4), (100000, 16)]:
    flips = np.random.default_rng(2).integers(0, 2, N).astype(np.int64)
    for serial in ("1", "0"):
        os.environ["BNMC_HMM_SERIAL"] = serial
        e = g.Engine("hmm", {"N": N, "S": S}, g.RunConfig(seed=21))
        s = e.allocate()
        s["flips"] = flips
        e.prior_init(s, 21)
        e.sweep(s, 0)
        n = 5 if serial == "1" else 50
        t = time.perf_counter()
        tr = e.run(s, n)
        dt = (time.perf_counter() - t) / n
        print(json.dumps({"N": N, "S": S, "serial": serial, "ms_per_sweep": round(dt * 1e3, 4),
                          "device_ms": round(float(np.mean(tr["timing_ms"])), 4) if "timing_ms" in tr else None}),
              flush=True)
        e.close()
