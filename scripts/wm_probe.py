"""Sweep time of the word-major vs document-major z-step order (BNMC_ZSTEP_WM) on a few
synthetic LDA shapes (device generator), to check the automatic switch (fp32 rows > 64 MB)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1312_3613_b200 as g  # noqa: E402

SHAPES = [  # K, V, docs, doc_len
    (200, 100000, 50000, 400),
    (300, 30000, 50000, 400),
    (600, 60000, 40000, 500),
    (1000, 20000, 40000, 500),
    (200, 5000, 20000, 300),
    (500, 10000, 10000, 1000),
    (1000, 5000, 5000, 1000),
    (150, 12419, 1500, 1267),
    (400, 12419, 1500, 1267),
    (100, 200000, 50000, 400),
    (100, 80000, 50000, 400),
    (100, 40000, 50000, 400),
    (100, 12419, 1500, 1267),
    (50, 100000, 50000, 400),
]
if len(sys.argv) > 1:
    SHAPES = SHAPES[int(sys.argv[1]):]
for K, V, M, L in SHAPES:
    res = {"K": K, "V": V, "docs": M, "doc_len": L, "rows32_MB": round(4 * V * (-(-K // 32) * 32) / 2**20, 1)}
    for wm in ("0", "1"):
        os.environ["BNMC_ZSTEP_WM"] = wm
        e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=3))
        e.lda_generate(3)
        e.run_device(0, 3)
        torch.cuda.synchronize()
        t = time.perf_counter()
        lj, _ = e.run_device(3, 10)
        res[f"ms_wm{wm}"] = round((time.perf_counter() - t) / 10 * 1e3, 3)
        res[f"lj_wm{wm}"] = float(lj[-1])
        e.close()
    print(json.dumps(res), flush=True)
