"""Breakdown of the bound-store Engine.sweep path on the NIPS shape (host timers)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1312_3613_b200 as g
from bench import gen_lda_corpus, pinned_like

docs, V, K, L = 1500, 12419, 100, 1267
e = g.Engine("lda", {"K": K, "V": V, "M": docs, "N": [L] * docs}, g.RunConfig(seed=1))
s = e.allocate()
s["w"] = gen_lda_corpus(docs, V, K, L, 1)
e.prior_init(s, 1)
pins = []
if "--pageable" not in sys.argv:
    for n in s.names:
        if not s.observed[n]:
            a, t = pinned_like(s.arrays[n])
            s.arrays[n] = a
            pins.append(t)
e.sweep(s, 0)
e.sweep(s, 1)
L_ = g.lib()


def tm(f, n=30):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


st = s._view()
print("transfer bytes", e.transfer_stats())
print("upload_sweep_inputs ms %.3f" % tm(lambda: (L_.bnmc_gpu_upload_sweep_inputs(e._h, ctypes.byref(st)), torch.cuda.synchronize())))
print("sweep_device ms %.3f" % tm(lambda: e.sweep_device(1)))
print("download ms %.3f" % tm(lambda: e.download(s)))
print("full sweep ms %.3f" % tm(lambda: e.sweep(s, 2)))
z = s["z"]
buf = np.empty(len(z), dtype=np.uint8)
t0 = time.perf_counter()
for _ in range(10):
    np.copyto(buf, z, casting="unsafe")
print("numpy 1-thread pack ms %.3f" % ((time.perf_counter() - t0) / 10 * 1e3))
t0 = time.perf_counter()
for _ in range(10):
    np.copyto(z, buf, casting="unsafe")
print("numpy 1-thread expand ms %.3f" % ((time.perf_counter() - t0) / 10 * 1e3))
