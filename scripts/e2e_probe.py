import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1312_3613_b200 as g
from bench import gen_lda_corpus, pinned_like
docs, V, K, L = 1500, 12419, 100, 1267
e = g.Engine("lda", {"K": K, "V": V, "M": docs, "N": [L] * docs}, g.RunConfig(seed=1))
s = e.allocate(); s["w"] = gen_lda_corpus(docs, V, K, L, 1); e.prior_init(s, 1)
pins = []
for n in s.names:
    if not s.observed[n]:
        a, t = pinned_like(s.arrays[n]); s.arrays[n] = a; pins.append(t)
e.sweep(s, 0)
import ctypes
L_ = g.lib()
def tm(f, n=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
st = s._view()
print("upload_sweep_inputs ms", tm(lambda: L_.bnmc_gpu_upload_sweep_inputs(e._h, ctypes.byref(st))))
print("sweep_device ms", tm(lambda: e.sweep_device(1)))
print("download ms", tm(lambda: e.download(s)))
print("full sweep ms", tm(lambda: e.sweep(s, 2)))
