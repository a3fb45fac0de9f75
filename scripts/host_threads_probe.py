import numpy as np, time, os, concurrent.futures as cf
z = np.random.randint(0, 100, 1900500).astype(np.int64)
buf = np.empty(len(z), np.uint8)
print("sched_getaffinity", len(os.sched_getaffinity(0)))
try:
    print("cpu.max", open("/sys/fs/cgroup/cpu.max").read().strip())
except Exception as e:
    print("cpu.max n/a", e)
for T in (1, 2, 4, 8, 16):
    ex = cf.ThreadPoolExecutor(T)
    sl = [(len(z) * i // T, len(z) * (i + 1) // T) for i in range(T)]
    def job(a):
        np.copyto(buf[a[0]:a[1]], z[a[0]:a[1]], casting="unsafe")
    list(ex.map(job, sl))
    t0 = time.perf_counter()
    for _ in range(50):
        list(ex.map(job, sl))
    print(T, "threads pack ms %.3f" % ((time.perf_counter() - t0) / 50 * 1e3))
    ex.shutdown()
