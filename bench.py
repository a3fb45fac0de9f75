#!/usr/bin/env python
"""bench.py -- sampled sites/s of one Gibbs sweep on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload nips|kos|1b|gmm|logreg]
    python bench.py --impl reference ...     # the reference CPU sampler on this host

Default workload: LDA uncollapsed Gibbs on the NIPS-shaped corpus (D=1500, V=12419,
K=100, 1267 tokens/doc = 1,900,500 sites per sweep), the configuration the
north_star's per-GPU target is stated on.  A "step" is one full sweep (phi block,
theta block, z block, log-joint), exactly Engine::sweep (sampler.cpp:390-405).

Prints ONE JSON line (rank 0).  Fields beyond the base contract:
  roofline     the dominant kernel (zstep: the z block) against the measured HBM copy
               bandwidth (MEASURED_PEAKS.json).  achieved = the kernel's compulsory DRAM
               bytes per launch / its CUDA-event duration: at NIPS/KOS the working set
               (w, z, the fp32 screen rows, theta, counts) lives in the 126 MB L2, so the
               HBM fraction is small and `binding` names the unit that bounds the kernel
               (ncu: the L1TEX data pipe); `l2` relates the operand bytes the kernel
               actually streams to the L2 -> SM read bandwidth measured in this run.
  roofline_1b  (default NIPS run, N=1) a short pass over the 1B-token config (410 MB of
               screen rows): the z-step runs in the word-major order (tokens sorted by
               document block x word, theta/S rows L2-resident per block), so like NIPS
               it reports its compulsory DRAM fraction, the binding unit and the L2
               operand fraction, with its own clocks
  cpu_baseline the compiled reference (oracle/_ref) timed on one host core on half of
               the same corpus (identical documents)
  e2e          the same metric through the public API with HOST buffers: every step
               uploads what the sweep reads from the caller's store (LDA: z; its phi and
               theta blocks redraw phi and theta first), sweeps, and downloads the whole
               latent state + log-joint (Engine::sweep borrow semantics).  The store is
               plain numpy memory the engine page-locks once per binding (as the
               reference-side adapter does for its std::vector store); `e2e_pageable`
               is the same loop with pin_host=False.
Both arms run on identical inputs: the corpus is drawn by gen_lda_corpus (seeded) and
the reference arm reads it from a binary corpus file (oracle/ref_bench lda-file).
Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) when not already
under torchrun; documents sharded across ranks (weak scaling: each rank holds a
NIPS-shaped shard), one NCCL all-reduce of the K x V counts per sweep inside the graph.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled sites/sec per Gibbs sweep"
UNIT = "sites/s"

WORKLOADS = {
    "nips": dict(model="lda", docs=1500, vocab=12419, topics=100, doc_len=1267, scaling="weak"),
    "kos": dict(model="lda", docs=3430, vocab=6906, topics=50, doc_len=136, scaling="weak"),
    "1b": dict(model="lda", docs=1_000_000, vocab=100_000, topics=1000, doc_len=1000, scaling="strong"),
    "gmm": dict(model="gmm", points=100_000, topics=4, scaling="weak"),
    "logreg": dict(model="logreg", rows=10_000_000, features=64, scaling="weak"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ----------------------------------------------------------------------------------------
# measurement helpers
# ----------------------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons sampled while the timed region runs.

    NVML (libnvidia-ml, the library nvidia-smi reads) polled from a background thread
    every ~0.5 ms, so even a timed region of a few tens of ms gets dozens of samples;
    only samples taken between __enter__ and __exit__ are kept.  Falls back to
    `nvidia-smi -lms 20` when NVML cannot be loaded."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.rows = []  # (sm_mhz, sm_max_mhz, [flag names active])
        self.source = None

    def _nvml_loop(self, nv, h, bits):
        import time as _t

        while not self._stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), [n for n, b in zip(self.NAMES, bits) if r & b]))
            except Exception:
                break
            _t.sleep(0.0005)

    def __enter__(self):
        self._stop = False
        self.thread = None
        try:
            import threading

            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h, bits), daemon=True)
            self.source = "nvml"
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self._stop = True
        if self.thread is not None:
            self.thread.join(timeout=5)
        out = ""
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
        for line in (out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                flags = [n for n, f in zip(self.NAMES, parts[3:]) if f.lower() == "active"]
                self.rows.append((float(parts[0]), float(parts[1]), flags))
            except ValueError:
                continue

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        reasons = sorted({n for _, _, flags in rows for n in flags})
        loaded = [r[0] for r in rows if r[0] > 500] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": self.source}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_profile(key: str):
    """The committed `ncu --set full` summary of kernel `workload:kernel`
    (profiles/ncu_traffic.json): {"dram_bytes": per launch, "l1tex_pct", "lts_pct",
    "source"}; None when that capture does not exist."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            v = json.load(f).get(key)
    except Exception:
        return None
    if isinstance(v, (int, float)):
        return {"dram_bytes": float(v)}
    return v


def binding_of(prof):
    """The unit that bounds a kernel in its committed ncu capture: the busier of the L1TEX
    data pipe and instruction issue (with the L2 throughput beside them)."""
    units = {"l1tex data pipe": prof.get("l1tex_pct"), "instruction issue": prof.get("issue_pct")}
    name, pct = max(((k, v) for k, v in units.items() if v is not None), key=lambda kv: kv[1])
    return {"unit": name, "pct_of_peak": pct, "l1tex_pct_of_peak": prof.get("l1tex_pct"),
            "issue_pct_of_peak": prof.get("issue_pct"), "lts_pct_of_peak": prof.get("lts_pct"),
            "source": prof.get("source")}


# ----------------------------------------------------------------------------------------
# synthetic inputs (host side, gen_lda's generative process, gen.cpp:21-60)
# ----------------------------------------------------------------------------------------
def gen_lda_corpus(docs, vocab, topics, doc_len, seed):
    """phi_k ~ Dir(0.05), theta_d ~ Dir(0.3), uniform document length, z ~ Cat(theta_d),
    w ~ Cat(phi_z) -- the process of the reference's gen_lda, drawn with numpy."""
    rs = np.random.default_rng(seed)
    phi = rs.dirichlet(np.full(vocab, 0.05), size=topics)
    cphi = np.cumsum(phi, axis=1)
    w = np.empty(docs * doc_len, dtype=np.int64)
    chunk = max(1, 500_000 // max(doc_len, 1))
    for d0 in range(0, docs, chunk):
        d1 = min(docs, d0 + chunk)
        th = rs.dirichlet(np.full(topics, 0.3), size=d1 - d0)
        cth = np.cumsum(th, axis=1)
        u = rs.random((d1 - d0, doc_len))
        z = np.minimum((u[:, :, None] >= cth[:, None, :]).sum(-1), topics - 1) if topics <= 128 else \
            np.stack([np.minimum(np.searchsorted(cth[i], u[i], side="right"), topics - 1) for i in range(d1 - d0)])
        z = z.reshape(-1)
        uw = rs.random(z.size)
        ww = np.empty(z.size, dtype=np.int64)
        for k in np.unique(z):
            sel = z == k
            ww[sel] = np.minimum(np.searchsorted(cphi[k], uw[sel] * cphi[k, -1], side="right"), vocab - 1)
        w[d0 * doc_len:d1 * doc_len] = ww
    return w


E2E_NOTES = {
    "lda": "; the sweep starts from the written-back state while z uploads (compared on the device "
           "after the sweep, redone if the caller changed it); phi/theta copies overlap the z-step",
    "logreg": "; w, b uploaded every call, the likelihood refresh pass skipped when they equal the "
              "written-back state",
}


def pinned_like(arr):
    import torch

    t = torch.empty(arr.size, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True)
    a = t.numpy()
    a[:] = arr
    return a, t


L2_NOTE = ("GPU arm: 256 MiB written before every timed sweep (L2 flushed; NIPS/KOS fit the "
           "126 MB L2 within a sweep); CPU arm: not applicable")


def write_corpus_file(path, offsets, w, V):
    """The binary corpus format of bnmc_gpu_lda_load_corpus (include/bnmc_gpu.h), read by
    oracle/ref_bench lda-file (kept here so the reference arm imports nothing of ours)."""
    with open(path, "wb") as f:
        f.write(b"BNMCCORP")
        f.write(np.array([1, 0], dtype=np.uint32).tobytes())
        f.write(np.array([len(offsets) - 1, len(w), V], dtype=np.int64).tobytes())
        f.write(np.ascontiguousarray(offsets, dtype=np.int64).tobytes())
        f.write(np.ascontiguousarray(w, dtype=np.int32).tobytes())


def gmm_points(n, seed):
    """gen_gmm's process (gen.cpp:90-107): centres -5, -1, 1, 5 with sd 1, 0.1, 2, 1."""
    rs = np.random.default_rng(seed)
    c, sd = np.array([-5.0, -1.0, 1.0, 5.0]), np.array([1.0, 0.1, 2.0, 1.0])
    zt = rs.integers(0, 4, n)
    return c[zt] + sd[zt] * rs.normal(size=n)


def shared_config(args, world):
    """The `config` both arms print (identical dicts: same workload, same inputs)."""
    wl = WORKLOADS[args.workload]
    if wl["model"] == "lda":
        docs = wl["docs"] * (world if wl["scaling"] == "weak" else 1)
        cfg = {"workload": f"lda-{args.workload}", "model": "lda (proj/models/lda.bn)", "docs": docs,
               "vocab": wl["vocab"], "topics": wl["topics"], "doc_len": wl["doc_len"],
               "tokens": docs * wl["doc_len"], "seed": args.seed,
               "init": "prior_init(seed) (sampler.cpp:542-555)", "l2": L2_NOTE}
        if args.workload == "1b":
            cfg["corpus"] = ("GPU arm: device generator (gen_lda's process, gen_tokens_kernel); "
                             "CPU arm: reference gen_lda on a sample (the host cannot hold 1e9 tokens)")
        else:
            cfg["corpus"] = ("gen_lda_corpus (numpy, seeded; gen_lda's process gen.cpp:21-60: phi_k ~ "
                             "Dir(0.05), theta_d ~ Dir(0.3)); identical documents in both arms")
        return cfg
    if wl["model"] == "gmm":
        return {"workload": "gmm-100k", "model": "gmm (proj/models/gmm.bn)", "points": wl["points"],
                "components": wl["topics"], "seed": args.seed, "init": "prior_init(seed)",
                "data": "gmm_points (numpy, seeded; gen_gmm's process); identical points in both arms",
                "l2": L2_NOTE}
    return {"workload": "logreg-mh-10m", "model": "logistic regression MH", "rows": wl["rows"] * world,
            "features": wl["features"], "seed": args.seed, "l2": L2_NOTE,
            "data": "GPU arm: logistic rows; CPU arm: regression.bn (the reference has no logistic model)"}


# ----------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1312_3613_b200 as g

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wl = dict(WORKLOADS[args.workload])
    stream = torch.cuda.Stream()  # the engine runs on this stream; events and flushes too
    with torch.cuda.stream(stream):
        return _run_ours(args, rank, world, local_rank, g, torch, dist, wl, stream)


def gpu_index_of(local_rank):
    gi = local_rank
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gi = int(vis.split(",")[local_rank])
        except (ValueError, IndexError):
            pass
    return gi


def time_sweeps(eng, torch, stream, flush, it, steps, gpu_index, dist=None):
    """`steps` sweeps, each bracketed by CUDA events on the engine's stream after an L2
    flush; clocks sampled during the timed region.  Returns (mean ms, clocks, wall s)."""
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu_index) as clk:
        w0 = time.perf_counter()
        for i in range(steps):
            flush.zero_()                      # > 126 MB L2: every sweep starts cold
            starts[i].record(stream)
            eng.enqueue(it + i, 1)
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    ms = float(np.mean([s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]))
    return ms, clk.summary(), wall


def phase_times(eng, torch, flush, it, n):
    """The same sweep launched kernel by kernel with events (bnmc_gpu_sweep_phases)."""
    phase_ms = {}
    for i in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        for name, t in eng.sweep_phases(it + i):
            phase_ms.setdefault(name, []).append(t)
    return {k: float(np.mean(v)) for k, v in phase_ms.items()}


def lda_zstep_bytes(docs, V, K, L):
    """Per z-step launch: (compulsory DRAM bytes of its working set, operand bytes it
    streams).  Working set: w, z (4 + 4 B per token), the fp32 screen rows (V x Kp32),
    theta/S (M x K), both count arrays written (V x Kp, M x K int32).  Operands: per
    token its fp32 row (4 Kp32 B) + w, z, 2 count updates (16 B), per document its
    theta row (8 K B)."""
    N = docs * L
    kp32 = -(-K // 32) * 32
    kp = -(-K // 4) * 4
    compulsory = 8 * N + 4 * V * kp32 + 8 * docs * K + 4 * V * kp + 4 * docs * K
    operand = N * (4 * kp32 + 16) + 8 * docs * K
    return compulsory, operand


def lda_wm_bytes(docs, V, K, L):
    """Compulsory DRAM bytes per z-step launch in the word-major order (K > 128 corpora
    whose fp32 rows exceed the L2, lda.cu build_word_major): per token its sorted index,
    document and z (12 B); theta/S fp32 rows read once (4 Kp32 per document, the blocks'
    rows then stay in L2); the doc-topic counts read and written (8 K per document); each
    word's fp32 row once per document block (the words of a ~24 MB block of theta/S rows).
    The operand stream (a theta/S row per token) is served by L2."""
    N = docs * L
    kp32 = -(-K // 32) * 32
    block_docs = max(1, (24 << 20) // (4 * kp32))
    nblocks = -(-docs // block_docs)
    words_per_block = min(V, block_docs * L)
    return 12 * N + 4 * kp32 * docs + 8 * K * docs + 4 * kp32 * words_per_block * nblocks


def _run_ours(args, rank, world, local_rank, g, torch, dist, wl, stream):
    nccl_id = None
    if world > 1:
        obj = [g.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    model = wl["model"]
    config = shared_config(args, world)
    t_setup = time.perf_counter()
    extra = {}
    if model == "lda":
        docs = config["docs"]
        V, K, L = wl["vocab"], wl["topics"], wl["doc_len"]
        hyper = {"K": K, "V": V, "M": docs, "N": [L] * docs}
        exact = args.weights == "exact"
        cfg = g.RunConfig(seed=args.seed, device=local_rank, exact_weights=exact)
        eng = g.Engine("lda", hyper, cfg, rank=rank, world_size=world, nccl_id=nccl_id,
                       stream=stream.cuda_stream)
        sites_total = docs * L
        host_corpus = args.workload != "1b"
        if host_corpus:
            store = eng.allocate()
            store["w"] = gen_lda_corpus(docs, V, K, L, args.seed)
            eng.prior_init(store, args.seed)       # device prior_init, written back to the host store
        else:
            eng.lda_generate(args.seed)            # device generator + device prior_init
            store = None
        b, e = g.partition(np.arange(docs + 1, dtype=np.int64) * L, world, rank)
        sites_local = (e - b) * L
        # conj_pool, colsum_rows, z-step screen, z-step fallback, wterm<FINAL>
        # (sharded: + finalize after the log-joint all-reduce; NCCL's own kernels not counted)
        per_sweep_kernels = 5 + (1 if world > 1 else 0)
        # exact: the same kernels; the fallback is the log-space one (zfallback_log_kernel)
        dominant = "zstep"
        compulsory, operand = lda_zstep_bytes(e - b, V, K, L)
        if args.workload == "1b":
            # word-major order: theta/S rows of a document block stay in L2
            compulsory = lda_wm_bytes(e - b, V, K, L)
        extra["weights"] = ("log-space exp(log theta + log phi - max): the reference's arithmetic "
                            "(draw_from_log_weights, dist.cpp:202-215), fp64, no screen" if exact else
                            "product theta*phi (fp64; fp32 screen + fp64 fallback, z bit-exact)")
        if exact:
            config = dict(config, weights="log-space (BNMC_GPU_EXACT_WEIGHTS)")
    elif model == "gmm":
        N, K = wl["points"], wl["topics"]
        hyper = {"N": N, "K": K}
        eng = g.Engine("gmm", hyper, g.RunConfig(seed=args.seed, device=local_rank), stream=stream.cuda_stream)
        store = eng.allocate()
        store["x"] = gmm_points(N, args.seed)
        eng.prior_init(store, args.seed)
        sites_total, sites_local = N * world, N  # replicas
        # K <= 8: the fused sweep -- draw_params, z (+ next-sweep statistics), finalize
        fused = K <= 8 and os.environ.get("BNMC_GMM_FUSED", "1") != "0"
        per_sweep_kernels, dominant = (3, "z_stats") if fused else (6, "z")
        compulsory = operand = 16 * N
        host_corpus = True
        extra["parallelism"] = f"replicas x{world}"
    else:
        N, Kf = wl["rows"], wl["features"]
        Nt = N * world
        rs = np.random.default_rng(args.seed)
        x = rs.uniform(-1, 1, size=(Nt, Kf))
        wt = 0.3 * rs.normal(size=Kf)
        y = (rs.random(Nt) < 1 / (1 + np.exp(-(x @ wt + 0.1)))).astype(np.float64)
        hyper = {"N": Nt, "K": Kf, "l": -1.0, "u": 1.0}
        eng = g.Engine("logreg", hyper, g.RunConfig(seed=args.seed, device=local_rank, mh_scale=0.01),
                       rank=rank, world_size=world, nccl_id=nccl_id, stream=stream.cuda_stream)
        store = eng.allocate()
        store["x"], store["y"] = x.ravel(), y
        del x
        eng.upload(store)
        sites_total, sites_local = Nt, Nt // world
        per_sweep_kernels, dominant = 3, "lik"
        compulsory = operand = sites_local * (8 * Kf + 8)
        host_corpus = True
    setup_s = time.perf_counter() - t_setup

    # --- device-resident timing (value): per-sweep CUDA events, L2 flushed in between ---
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    it = 0
    eng.enqueue(it, args.warmup)
    it += args.warmup
    eng.synchronize()
    gpu_index = gpu_index_of(local_rank)
    ms_step, clocks, wall = time_sweeps(eng, torch, stream, flush, it, args.steps, gpu_index, dist)
    lj_last, _ = eng.synchronize()
    it += args.steps
    if dist:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        dist.barrier()
    value = sites_total / (ms_step / 1e3)

    # --- per-kernel pass (same sweep, launched phase by phase with events) ---
    nph = max(3, min(args.steps, 20))
    phases = phase_times(eng, torch, flush, it, nph)
    it += nph
    dom_ms = phases.get(dominant)
    peak, peak_src = measured_peak_hbm()
    roofline = None
    if dom_ms:
        prof = ncu_profile(f"{args.workload}:{dominant}") or {}
        achieved = compulsory / (dom_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
                    "traffic": prof.get("dram_bytes"), "algorithmic_bytes_per_launch": compulsory,
                    "kernel_ms": round(dom_ms, 5), "share_of_sweep": round(dom_ms / sum(phases.values()), 3)}
        if model == "lda" and args.workload == "1b":
            roofline["algorithmic_bytes_note"] = (
                "compulsory DRAM bytes of the word-major z-step (sorted token index, document and z per "
                "token; theta/S rows once; doc-topic counts; each word's row once per document block); "
                "the theta/S operand rows stream from L2")
            if prof.get("dram_bytes"):
                roofline["dram_frac"] = round(prof["dram_bytes"] / (dom_ms / 1e3) / 1e9 / peak, 4)
        elif model == "lda":
            roofline["algorithmic_bytes_note"] = (
                "compulsory DRAM bytes of the z-step's working set (w, z, fp32 screen rows, theta, "
                "both count arrays); the rows are re-read per token from L2, not HBM")
        elif model == "logreg":
            roofline["algorithmic_bytes_note"] = (
                "x row + y per data row, read once per step (a read-only stream; the copy peak counts "
                "read + write traffic, so a pure read stream can reach slightly above it)")
        if model == "lda":
            if prof.get("l1tex_pct") is not None:
                roofline["binding"] = binding_of(prof)
            # the operand bytes the kernel streams (fp32 row per token) against the L2 -> SM
            # read bandwidth measured in this run by one long launch over 24 MB
            try:
                l2_bw = g.read_bandwidth(24 << 20, 200)
                hbm_bw = g.read_bandwidth(4 << 30, 3)
                ach_l2 = operand / (dom_ms / 1e3) / 1e9
                roofline["l2"] = {"achieved": round(ach_l2, 1), "peak": round(l2_bw, 1), "unit": "GB/s",
                                  "frac": round(ach_l2 / l2_bw, 4), "operand_bytes_per_launch": operand,
                                  "peak_source": "measured in this run: one persistent launch re-reading a 24 MB "
                                                 "buffer 200 times (256-bit ld.global.cg loads)",
                                  "hbm_read_measured": round(hbm_bw, 1)}
            except Exception as ex:  # reported, never fatal
                roofline["l2"] = {"error": str(ex)}

    # --- e2e through the public API with host buffers ---
    e2e = None
    e2e_pageable = None
    if host_corpus and store is not None:
        # bytes per step, counted by the library (bnmc_gpu_transfer_stats) on the call after
        # the bind: LDA this rank's z slice up (the sweep reads only z of the latent state),
        # z and theta slices + the global phi + lj down; MH w, b up and down; GMM z, pi,
        # mu, sigma2 up and down
        def e2e_loop(e_, s_, it_):
            e_.sweep(s_, it_)  # bind (page-locks the store, uploads the observed data once)
            e_.sweep(s_, it_ + 1)
            up, down = e_.transfer_stats()
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(args.steps):
                e_.sweep(s_, it_ + 2 + i)
            torch.cuda.synchronize()
            sec = (time.perf_counter() - t0) / args.steps
            if dist:
                t = torch.tensor([sec], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                sec = float(t.item())
            return sec, up, down, it_ + 2 + args.steps

        e2e_s, up, down, it = e2e_loop(eng, store, it)
        e2e = {"value": sites_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(up),
               "d2h_bytes_per_step": int(down), "ms_per_step": e2e_s * 1e3,
               "path": "Engine.sweep(store, iter) on the caller's numpy store, page-locked once at binding "
                       "(RunConfig.pin_host): bnmc_gpu_sweep_store (upload of what the sweep reads, sweep, "
                       "write-back)" + E2E_NOTES.get(model, "")}
        if model in ("lda", "gmm") and world == 1:
            # the same loop with the store left pageable (pin_host=False): a fresh engine on
            # the same stream, the store's state as the pinned loop left it
            eng.close()
            eng = g.Engine(model, hyper, g.RunConfig(seed=args.seed, device=local_rank, pin_host=False,
                                                     exact_weights=args.weights == "exact" and model == "lda"),
                           stream=stream.cuda_stream)
            sp, up2, down2, it = e2e_loop(eng, store, it)
            e2e_pageable = {"value": sites_total / sp, "unit": UNIT, "ms_per_step": sp * 1e3,
                            "h2d_bytes_per_step": int(up2), "d2h_bytes_per_step": int(down2)}
    else:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "1B corpus is generated and kept on the device (host cannot hold it)"}
    eng.close()

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (gen_lda process, numpy; device prior_init)" if model == "lda" else "synthetic",
           "config": config, "execution": {**extra, "parallelism": extra.get(
               "parallelism", f"{'documents' if model == 'lda' else 'rows'} sharded x{world}")},
           "roofline": roofline, "phases_ms": {k: round(v, 5) for k, v in phases.items()},
           "e2e": e2e, "e2e_pageable": e2e_pageable, "gpu_launches": per_sweep_kernels * args.steps,
           "clocks": clocks, "wall_s_timed": wall, "setup_s": setup_s, "last_log_joint": lj_last}
    if rank == 0 and world == 1 and model == "lda" and host_corpus and args.weights == "product":
        out["e2e_reference_engine"] = e2e_reference_engine(args, config, store["w"])
    if rank == 0 and world == 1 and args.workload == "nips" and not args.no_1b and args.weights == "product":
        out["roofline_1b"] = roofline_1b(args, g, torch, stream, flush, gpu_index)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    if dist:
        dist.destroy_process_group()
    return out if rank == 0 else None


def e2e_reference_engine(args, config, w):
    """The reference's OWN bnmc::Engine::sweep with RunConfig::device = B200
    (integration/: reference_b200.patch + gpu_backend.cpp, linked to libbnmc_gpu.so) on
    its std::vector ParamStore -- pageable memory the backend page-locks once at binding --
    timed per call in C++ (b2r_sweeps_timed) on this run's corpus: what a caller of the
    unchanged reference API sees."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "integration"))
        import b200ref

        R = b200ref.B200Ref()
        hyper = {"K": config["topics"], "V": config["vocab"], "M": config["docs"],
                 "N": [config["doc_len"]] * config["docs"]}
        e = R.open("lda", hyper, "gibbs", args.seed, device="b200")
        if not e.on_device:
            return {"error": "the reference Engine did not select the B200 backend"}
        e.set("w", w)
        e.prior_init(args.seed)
        e.sweeps_timed(0, 3)  # bind (page-lock, observed data up) + warm calls
        lj, ms = e.sweeps_timed(3, args.steps)
        e.close()
        mean = float(np.mean(ms))
        return {"value": config["tokens"] / (mean / 1e3), "unit": UNIT, "ms_per_step": mean,
                "ms_min": float(np.min(ms)), "last_log_joint": float(lj[-1]),
                "path": "bnmc::Engine::sweep of the patched reference (RunConfig::device = B200) on its own "
                        "std::vector ParamStore, C++ steady_clock per call (integration/b200_driver.cpp)"}
    except Exception as ex:  # reported, never fatal
        return {"error": str(ex)}


def roofline_1b(args, g, torch, stream, flush, gpu_index):
    """A short pass over the 1B-token config (K=1000, V=1e5, 1e6 documents x 1000 tokens;
    device generator + device prior_init): 3 warm + 3 timed sweeps, the z-step's time from
    the phase pass, its DRAM fraction from the committed ncu capture's bytes per launch."""
    try:
        wl = WORKLOADS["1b"]
        docs, V, K, L = wl["docs"], wl["vocab"], wl["topics"], wl["doc_len"]
        t0 = time.perf_counter()
        eng = g.Engine("lda", {"K": K, "V": V, "M": docs, "N": [L] * docs},
                       g.RunConfig(seed=args.seed, device=torch.cuda.current_device()), stream=stream.cuda_stream)
        eng.lda_generate(args.seed)
        eng.enqueue(0, 3)
        eng.synchronize()
        setup = time.perf_counter() - t0
        ms, clocks, _ = time_sweeps(eng, torch, stream, flush, 3, 3, gpu_index)
        phases = phase_times(eng, torch, flush, 6, 2)
        eng.close()
        zms = phases["zstep"]
        N = docs * L
        peak, peak_src = measured_peak_hbm()
        _, operand = lda_zstep_bytes(docs, V, K, L)
        compulsory = lda_wm_bytes(docs, V, K, L)
        ach = compulsory / (zms / 1e3) / 1e9
        prof = ncu_profile("1b:zstep") or {}
        dram = prof.get("dram_bytes")
        out = {"bound": "hbm", "kernel": "zstep", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
               "frac": round(ach / peak, 4), "peak_source": peak_src, "algorithmic_bytes_per_launch": compulsory,
               "algorithmic_bytes_note": (
                   "compulsory DRAM bytes of the word-major z-step (tokens sorted by document block x word: "
                   "12 B per token, theta/S rows once, doc-topic counts, each word's row once per block); "
                   "the per-token operand rows (theta/S, 4 Kp32 B) are served by L2"),
               "traffic": dram, "kernel_ms": round(zms, 3), "sweep_ms": round(ms, 3),
               "sites_per_s": N / (ms / 1e3), "phases_ms": {k: round(v, 3) for k, v in phases.items()},
               "clocks": clocks, "setup_s": round(setup, 2),
               "config": {"workload": "lda-1b", "docs": docs, "vocab": V, "topics": K, "doc_len": L, "tokens": N}}
        if dram:
            out["dram_frac"] = round(dram / (zms / 1e3) / 1e9 / peak, 4)
        if prof.get("l1tex_pct") is not None:
            out["binding"] = binding_of(prof)
        try:
            l2_bw = g.read_bandwidth(24 << 20, 200)
            ach_l2 = operand / (zms / 1e3) / 1e9
            out["l2"] = {"achieved": round(ach_l2, 1), "peak": round(l2_bw, 1), "unit": "GB/s",
                         "frac": round(ach_l2 / l2_bw, 4), "operand_bytes_per_launch": operand}
        except Exception as ex:  # reported, never fatal
            out["l2"] = {"error": str(ex)}
        return out
    except Exception as ex:  # reported, never fatal for the NIPS line
        return {"error": str(ex)}


# ----------------------------------------------------------------------------------------
# reference arm / cpu baseline (the compiled, unmodified reference: oracle/_ref)
# ----------------------------------------------------------------------------------------
def ref_bench(argv, timeout, retries=3):
    from oracle import REF_BENCH

    if not os.path.exists(REF_BENCH):
        raise FileNotFoundError("oracle/_ref/ref_bench not built (make -C oracle ref)")
    last = None
    for attempt in range(retries):
        try:
            r = subprocess.run([REF_BENCH, *map(str, argv)], capture_output=True, text=True, timeout=timeout)
            if r.returncode == 0:
                return json.loads(r.stdout.strip().splitlines()[-1]), attempt
            last = f"exit {r.returncode}: {r.stderr.strip()[-200:]}"
        except subprocess.TimeoutExpired:
            last = f"timeout after {timeout}s (reference thread-pool hang, SURVEY.md section 5)"
    raise RuntimeError(last)


def shared_inputs(args, world, tmp):
    """The arm-independent input file for the reference (`lda-file` / `gmm-file`), written
    from the same seeded generators the GPU arm uses; None for the workloads whose
    reference run draws its own sample (1b, logreg)."""
    wl = WORKLOADS[args.workload]
    if wl["model"] == "lda" and args.workload != "1b":
        cfg = shared_config(args, world)
        docs, L = cfg["docs"], wl["doc_len"]
        path = os.path.join(tmp, "corpus.bnc")
        write_corpus_file(path, np.arange(docs + 1, dtype=np.int64) * L,
                          gen_lda_corpus(docs, wl["vocab"], wl["topics"], L, args.seed), wl["vocab"])
        return path
    if wl["model"] == "gmm":
        path = os.path.join(tmp, "points.f64")
        gmm_points(wl["points"], args.seed).tofile(path)
        return path
    return None


def cpu_baseline(args):
    """The reference on ONE host core on half of the same corpus (the first 750 of the
    1500 NIPS documents), 2 timed sweeps (~25 s)."""
    import tempfile

    wl = WORKLOADS[args.workload]
    try:
        with tempfile.TemporaryDirectory() as tmp:
            path = shared_inputs(args, 1, tmp)
            if wl["model"] == "lda" and path:
                docs = wl["docs"] // 2
                res, retries = ref_bench(["lda-file", path, wl["topics"], args.seed, 1, 0, 2, docs], timeout=300)
                sample = (f"the first {docs} of the {wl['docs']} documents of this run's corpus "
                          f"({docs * wl['doc_len']} sites), reference prior_init, 2 timed sweeps, "
                          f"Engine::sweep incl. log-joint")
            elif wl["model"] == "lda":
                res, retries = ref_bench(["lda", 8, wl["vocab"], wl["topics"], 10_000, args.seed, 1, 1, 2], timeout=300)
                sample = "8 documents x 10000 tokens of the 1b shape (reference gen_lda), 1 warm + 2 timed sweeps"
            elif wl["model"] == "gmm":
                res, retries = ref_bench(["gmm-file", path, args.seed, 1, 1, 5], timeout=300)
                sample = f"this run's {wl['points']} points, 1 warm + 5 timed sweeps"
            else:
                n = 20_000
                res, retries = ref_bench(["regression", n, wl["features"], args.seed, 1, 1, 3, 0.01], timeout=300)
                sample = (f"regression.bn MH (linear twin; no logistic reference), {n} rows x {wl['features']} "
                          f"features, 1 warm + 3 timed steps")
        s_ = float(np.mean(res["ms"])) / 1e3
        return {"value": res["sites"] / s_, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": sample, "s_per_sweep": s_, "retries": retries}
    except Exception as e:  # reported, never fatal for the GPU line
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": None, "error": str(e)}


def run_reference(args, world):
    import tempfile

    wl = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    budget_s = 150.0
    steps, warm = args.steps, args.warmup
    cfg = shared_config(args, world)
    with tempfile.TemporaryDirectory() as tmp:
        path = shared_inputs(args, world, tmp)
        if wl["model"] == "lda":
            K = wl["topics"]
            L = wl["doc_len"] if args.workload != "1b" else 10_000
            full_docs = cfg["docs"] if args.workload != "1b" else 8
            # ~252 ns per token-candidate single-threaded, ~60 % parallel efficiency
            per_doc_s = L * K * 252e-9 / max(1.0, 0.6 * threads)
            fixed_s = 1.5 * K * wl["vocab"] / 1.24e6 / max(1.0, 0.6 * threads)
            docs = int(max(1, min(full_docs, (budget_s / (steps + warm) - fixed_s) / per_doc_s)))
            if path:
                argv, tail = ["lda-file", path, K, args.seed], [warm, steps, docs]
                sample = (f"{docs} of {full_docs} documents x {L} tokens of this run's corpus (the GPU arm's "
                          f"documents), V={wl['vocab']}, K={K}; reference prior_init; Engine::sweep incl. log-joint")
            else:
                argv, tail = ["lda", docs, wl["vocab"], K, L, args.seed], [warm, steps]
                sample = (f"{docs} documents x {L} tokens of the 1b shape, reference gen_lda + prior_init; "
                          f"Engine::sweep incl. log-joint")
            est = (steps + warm) * (fixed_s + docs * per_doc_s)
        elif wl["model"] == "gmm":
            argv, tail = ["gmm-file", path, args.seed], [warm, steps]
            sample, est = f"this run's {wl['points']} points (full workload)", (steps + warm) * 0.1
        else:
            n = int(min(wl["rows"], max(10_000, 1e8 / (steps + warm))))
            argv, tail = ["regression", n, wl["features"], args.seed], [warm, steps]
            sample, est = f"regression.bn MH (linear twin), {n} rows x {wl['features']}", (steps + warm) * n * 1.6e-5
        res, retries, used, last = None, 0, threads, None
        for t in (threads, max(1, threads // 2), 1):
            try:
                if wl["model"] == "lda" and path:
                    a = argv + [t] + tail
                else:
                    a = argv + [t] + tail + ([0.01] if wl["model"] == "logreg" else [])
                res, retries = ref_bench(a, timeout=int(60 + 4 * est * max(1, threads / t)))
                used = t
                break
            except Exception as e:
                last = str(e)
                continue
    if res is None:
        return {"impl": "reference", "unavailable": f"reference sampler failed on this host: {last}"}
    s_ = float(np.mean(res["ms"])) / 1e3
    value = res["sites"] / s_
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": s_ * 1e3, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_lda process, numpy; device prior_init)" if wl["model"] == "lda" else "synthetic",
            "config": cfg, "execution": {"sample": sample, "threads": used},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "reference", "sample": sample,
                             "retries": retries},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn_ranks(n):
    """`--gpus N` outside torchrun: launch this script under torch.distributed.run with N
    ranks (one per GPU), rank 0 prints the line."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="nips", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-1b", action="store_true", help="skip the 1B-token roofline pass of the NIPS run")
    ap.add_argument("--weights", default="product", choices=["product", "exact"],
                    help="LDA z-step arithmetic: product form (default) or the reference's log-space form")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return
    out = run_ours(args, rank, world, local)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
