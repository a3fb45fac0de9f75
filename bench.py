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
               bandwidth; achieved = algorithmic bytes per launch (phi row
               8K + 16 B of token state per site + the theta row per 512-token unit) /
               its CUDA-event duration
  cpu_baseline the compiled reference (oracle/_ref) timed on this host's cores on a
               bounded sample of the same workload
  e2e          the same metric through the public API with HOST buffers: every step
               uploads what the sweep reads from the caller's store (LDA: z; its phi and
               theta blocks redraw phi and theta first), sweeps, and downloads the whole
               latent state + log-joint (Engine::sweep borrow semantics), pinned memory
Multi-GPU (torchrun): documents sharded across ranks (weak scaling: each rank holds a
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


def ncu_traffic(key: str):
    """dram bytes per launch of the kernel `workload:kernel` from the committed ncu summaries
    (profiles/ncu_traffic.json; one `ncu --set full` capture per workload), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


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


def _run_ours(args, rank, world, local_rank, g, torch, dist, wl, stream):
    nccl_id = None
    if world > 1:
        obj = [g.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    model = wl["model"]
    t_setup = time.perf_counter()
    if model == "lda":
        docs = wl["docs"] * (world if wl["scaling"] == "weak" else 1)
        V, K, L = wl["vocab"], wl["topics"], wl["doc_len"]
        hyper = {"K": K, "V": V, "M": docs, "N": [L] * docs}
        cfg = g.RunConfig(seed=args.seed, device=local_rank)
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
        # phi_gamma2, phi_colsum2, theta2, z-step screen, z-step fallback, wterm<FINAL>
        # (sharded: + finalize after the log-joint all-reduce; NCCL's own kernels not counted)
        per_sweep_kernels = 6 + (1 if world > 1 else 0)
        dominant = "zstep"
        # SURVEY 8(d), per token: phi row 8K (fp64) + w 4 + z 4 + topic-word count 4 +
        # doc-topic count 4, theta row 8K per work unit (a document, <= 2048 tokens)
        bytes_per_site_dom = 8 * K + 16 + 8 * K / min(L, 2048)
        # what the implementation moves per token: the fp32 screen row (4K) + the same 16
        impl_bytes_per_site = 4 * K + 16
        bytes_per_site_sweep = 8 * K + 16 * K / L + 16 + 20 * K * V / (docs * L)
        config = {"workload": f"lda-{args.workload}", "model": "lda (proj/models/lda.bn)", "docs": docs,
                  "vocab": V, "topics": K, "doc_len": L, "tokens": sites_total, "seed": args.seed,
                  "weights": "product theta*phi (fp64)", "parallelism": f"docs sharded x{world} (NCCL allreduce K x V counts)"}
    elif model == "gmm":
        N, K = wl["points"], wl["topics"]
        rs = np.random.default_rng(args.seed)
        c, sd = np.array([-5.0, -1.0, 1.0, 5.0]), np.array([1.0, 0.1, 2.0, 1.0])
        zt = rs.integers(0, 4, N)
        hyper = {"N": N, "K": K}
        eng = g.Engine("gmm", hyper, g.RunConfig(seed=args.seed, device=local_rank), stream=stream.cuda_stream)
        store = eng.allocate()
        store["x"] = c[zt] + sd[zt] * rs.normal(size=N)
        eng.prior_init(store, args.seed)
        sites_total = sites_local = N * world  # replicas
        sites_local = N
        # K <= 8: the fused sweep -- draw_params, z (+ next-sweep statistics), finalize
        fused = K <= 8 and os.environ.get("BNMC_GMM_FUSED", "1") != "0"
        per_sweep_kernels, dominant = (3, "z_stats") if fused else (6, "z")
        bytes_per_site_dom = bytes_per_site_sweep = impl_bytes_per_site = 16
        host_corpus = True
        config = {"workload": "gmm-100k", "model": "gmm (proj/models/gmm.bn)", "points": N, "components": K,
                  "seed": args.seed, "parallelism": f"replicas x{world}"}
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
        bytes_per_site_dom = bytes_per_site_sweep = impl_bytes_per_site = 8 * Kf + 8
        host_corpus = True
        config = {"workload": "logreg-mh-10m", "model": "logistic regression MH", "rows": Nt, "features": Kf,
                  "seed": args.seed, "parallelism": f"rows sharded x{world}"}
    setup_s = time.perf_counter() - t_setup

    # --- device-resident timing (value): per-sweep CUDA events, L2 flushed in between ---
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    it = 0
    eng.enqueue(it, args.warmup)
    it += args.warmup
    eng.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    gpu_index = env_int("LOCAL_RANK", 0)
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_index = int(vis.split(",")[local_rank])
        except (ValueError, IndexError):
            pass
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu_index) as clk:
        w0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                      # > 126 MB L2: every sweep starts cold
            starts[i].record(stream)
            eng.enqueue(it + i, 1)
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    lj_last, _ = eng.synchronize()
    it += args.steps
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_step = float(np.mean(ms))
    if dist:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        dist.barrier()
    value = sites_total / (ms_step / 1e3)

    # --- per-kernel pass (same sweep, launched phase by phase with events) ---
    phase_ms = {}
    for i in range(max(3, min(args.steps, 20))):
        flush.zero_()
        torch.cuda.synchronize()
        for name, t in eng.sweep_phases(it):
            phase_ms.setdefault(name, []).append(t)
        it += 1
    phases = {k: float(np.mean(v)) for k, v in phase_ms.items()}
    dom_ms = phases.get(dominant)
    peak, peak_src = measured_peak_hbm()
    roofline = roofline_l2 = None
    if dom_ms:
        achieved = sites_local * bytes_per_site_dom / (dom_ms / 1e3) / 1e9
        traffic = ncu_traffic(f"{args.workload}:{dominant}")
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
                    "traffic": traffic, "algorithmic_bytes_per_site": round(bytes_per_site_dom, 2),
                    "kernel_ms": round(dom_ms, 5), "share_of_sweep": round(dom_ms / sum(phases.values()), 3),
                    "sweep_effective_frac": round(value / world * bytes_per_site_sweep / 1e9 / peak, 4),
                    "sweep_bytes_per_site": round(bytes_per_site_sweep, 2),
                    "note": "KOS/NIPS working sets fit the 126 MB L2 within a sweep (L2 is flushed before every "
                            "timed sweep, so reads start in HBM): frac > 1 means the kernel is fed from L2 -- "
                            "see roofline_l2"}
        # Secondary roofline: the bytes the implementation moves / the kernel time against
        # the device's L2 -> SM read bandwidth, measured here (bnmc_gpu_probe_read_bandwidth
        # over a 48 MB buffer); the HBM read bandwidth is measured the same way for context.
        try:
            l2_bw = g.read_bandwidth(48 << 20, 50)
            hbm_bw = g.read_bandwidth(4 << 30, 5)
            ach_impl = sites_local * impl_bytes_per_site / (dom_ms / 1e3) / 1e9
            roofline_l2 = {"bound": "l2", "kernel": dominant, "achieved": round(ach_impl, 1),
                           "peak": round(l2_bw, 1), "unit": "GB/s", "frac": round(ach_impl / l2_bw, 4),
                           "implementation_bytes_per_site": impl_bytes_per_site,
                           "peak_source": "measured in this run: 256-bit read stream over a 48 MB buffer",
                           "hbm_read_measured": round(hbm_bw, 1)}
        except Exception as ex:  # reported, never fatal
            roofline_l2 = {"error": str(ex)}

    # --- e2e through the public API with host buffers ---
    e2e = None
    if host_corpus and store is not None:
        for name in store.names:
            if not store.observed[name]:
                arr, t = pinned_like(store.arrays[name])
                store.arrays[name] = arr
                store.__dict__.setdefault("_pins", []).append(t)
        # bytes per step, counted by the library (bnmc_gpu_transfer_stats) on the call after
        # the bind: LDA this rank's z slice up (the sweep reads only z of the latent state),
        # z and theta slices + the global phi + lj down; MH w, b up and down; GMM z, pi,
        # mu, sigma2 up and down
        eng.sweep(store, it)  # bind (uploads the observed data once, outside the timed region)
        it += 1
        eng.sweep(store, it)
        it += 1
        up, down = eng.transfer_stats()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            eng.sweep(store, it + i)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.steps
        it += args.steps
        if dist:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": sites_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(up),
               "d2h_bytes_per_step": int(down), "ms_per_step": e2e_s * 1e3,
               "path": "Engine.sweep(store, iter) with pinned host arrays: bnmc_gpu_sweep_store (upload of "
                       "what the sweep reads, sweep, write-back)" + E2E_NOTES.get(model, "")}
    else:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "1B corpus is generated and kept on the device (host cannot hold it)"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (gen_lda process, numpy; device prior_init)" if model == "lda" else "synthetic",
           "config": {**config, "l2": "flushed before every timed sweep (256 MiB write)"},
           "roofline": roofline, "roofline_l2": roofline_l2, "phases_ms": {k: round(v, 5) for k, v in phases.items()},
           "e2e": e2e, "gpu_launches": per_sweep_kernels * args.steps,
           "clocks": clk.summary(), "wall_s_timed": wall, "setup_s": setup_s, "last_log_joint": lj_last}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    eng.close()
    if dist:
        dist.destroy_process_group()
    return out if rank == 0 else None


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


def cpu_baseline(args):
    wl = WORKLOADS[args.workload]
    if wl["model"] != "lda" or args.workload == "1b":
        docs = None
    try:
        if wl["model"] == "lda":
            docs = 150 if args.workload == "nips" else (600 if args.workload == "kos" else 8)
            L = wl["doc_len"] if args.workload != "1b" else 10_000
            res, retries = ref_bench(["lda", docs, wl["vocab"], wl["topics"], L, args.seed, 1, 1, 2], timeout=300)
            sample = (f"{docs} documents x {L} tokens ({docs * L} sites) of the {args.workload} shape "
                      f"(V={wl['vocab']}, K={wl['topics']}), reference gen_lda + prior_init, 1 warm + 2 timed "
                      f"sweeps, Engine::sweep incl. log-joint")
        elif wl["model"] == "gmm":
            res, retries = ref_bench(["gmm", wl["points"], args.seed, 1, 1, 5], timeout=300)
            sample = f"{wl['points']} points, 1 warm + 5 timed sweeps"
        else:
            n = 20_000
            res, retries = ref_bench(["regression", n, wl["features"], args.seed, 1, 1, 3, 0.01], timeout=300)
            sample = (f"regression.bn MH (linear twin; no logistic reference), {n} rows x {wl['features']} "
                      f"features, 1 warm + 3 timed steps")
        s = float(np.mean(res["ms"])) / 1e3
        return {"value": res["sites"] / s, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": sample, "s_per_sweep": s, "retries": retries}
    except Exception as e:  # reported, never fatal for the GPU line
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": None, "error": str(e)}


def run_reference(args, world):
    wl = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    budget_s = 150.0
    steps, warm = args.steps, args.warmup
    if wl["model"] == "lda":
        K, L = wl["topics"], wl["doc_len"] if args.workload != "1b" else 10_000
        full_docs = wl["docs"] * (world if wl["scaling"] == "weak" else 1) if args.workload != "1b" else 8
        # ~252 ns per token-candidate single-threaded, ~60 % parallel efficiency
        per_doc_s = L * K * 252e-9 / max(1.0, 0.6 * threads)
        fixed_s = 1.5 * K * wl["vocab"] / 1.24e6 / max(1.0, 0.6 * threads)
        docs = int(max(1, min(full_docs, (budget_s / (steps + warm) - fixed_s) / per_doc_s)))
        argv = ["lda", docs, wl["vocab"], K, L, args.seed]
        sample = (f"{docs} of {full_docs} documents x {L} tokens, V={wl['vocab']}, K={K}; reference gen_lda + "
                  f"prior_init; Engine::sweep incl. log-joint")
        tail = [warm, steps]
        est = (steps + warm) * (fixed_s + docs * per_doc_s)
    elif wl["model"] == "gmm":
        argv, tail = ["gmm", wl["points"], args.seed], [warm, steps]
        sample, est = f"{wl['points']} points (full workload)", (steps + warm) * 0.1
    else:
        n = int(min(wl["rows"], max(10_000, 1e8 / (steps + warm))))
        argv, tail = ["regression", n, wl["features"], args.seed], [warm, steps]
        sample, est = f"regression.bn MH (linear twin), {n} rows x {wl['features']}", (steps + warm) * n * 1.6e-5
    res, retries, used = None, 0, threads
    for t in (threads, max(1, threads // 2), 1):
        try:
            a = argv + [t] + tail + ([0.01] if wl["model"] == "logreg" else [])
            res, retries = ref_bench(a, timeout=int(60 + 4 * est * max(1, threads / t)))
            used = t
            break
        except Exception as e:
            last = str(e)
            continue
    if res is None:
        return {"impl": "reference", "unavailable": f"reference sampler failed on this host: {last}"}
    s = float(np.mean(res["ms"])) / 1e3
    value = res["sites"] / s
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": s * 1e3, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generators)",
            "config": {"workload": f"{wl['model']}-{args.workload}", "sample": sample, "threads": used},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "reference", "sample": sample,
                             "retries": retries},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="nips", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.gpus > 1 and world == 1:
        sys.exit("bench.py --gpus N>1 must be launched with torch.distributed.run (one rank per GPU)")
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return
    out = run_ours(args, rank, world, local)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
