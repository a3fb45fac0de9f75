"""TEST INFRASTRUCTURE: run a chain of the compiled, unmodified reference
(oracle/_ref/libbnmc_ref.so) in a child process.

The reference's worker pool can crash or hang when it runs multi-threaded (SURVEY.md
section 5: the ParallelExecutor generation race; surviving runs are bit-identical at any
thread count).  The at-size parity tests want its multi-threaded speed, so the chain runs
in a child process under a timeout and is retried -- with fewer threads after a failure,
finally single-threaded -- without taking the test runner down.

    spec = {"model": "lda", "hyper": {...}, "method": "gibbs", "seed": 42, "threads": 16,
            "mh_scale": 0.5, "gen": ["lda", [M, V, K, L, seed]] | ["gmm", [...]] |
            ["regression", [...]] | None, "data": {name: array} (observed data when no gen),
            "init": "prior" | {name: array}, "sweeps": n, "record": [names]}
    out = run_chain(spec)   # {"<gen output>", "<var>_init", "<var>" [n, ...], "lj" [n], "acc" [n]}
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _child(spec_path: str, out_path: str) -> None:
    sys.path.insert(0, ROOT)
    from oracle import Reference

    with open(spec_path) as f:
        spec = json.load(f)
    data = dict(np.load(spec_path + ".npz")) if os.path.exists(spec_path + ".npz") else {}
    R = Reference()
    out = {}
    t0 = time.time()
    gen = spec.get("gen")
    if gen:
        kind, args = gen
        if kind == "lda":
            M, V, K, L, s = args
            w, _, _ = R.gen_lda(M, V, K, L, s)
            out["w"] = data["w"] = w
        elif kind == "gmm":
            n, centers, stds, s = args
            out["x"] = data["x"] = R.gen_gmm(n, centers, stds, s)
        elif kind == "regression":
            n, k, noise, s = args
            x, y, wt, bt = R.gen_regression(n, k, noise, s)
            out["x"] = data["x"] = x
            out["y"] = data["y"] = y
        else:
            raise ValueError(kind)
    out["t_gen"] = np.array(time.time() - t0)
    e = R.open(spec["model"], spec["hyper"], spec.get("method", "gibbs"), spec["seed"], spec["threads"],
               spec.get("mh_scale", 0.5), spec.get("observe", ()))
    for name in spec.get("observed", []):
        e.set(name, data[name])
    init = spec["init"]
    if init == "prior":
        e.prior_init(spec["seed"])
    else:
        for name in init:
            e.set(name, data[name])
    rec = spec["record"]
    for name in rec:
        out[name + "_init"] = e.get(name)
    out["lj_init"] = np.array(e.log_joint())
    n = spec["sweeps"]
    hist = {name: [] for name in rec}
    lj, acc, ms = [], [], []
    for it in range(n):
        t = time.time()
        v, a = e.sweep(it)
        ms.append(1e3 * (time.time() - t))
        lj.append(v)
        acc.append(a)
        for name in rec:
            hist[name].append(e.get(name))
    for name in rec:
        out[name] = np.array(hist[name])
    out["lj"], out["acc"], out["ms"] = np.array(lj), np.array(acc), np.array(ms)
    e.close()
    np.savez(out_path, **out)


def run_chain(spec: dict, timeout: float = 900.0, data: dict | None = None) -> dict:
    threads = int(spec.get("threads", 1))
    attempts = [threads, threads, max(1, threads // 2), 1] if threads > 1 else [1]
    errors = []
    with tempfile.TemporaryDirectory() as d:
        sp, op = os.path.join(d, "spec.json"), os.path.join(d, "out.npz")
        if data:
            np.savez(sp + ".npz", **data)
        for th in attempts:
            s = dict(spec, threads=th)
            with open(sp, "w") as f:
                json.dump(s, f)
            try:
                r = subprocess.run([sys.executable, os.path.abspath(__file__), sp, op], cwd=ROOT,
                                   capture_output=True, text=True, timeout=timeout)
            except subprocess.TimeoutExpired:
                errors.append(f"threads={th}: timeout")
                continue
            if r.returncode == 0 and os.path.exists(op):
                res = dict(np.load(op))
                res["threads"] = th
                res["failed_attempts"] = errors
                return res
            errors.append(f"threads={th}: rc={r.returncode} {r.stderr[-300:]}")
    raise RuntimeError("reference chain failed: " + "; ".join(errors))


if __name__ == "__main__":
    _child(sys.argv[1], sys.argv[2])
