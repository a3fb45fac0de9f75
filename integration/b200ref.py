"""ctypes facade over integration/_build/libbnmc_b200ref.so -- the REFERENCE (its own
sources, patched by integration/reference_b200.patch) with the B200 backend behind its
Engine.  Used by tests/test_gpu_integration.py and bench.py to drive the reference's
public API (Engine, sample, map_estimate, lpp_curve) with RunConfig::device = Cpu or B200.
"""
from __future__ import annotations

import ctypes
import json
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_longlong, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libbnmc_b200ref.so")
CLI = os.path.join(HERE, "_build", "bnmc")

_ip, _dp = POINTER(c_int64), POINTER(c_double)

# variable names of the zoo models, declaration order (= the reference's var ids)
VARS = {"lda": ["phi", "theta", "z", "w"], "gmm": ["pi", "mu", "sigma2", "z", "x"],
        "regression": ["w", "b", "tau", "x", "y"], "catmix": ["theta", "phi", "z", "x"],
        "naivebayes": ["pC", "c", "pF", "f"], "hmm": ["T", "bias", "s", "flips"],
        "polyreg": ["w", "bias", "x", "y"], "regprec": ["w", "b", "tau", "x", "y"]}


class RefError(RuntimeError):
    pass


def build() -> None:
    import subprocess

    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


class B200Ref:
    def __init__(self, path: str = LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C integration` where /root/reference exists")
        L = self.lib = ctypes.CDLL(path)
        L.b2r_last_error.restype = c_char_p
        L.b2r_canonical_model.restype = c_char_p
        L.b2r_canonical_model.argtypes = [c_char_p]
        L.b2r_set_default_device.argtypes = [c_int]
        L.b2r_open.restype = c_void_p
        L.b2r_open.argtypes = [c_char_p, c_char_p, c_char_p, c_char_p, c_uint64, c_int, c_double, c_char_p, c_int,
                               c_longlong, c_longlong]
        L.b2r_close.argtypes = [c_void_p]
        L.b2r_on_device.argtypes = [c_void_p]
        L.b2r_var_info.argtypes = [c_void_p, c_char_p, _ip, _ip, POINTER(c_int), POINTER(c_int)]
        L.b2r_set.argtypes = [c_void_p, c_char_p, c_void_p, c_int64]
        L.b2r_get.argtypes = [c_void_p, c_char_p, c_void_p, c_int64]
        L.b2r_prior_init.argtypes = [c_void_p, c_uint64]
        L.b2r_sweep.argtypes = [c_void_p, c_int64, _dp, POINTER(c_int)]
        L.b2r_sweeps_timed.argtypes = [c_void_p, c_int64, c_int64, _dp, _dp]
        L.b2r_log_joint.argtypes = [c_void_p, _dp]
        L.b2r_run.argtypes = [c_void_p, c_longlong]
        L.b2r_sample.argtypes = [c_void_p, c_longlong]
        L.b2r_map_estimate.argtypes = [c_void_p, c_longlong, c_char_p]
        L.b2r_trace_info.argtypes = [c_void_p, _ip, _ip, _dp, POINTER(c_int)]
        L.b2r_trace_lj.argtypes = [c_void_p, _dp, _dp]
        L.b2r_trace_value.argtypes = [c_void_p, c_int64, c_char_p, c_void_p, c_int64]
        L.b2r_lpp_curve.argtypes = [c_void_p, _ip, _ip, c_int64, _ip, _ip, c_int64, c_longlong, c_uint64, c_int, _ip]
        L.b2r_lpp_point.argtypes = [c_void_p, c_int64, POINTER(c_longlong), _dp, _dp]

    def check(self, rc):
        if rc != 0:
            raise RefError(self.lib.b2r_last_error().decode())

    def canonical_model(self, name: str) -> str:
        s = self.lib.b2r_canonical_model(name.encode())
        if s is None:
            raise KeyError(name)
        return s.decode()

    def set_default_device(self, device: str):
        self.lib.b2r_set_default_device(1 if device == "b200" else 0)

    def open(self, model, hyper, method="gibbs", seed=0, threads=1, mh_scale=0.5, observe=(), device="b200",
             thin=1, burnin=0, source=None):
        return RefEngine(self, model, hyper, method, seed, threads, mh_scale, observe, device, thin, burnin, source)


class RefEngine:
    """One bnmc::Engine of the patched reference, with its own ParamStore."""

    def __init__(self, ref, model, hyper, method, seed, threads, mh_scale, observe, device, thin, burnin, source):
        self.ref, self.L = ref, ref.lib
        self.h = self.L.b2r_open(model.encode(), source.encode() if source else None, json.dumps(hyper).encode(),
                                 method.encode(), seed, threads, mh_scale, ",".join(observe).encode(),
                                 1 if device == "b200" else 0, thin, burnin)
        if not self.h:
            raise RefError(self.L.b2r_last_error().decode())
        self.names = VARS.get(model, [])

    def close(self):
        if self.h:
            self.L.b2r_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def on_device(self) -> bool:
        return bool(self.L.b2r_on_device(self.h))

    def info(self, name):
        i, n, isint, obs = c_int64(), c_int64(), c_int(), c_int()
        self.ref.check(self.L.b2r_var_info(self.h, name.encode(), ctypes.byref(i), ctypes.byref(n),
                                           ctypes.byref(isint), ctypes.byref(obs)))
        return i.value, n.value, bool(isint.value), bool(obs.value)

    def get(self, name):
        _, n, isint, _ = self.info(name)
        a = np.empty(n, dtype=np.int64 if isint else np.float64)
        self.ref.check(self.L.b2r_get(self.h, name.encode(), a.ctypes.data, n))
        return a

    def set(self, name, arr):
        _, n, isint, _ = self.info(name)
        a = np.ascontiguousarray(arr, dtype=np.int64 if isint else np.float64)
        self.ref.check(self.L.b2r_set(self.h, name.encode(), a.ctypes.data, n))

    def prior_init(self, seed):
        self.ref.check(self.L.b2r_prior_init(self.h, seed))

    def sweep(self, it):
        lj, acc = c_double(), c_int()
        self.ref.check(self.L.b2r_sweep(self.h, it, ctypes.byref(lj), ctypes.byref(acc)))
        return lj.value, bool(acc.value)

    def sweeps_timed(self, it0, n):
        lj, ms = np.empty(n), np.empty(n)
        self.ref.check(self.L.b2r_sweeps_timed(self.h, it0, n, lj.ctypes.data_as(_dp), ms.ctypes.data_as(_dp)))
        return lj, ms

    def log_joint(self):
        lj = c_double()
        self.ref.check(self.L.b2r_log_joint(self.h, ctypes.byref(lj)))
        return lj.value

    def run(self, n):
        self.ref.check(self.L.b2r_run(self.h, n))
        return self.trace()

    def sample(self, n):
        self.ref.check(self.L.b2r_sample(self.h, n))
        return self.trace()

    def map_estimate(self, n, observe=()):
        self.ref.check(self.L.b2r_map_estimate(self.h, n, ",".join(observe).encode()))

    def trace(self, names=None):
        nlj, ns, mlj, hm = c_int64(), c_int64(), c_double(), c_int()
        self.ref.check(self.L.b2r_trace_info(self.h, ctypes.byref(nlj), ctypes.byref(ns), ctypes.byref(mlj),
                                             ctypes.byref(hm)))
        lj, ms = np.empty(nlj.value), np.empty(nlj.value)
        self.L.b2r_trace_lj(self.h, lj.ctypes.data_as(_dp), ms.ctypes.data_as(_dp))
        out = {"log_joint": lj, "timing_ms": ms, "map_log_joint": mlj.value, "samples": [], "map_state": {}}
        latent = names if names is not None else [n for n in self.names if not self.info(n)[3]]
        for j in range(ns.value):
            out["samples"].append({v: self._trace_value(j, v) for v in latent})
        if hm.value:
            out["map_state"] = {v: self._trace_value(-1, v) for v in latent}
        return out

    def _trace_value(self, j, name):
        _, n, isint, _ = self.info(name)
        a = np.empty(n, dtype=np.int64 if isint else np.float64)
        self.ref.check(self.L.b2r_trace_value(self.h, j, name.encode(), a.ctypes.data, n))
        return a

    def lpp_curve(self, fit_w, fit_lengths, test_w, test_off, fit_sweeps, seed, threads=1):
        fw = np.ascontiguousarray(fit_w, dtype=np.int64)
        fl = np.ascontiguousarray(fit_lengths, dtype=np.int64)
        tw = np.ascontiguousarray(test_w, dtype=np.int64)
        to = np.ascontiguousarray(test_off, dtype=np.int64)
        cnt = c_int64()
        self.ref.check(self.L.b2r_lpp_curve(self.h, fw.ctypes.data_as(_ip), fl.ctypes.data_as(_ip), fl.size,
                                            tw.ctypes.data_as(_ip), to.ctypes.data_as(_ip), to.size - 1, fit_sweeps,
                                            seed, threads, ctypes.byref(cnt)))
        pts = []
        for i in range(cnt.value):
            s, l, sec = c_longlong(), c_double(), c_double()
            self.ref.check(self.L.b2r_lpp_point(self.h, i, ctypes.byref(s), ctypes.byref(l), ctypes.byref(sec)))
            pts.append({"samples": s.value, "lpp": l.value, "seconds": sec.value})
        return pts
