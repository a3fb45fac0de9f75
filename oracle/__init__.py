"""oracle -- TEST INFRASTRUCTURE ONLY: the CPU checkers for the CUDA sweep.

Two checkers, both CPU-only, both loaded through ctypes:

* ``Restatement`` -- ``oracle/liboracle.so``, the plain-C restatement of the
  reference hot path (``oracle/bnmc_oracle.c``; every function cites the
  reference file:line it follows).
* ``Reference``   -- ``oracle/_ref/libbnmc_ref.so``, the UNMODIFIED reference
  sampler compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``,
  driven through its own public API (parse/validate/prior_init/Engine::sweep).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference`` arm) may import this package.  The product package
``paper_1312_3613_b200`` never imports it and has no CPU fallback.
"""
from __future__ import annotations

import ctypes
import json
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libbnmc_ref.so")
REF_BENCH = os.path.join(HERE, "_ref", "ref_bench")

_dp = POINTER(c_double)
_ip = POINTER(c_int64)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def build(reference: bool = True) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    import subprocess

    targets = ["restatement"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def doc_offsets(lengths) -> np.ndarray:
    off = np.zeros(len(lengths) + 1, dtype=np.int64)
    off[1:] = np.cumsum(np.asarray(lengths, dtype=np.int64))
    return off


# --------------------------------------------------------------------------------------
# Restatement (liboracle.so)
# --------------------------------------------------------------------------------------
class _Lda(ctypes.Structure):
    _fields_ = [("K", c_int64), ("V", c_int64), ("M", c_int64), ("offsets", _ip), ("w", _ip),
                ("alpha", c_double), ("beta", c_double),
                ("var_phi", c_int32), ("var_theta", c_int32), ("var_z", c_int32)]


class _Gmm(ctypes.Structure):
    _fields_ = [("N", c_int64), ("K", c_int64), ("x", _dp), ("alpha", c_double),
                ("mu0", c_double), ("v0", c_double), ("a0", c_double), ("b0", c_double),
                ("var_pi", c_int32), ("var_mu", c_int32), ("var_sigma2", c_int32), ("var_z", c_int32)]


class _Mh(ctypes.Structure):
    _fields_ = [("N", c_int64), ("K", c_int64), ("x", _dp), ("y", _dp),
                ("lo", c_double), ("hi", c_double), ("w_var", c_double), ("b_var", c_double),
                ("tau_a", c_double), ("tau_b", c_double), ("mh_scale", c_double),
                ("var_w", c_int32), ("var_b", c_int32), ("var_tau", c_int32), ("logistic", c_int32)]


class OracleError(RuntimeError):
    pass


class Restatement:
    """ctypes facade over oracle/liboracle.so (see oracle/bnmc_oracle.h)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = self.lib = ctypes.CDLL(path)
        L.bo_last_error.restype = c_char_p
        for n, a in [("bo_mix", [c_uint64]), ("bo_fold", [c_uint64, c_uint64]),
                     ("bo_keyed", [c_uint64] * 5), ("bo_derive", [c_uint64] * 3)]:
            getattr(L, n).restype = c_uint64
            getattr(L, n).argtypes = a
        L.bo_draw_gamma.restype = c_double
        L.bo_draw_from_log_weights.restype = c_int64
        L.bo_lda_log_joint.restype = c_double
        L.bo_gmm_log_joint.restype = c_double
        L.bo_mh_log_joint.restype = c_double
        L.bo_mh_blanket.restype = c_double
        L.bo_lda_lpp.restype = c_double
        L.bo_log_pdf_dirichlet.restype = c_double

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.bo_last_error().decode())

    # -- rng / primitives --------------------------------------------------------------
    def keyed(self, seed, a=0, b=0, c=0, d=0) -> int:
        return self.lib.bo_keyed(seed, a, b, c, d)

    def derive(self, key, a, b=0) -> int:
        return self.lib.bo_derive(key, a, b)

    def draw_gamma(self, key: int, shape: float) -> float:
        class R(ctypes.Structure):
            _fields_ = [("key", c_uint64), ("counter", c_uint64)]
        r = R(key, 0)
        self.lib.bo_draw_gamma.argtypes = [POINTER(R), c_double]
        return self.lib.bo_draw_gamma(ctypes.byref(r), shape)

    # -- LDA ----------------------------------------------------------------------------
    def _lda(self, K, V, offsets, w, alpha=0.1, beta=0.1):
        return _Lda(K, V, len(offsets) - 1, _i(offsets), _i(w), alpha, beta, 0, 1, 2)

    def lda_prior_init(self, K, V, offsets, w, seed):
        M, N = len(offsets) - 1, int(offsets[-1])
        phi = np.empty(K * V); theta = np.empty(M * K); z = np.empty(N, dtype=np.int64)
        m = self._lda(K, V, offsets, w)
        self._check(self.lib.bo_lda_prior_init(ctypes.byref(m), c_uint64(seed), _d(phi), _d(theta), _i(z)))
        return phi, theta, z

    def lda_sweep(self, K, V, offsets, w, z, phi, theta, seed, it, observe_phi=False):
        """In place on (z, phi, theta); returns the post-sweep log-joint."""
        m = self._lda(K, V, offsets, w)
        lj = c_double()
        self._check(self.lib.bo_lda_sweep(ctypes.byref(m), _i(z), _d(phi), _d(theta), c_uint64(seed),
                                          c_int64(it), c_int(1 if observe_phi else 0), ctypes.byref(lj)))
        return lj.value

    def lda_log_joint(self, K, V, offsets, w, z, phi, theta):
        m = self._lda(K, V, offsets, w)
        return self.lib.bo_lda_log_joint(ctypes.byref(m), _i(z), _d(phi), _d(theta))

    def lda_count_phi(self, K, V, offsets, w, z, d0, d1):
        m = self._lda(K, V, offsets, w)
        nkw = np.zeros(K * V, dtype=np.int64)
        self._check(self.lib.bo_lda_count_phi(ctypes.byref(m), _i(z), c_int64(d0), c_int64(d1), _i(nkw)))
        return nkw

    def lda_draw_phi(self, K, V, offsets, w, nkw, seed, it):
        m = self._lda(K, V, offsets, w)
        phi = np.empty(K * V)
        self._check(self.lib.bo_lda_draw_phi(ctypes.byref(m), _i(nkw), c_uint64(seed), c_int64(it), _d(phi)))
        return phi

    def lda_phi_gammas(self, K, V, offsets, w, nkw, seed, it, v0, v1):
        """Unnormalised phi cells of vocabulary columns [v0, v1) (zeros elsewhere)."""
        m = self._lda(K, V, offsets, w)
        g = np.zeros(K * V)
        self._check(self.lib.bo_lda_phi_gammas(ctypes.byref(m), _i(nkw), c_uint64(seed), c_int64(it),
                                               c_int64(v0), c_int64(v1), _d(g)))
        return g

    def lda_theta_z(self, K, V, offsets, w, z, phi, theta, seed, it, d0, d1):
        m = self._lda(K, V, offsets, w)
        self._check(self.lib.bo_lda_theta_z(ctypes.byref(m), _i(z), _d(phi), _d(theta), c_uint64(seed),
                                            c_int64(it), c_int64(d0), c_int64(d1)))

    def lda_lpp(self, phi, theta, K, V, w, offsets):
        return self.lib.bo_lda_lpp(_d(phi), _d(theta), c_int64(K), c_int64(V), _i(w), _i(offsets),
                                   c_int64(len(offsets) - 1))

    # -- GMM ----------------------------------------------------------------------------
    def _gmm(self, x, K):
        return _Gmm(len(x), K, _d(x), 0.1, 0.0, 10.0, 1.0, 1.0, 0, 1, 2, 3)

    def gmm_prior_init(self, x, K, seed):
        pi = np.empty(K); mu = np.empty(K); s2 = np.empty(K); z = np.empty(len(x), dtype=np.int64)
        m = self._gmm(x, K)
        self._check(self.lib.bo_gmm_prior_init(ctypes.byref(m), c_uint64(seed), _d(pi), _d(mu), _d(s2), _i(z)))
        return pi, mu, s2, z

    def gmm_sweep(self, x, K, z, pi, mu, s2, seed, it):
        m = self._gmm(x, K)
        lj = c_double()
        self._check(self.lib.bo_gmm_sweep(ctypes.byref(m), _i(z), _d(pi), _d(mu), _d(s2), c_uint64(seed),
                                          c_int64(it), ctypes.byref(lj)))
        return lj.value

    # -- MH -----------------------------------------------------------------------------
    def _mh(self, x, y, K, logistic, mh_scale=0.5, lo=-1.0, hi=1.0):
        return _Mh(len(y), K, _d(x), _d(y), lo, hi, 10.0, 10.0, 3.0, 1.0, mh_scale, 0, 1, 2,
                   1 if logistic else 0)

    def mh_step(self, x, y, K, w, b, tau, seed, it, logistic=False, mh_scale=0.5):
        """In place on w; returns (b, tau, log_joint, accepted)."""
        m = self._mh(x, y, K, logistic, mh_scale)
        bb, tt, lj, acc = c_double(b), c_double(tau), c_double(), c_int()
        self._check(self.lib.bo_mh_step(ctypes.byref(m), _d(w), ctypes.byref(bb), ctypes.byref(tt),
                                        c_uint64(seed), c_int64(it), ctypes.byref(lj), ctypes.byref(acc)))
        return bb.value, tt.value, lj.value, bool(acc.value)

    def mh_log_joint(self, x, y, K, w, b, tau, logistic=False):
        m = self._mh(x, y, K, logistic)
        return self.lib.bo_mh_log_joint(ctypes.byref(m), _d(w), c_double(b), c_double(tau))


# --------------------------------------------------------------------------------------
# Compiled reference (oracle/_ref/libbnmc_ref.so)
# --------------------------------------------------------------------------------------
class Reference:
    """ctypes facade over the compiled, unmodified reference (oracle/ref_driver.cpp)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = ctypes.CDLL(path)
        L.bref_last_error.restype = c_char_p
        L.bref_open.restype = c_void_p
        L.bref_open.argtypes = [c_char_p, c_char_p, c_char_p, c_uint64, c_int, c_double, c_char_p]
        L.bref_close.argtypes = [c_void_p]
        L.bref_var_info.argtypes = [c_void_p, c_char_p, _ip, _ip, POINTER(c_int), POINTER(c_int)]
        for n, t in [("bref_set_real", _dp), ("bref_get_real", _dp), ("bref_set_int", _ip), ("bref_get_int", _ip)]:
            getattr(L, n).argtypes = [c_void_p, c_char_p, t, c_int64]
        L.bref_prior_init.argtypes = [c_void_p, c_uint64]
        L.bref_sweep.argtypes = [c_void_p, c_int64, _dp, POINTER(c_int)]
        L.bref_sweeps_timed.argtypes = [c_void_p, c_int64, c_int64, _dp, _dp]
        L.bref_log_joint.argtypes = [c_void_p, _dp]
        L.bref_describe.argtypes = [c_void_p, c_char_p, c_int64]
        L.bref_gen_lda.argtypes = [c_int64] * 5 + [c_uint64, _ip, _dp, _ip]
        L.bref_gen_gmm.argtypes = [c_int64, _dp, _dp, c_int64, c_uint64, _dp]
        L.bref_gen_regression.argtypes = [c_int64, c_int64, c_double, c_uint64, _dp, _dp, _dp, _dp]
        for n, a in [("bref_keyed", [c_uint64] * 5), ("bref_derive", [c_uint64] * 3)]:
            getattr(L, n).restype = c_uint64
            getattr(L, n).argtypes = a
        L.bref_stream_u64.argtypes = [c_uint64, c_int64, POINTER(c_uint64)]
        L.bref_stream_unit.argtypes = [c_uint64, c_int64, _dp]
        L.bref_stream_gaussian.argtypes = [c_uint64, c_int64, _dp]
        L.bref_draw_gamma.restype = c_double
        L.bref_draw_gamma.argtypes = [c_uint64, c_double, POINTER(c_uint64)]
        L.bref_draw_from_log_weights.restype = c_int64
        L.bref_draw_from_log_weights.argtypes = [c_uint64, _dp, c_int64]
        L.bref_dirichlet_batch.argtypes = [c_int64, c_int64, _dp, c_int, c_uint64, c_int, c_int, _dp]
        L.bref_log_pdf_dirichlet.restype = c_double
        L.bref_log_pdf_dirichlet.argtypes = [_dp, _dp, c_int64]
        L.bref_lpp.argtypes = [_dp, _dp, c_int64, c_int64, _ip, _ip, c_int64, _dp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.bref_last_error().decode())

    # -- generators ---------------------------------------------------------------------
    def gen_lda(self, docs, vocab, topics, length, seed, heldout=0):
        w = np.empty(docs * length, dtype=np.int64)
        phi = np.empty(topics * vocab)
        wh = np.empty(max(heldout * length, 1), dtype=np.int64)
        self._check(self.lib.bref_gen_lda(docs, vocab, topics, length, heldout, seed, _i(w), _d(phi), _i(wh)))
        return w, phi, wh[: heldout * length]

    def gen_gmm(self, n, centers, stds, seed):
        c = np.asarray(centers, dtype=np.float64); s = np.asarray(stds, dtype=np.float64)
        x = np.empty(n)
        self._check(self.lib.bref_gen_gmm(n, _d(c), _d(s), len(c), seed, _d(x)))
        return x

    def gen_regression(self, n, k, noise_var, seed):
        x = np.empty(n * k); y = np.empty(n); w = np.empty(k); b = c_double()
        self._check(self.lib.bref_gen_regression(n, k, noise_var, seed, _d(x), _d(y), _d(w), ctypes.byref(b)))
        return x, y, w, b.value

    # -- engine -------------------------------------------------------------------------
    def open(self, model: str, hyper: dict, method: str = "gibbs", seed: int = 0, threads: int = 1,
             mh_scale: float = 0.5, observe=()):
        return RefEngine(self, model, hyper, method, seed, threads, mh_scale, observe)

    def keyed(self, seed, a=0, b=0, c=0, d=0):
        return self.lib.bref_keyed(seed, a, b, c, d)

    def derive(self, key, a, b=0):
        return self.lib.bref_derive(key, a, b)


class RefEngine:
    def __init__(self, ref: Reference, model, hyper, method, seed, threads, mh_scale, observe):
        self.ref, self.L = ref, ref.lib
        self.h = self.L.bref_open(model.encode(), json.dumps(hyper).encode(), method.encode(), seed,
                                  threads, mh_scale, ",".join(observe).encode())
        if not self.h:
            raise OracleError(self.L.bref_last_error().decode())

    def close(self):
        if self.h:
            self.L.bref_close(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def info(self, name):
        i, n, isint, obs = c_int64(), c_int64(), c_int(), c_int()
        self.ref._check(self.L.bref_var_info(self.h, name.encode(), ctypes.byref(i), ctypes.byref(n),
                                             ctypes.byref(isint), ctypes.byref(obs)))
        return i.value, n.value, bool(isint.value), bool(obs.value)

    def get(self, name):
        _, n, isint, _ = self.info(name)
        if isint:
            a = np.empty(n, dtype=np.int64)
            self.ref._check(self.L.bref_get_int(self.h, name.encode(), _i(a), n))
        else:
            a = np.empty(n)
            self.ref._check(self.L.bref_get_real(self.h, name.encode(), _d(a), n))
        return a

    def set(self, name, arr):
        _, n, isint, _ = self.info(name)
        if isint:
            a = np.ascontiguousarray(arr, dtype=np.int64)
            self.ref._check(self.L.bref_set_int(self.h, name.encode(), _i(a), n))
        else:
            a = np.ascontiguousarray(arr, dtype=np.float64)
            self.ref._check(self.L.bref_set_real(self.h, name.encode(), _d(a), n))

    def prior_init(self, seed):
        self.ref._check(self.L.bref_prior_init(self.h, seed))

    def sweep(self, it):
        lj, acc = c_double(), c_int()
        self.ref._check(self.L.bref_sweep(self.h, it, ctypes.byref(lj), ctypes.byref(acc)))
        return lj.value, bool(acc.value)

    def log_joint(self):
        lj = c_double()
        self.ref._check(self.L.bref_log_joint(self.h, ctypes.byref(lj)))
        return lj.value

    def describe(self):
        buf = ctypes.create_string_buffer(1 << 16)
        self.ref._check(self.L.bref_describe(self.h, buf, len(buf)))
        return buf.value.decode()
