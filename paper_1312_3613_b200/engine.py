"""Python host layer over the C-ABI (include/bnmc_gpu.h) -- mirrors the reference's
sampler API (proj/include/bnmc/sampler.hpp) for the models the GPU path serves.

Reference name            -> here
  RunConfig (:14-22)          RunConfig
  ParamStore (store.hpp:74)   ParamStore (flat arrays per variable id + observed mask)
  Engine (:45-86)             Engine: sweep / run / eval_log_joint / allocate
  prior_init (:97-99)         Engine.prior_init (on the device)
  sample (:103-104)           sample
  map_estimate (:108-110)     map_estimate
  RuntimeError (store.hpp:14) RuntimeError (also std::domain_error -> DomainError,
                              std::invalid_argument -> ValueError)

Every call runs on the GPU through libbnmc_gpu.so; there is no CPU path.  If the
library is missing or no CUDA device exists, construction raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNMC_GPU_LIB") or os.path.join(HERE, "libbnmc_gpu.so")
ABI_VERSION = 2

LDA, GMM, MH_LINREG, MH_LOGREG, CATMIX, NAIVEBAYES, HMM, MH_POLYREG = 1, 2, 3, 4, 5, 6, 7, 8
OBSERVE_PHI, EXACT_WEIGHTS, NO_GRAPH, GIBBS, MWG, TAU_PRECISION = 1, 2, 4, 8, 16, 32


class BnmcError(RuntimeError):
    """Base of the errors raised from C-ABI status codes."""


class DomainError(BnmcError, ArithmeticError):
    """std::domain_error in the reference (e.g. all candidate log-weights -inf)."""


class CudaError(BnmcError):
    pass


class _Desc(ctypes.Structure):
    _fields_ = [("abi_version", c_int32), ("kind", c_int32), ("seed", c_uint64), ("device", c_int32),
                ("flags", c_uint32), ("K", c_int64), ("V", c_int64), ("M", c_int64), ("N", c_int64),
                ("doc_offsets", POINTER(c_int64)), ("hyper", c_double * 8), ("var_ids", c_int32 * 8),
                ("mh_scale", c_double), ("rank", c_int32), ("world_size", c_int32),
                ("nccl_id", c_void_p), ("stream", c_void_p), ("group", c_void_p)]


class _Store(ctypes.Structure):
    _fields_ = [("n_vars", c_int32), ("real", POINTER(POINTER(c_double))), ("ival", POINTER(POINTER(c_int64))),
                ("len", POINTER(c_int64)), ("observed", POINTER(c_char))]


class _Trace(ctypes.Structure):
    _fields_ = [("burnin", c_int64), ("n", c_int64), ("thin", c_int64), ("log_joints", POINTER(c_double)),
                ("timing_ms", POINTER(c_double)), ("accepted", POINTER(c_int)), ("samples", POINTER(_Store)),
                ("map_state", POINTER(_Store)), ("map_log_joint", POINTER(c_double))]


_lib = None


def lib():
    """Load libbnmc_gpu.so (built in-tree by paper_1312_3613_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1312_3613_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.bnmc_gpu_abi_version.restype = c_int
    L.bnmc_gpu_last_error.restype = c_char_p
    L.bnmc_gpu_last_error.argtypes = [c_void_p]
    L.bnmc_gpu_create.argtypes = [POINTER(_Desc), POINTER(c_void_p)]
    L.bnmc_gpu_destroy.argtypes = [c_void_p]
    L.bnmc_gpu_upload.argtypes = [c_void_p, POINTER(_Store)]
    L.bnmc_gpu_upload_state.argtypes = [c_void_p, POINTER(_Store)]
    L.bnmc_gpu_upload_sweep_inputs.argtypes = [c_void_p, POINTER(_Store)]
    L.bnmc_gpu_sweep_store.argtypes = [c_void_p, POINTER(_Store), c_int64, POINTER(c_double), POINTER(c_int)]
    L.bnmc_gpu_transfer_stats.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_int64)]
    L.bnmc_gpu_sweep_phases.argtypes = [c_void_p, c_int64, POINTER(c_double), POINTER(c_char_p), c_int,
                                        POINTER(c_int)]
    L.bnmc_gpu_nccl_unique_id.argtypes = [c_void_p]
    L.bnmc_gpu_group_create.argtypes = [c_int32, POINTER(c_void_p)]
    L.bnmc_gpu_group_destroy.argtypes = [c_void_p]
    L.bnmc_gpu_register_host.argtypes = [c_void_p, POINTER(_Store)]
    L.bnmc_gpu_unregister_host.argtypes = [c_void_p]
    L.bnmc_gpu_download.argtypes = [c_void_p, POINTER(_Store)]
    L.bnmc_gpu_sweep.argtypes = [c_void_p, c_int64, POINTER(c_double), POINTER(c_int)]
    L.bnmc_gpu_run.argtypes = [c_void_p, c_int64, c_int64, POINTER(c_double), POINTER(c_int)]
    L.bnmc_gpu_enqueue.argtypes = [c_void_p, c_int64, c_int64]
    L.bnmc_gpu_run_trace.argtypes = [c_void_p, c_int64, POINTER(_Trace)]
    L.bnmc_gpu_synchronize.argtypes = [c_void_p, POINTER(c_double), POINTER(c_int)]
    L.bnmc_gpu_eval_log_joint.argtypes = [c_void_p, POINTER(c_double)]
    L.bnmc_gpu_prior_init.argtypes = [c_void_p, c_uint64]
    L.bnmc_gpu_lda_counts.argtypes = [c_void_p, POINTER(c_int32), POINTER(c_int32)]
    L.bnmc_gpu_lda_generate.argtypes = [c_void_p, c_uint64, c_double, c_double]
    L.bnmc_gpu_save_checkpoint.argtypes = [c_void_p, c_char_p]
    L.bnmc_gpu_load_checkpoint.argtypes = [c_void_p, c_char_p]
    L.bnmc_gpu_checkpoint_iter.argtypes = [c_void_p, POINTER(c_int64)]
    L.bnmc_gpu_lda_load_corpus.argtypes = [c_void_p, c_char_p]
    L.bnmc_gpu_partition.argtypes = [POINTER(c_int64), c_int64, c_int32, c_int32, POINTER(c_int64), POINTER(c_int64)]
    L.bnmc_gpu_lpp.argtypes = [POINTER(c_double), POINTER(c_double), c_int64, c_int64, POINTER(c_int64),
                               POINTER(c_int64), c_int64, POINTER(c_double)]
    L.bnmc_gpu_dirichlet_batch.argtypes = [c_int64, c_int64, POINTER(c_double), c_uint64, POINTER(c_double)]
    L.bnmc_gpu_probe_rng.argtypes = [POINTER(c_uint64), c_int64, c_int64, POINTER(c_uint64), POINTER(c_double),
                                     POINTER(c_double)]
    L.bnmc_gpu_probe_gamma.argtypes = [POINTER(c_uint64), POINTER(c_double), c_int64, POINTER(c_double),
                                       POINTER(c_uint64)]
    L.bnmc_gpu_probe_read_bandwidth.argtypes = [c_int64, c_int32, POINTER(c_double)]
    L.bnmc_gpu_probe_log_weights.argtypes = [POINTER(c_uint64), POINTER(c_double), c_int64, c_int64,
                                             POINTER(c_int64)]
    if L.bnmc_gpu_abi_version() != ABI_VERSION:
        raise ImportError("libbnmc_gpu.so ABI version mismatch")
    _lib = L
    return L


def _raise(rc: int, ctx=None):
    if rc == 0:
        return
    msg = lib().bnmc_gpu_last_error(ctx).decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise DomainError(msg)
    if rc == 4:
        raise CudaError(msg)
    raise BnmcError(msg)


def _p(a, t):
    return a.ctypes.data_as(POINTER(t)) if a is not None else None


# --------------------------------------------------------------------------------------
# Models the GPU path serves: variable names in declaration order (= reference var ids).
# --------------------------------------------------------------------------------------
MODELS = {
    "lda": dict(kind=LDA, method="gibbs", vars=["phi", "theta", "z", "w"], ints={"z", "w"},
                observed={"w"}),
    "gmm": dict(kind=GMM, method="gibbs", vars=["pi", "mu", "sigma2", "z", "x"], ints={"z"},
                observed={"x"}),
    "regression": dict(kind=MH_LINREG, method="mh", vars=["w", "b", "tau", "x", "y"], ints=set(),
                       observed={"x", "y"}),
    # regression with a Gamma-distributed noise PRECISION, y ~ N(mean, pow(tau, -1))
    # (oracle/models/regprec.bn): the GammaPrecision conjugate kind
    "regprec": dict(kind=MH_LINREG, method="mh", vars=["w", "b", "tau", "x", "y"], ints=set(),
                    observed={"x", "y"}, flags=TAU_PRECISION),
    "logreg": dict(kind=MH_LOGREG, method="mh", vars=["w", "b", "x", "y"], ints=set(), observed={"x", "y"}),
    # the rest of the reference zoo
    "catmix": dict(kind=CATMIX, method="gibbs", vars=["theta", "phi", "z", "x"], ints={"z", "x"},
                   observed={"x"}),
    "naivebayes": dict(kind=NAIVEBAYES, method="gibbs", vars=["pC", "c", "pF", "f"], ints={"c", "f"},
                       observed={"c", "f"}),
    "hmm": dict(kind=HMM, method="gibbs", vars=["T", "bias", "s", "flips"], ints={"s", "flips"},
                observed={"flips"}),
    "polyreg": dict(kind=MH_POLYREG, method="mh", vars=["w", "bias", "x", "y"], ints=set(), observed={"x", "y"}),
}


@dataclass
class RunConfig:
    """proj/include/bnmc/sampler.hpp:14-22 (threads is accepted and ignored: the GPU grid
    replaces the worker pool)."""
    method: str = ""
    seed: int = 0
    threads: int = 1
    thin: int = 1
    burnin: int = 0
    mh_scale: float = 0.5
    observe_extra: list = field(default_factory=list)
    exact_weights: bool = False   # LDA: reference log-space weights instead of theta*phi
    device: int = -1
    use_graph: bool = True
    # page-lock the bound store's arrays once per binding (bnmc_gpu_register_host), as
    # the reference-side adapter does for its std::vector store (integration/): the
    # per-call copies then run at pinned-memory speed from the caller's own arrays
    pin_host: bool = True


def layout_lengths(model: str, hyper: dict) -> dict:
    """Flat length of every variable (VarLayout::flat_values, eval.cpp:91-136)."""
    if model == "lda":
        K, V, M = int(hyper["K"]), int(hyper["V"]), int(hyper["M"])
        N = int(np.sum(np.asarray(hyper["N"], dtype=np.int64))) if M else 0
        return {"phi": K * V, "theta": M * K, "z": N, "w": N}
    if model == "gmm":
        N, K = int(hyper["N"]), int(hyper["K"])
        return {"pi": K, "mu": K, "sigma2": K, "z": N, "x": N}
    if model == "catmix":
        N, K, V = int(hyper["N"]), int(hyper["K"]), int(hyper["V"])
        return {"theta": K * V, "phi": K, "z": N, "x": N}
    if model == "naivebayes":
        N, K = int(hyper["N"]), int(hyper["K"])
        return {"pC": 1, "c": N, "pF": 2 * K, "f": N * K}
    if model == "hmm":
        N, S = int(hyper["N"]), int(hyper["S"])
        return {"T": S * S, "bias": S, "s": N, "flips": N}
    if model == "polyreg":
        N, M = int(hyper["N"]), int(hyper["M"])
        return {"w": M, "bias": 1, "x": N, "y": N}
    if model in ("regression", "regprec", "logreg"):
        N, K = int(hyper["N"]), int(hyper["K"])
        d = {"w": K, "b": 1, "x": N * K, "y": N}
        if model in ("regression", "regprec"):
            d["tau"] = 1
        return d
    raise ValueError(f"model '{model}' has no GPU path")


class ParamStore:
    """Flat typed arrays per variable id + the observed mask (store.hpp:74-83)."""

    def __init__(self, model: str, hyper: dict):
        spec = MODELS[model]
        self.model = model
        self.names = list(spec["vars"])
        lens = layout_lengths(model, hyper)
        self.arrays = {}
        for n in self.names:
            dt = np.int64 if n in spec["ints"] else np.float64
            self.arrays[n] = np.zeros(lens[n], dtype=dt)
        self.observed = {n: (n in spec["observed"]) for n in self.names}

    def __getitem__(self, name):
        return self.arrays[name]

    def __setitem__(self, name, value):
        a = self.arrays[name]
        v = np.array(value, dtype=a.dtype, copy=True).reshape(-1)  # the store owns its arrays
        if v.shape != a.shape:
            raise BnmcError(f"variable '{name}' has flat length {v.size}, expected {a.size}")
        self.arrays[name] = v

    def copy(self):
        s = object.__new__(ParamStore)
        s.model, s.names = self.model, list(self.names)
        s.arrays = {k: v.copy() for k, v in self.arrays.items()}
        s.observed = dict(self.observed)
        return s

    def _latent_copy(self):
        """A store for the engine to write a snapshot into: fresh (uninitialised) arrays
        for the unobserved variables, the observed arrays shared (the engine never writes
        observed variables)."""
        s = ParamStore.__new__(ParamStore)
        s.__dict__.update({k: v for k, v in self.__dict__.items() if k not in ("arrays", "observed", "_vcache")})
        s.arrays = {k: (v if self.observed[k] else np.empty_like(v)) for k, v in self.arrays.items()}
        s.observed = dict(self.observed)
        return s

    def _view(self):
        # cached per array identity (an array object's buffer and layout never change) and
        # observed mask; the cache holds the arrays, so an id cannot be reused by a
        # replacement while the cached view points at the old one (~30 us per call saved
        # on every Engine.sweep)
        c = self.__dict__.get("_vcache")
        if c is not None:
            arrs, obs, st = c
            a = self.arrays
            if all(a[n] is x for n, x in zip(self.names, arrs)) and obs == tuple(self.observed[n] for n in self.names):
                return st
        st = self._build_view()  # (may replace non-contiguous arrays by contiguous copies)
        self._vcache = (tuple(self.arrays[n] for n in self.names), tuple(self.observed[n] for n in self.names), st)
        return st

    def _build_view(self):
        n = len(self.names)
        real = (POINTER(c_double) * n)()
        ival = (POINTER(c_int64) * n)()
        lens = (c_int64 * n)()
        obs = (c_char * n)()
        for i, name in enumerate(self.names):
            a = self.arrays[name]
            if not a.flags["C_CONTIGUOUS"]:
                a = self.arrays[name] = np.ascontiguousarray(a)
            lens[i] = a.size
            obs[i] = b"\x01" if self.observed[name] else b"\x00"
            if a.dtype == np.int64:
                ival[i] = a.ctypes.data_as(POINTER(c_int64))
            else:
                real[i] = a.ctypes.data_as(POINTER(c_double))
        st = _Store(n, real, ival, lens, obs)
        st._keep = (real, ival, lens, obs)
        return st


def write_corpus(path: str, offsets, w, V: int):
    """The binary LDA corpus format of bnmc_gpu_lda_load_corpus (include/bnmc_gpu.h)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    ww = np.ascontiguousarray(w, dtype=np.int32)
    if off[0] != 0 or off[-1] != ww.size:
        raise BnmcError("offsets must run from 0 to len(w)")
    with open(path, "wb") as f:
        f.write(b"BNMCCORP")
        f.write(np.array([1, 0], dtype=np.uint32).tobytes())
        f.write(np.array([off.size - 1, ww.size, V], dtype=np.int64).tobytes())
        f.write(off.tobytes())
        f.write(ww.tobytes())


def read_bandwidth(nbytes: int, reps: int = 20) -> float:
    """Device read bandwidth in GB/s over an `nbytes` buffer (bnmc_gpu_probe_read_bandwidth)."""
    out = c_double()
    _raise(lib().bnmc_gpu_probe_read_bandwidth(int(nbytes), int(reps), ctypes.byref(out)))
    return out.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _raise(lib().bnmc_gpu_nccl_unique_id(buf))
    return buf.raw


class PeerGroup:
    """A single-process peer group (bnmc_gpu_group): `world` Engines created with
    group=this share collectives over our own peer-memory all-reduce instead of NCCL --
    one host thread per rank (each rank's calls from its own thread), the ranks on one
    GPU or one GPU each.  Keep the group alive while its engines live."""

    def __init__(self, world: int):
        h = c_void_p()
        _raise(lib().bnmc_gpu_group_create(int(world), ctypes.byref(h)))
        self._h, self.world = h, int(world)

    def close(self):
        if getattr(self, "_h", None):
            lib().bnmc_gpu_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition(doc_offsets, world: int, rank: int):
    """Documents [begin, end) owned by `rank` (bnmc_gpu_partition)."""
    off = np.ascontiguousarray(doc_offsets, dtype=np.int64)
    b, e = c_int64(), c_int64()
    _raise(lib().bnmc_gpu_partition(_p(off, c_int64), len(off) - 1, world, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


class Engine:
    """GPU twin of bnmc::Engine (sampler.hpp:45-86) for LDA / GMM Gibbs and MH regression."""

    def __init__(self, model: str, hyper: dict, cfg: RunConfig | None = None, *, rank: int = 0,
                 world_size: int = 1, nccl_id: bytes | None = None, stream: int | None = None,
                 group: PeerGroup | None = None):
        if model not in MODELS:
            raise ValueError(f"model '{model}' has no GPU path (supported: {sorted(MODELS)})")
        self.model, self.hyper = model, dict(hyper)
        self.cfg = cfg or RunConfig()
        spec = MODELS[model]
        method = self.cfg.method or spec["method"]
        # regression.bn / polyreg.bn also run their Gibbs plan (an MH block per variable,
        # conjugate tau) and their MWG plan (single-site blocks): BNMC_GPU_GIBBS / _MWG
        methods = {spec["method"], "gibbs", "mwg"} if model in ("regression", "regprec", "polyreg") else {spec["method"]}
        if method not in methods:
            raise ValueError(f"the GPU path runs {model} with method {sorted(methods)}, not '{method}'")
        self.method = method
        self.spec = spec
        L = lib()
        d = _Desc()
        d.abi_version = ABI_VERSION
        d.kind = spec["kind"]
        d.seed = self.cfg.seed
        d.device = self.cfg.device
        flags = 0
        observe = set(self.cfg.observe_extra)
        unknown = observe - set(spec["vars"])
        if unknown:
            raise BnmcError(f"cannot observe unknown variable '{sorted(unknown)[0]}'")
        # The device sweeps implement the reference plans of the served models plus one
        # clamped latent variable: LDA's phi (the lpp protocol, bench.cpp:30-77).  Any
        # other observe_extra entry would change the plan (plan.cpp drops observed
        # variables from the blocks) and is refused instead of silently resampled.
        clampable = set(spec["observed"]) | ({"phi"} if model == "lda" else set())
        unsupported = observe - clampable
        if unsupported:
            raise ValueError(f"observe_extra {sorted(unsupported)} is not supported on the GPU path for '{model}' "
                             f"(clampable: {sorted(clampable)})")
        if model == "lda" and "phi" in observe:
            flags |= OBSERVE_PHI
        if self.cfg.exact_weights:
            flags |= EXACT_WEIGHTS
        if not self.cfg.use_graph:
            flags |= NO_GRAPH
        if method == "gibbs" and spec["method"] == "mh":
            flags |= GIBBS
        if method == "mwg":
            flags |= MWG
        flags |= spec.get("flags", 0)
        d.flags = flags
        self._offsets = None
        if model == "lda":
            K, V, M = int(hyper["K"]), int(hyper["V"]), int(hyper["M"])
            lengths = np.asarray(hyper["N"], dtype=np.int64).reshape(-1)
            if lengths.size != M:
                raise BnmcError("hyperparameter N must have M entries")
            off = np.zeros(M + 1, dtype=np.int64)
            off[1:] = np.cumsum(lengths)
            self._offsets = off
            d.K, d.V, d.M, d.N = K, V, M, int(off[-1])
            d.doc_offsets = _p(off, c_int64)
            d.hyper[0], d.hyper[1] = float(hyper.get("alpha", 0.1)), float(hyper.get("beta", 0.1))
        elif model == "gmm":
            d.K, d.N = int(hyper["K"]), int(hyper["N"])
            for i, v in enumerate([hyper.get("alpha", 0.1), hyper.get("mu0", 0.0), hyper.get("v0", 10.0),
                                   hyper.get("a0", 1.0), hyper.get("b0", 1.0)]):
                d.hyper[i] = float(v)
        elif model == "catmix":
            d.K, d.V, d.N = int(hyper["K"]), int(hyper["V"]), int(hyper["N"])
            d.hyper[0], d.hyper[1] = float(hyper.get("alpha", 0.5)), float(hyper.get("beta", 0.5))
        elif model == "naivebayes":
            d.K, d.N = int(hyper["K"]), int(hyper["N"])
        elif model == "hmm":
            d.K, d.N = int(hyper["S"]), int(hyper["N"])
            d.hyper[0] = float(hyper.get("v", 0.1))
        elif model == "polyreg":
            d.K, d.N = int(hyper["M"]), int(hyper["N"])
            for i, v in enumerate([0.0, 2.0, 1.0, 1.0]):
                d.hyper[i] = v
        else:
            d.K, d.N = int(hyper["K"]), int(hyper["N"])
            for i, v in enumerate([hyper.get("l", -1.0), hyper.get("u", 1.0), hyper.get("w_var", 10.0),
                                   hyper.get("b_var", 10.0), hyper.get("tau_a", 3.0), hyper.get("tau_b", 1.0)]):
                d.hyper[i] = float(v)
        for i in range(len(spec["vars"])):
            d.var_ids[i] = i
        d.mh_scale = self.cfg.mh_scale
        d.rank, d.world_size = rank, world_size
        self._rank, self._world = rank, world_size
        self._nccl = None
        self._group = group
        if group is not None:
            if group.world != world_size:
                raise ValueError("the peer group's world size differs from world_size")
            d.group = group._h
        elif world_size > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("world_size > 1 needs a 128-byte ncclUniqueId or a PeerGroup")
            self._nccl = ctypes.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = ctypes.cast(self._nccl, c_void_p)
        d.stream = stream
        h = c_void_p()
        _raise(L.bnmc_gpu_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._bound = None  # the ParamStore whose state is on the device
        self._registered = None  # the store view whose arrays are page-locked
        self._registered_arrays = None

    # -- lifetime -----------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().bnmc_gpu_unregister_host(self._h)
            self._registered = self._registered_arrays = None
            lib().bnmc_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- reference API ------------------------------------------------------------------
    def allocate(self) -> ParamStore:
        """Zero-initialised store with the layouts' shapes (Engine::allocate)."""
        s = ParamStore(self.model, self.hyper)
        for n in self.cfg.observe_extra:
            s.observed[n] = True
        return s

    def _register(self, store: ParamStore, st):
        # once per view (the view is cached per array identity: a replaced array builds a
        # new view, which re-registers; ranges no longer bound are released by the C side).
        # The registered arrays are kept alive until then: numpy must not free page-locked
        # memory under the driver.
        if self.cfg.pin_host and self._registered is not st:
            _raise(lib().bnmc_gpu_register_host(self._h, ctypes.byref(st)), self._h)
            self._registered = st
            self._registered_arrays = tuple(store.arrays.values())

    def upload(self, store: ParamStore):
        st = store._view()
        self._register(store, st)
        _raise(lib().bnmc_gpu_upload(self._h, ctypes.byref(st)), self._h)
        self._bound = store

    def upload_state(self, store: ParamStore):
        """Latent variables only; the observed data stays as bound (bnmc_gpu_upload_state)."""
        st = store._view()
        _raise(lib().bnmc_gpu_upload_state(self._h, ctypes.byref(st)), self._h)
        self._bound = store

    def download(self, store: ParamStore):
        st = store._view()
        _raise(lib().bnmc_gpu_download(self._h, ctypes.byref(st)), self._h)

    def prior_init(self, store: ParamStore, seed: int):
        """prior_init(skip_observed=True) on the device, then written back into `store`."""
        self.upload(store)
        _raise(lib().bnmc_gpu_prior_init(self._h, seed), self._h)
        self.download(store)

    def sweep(self, store: ParamStore, it: int, mh_accepted: list | None = None) -> float:
        """Engine::sweep: the store is advanced in place; returns the post-sweep log-joint.

        Borrow semantics of the reference: the caller's latent state is read on every
        call (the caller may have changed it) and written back after the sweep; the
        observed data is uploaded once per bound store."""
        lj, acc = c_double(), c_int()
        if self._bound is not store:
            self.upload(store)
            _raise(lib().bnmc_gpu_sweep(self._h, it, ctypes.byref(lj), ctypes.byref(acc)), self._h)
            self.download(store)
        else:
            # upload what the sweep reads, sweep, write back (phi / theta copies overlap
            # the z-step): bnmc_gpu_sweep_store
            st = store._view()
            self._register(store, st)
            _raise(lib().bnmc_gpu_sweep_store(self._h, ctypes.byref(st), it, ctypes.byref(lj), ctypes.byref(acc)),
                   self._h)
        if mh_accepted is not None:
            mh_accepted.append(bool(acc.value))
        return lj.value

    def transfer_stats(self) -> tuple[int, int]:
        """(host->device, device->host) bytes of the last bound-store sweep call."""
        up, down = c_int64(), c_int64()
        _raise(lib().bnmc_gpu_transfer_stats(self._h, ctypes.byref(up), ctypes.byref(down)), self._h)
        return up.value, down.value

    def sweep_device(self, it: int):
        """One sweep on the device-resident state (no host copies); returns (lj, accepted)."""
        lj, acc = c_double(), c_int()
        _raise(lib().bnmc_gpu_sweep(self._h, it, ctypes.byref(lj), ctypes.byref(acc)), self._h)
        return lj.value, bool(acc.value)

    def run_device(self, it0: int, n: int):
        """n sweeps it0..it0+n-1 with one host sync; returns (log_joints, accepted)."""
        lj = np.empty(n)
        acc = np.empty(n, dtype=np.int32)
        _raise(lib().bnmc_gpu_run(self._h, it0, n, _p(lj, c_double), _p(acc, c_int)), self._h)
        return lj, acc.astype(bool)

    def enqueue(self, it0: int, n: int):
        _raise(lib().bnmc_gpu_enqueue(self._h, it0, n), self._h)

    def synchronize(self):
        lj, acc = c_double(), c_int()
        _raise(lib().bnmc_gpu_synchronize(self._h, ctypes.byref(lj), ctypes.byref(acc)), self._h)
        return lj.value, bool(acc.value)

    def sweep_phases(self, it: int):
        """One sweep launched phase by phase with CUDA events: [(phase, ms), ...]."""
        ms = (c_double * 32)()
        names = (c_char_p * 32)()
        n = c_int()
        _raise(lib().bnmc_gpu_sweep_phases(self._h, it, ms, names, 32, ctypes.byref(n)), self._h)
        return [(names[i].decode(), ms[i]) for i in range(n.value)]

    def eval_log_joint(self, store: ParamStore | None = None) -> float:
        """Engine::eval_log_joint(store): the store's current state (re-read every call, as
        the reference does; without a store: the device state)."""
        if store is not None:
            if self._bound is not store:
                self.upload(store)
            else:
                self.upload_state(store)  # the caller may have changed its latent state
        lj = c_double()
        _raise(lib().bnmc_gpu_eval_log_joint(self._h, ctypes.byref(lj)), self._h)
        return lj.value

    def run(self, store: ParamStore, n: int) -> dict:
        """Engine::run (sampler.cpp:426-455): burn-in + n kept sweeps, thinned samples,
        MAP state, per-sweep log-joints and timings -- through bnmc_gpu_run_trace, which
        keeps the MAP state on the device (no host round trip per sweep); only the
        thinned samples are downloaded as they are taken."""
        if self._bound is not store:
            self.upload(store)
        else:
            self.upload_state(store)  # the chain starts from the store's current state
        cfg = self.cfg
        if n < 0 or cfg.thin < 1:
            raise BnmcError("run needs n >= 0 and thin >= 1")
        unobs = [v for v in store.names if not store.observed[v]]
        n_samples = (n + cfg.thin - 1) // cfg.thin
        samples = [store._latent_copy() for _ in range(n_samples)]
        map_store = store._latent_copy()
        views = (_Store * max(n_samples, 1))()
        keep = []
        for i, smp in enumerate(samples):
            v = smp._view()
            views[i] = v
            keep.append(v)
        mv = map_store._view()
        lj = np.full(max(n, 1), np.nan)
        tm = np.zeros(max(n, 1))
        acc = np.zeros(max(n, 1), dtype=np.int32)
        map_lj = c_double(-np.inf)
        tr = _Trace(cfg.burnin, n, cfg.thin, _p(lj, c_double), _p(tm, c_double), _p(acc, c_int),
                    ctypes.cast(views, POINTER(_Store)), ctypes.pointer(mv), ctypes.pointer(map_lj))
        _raise(lib().bnmc_gpu_run_trace(self._h, 0, ctypes.byref(tr)), self._h)
        trace = dict(model=self.model, method=self.method, seed=cfg.seed, var_names=unobs,
                     samples=[{v: smp[v] for v in unobs} for smp in samples],
                     log_joint=lj[:n].tolist(), timing_ms=tm[:n].tolist(),
                     map_state={v: map_store[v] for v in unobs} if n > 0 else {},
                     map_log_joint=map_lj.value)
        if self.method != "gibbs" or self.spec["method"] == "mh":
            trace["accepted"] = acc[:n].astype(bool).tolist()
        self.download(store)
        return trace

    # -- LDA extras -----------------------------------------------------------------------
    def lda_counts(self):
        """(topic-word counts K x V, this shard's doc-topic counts) of the current z."""
        K, V = int(self.hyper["K"]), int(self.hyper["V"])
        b, e = partition(self._offsets, self._world, self._rank)
        Ml = e - b
        nkw = np.empty(K * V, dtype=np.int32)
        nmk = np.empty(max(Ml, 1) * K, dtype=np.int32)
        _raise(lib().bnmc_gpu_lda_counts(self._h, _p(nkw, c_int32), _p(nmk, c_int32)), self._h)
        return nkw.reshape(K, V), nmk[: Ml * K].reshape(Ml, K)

    # -- checkpoint / binary corpus ------------------------------------------------------
    def save_checkpoint(self, path: str):
        """Device state + next iteration to a binary file (bnmc_gpu_save_checkpoint)."""
        _raise(lib().bnmc_gpu_save_checkpoint(self._h, os.fsencode(path)), self._h)

    def load_checkpoint(self, path: str, store: ParamStore | None = None) -> int:
        """Restore a checkpoint of the same model / sizes / seed / configuration; returns
        the iteration the next sweep runs.  The chain resumes exactly from the device
        state (sweep_device / run_device), or -- given `store`, whose observed data must
        be the checkpointed run's -- the restored latent state is written into `store`,
        which becomes the bound store, so sweep(store, it) / run(store) resume too."""
        _raise(lib().bnmc_gpu_load_checkpoint(self._h, os.fsencode(path)), self._h)
        it = c_int64()
        _raise(lib().bnmc_gpu_checkpoint_iter(self._h, ctypes.byref(it)), self._h)
        self._bound = None
        if store is not None:
            self.download(store)
            self.upload(store)  # binds the observed data; the latent state round-trips unchanged
        return it.value

    def rebind(self, store: ParamStore):
        """Re-upload everything, observed data included.  The observed arrays of a bound
        store are uploaded once per binding (the engine never writes them); a caller who
        edits observed data in place between calls rebinds, or passes a new store."""
        self.upload(store)

    def lda_load_corpus(self, path: str):
        """Stream a binary corpus (write_corpus) into device memory (bnmc_gpu_lda_load_corpus)."""
        _raise(lib().bnmc_gpu_lda_load_corpus(self._h, os.fsencode(path)), self._h)
        self._bound = None

    def prior_init_device(self, seed: int):
        """prior_init on the device-resident state (no host store involved)."""
        _raise(lib().bnmc_gpu_prior_init(self._h, seed), self._h)
        self._bound = None

    def lda_generate(self, seed: int, phi_conc: float = 0.05, theta_conc: float = 0.3):
        _raise(lib().bnmc_gpu_lda_generate(self._h, seed, phi_conc, theta_conc), self._h)
        self._bound = None


def sample(model: str, hyper: dict, store: ParamStore, n: int, cfg: RunConfig) -> dict:
    """sample() (sampler.cpp:557-568)."""
    if n < 1:
        raise BnmcError("sample count must be at least 1")
    for name in cfg.observe_extra:
        store.observed[name] = True
    with Engine(model, hyper, cfg) as e:
        return e.run(store, n)


def map_estimate(model: str, observe_extra, hyper: dict, store: ParamStore, n: int, cfg: RunConfig):
    """map_estimate() (sampler.cpp:570-584): overwrite unobserved vars with the MAP state."""
    cfg = RunConfig(**{**cfg.__dict__, "observe_extra": sorted(set(observe_extra))})
    tr = sample(model, hyper, store, n, cfg)
    for k, v in (tr["map_state"] or {}).items():
        store[k] = v
    return store


def lpp_curve(phi_samples, timing_ms, heldout_hyper: dict, heldout_w, heldout_docs, fit_sweeps: int, seed: int,
              cfg: RunConfig | None = None):
    """lpp_curve (bench.cpp:30-77), the Fig. 3 protocol, on the device: for checkpoints
    c = 1, 2, 4, ... (and the last sample) clamp phi to training sample c - 1, prior_init
    the held-out documents' theta and z with seed + c, map_estimate them over `fit_sweeps`
    Gibbs sweeps (blocks theta, z), and score log_predictive_probability on the held-out
    tokens.  heldout_docs = (w, offsets) of the held-out tokens.  Returns
    [{"samples": c, "lpp": ..., "seconds": sum of the first c sweep times}]."""
    n = len(phi_samples)
    checkpoints = []
    c = 1
    while c <= n:
        checkpoints.append(c)
        c *= 2
    if not checkpoints or checkpoints[-1] != n:
        checkpoints.append(n)
    K, V = int(heldout_hyper["K"]), int(heldout_hyper["V"])
    hw, hoff = heldout_docs
    out = []
    for c in checkpoints:
        phi = np.asarray(phi_samples[c - 1], dtype=np.float64)
        run = RunConfig(**{**(cfg or RunConfig()).__dict__, "seed": seed + c, "method": "gibbs",
                           "observe_extra": ["phi"]})
        with Engine("lda", heldout_hyper, run) as e:
            store = e.allocate()
            store["w"] = heldout_w
            store["phi"] = phi
            e.prior_init(store, seed + c)  # skip_observed: theta and z only
        map_estimate("lda", {"phi"}, heldout_hyper, store, fit_sweeps, run)
        lpp = log_predictive_probability(phi, store["theta"], K, V, hw, hoff)
        secs = float(np.sum(np.asarray(timing_ms[:c], dtype=np.float64)) / 1000.0) if timing_ms is not None else 0.0
        out.append({"samples": c, "lpp": lpp, "seconds": secs})
    return out


# -- primitive operators (device) -------------------------------------------------------
def probe_rng(keys, per: int):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n = keys.size
    u = np.empty(n * per, dtype=np.uint64)
    un = np.empty(n * per)
    g = np.empty(n * per)
    _raise(lib().bnmc_gpu_probe_rng(_p(keys, c_uint64), n, per, _p(u, c_uint64), _p(un, c_double), _p(g, c_double)))
    return u.reshape(n, per), un.reshape(n, per), g.reshape(n, per)


def probe_gamma(keys, shapes):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    shapes = np.ascontiguousarray(shapes, dtype=np.float64)
    out = np.empty(keys.size)
    cnt = np.empty(keys.size, dtype=np.uint64)
    _raise(lib().bnmc_gpu_probe_gamma(_p(keys, c_uint64), _p(shapes, c_double), keys.size, _p(out, c_double),
                                      _p(cnt, c_uint64)))
    return out, cnt


def probe_log_weights(keys, logw):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    logw = np.ascontiguousarray(logw, dtype=np.float64)
    picks = np.empty(keys.size, dtype=np.int64)
    _raise(lib().bnmc_gpu_probe_log_weights(_p(keys, c_uint64), _p(logw, c_double), logw.shape[0], logw.shape[1],
                                            _p(picks, c_int64)))
    return picks


def dirichlet_batch(alpha, key: int):
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    out = np.empty_like(alpha)
    _raise(lib().bnmc_gpu_dirichlet_batch(alpha.shape[0], alpha.shape[1], _p(alpha, c_double), key, _p(out, c_double)))
    return out


def log_predictive_probability(phi, theta, K: int, V: int, w, offsets) -> float:
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.int64)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    out = c_double()
    _raise(lib().bnmc_gpu_lpp(_p(phi, c_double), _p(theta, c_double), K, V, _p(w, c_int64), _p(off, c_int64),
                              len(off) - 1, ctypes.byref(out)))
    return out.value
