"""Generate the committed golden fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists and `make -C oracle ref`
has produced oracle/_ref/libbnmc_ref.so):

    python tests/golden/make_golden.py

Every array in tests/golden/*.npz is an output of the compiled reference sampler
(proj/src/*.cpp) through its own public API -- RngStream (rng.hpp), draw_gamma
(dist.cpp:136-155), draw_from_log_weights (dist.cpp:202-215),
sample_dirichlet_batch (batch.cpp:45-83), gen_lda/gen_gmm/gen_regression
(gen.cpp), prior_init (sampler.cpp:542-555) and Engine::sweep
(sampler.cpp:390-405).  The fixtures let the GPU box (which has no
/root/reference) check the restatement and the CUDA path against reference
outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference, doc_offsets  # noqa: E402


def rng_kats(F: Reference):
    keys = []
    for t in [(42, 1, 2, 3, 0), (99, 3, 2, 0, 3), (99, 4, 0, 3, 0), (7, 0, 0, 0, 0), (13, 0, 0, 0, 0),
              (0, 0, 0, 0, 0), (2**64 - 1, 5, 2, 123456789, 77), (1234, 3, 2, 10**9 - 1, 511)]:
        keys.append(F.keyed(*t))
    tuples = np.array([[42, 1, 2, 3, 0], [99, 3, 2, 0, 3], [99, 4, 0, 3, 0], [7, 0, 0, 0, 0],
                       [13, 0, 0, 0, 0], [0, 0, 0, 0, 0], [2**64 - 1, 5, 2, 123456789, 77],
                       [1234, 3, 2, 10**9 - 1, 511]], dtype=np.uint64)
    keys = np.array(keys, dtype=np.uint64)
    derive_args = np.array([[5, 7], [0, 0], [123, 4567], [2**40, 3]], dtype=np.uint64)
    derived = np.array([[F.derive(int(k), int(a), int(b)) for a, b in derive_args] for k in keys],
                       dtype=np.uint64)
    import ctypes
    u64 = np.empty((len(keys), 16), dtype=np.uint64)
    unit = np.empty((len(keys), 16))
    gauss = np.empty((len(keys), 16))
    for i, k in enumerate(keys):
        F.lib.bref_stream_u64(int(k), 16, u64[i].ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        F.lib.bref_stream_unit(int(k), 16, unit[i].ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        F.lib.bref_stream_gaussian(int(k), 16, gauss[i].ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    # gamma draws: shapes across the <1 boost branch and the M-T branch
    shapes = np.array([0.01, 0.05, 0.1, 0.3, 0.5, 0.999, 1.0, 1.1, 2.5, 3.5, 10.1, 100.1, 1000.1, 12345.1])
    gkeys = np.array([F.keyed(13, i) for i in range(64)], dtype=np.uint64)
    gam = np.empty((len(shapes), len(gkeys)))
    cnt = np.empty((len(shapes), len(gkeys)), dtype=np.uint64)
    c = ctypes.c_uint64()
    for a, s in enumerate(shapes):
        for b, k in enumerate(gkeys):
            gam[a, b] = F.lib.bref_draw_gamma(int(k), float(s), ctypes.byref(c))
            cnt[a, b] = c.value
    # draw_from_log_weights
    rs = np.random.default_rng(3)
    lw = rs.normal(size=(200, 37)) * 5.0
    lw[5, :] = -np.inf
    lw[5, 17] = -3.0
    lw[7, ::2] = -np.inf
    lkeys = np.array([F.keyed(31, 3, 2, i, 9) for i in range(200)], dtype=np.uint64)
    picks = np.array([F.lib.bref_draw_from_log_weights(int(k), np.ascontiguousarray(lw[i]).ctypes.data_as(
        ctypes.POINTER(ctypes.c_double)), lw.shape[1]) for i, k in enumerate(lkeys)], dtype=np.int64)
    # Dirichlet batch (rows x cols) with per-row concentrations
    alpha = 0.1 + rs.integers(0, 5, size=(6, 40)).astype(np.float64)
    dkey = F.keyed(77, 4, 0, 3)
    dout = np.empty(alpha.size)
    F._check(F.lib.bref_dirichlet_batch(6, 40, np.ascontiguousarray(alpha.ravel()).ctypes.data_as(
        ctypes.POINTER(ctypes.c_double)), 1, dkey, 1, 0, dout.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    np.savez_compressed(os.path.join(HERE, "rng_dist.npz"), tuples=tuples, keys=keys, derive_args=derive_args,
                        derived=derived, u64=u64, unit=unit, gauss=gauss, gamma_shapes=shapes,
                        gamma_keys=gkeys, gamma=gam, gamma_counters=cnt, logw=lw, logw_keys=lkeys,
                        logw_picks=picks, dir_alpha=alpha, dir_key=np.uint64(dkey), dir_out=dout.reshape(6, 40))


def lda_fixture(F: Reference, name, M, V, K, L, seed, sweeps, lengths=None):
    if lengths is None:
        w, _, _ = F.gen_lda(M, V, K, L, seed)
        lengths = [L] * M
    else:
        rs = np.random.default_rng(seed)
        w = rs.integers(0, V, int(sum(lengths))).astype(np.int64)
    e = F.open("lda", {"K": K, "V": V, "M": M, "N": list(map(int, lengths))}, seed=seed)
    e.set("w", w)
    e.prior_init(seed)
    out = dict(K=K, V=V, M=M, seed=seed, offsets=doc_offsets(lengths), w=w,
               phi0=e.get("phi"), theta0=e.get("theta"), z0=e.get("z"), lj0=e.log_joint())
    zs, phis, thetas, ljs = [], [], [], []
    for it in range(sweeps):
        lj, _ = e.sweep(it)
        zs.append(e.get("z")); phis.append(e.get("phi")); thetas.append(e.get("theta")); ljs.append(lj)
    out.update(z=np.stack(zs), phi=np.stack(phis), theta=np.stack(thetas), lj=np.array(ljs))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def gmm_fixture(F: Reference, name, N, seed, sweeps):
    x = F.gen_gmm(N, [-5.0, -1.0, 1.0, 5.0], [1.0, 0.1, 2.0, 1.0], seed)
    e = F.open("gmm", {"N": N, "K": 4}, seed=seed)
    e.set("x", x)
    e.prior_init(seed)
    out = dict(N=N, K=4, seed=seed, x=x, pi0=e.get("pi"), mu0=e.get("mu"), sigma20=e.get("sigma2"),
               z0=e.get("z"))
    acc = {k: [] for k in ("z", "pi", "mu", "sigma2", "lj")}
    for it in range(sweeps):
        lj, _ = e.sweep(it)
        for k in ("z", "pi", "mu", "sigma2"):
            acc[k].append(e.get(k))
        acc["lj"].append(lj)
    out.update({k: np.array(v) for k, v in acc.items()})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def mh_fixture(F: Reference, name, N, K, seed, steps):
    x, y, wt, bt = F.gen_regression(N, K, 0.1, seed)
    e = F.open("regression", {"K": K, "N": N, "l": -1.0, "u": 1.0}, method="mh", seed=seed)
    e.set("x", x)
    e.set("y", y)
    e.prior_init(seed)
    out = dict(N=N, K=K, seed=seed, x=x, y=y, w0=e.get("w"), b0=e.get("b")[0], tau0=e.get("tau")[0],
               lj0=e.log_joint())
    ws, bs, ts, ljs, accs = [], [], [], [], []
    for it in range(steps):
        lj, a = e.sweep(it)
        ws.append(e.get("w")); bs.append(e.get("b")[0]); ts.append(e.get("tau")[0]); ljs.append(lj); accs.append(a)
    out.update(w=np.array(ws), b=np.array(bs), tau=np.array(ts), lj=np.array(ljs), accepted=np.array(accs))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def zoo_fixture(F: Reference, name, model, hyper, data, seed, sweeps, method="gibbs", mh_scale=0.5):
    """catmix / naivebayes / hmm / polyreg: observed data from numpy,
    the reference's prior_init, then `sweeps` reference sweeps (state + log-joint each)."""
    e = F.open(model, hyper, method=method, seed=seed, mh_scale=mh_scale)
    for k, v in data.items():
        e.set(k, v)
    e.prior_init(seed)
    import paper_1312_3613_b200.engine as eng  # names only (no device): variable order
    names = eng.MODELS[model]["vars"]
    latent = [n for n in names if n not in eng.MODELS[model]["observed"]]
    out = dict(seed=seed, hyper=np.array(repr(hyper)), method=np.array(method), mh_scale=mh_scale, lj0=e.log_joint(),
               **{f"data_{k}": v for k, v in data.items()}, **{f"{n}0": e.get(n) for n in latent})
    hist = {n: [] for n in latent}
    ljs, accs = [], []
    for it in range(sweeps):
        lj, a = e.sweep(it)
        for n in latent:
            hist[n].append(e.get(n))
        ljs.append(lj)
        accs.append(a)
    out.update({n: np.stack(v) for n, v in hist.items()})
    out.update(lj=np.array(ljs), accepted=np.array(accs))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def zoo(F: Reference):
    rs = np.random.default_rng(99)
    zoo_fixture(F, "catmix_small", "catmix", {"N": 500, "K": 4, "V": 12},
                {"x": rs.integers(0, 12, 500)}, seed=31, sweeps=4)
    zoo_fixture(F, "naivebayes_small", "naivebayes", {"N": 400, "K": 6},
                {"c": rs.integers(0, 2, 400), "f": (rs.random(2400) < 0.3).astype(np.int64)}, seed=37, sweeps=4)
    flips = (rs.random(300) < np.repeat([0.2, 0.8, 0.5], 100)).astype(np.int64)
    zoo_fixture(F, "hmm_small", "hmm", {"N": 300, "S": 3}, {"flips": flips}, seed=41, sweeps=4)
    x = rs.uniform(0.0, 2.0, 800)
    y = 0.5 + 0.3 * x - 0.7 * x ** 2 + 0.2 * x ** 3 + rs.normal(size=800)
    zoo_fixture(F, "polyreg_small", "polyreg", {"N": 800, "M": 3}, {"x": x, "y": y}, seed=43, sweeps=12,
                method="mh", mh_scale=0.05)
    # Gibbs plans of the MH models: single-site MWG for w and b, conjugate tau
    zoo_fixture(F, "polyreg_gibbs", "polyreg", {"N": 600, "M": 3}, {"x": x[:600], "y": y[:600]}, seed=47,
                sweeps=6, method="gibbs", mh_scale=0.05)
    xr = rs.uniform(-1.0, 1.0, (700, 5))
    yr = xr @ np.array([0.5, -1.0, 0.3, 0.0, 2.0]) + 0.2 + 0.3 * rs.normal(size=700)
    zoo_fixture(F, "regression_gibbs", "regression", {"K": 5, "N": 700, "l": -1.0, "u": 1.0},
                {"x": xr.ravel(), "y": yr}, seed=53, sweeps=6, method="gibbs", mh_scale=0.1)
    zoo_fixture(F, "polyreg_mwg", "polyreg", {"N": 600, "M": 3}, {"x": x[:600], "y": y[:600]}, seed=59,
                sweeps=4, method="mwg", mh_scale=0.05)
    zoo_fixture(F, "regression_mwg", "regression", {"K": 5, "N": 700, "l": -1.0, "u": 1.0},
                {"x": xr.ravel(), "y": yr}, seed=61, sweeps=4, method="mwg", mh_scale=0.1)


def regprec(F: Reference):
    """The GammaPrecision conjugate kind (rewrite.cpp:538-549, sampler.cpp:205-207) through our
    test model oracle/models/regprec.bn (regression with y ~ N(mean, pow(tau, -1)), tau ~
    Gamma(3, 1)) under its MH, Gibbs (conjugate Gamma tau) and MWG plans."""
    rs = np.random.default_rng(101)
    xr = rs.uniform(-1.0, 1.0, (700, 5))
    yr = xr @ np.array([0.5, -1.0, 0.3, 0.0, 2.0]) + 0.2 + 0.3 * rs.normal(size=700)
    hyper = {"K": 5, "N": 700, "l": -1.0, "u": 1.0}
    data = {"x": xr.ravel(), "y": yr}
    zoo_fixture(F, "regprec_mh", "regprec", hyper, data, seed=67, sweeps=12, method="mh", mh_scale=0.1)
    zoo_fixture(F, "regprec_gibbs", "regprec", hyper, data, seed=71, sweeps=6, method="gibbs", mh_scale=0.1)
    zoo_fixture(F, "regprec_mwg", "regprec", hyper, data, seed=73, sweeps=4, method="mwg", mh_scale=0.1)


def describe(F: Reference):
    # Block order of the LDA plan (phi, theta, z) as the reference reports it.
    with open(os.path.join(HERE, "describe_lda.txt"), "w") as f:
        f.write(F.open("lda", {"K": 3, "V": 5, "M": 2, "N": [1, 2]}).describe())


if __name__ == "__main__":
    F = Reference()
    rng_kats(F)
    lda_fixture(F, "lda_desk", M=60, V=150, K=8, L=40, seed=2024, sweeps=4)
    lda_fixture(F, "lda_ragged", M=7, V=40, K=5, L=0, seed=7, sweeps=3, lengths=[5, 0, 17, 1, 33, 0, 9])
    lda_fixture(F, "lda_k1", M=5, V=30, K=1, L=12, seed=5, sweeps=2)
    gmm_fixture(F, "gmm_small", N=3000, seed=17, sweeps=5)
    mh_fixture(F, "mh_linreg", N=1500, K=16, seed=23, steps=12)
    zoo(F)
    regprec(F)
    describe(F)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
