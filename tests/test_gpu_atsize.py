"""At-size parity: every BASELINE.json config the reference can run, on the GPU against
the LIVE compiled reference (oracle/_ref, the unmodified sampler) on the same inputs.

  GMM    gen_gmm(1e5, {-5,-1,1,5}, {1,0.1,2,1}) + prior_init, 100 sweeps   (sampler.cpp:114-130,222-265)
  LDA    NIPS gen_lda(1500, 12419, 100, 1267) + prior_init, 3 sweeps,
         product-form (default) and log-space (EXACT_WEIGHTS) modes       (sampler.cpp:52-265)
  LDA    the 1B shape K=1000, V=1e5 on an 8 x 10k-token slice, 1 sweep (both weight modes),
         and the device prior_init of that slice                          (batch.cpp:45-83)
  MH     regression.bn on gen_regression(1e5, 64), 10 steps               (sampler.cpp:284-340)
  HMM    hmm.bn on 1e5 random flips, S = 4 and 16, 5 sweeps (the chunked s-scan vs the
         reference's sequential scan)                                      (sampler.cpp:259-264)
  catmix catmix.bn on 1e5 categorical points, K = 8, V = 200, 5 sweeps
  NB     naivebayes.bn on 2e4 rows x 32 features, 5 sweeps

Contract: z / counts / accept decisions bit-exact on every sweep (0
mismatches); phi, theta, pi <= 1e-12 relative; GMM mu, sigma2 <= 1e-10; log-joint <= 1e-10.
The reference chain runs in a child process (tests/refrun.py: multi-threaded where its
pool survives, retried, else single-threaded).
"""
import os

import numpy as np
import pytest

from refrun import run_chain

pytestmark = pytest.mark.gpu

RTOL_PARAM = 1e-12
RTOL_MU = 1e-10
RTOL_LJ = 1e-10
THREADS = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def g():
    import paper_1312_3613_b200 as g

    g.lib()
    return g


@pytest.fixture(scope="module", autouse=True)
def _needs_reference():
    from oracle import REFERENCE_SO

    if not os.path.exists(REFERENCE_SO):
        pytest.skip("oracle/_ref/libbnmc_ref.so not built")


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def _lj_ok(a, b):
    return abs(a - b) <= RTOL_LJ * abs(b)


# ----------------------------------------------------------------------------------------
# GMM, N = 1e5, the paper's 4-centre set, 100 sweeps
# ----------------------------------------------------------------------------------------
def test_gmm_1e5_100_sweeps(g):
    N, K, seed, n = 100000, 4, 2024, 100
    ref = run_chain({"model": "gmm", "hyper": {"N": N, "K": K}, "method": "gibbs", "seed": seed, "threads": 1,
                     "gen": ["gmm", [N, [-5.0, -1.0, 1.0, 5.0], [1.0, 0.1, 2.0, 1.0], seed]],
                     "observed": ["x"], "init": "prior", "sweeps": n,
                     "record": ["z", "pi", "mu", "sigma2"]})
    e = g.Engine("gmm", {"N": N, "K": K}, g.RunConfig(seed=seed))
    s = e.allocate()
    s["x"] = ref["x"]
    e.prior_init(s, seed)                  # the device prior_init must equal the reference's
    assert np.array_equal(s["z"], ref["z_init"])
    for v, tol in (("pi", RTOL_PARAM), ("mu", RTOL_PARAM), ("sigma2", RTOL_PARAM)):
        assert rel(s[v], ref[v + "_init"]) < tol, v
    s["z"], s["pi"], s["mu"], s["sigma2"] = ref["z_init"], ref["pi_init"], ref["mu_init"], ref["sigma2_init"]
    worst = {"pi": 0.0, "mu": 0.0, "sigma2": 0.0}
    for it in range(n):
        lj = e.sweep(s, it)
        mism = int((s["z"] != ref["z"][it]).sum())
        assert mism == 0, f"sweep {it}: {mism} z mismatches of {N}"
        for v in worst:
            worst[v] = max(worst[v], rel(s[v], ref[v][it]))
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    assert worst["pi"] < RTOL_PARAM and worst["mu"] < RTOL_MU and worst["sigma2"] < RTOL_MU, worst
    e.close()


# ----------------------------------------------------------------------------------------
# LDA, NIPS-shaped, 3 consecutive sweeps, both weight modes
# ----------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def nips_ref():
    M, V, K, L, seed = 1500, 12419, 100, 1267, 42
    return run_chain({"model": "lda", "hyper": {"K": K, "V": V, "M": M, "N": [L] * M}, "method": "gibbs",
                      "seed": seed, "threads": THREADS, "gen": ["lda", [M, V, K, L, seed]], "observed": ["w"],
                      "init": "prior", "sweeps": 3, "record": ["z", "phi", "theta"]}, timeout=1800)


@pytest.mark.parametrize("exact", [False, True], ids=["product-form", "log-space"])
def test_lda_nips_3_sweeps(g, nips_ref, exact):
    M, V, K, L, seed = 1500, 12419, 100, 1267, 42
    ref = nips_ref
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=seed, exact_weights=exact))
    s = e.allocate()
    s["w"] = ref["w"]
    e.prior_init(s, seed)
    assert np.array_equal(s["z"], ref["z_init"])
    assert rel(s["phi"], ref["phi_init"]) < RTOL_PARAM and rel(s["theta"], ref["theta_init"]) < RTOL_PARAM
    assert _lj_ok(e.eval_log_joint(s), float(ref["lj_init"]))
    for it in range(3):
        lj = e.sweep(s, it)
        mism = int((s["z"] != ref["z"][it]).sum())
        assert mism == 0, f"sweep {it}: {mism} z mismatches of {M * L}"
        assert rel(s["phi"], ref["phi"][it]) < RTOL_PARAM, it
        assert rel(s["theta"], ref["theta"][it]) < RTOL_PARAM, it
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    # the topic-word counts of the final z (the next sweep's phi block input)
    nkw, nmk = e.lda_counts()
    want = np.zeros((K, V), dtype=np.int64)
    np.add.at(want, (ref["z"][-1], ref["w"]), 1)
    assert np.array_equal(nkw, want)
    e.close()


# ----------------------------------------------------------------------------------------
# LDA at the 1B shape (K = 1000, V = 1e5): an 8-document x 10k-token slice, one sweep
# ----------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def k1000_ref():
    M, V, K, L, seed = 8, 100000, 1000, 10000, 7
    return run_chain({"model": "lda", "hyper": {"K": K, "V": V, "M": M, "N": [L] * M}, "method": "gibbs",
                      "seed": seed, "threads": THREADS, "gen": ["lda", [M, V, K, L, seed]], "observed": ["w"],
                      "init": "prior", "sweeps": 1, "record": ["z", "phi", "theta"]}, timeout=1800)


@pytest.mark.parametrize("exact", [False, True], ids=["product-form", "log-space"])
def test_lda_k1000_v1e5_slice(g, k1000_ref, exact):
    """(word-major z-step order: > 32 MB of fp32 rows; log-space: the screen + the
    log-space fallback)"""
    M, V, K, L, seed = 8, 100000, 1000, 10000, 7
    ref = k1000_ref
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=seed, exact_weights=exact))
    s = e.allocate()
    s["w"] = ref["w"]
    e.prior_init(s, seed)
    assert np.array_equal(s["z"], ref["z_init"])
    assert rel(s["phi"], ref["phi_init"]) < RTOL_PARAM and rel(s["theta"], ref["theta_init"]) < RTOL_PARAM
    lj = e.sweep(s, 0)
    mism = int((s["z"] != ref["z"][0]).sum())
    assert mism == 0, f"{mism} z mismatches of {M * L}"
    assert rel(s["phi"], ref["phi"][0]) < RTOL_PARAM
    assert rel(s["theta"], ref["theta"][0]) < RTOL_PARAM
    assert _lj_ok(lj, ref["lj"][0]), (lj, ref["lj"][0])
    e.close()


# ----------------------------------------------------------------------------------------
# Metropolis-Hastings, regression.bn, N = 1e5 rows x 64 features, 10 steps
# ----------------------------------------------------------------------------------------
def test_mh_linreg_1e5x64_10_steps(g):
    N, K, seed, n = 100000, 64, 11, 10
    # the reference's pool crashes on this model when multi-threaded: 1 thread
    ref = run_chain({"model": "regression", "hyper": {"N": N, "K": K, "l": -1.0, "u": 1.0}, "method": "mh",
                     "seed": seed, "threads": 1, "mh_scale": 0.5, "gen": ["regression", [N, K, 0.1, seed]],
                     "observed": ["x", "y"], "init": "prior", "sweeps": n, "record": ["w", "b", "tau"]},
                    timeout=1800)
    assert 0 < ref["acc"].sum() < n  # both branches of the accept test are exercised
    e = g.Engine("regression", {"N": N, "K": K, "l": -1.0, "u": 1.0}, g.RunConfig(seed=seed, mh_scale=0.5))
    s = e.allocate()
    s["x"], s["y"] = ref["x"], ref["y"]
    e.prior_init(s, seed)
    for v in ("w", "b", "tau"):
        assert rel(s[v], ref[v + "_init"]) < RTOL_PARAM, v
    s["w"], s["b"], s["tau"] = ref["w_init"], ref["b_init"], ref["tau_init"]
    assert _lj_ok(e.eval_log_joint(s), float(ref["lj_init"]))
    for it in range(n):
        acc = []
        lj = e.sweep(s, it, acc)
        assert acc[0] == bool(ref["acc"][it]), f"accept decision differs at step {it}"
        for v in ("w", "b", "tau"):
            assert rel(s[v], ref[v][it]) < RTOL_PARAM, (it, v)
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    e.close()


# ----------------------------------------------------------------------------------------
# A long LDA chain: 300 sweeps from the reference's prior_init, posterior summaries
# ----------------------------------------------------------------------------------------
def test_lda_long_chain_posterior_vs_reference(g):
    """north_star (b): posterior summaries over many sweeps.  A 300-sweep chain on a
    gen_lda corpus (200 documents x 60 tokens, V = 500, K = 10): z equal to the live
    reference's on EVERY sweep (the whole chain, not one step), the log-joint trajectory
    within 1e-10, and the posterior means of phi and theta over the last 150 sweeps within
    1e-10 relative."""
    M, V, K, L, seed, n = 200, 500, 10, 60, 11, 300
    ref = run_chain({"model": "lda", "hyper": {"K": K, "V": V, "M": M, "N": [L] * M}, "method": "gibbs",
                     "seed": seed, "threads": 1, "gen": ["lda", [M, V, K, L, seed]], "observed": ["w"],
                     "init": "prior", "sweeps": n, "record": ["z", "phi", "theta"]}, timeout=1800)
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=seed))
    s = e.allocate()
    s["w"] = ref["w"]
    e.prior_init(s, seed)
    assert np.array_equal(s["z"], ref["z_init"])
    phis, thetas = [], []
    for it in range(n):
        lj = e.sweep(s, it)
        assert np.array_equal(s["z"], ref["z"][it]), f"z differs at sweep {it}"
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
        if it >= n // 2:
            phis.append(s["phi"].copy())
            thetas.append(s["theta"].copy())
    assert rel(np.mean(phis, axis=0), ref["phi"][n // 2:].mean(axis=0)) < 1e-10
    assert rel(np.mean(thetas, axis=0), ref["theta"][n // 2:].mean(axis=0)) < 1e-10
    e.close()


# ----------------------------------------------------------------------------------------
# HMM: the chunked s-scan (composed chunk maps) against the reference's sequential scan
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("S", [4, 16])
def test_hmm_1e5_5_sweeps(g, S):
    N, seed, n = 100000, 77, 5
    flips = np.random.default_rng(seed).integers(0, 2, N).astype(np.int64)
    ref = run_chain({"model": "hmm", "hyper": {"N": N, "S": S}, "method": "gibbs", "seed": seed, "threads": 1,
                     "observed": ["flips"], "init": "prior", "sweeps": n, "record": ["s", "T", "bias"]},
                    data={"flips": flips})
    e = g.Engine("hmm", {"N": N, "S": S}, g.RunConfig(seed=seed))
    st = e.allocate()
    st["flips"] = flips
    e.prior_init(st, seed)                 # the chunked prior chain against the reference's
    assert np.array_equal(st["s"], ref["s_init"])
    assert rel(st["T"], ref["T_init"]) < RTOL_PARAM and rel(st["bias"], ref["bias_init"]) < RTOL_PARAM
    st["s"], st["T"], st["bias"] = ref["s_init"], ref["T_init"], ref["bias_init"]
    for it in range(n):
        lj = e.sweep(st, it)
        mism = int((st["s"] != ref["s"][it]).sum())
        assert mism == 0, f"sweep {it}: {mism} s mismatches of {N}"
        assert rel(st["T"], ref["T"][it]) < RTOL_PARAM and rel(st["bias"], ref["bias"][it]) < RTOL_PARAM
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    e.close()


# ----------------------------------------------------------------------------------------
# catmix and naive Bayes at size: parallel prior_init, the per-block log-joint partials
# ----------------------------------------------------------------------------------------
def test_catmix_1e5_5_sweeps(g):
    N, K, V, seed, n = 100000, 8, 200, 91, 5
    x = np.random.default_rng(seed).integers(0, V, N).astype(np.int64)
    ref = run_chain({"model": "catmix", "hyper": {"N": N, "K": K, "V": V}, "method": "gibbs", "seed": seed,
                     "threads": 1, "observed": ["x"], "init": "prior", "sweeps": n,
                     "record": ["z", "theta", "phi"]}, data={"x": x})
    e = g.Engine("catmix", {"N": N, "K": K, "V": V}, g.RunConfig(seed=seed))
    st = e.allocate()
    st["x"] = x
    e.prior_init(st, seed)
    assert np.array_equal(st["z"], ref["z_init"])
    assert rel(st["theta"], ref["theta_init"]) < RTOL_PARAM and rel(st["phi"], ref["phi_init"]) < RTOL_PARAM
    for it in range(n):
        lj = e.sweep(st, it)
        assert np.array_equal(st["z"], ref["z"][it]), it
        assert rel(st["theta"], ref["theta"][it]) < RTOL_PARAM and rel(st["phi"], ref["phi"][it]) < RTOL_PARAM
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    e.close()


def test_naivebayes_2e4x32_5_sweeps(g):
    N, K, seed, n = 20000, 32, 93, 5
    rs = np.random.default_rng(seed)
    c = rs.integers(0, 2, N).astype(np.int64)
    f = rs.integers(0, 2, N * K).astype(np.int64)
    ref = run_chain({"model": "naivebayes", "hyper": {"N": N, "K": K}, "method": "gibbs", "seed": seed,
                     "threads": 1, "observed": ["c", "f"], "init": "prior", "sweeps": n,
                     "record": ["pC", "pF"]}, data={"c": c, "f": f})
    e = g.Engine("naivebayes", {"N": N, "K": K}, g.RunConfig(seed=seed))
    st = e.allocate()
    st["c"], st["f"] = c, f
    e.prior_init(st, seed)
    assert rel(st["pC"], ref["pC_init"]) < RTOL_PARAM and rel(st["pF"], ref["pF_init"]) < RTOL_PARAM
    for it in range(n):
        lj = e.sweep(st, it)
        assert rel(st["pC"], ref["pC"][it]) < RTOL_PARAM and rel(st["pF"], ref["pF"][it]) < RTOL_PARAM
        assert _lj_ok(lj, ref["lj"][it]), (it, lj, ref["lj"][it])
    e.close()
