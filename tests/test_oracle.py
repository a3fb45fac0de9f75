"""CPU: pin the oracle restatement against the reference's own outputs.

Two sources of truth, both produced by the UNMODIFIED reference:
* the committed golden fixtures (tests/golden/*.npz, made by make_golden.py);
* the compiled reference itself (oracle/_ref), when it is present.
Everything here is bit-exact: the restatement follows the reference's
arithmetic expression for expression on the same libm.
"""
import ctypes
import os

import numpy as np
import pytest

from conftest import ROOT, golden


class _R(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint64), ("counter", ctypes.c_uint64)]


def _lib(restatement):
    L = restatement.lib
    L.bo_next_u64.restype = ctypes.c_uint64
    L.bo_next_u64.argtypes = [ctypes.POINTER(_R)]
    L.bo_next_unit.restype = ctypes.c_double
    L.bo_next_unit.argtypes = [ctypes.POINTER(_R)]
    L.bo_next_gaussian.restype = ctypes.c_double
    L.bo_next_gaussian.argtypes = [ctypes.POINTER(_R)]
    L.bo_draw_gamma.restype = ctypes.c_double
    L.bo_draw_gamma.argtypes = [ctypes.POINTER(_R), ctypes.c_double]
    L.bo_draw_from_log_weights.restype = ctypes.c_int64
    L.bo_draw_from_log_weights.argtypes = [ctypes.POINTER(_R), ctypes.POINTER(ctypes.c_double), ctypes.c_int64]
    return L


def test_rng_known_answers(restatement):
    """SURVEY.md 8c KAT table (rng.hpp:12-51)."""
    R = restatement
    assert R.keyed(42, 1, 2, 3) == 0x41F2B17275622A47
    assert R.keyed(99, 3, 2, 0, 3) == 0xB55297D6128BFC45
    assert R.derive(R.keyed(99, 4, 0, 3), 5, 7) == 0xB5278FD3D79F0EA8
    L = _lib(R)
    r = _R(R.keyed(42, 1, 2, 3), 0)
    # SURVEY.md lists these two in swapped order; the compiled reference emits this order.
    assert L.bo_next_u64(ctypes.byref(r)) == 0x0F7C1C79CBE2C665
    assert L.bo_next_u64(ctypes.byref(r)) == 0x84C0AD9731388361
    r = _R(R.keyed(99, 3, 2, 0, 3), 0)
    assert L.bo_next_unit(ctypes.byref(r)) == 0.74121406422902969
    r = _R(R.keyed(7), 0)
    assert L.bo_next_gaussian(ctypes.byref(r)) == -1.8393998306609216
    r = _R(R.keyed(13, 0), 0)
    assert L.bo_draw_gamma(ctypes.byref(r), 0.1) == 0.00023006744857612197
    r = _R(R.keyed(13, 1), 0)
    assert L.bo_draw_gamma(ctypes.byref(r), 3.5) == 1.3082667264652144


def test_rng_streams_vs_golden(restatement):
    g = golden("rng_dist")
    R = restatement
    L = _lib(R)
    for t, k in zip(g["tuples"], g["keys"]):
        assert R.keyed(*[int(v) for v in t]) == int(k)
    for i, k in enumerate(g["keys"]):
        for j, (a, b) in enumerate(g["derive_args"]):
            assert R.derive(int(k), int(a), int(b)) == int(g["derived"][i, j])
        r = _R(int(k), 0)
        assert [L.bo_next_u64(ctypes.byref(r)) for _ in range(16)] == [int(v) for v in g["u64"][i]]
        r = _R(int(k), 0)
        assert np.array_equal([L.bo_next_unit(ctypes.byref(r)) for _ in range(16)], g["unit"][i])
        r = _R(int(k), 0)
        assert np.array_equal([L.bo_next_gaussian(ctypes.byref(r)) for _ in range(16)], g["gauss"][i])
        u = g["unit"][i]
        assert np.all((u > 0) & (u < 1))


def test_gamma_vs_golden(restatement):
    """draw_gamma (dist.cpp:136-155) incl. the shape<1 boost: values AND counters consumed."""
    g = golden("rng_dist")
    L = _lib(restatement)
    for a, s in enumerate(g["gamma_shapes"]):
        for b, k in enumerate(g["gamma_keys"]):
            r = _R(int(k), 0)
            v = L.bo_draw_gamma(ctypes.byref(r), float(s))
            assert v == g["gamma"][a, b]
            assert r.counter == int(g["gamma_counters"][a, b])


def test_draw_from_log_weights_vs_golden(restatement):
    g = golden("rng_dist")
    L = _lib(restatement)
    lw = g["logw"]
    for i, k in enumerate(g["logw_keys"]):
        r = _R(int(k), 0)
        row = np.ascontiguousarray(lw[i])
        got = L.bo_draw_from_log_weights(ctypes.byref(r), row.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(row))
        assert got == g["logw_picks"][i]
    # all -inf -> error (std::domain_error in the reference)
    r = _R(1, 0)
    row = np.full(4, -np.inf)
    assert L.bo_draw_from_log_weights(ctypes.byref(r), row.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 4) == -1


def test_dirichlet_batch_vs_golden(restatement):
    g = golden("rng_dist")
    a = np.ascontiguousarray(g["dir_alpha"].ravel())
    out = np.empty_like(a)
    dp = ctypes.POINTER(ctypes.c_double)
    restatement.lib.bo_dirichlet_batch.argtypes = [ctypes.c_int64, ctypes.c_int64, dp, ctypes.c_uint64, dp]
    assert restatement.lib.bo_dirichlet_batch(6, 40, a.ctypes.data_as(dp), int(g["dir_key"]), out.ctypes.data_as(dp)) == 0
    assert np.array_equal(out.reshape(6, 40), g["dir_out"])
    assert np.allclose(out.reshape(6, 40).sum(1), 1.0, atol=1e-12)


@pytest.mark.parametrize("name", ["lda_desk", "lda_ragged", "lda_k1"])
def test_lda_sweeps_vs_golden(restatement, name):
    g = golden(name)
    K, V = int(g["K"]), int(g["V"])
    off, w, seed = g["offsets"], g["w"], int(g["seed"])
    phi, theta, z = restatement.lda_prior_init(K, V, off, w, seed)
    assert np.array_equal(phi, g["phi0"]) and np.array_equal(theta, g["theta0"]) and np.array_equal(z, g["z0"])
    assert restatement.lda_log_joint(K, V, off, w, z, phi, theta) == g["lj0"]
    for it in range(len(g["lj"])):
        lj = restatement.lda_sweep(K, V, off, w, z, phi, theta, seed, it)
        assert np.array_equal(z, g["z"][it]), f"z mismatch at sweep {it}"
        assert np.array_equal(phi, g["phi"][it])
        assert np.array_equal(theta, g["theta"][it])
        assert lj == g["lj"][it]
    if name == "lda_k1":  # K=1 degenerate (test_runtime.cpp:360-386): theta = phi-row sums = 1, z = 0
        assert np.all(z == 0) and np.allclose(theta, 1.0)


def test_gmm_sweeps_vs_golden(restatement):
    g = golden("gmm_small")
    x, seed = g["x"], int(g["seed"])
    pi, mu, s2, z = restatement.gmm_prior_init(x, 4, seed)
    assert np.array_equal(z, g["z0"]) and np.array_equal(mu, g["mu0"])
    for it in range(len(g["lj"])):
        lj = restatement.gmm_sweep(x, 4, z, pi, mu, s2, seed, it)
        assert np.array_equal(z, g["z"][it])
        assert np.array_equal(pi, g["pi"][it]) and np.array_equal(mu, g["mu"][it])
        assert np.array_equal(s2, g["sigma2"][it])
        assert lj == g["lj"][it]


def test_mh_linreg_vs_golden(restatement):
    g = golden("mh_linreg")
    x, y, K, seed = g["x"], g["y"], int(g["K"]), int(g["seed"])
    w, b, tau = g["w0"].copy(), float(g["b0"]), float(g["tau0"])
    assert restatement.mh_log_joint(x, y, K, w, b, tau) == g["lj0"]
    for it in range(len(g["lj"])):
        b, tau, lj, acc = restatement.mh_step(x, y, K, w, b, tau, seed, it)
        assert acc == bool(g["accepted"][it])
        assert np.array_equal(w, g["w"][it]) and b == g["b"][it] and tau == g["tau"][it]
        assert lj == g["lj"][it]


def test_restatement_vs_live_reference_lda(restatement, reference):
    """Live cross-check on a fresh seed and a KOS-like shape (small)."""
    M, V, K, L = 30, 300, 12, 25
    w, _, _ = reference.gen_lda(M, V, K, L, 99)
    off = np.arange(M + 1, dtype=np.int64) * L
    e = reference.open("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, seed=99)
    e.set("w", w)
    e.prior_init(99)
    phi, theta, z = e.get("phi"), e.get("theta"), e.get("z")
    for it in range(3):
        lj, _ = e.sweep(it)
        lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, 99, it)
        assert lj == lj2 and np.array_equal(e.get("z"), z) and np.array_equal(e.get("phi"), phi)


def test_observed_phi_protocol(restatement, reference):
    """lpp_curve clamps phi (bench.cpp:30-77): the phi block is dropped, phi never written."""
    M, V, K, L = 10, 50, 4, 20
    w, true_phi, _ = reference.gen_lda(M, V, K, L, 5)
    off = np.arange(M + 1, dtype=np.int64) * L
    e = reference.open("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, seed=5, observe=("phi",))
    e.set("w", w)
    e.set("phi", true_phi)
    e.prior_init(5)
    phi, theta, z = e.get("phi"), e.get("theta"), e.get("z")
    assert np.array_equal(phi, true_phi)
    for it in range(3):
        lj, _ = e.sweep(it)
        lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, 5, it, observe_phi=True)
        assert lj == lj2 and np.array_equal(e.get("z"), z)
        assert np.array_equal(e.get("phi"), true_phi) and np.array_equal(phi, true_phi)


@pytest.mark.parametrize("name,model,method", [("catmix_small", "catmix", "gibbs"),
                                               ("naivebayes_small", "naivebayes", "gibbs"),
                                               ("hmm_small", "hmm", "gibbs"),
                                               ("polyreg_small", "polyreg", "mh"),
                                               ("polyreg_gibbs", "polyreg", "gibbs"),
                                               ("regression_gibbs", "regression", "gibbs"),
                                               ("polyreg_mwg", "polyreg", "mwg"),
                                               ("regression_mwg", "regression", "mwg"),
                                               ("regprec_mh", "regprec", "mh"),
                                               ("regprec_gibbs", "regprec", "gibbs"),
                                               ("regprec_mwg", "regprec", "mwg")])
def test_zoo_goldens_vs_live_reference(reference, name, model, method):
    """The zoo fixtures (tests/golden/make_golden.py) are outputs of the compiled
    reference: re-run its prior_init and two sweeps and compare bitwise."""
    import ast

    import numpy as np

    fx = golden(name)
    hyper = ast.literal_eval(str(fx["hyper"]))
    e = reference.open(model, hyper, method=method, seed=int(fx["seed"]), mh_scale=float(fx["mh_scale"]))
    for k in fx.files:
        if k.startswith("data_"):
            e.set(k[5:], fx[k])
    e.prior_init(int(fx["seed"]))
    latent = [k[:-1] for k in fx.files if k.endswith("0") and k[:-1] in fx.files and k != "lj0"]
    for n in latent:
        assert np.array_equal(e.get(n), fx[n + "0"]), n
    for it in range(2):
        lj, acc = e.sweep(it)
        assert lj == fx["lj"][it] and acc == bool(fx["accepted"][it])
        for n in latent:
            assert np.array_equal(e.get(n), fx[n][it]), (n, it)


def test_regprec_plans_tau_as_gamma_precision():
    """oracle/models/regprec.bn exercises the reference's GammaPrecision conjugate kind
    (rewrite.cpp:538-549): the reference CLI's `describe` of its Gibbs plan draws tau ~
    Gamma(3 + n/2, 1/(1/1 + rss/2))."""
    import subprocess

    cli = os.path.join(ROOT, "integration", "_build", "bnmc")
    if not os.path.exists(cli):
        pytest.skip("reference CLI not built (make -C integration)")
    d = subprocess.run([cli, "describe", "--model", os.path.join(ROOT, "oracle", "models", "regprec.bn"),
                        "--method", "gibbs"], capture_output=True, text=True, timeout=60).stdout
    assert "conjugate draw tau ~ Gamma(3 + n/2, 1/(1/(1) + rss/2))" in d, d
