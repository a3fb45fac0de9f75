"""The REFERENCE itself on the B200: its own sources, patched by
integration/reference_b200.patch (RunConfig::device, Engine::gpu_, the CLI's --device)
and linked to libbnmc_gpu.so through integration/gpu_backend.cpp.

Every test runs the reference's public API twice on the same inputs -- once with
RunConfig::device = Cpu (the reference's own CPU sweep), once with Device::B200 (the
Engine forwards sweep / eval_log_joint / run to the device) -- and requires the SURVEY.md
8c contract between the two: integer state bit-exact, reals <= 1e-12 (GMM mu / sigma2
1e-10), log-joints <= 1e-10.  Covered entry points: Engine::sweep, Engine::eval_log_joint,
Engine::run, sample() (sampler.cpp:557-568), map_estimate() (:570-584), lpp_curve
(bench.cpp:30-77) and the CLI `bnmc infer` (tools/main.cpp:68-130).
"""
import ast
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(ROOT, "integration"))
from b200ref import CLI, LIB, B200Ref  # noqa: E402

RTOL = 1e-12
RTOL_MU = 1e-10
RTOL_LJ = 1e-10


@pytest.fixture(scope="module")
def R():
    if not os.path.exists(LIB):
        pytest.skip("integration/_build not built (needs /root/reference at build time)")
    return B200Ref()


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def same_state(a: dict, b: dict, tol=RTOL):
    assert a.keys() == b.keys()
    for k in a:
        if np.asarray(a[k]).dtype == np.int64:
            assert np.array_equal(a[k], b[k]), f"{k}: {(np.asarray(a[k]) != np.asarray(b[k])).sum()} mismatches"
        else:
            assert rel(a[k], b[k]) < tol, (k, rel(a[k], b[k]))


def same_trace(t_gpu, t_cpu, tol=RTOL):
    assert len(t_gpu["log_joint"]) == len(t_cpu["log_joint"])
    assert rel(t_gpu["log_joint"], t_cpu["log_joint"]) < RTOL_LJ
    assert len(t_gpu["samples"]) == len(t_cpu["samples"])
    for a, b in zip(t_gpu["samples"], t_cpu["samples"]):
        same_state(a, b, tol)
    assert abs(t_gpu["map_log_joint"] - t_cpu["map_log_joint"]) <= RTOL_LJ * abs(t_cpu["map_log_joint"])
    same_state(t_gpu["map_state"], t_cpu["map_state"], tol)
    assert np.all(np.asarray(t_gpu["timing_ms"]) > 0)


def lda_pair(R, fx, **kw):
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    hyper = {"K": K, "V": V, "M": M, "N": np.diff(fx["offsets"]).tolist()}
    out = []
    for dev in ("b200", "cpu"):
        e = R.open("lda", hyper, "gibbs", int(fx["seed"]), device=dev, **kw)
        e.set("w", fx["w"])
        e.prior_init(int(fx["seed"]))
        out.append(e)
    assert out[0].on_device and not out[1].on_device
    return out


def test_engine_sweep_and_eval_log_joint(R):
    fx = golden("lda_desk")
    g, c = lda_pair(R, fx)
    assert abs(g.log_joint() - c.log_joint()) <= RTOL_LJ * abs(c.log_joint())
    for it in range(4):
        lg, _ = g.sweep(it)
        lc, _ = c.sweep(it)
        assert np.array_equal(g.get("z"), c.get("z")), it
        assert rel(g.get("phi"), c.get("phi")) < RTOL and rel(g.get("theta"), c.get("theta")) < RTOL
        assert abs(lg - lc) <= RTOL_LJ * abs(lc)
    # the reference's goldens, too (same seed, same prior_init): the first sweeps match
    assert np.array_equal(g.get("z"), fx["z"][3])


def test_engine_sweep_sees_caller_edits(R):
    """The store is borrowed per call: an edit of z between two sweeps is honoured."""
    fx = golden("lda_desk")
    g, c = lda_pair(R, fx)
    for e in (g, c):
        e.sweep(0)
        z = e.get("z")
        z[::7] = (z[::7] + 1) % int(fx["K"])
        e.set("z", z)
        e.sweep(1)
    assert np.array_equal(g.get("z"), c.get("z"))


@pytest.mark.parametrize("entry", ["run", "sample"])
def test_run_and_sample_traces(R, entry):
    fx = golden("lda_desk")
    g, c = lda_pair(R, fx, thin=2, burnin=1)
    tg = getattr(g, entry)(5)
    tc = getattr(c, entry)(5)
    assert len(tg["samples"]) == 3
    same_trace(tg, tc)
    assert np.array_equal(g.get("z"), c.get("z"))  # the store ends at the last sweep's state


def test_map_estimate_with_clamped_phi(R):
    fx = golden("lda_desk")
    g, c = lda_pair(R, fx)
    for e in (g, c):
        e.set("phi", fx["phi"][0])
        e.map_estimate(4, ["phi"])
    for v in ("z", "theta"):
        a, b = g.get(v), c.get(v)
        assert np.array_equal(a, b) if v == "z" else rel(a, b) < RTOL
    assert np.array_equal(g.get("phi"), fx["phi"][0])  # observed: never written


def test_lpp_curve_on_the_device(R):
    """lpp_curve builds its own RunConfig for every checkpoint's map_estimate: with the
    process default device B200 the fits run on the GPU."""
    fx = golden("lda_desk")
    _, c = lda_pair(R, fx)
    c.sample(5)  # the training trace (CPU), shared by both curves
    rs = np.random.default_rng(9)
    V = int(fx["V"])
    fit_len = np.full(10, 25)
    fit_w = rs.integers(0, V, fit_len.sum())
    test_off = np.arange(11) * 6
    test_w = rs.integers(0, V, 60)
    try:
        R.set_default_device("b200")
        pg = c.lpp_curve(fit_w, fit_len, test_w, test_off, 6, 77)
        R.set_default_device("cpu")
        pc = c.lpp_curve(fit_w, fit_len, test_w, test_off, 6, 77)
    finally:
        R.set_default_device("cpu")
    assert [p["samples"] for p in pg] == [1, 2, 4, 5]
    for a, b in zip(pg, pc):
        assert a["samples"] == b["samples"]
        assert abs(a["lpp"] - b["lpp"]) <= RTOL_LJ * abs(b["lpp"]), (a, b)


ZOO = [
    # model, golden, hyper, method, observed data names, mh_scale, tol for reals
    ("gmm", "gmm_small", {"N": 3000, "K": 4}, "gibbs", {"x": "x"}, 0.5, RTOL_MU),
    ("regression", "regression_gibbs", None, "mh", None, 0.1, RTOL),
    ("regression", "regression_gibbs", None, "gibbs", None, 0.1, RTOL),
    ("regression", "regression_gibbs", None, "mwg", None, 0.1, RTOL),
    ("catmix", "catmix_small", None, "gibbs", None, 0.5, RTOL),
    ("naivebayes", "naivebayes_small", None, "gibbs", None, 0.5, RTOL),
    ("hmm", "hmm_small", None, "gibbs", None, 0.5, RTOL),
    ("polyreg", "polyreg_small", None, "mh", None, 0.05, RTOL),
    ("polyreg", "polyreg_small", None, "gibbs", None, 0.05, RTOL),
    # the GammaPrecision kind through our test model oracle/models/regprec.bn
    ("regprec", "regprec_mh", None, "mh", None, 0.1, RTOL),
    ("regprec", "regprec_gibbs", None, "gibbs", None, 0.1, RTOL),
    ("regprec", "regprec_mwg", None, "mwg", None, 0.1, RTOL),
]


@pytest.mark.parametrize("model,gname,hyper,method,data,mh_scale,tol", ZOO,
                         ids=[f"{z[0]}-{z[3]}" for z in ZOO])
def test_zoo_sample_on_the_device(R, model, gname, hyper, method, data, mh_scale, tol):
    fx = golden(gname)
    hyper = hyper or ast.literal_eval(str(fx["hyper"]))
    data = data or {k[5:]: k for k in fx.files if k.startswith("data_")}
    seed = int(fx["seed"])
    traces = []
    for dev in ("b200", "cpu"):
        e = R.open(model, hyper, method, seed, mh_scale=mh_scale, device=dev, thin=1)
        for var, key in data.items():
            e.set(var, fx[key])
        e.prior_init(seed)
        traces.append(e.sample(4))
    same_trace(traces[0], traces[1], tol)


def test_unsupported_plans_are_refused(R):
    src = R.canonical_model("catmix").replace("beta = vector(K, 0.5)", "beta = vector(K, 0.7)")
    with pytest.raises(Exception, match="no device kernels"):
        R.open("catmix", {"N": 10, "K": 2, "V": 3}, source=src, device="b200")
    with pytest.raises(Exception, match="runs method"):
        R.open("lda", {"K": 2, "V": 5, "M": 1, "N": [3]}, "mh", device="b200")
    with pytest.raises(Exception, match="not supported on the device"):
        R.open("lda", {"K": 2, "V": 5, "M": 1, "N": [3]}, observe=["theta"], device="b200")
    # the same models run on the CPU device (the reference's own path)
    R.open("catmix", {"N": 10, "K": 2, "V": 3}, source=src, device="cpu").close()


def _cli(args, cwd):
    r = subprocess.run([CLI, *args], cwd=cwd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_cli_infer_with_lpp_metric(R, tmp_path):
    """bnmc gen + bnmc --device b200 infer --metric lpp: the reference's CLI end to end on
    the device; the trace and the lpp curve equal the CPU run's."""
    d = str(tmp_path)
    _cli(["gen", "--fixture", "lda", "--out", "train.json", "--docs", "40", "--vocab", "120", "--k", "5",
          "--doc-len", "50", "--heldout-docs", "8", "--heldout-out", "held.json", "--seed", "3"], d)
    outs = {}
    for dev in ("b200", "cpu"):
        _cli(["--device", dev, "infer", "--model", os.path.join(ROOT, "integration", "_build", "proj", "models",
                                                                 "lda.bn"),
              "--data", "train.json", "--samples", "6", "--seed", "5", "--omit-timing", "--out", f"t_{dev}.json",
              "--metric", "lpp", "--heldout", "held.json", "--fit-sweeps", "5", "--metric-out", f"lpp_{dev}.csv"], d)
        with open(os.path.join(d, f"t_{dev}.json")) as f:
            tr = json.load(f)
        lpp = np.loadtxt(os.path.join(d, f"lpp_{dev}.csv"), delimiter=",", skiprows=1)
        outs[dev] = (tr, lpp)
    (tg, lg), (tc, lc) = outs["b200"], outs["cpu"]
    assert rel(tg["log_joint"], tc["log_joint"]) < 1e-9  # printed with limited digits
    assert rel(lg[:, 1], lc[:, 1]) < 1e-9 and np.array_equal(lg[:, 0], lc[:, 0])
