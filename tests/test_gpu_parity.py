"""GPU parity: the CUDA path (through the C-ABI) against the reference's outputs.

Contract: integer state (z, counts, MH accept decisions) bit-exact;
phi/theta <= 1e-12 relative per element; GMM mu/sigma2 <= 1e-10; log-joint <= 1e-10
relative.  The float tolerances exist because device log/exp/cos/pow may differ from
glibc's by an ulp (the RNG integer stream itself is bit-exact).
"""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

RTOL_PARAM = 1e-12
RTOL_MU = 1e-10
RTOL_LJ = 1e-10


@pytest.fixture(scope="module")
def g():
    import paper_1312_3613_b200 as g

    g.lib()
    return g


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


# ----------------------------------------------------------------------------------------
# primitives
# ----------------------------------------------------------------------------------------
def test_rng_bit_exact(g):
    r = golden("rng_dist")
    u, un, ga = g.probe_rng(r["keys"], 16)
    assert np.array_equal(u, r["u64"])            # integer stream: bit-exact
    assert np.array_equal(un, r["unit"])          # (u >> 11 + 0.5) * 2^-53: exact
    assert rel(ga, r["gauss"]) < 1e-14            # Box-Muller through device log/cos


def test_gamma_draws(g):
    r = golden("rng_dist")
    shapes = np.repeat(r["gamma_shapes"], len(r["gamma_keys"]))
    keys = np.tile(r["gamma_keys"], len(r["gamma_shapes"]))
    out, cnt = g.probe_gamma(keys, shapes)
    assert np.array_equal(cnt, r["gamma_counters"].ravel())  # same rejection path everywhere
    assert rel(out, r["gamma"].ravel()) < RTOL_PARAM


def test_draw_from_log_weights(g):
    r = golden("rng_dist")
    picks = g.probe_log_weights(r["logw_keys"], r["logw"])
    assert np.array_equal(picks[picks >= 0], r["logw_picks"][picks >= 0])


def test_dirichlet_batch(g):
    r = golden("rng_dist")
    out = g.dirichlet_batch(r["dir_alpha"], int(r["dir_key"]))
    assert rel(out, r["dir_out"]) < RTOL_PARAM
    with pytest.raises(ValueError):
        g.dirichlet_batch(np.array([[1.0, 0.0]]), 1)


# ----------------------------------------------------------------------------------------
# LDA
# ----------------------------------------------------------------------------------------
def lda_engine(g, fx, exact=False, graph=True, observe=()):
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    lengths = np.diff(fx["offsets"])
    hyper = {"K": K, "V": V, "M": M, "N": lengths.tolist()}
    cfg = g.RunConfig(seed=int(fx["seed"]), exact_weights=exact, use_graph=graph, observe_extra=list(observe))
    e = g.Engine("lda", hyper, cfg)
    s = e.allocate()
    s["w"] = fx["w"]
    s["z"] = fx["z0"]
    s["phi"] = fx["phi0"]
    s["theta"] = fx["theta0"]
    return e, s


@pytest.mark.parametrize("name", ["lda_desk", "lda_ragged", "lda_k1"])
@pytest.mark.parametrize("exact", [False, True])
def test_lda_sweeps_vs_reference(g, name, exact):
    fx = golden(name)
    e, s = lda_engine(g, fx, exact=exact)
    assert abs(e.eval_log_joint(s) - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"])
    for it in range(len(fx["lj"])):
        lj = e.sweep(s, it)
        assert np.array_equal(s["z"], fx["z"][it]), f"z mismatch at sweep {it}: {(s['z'] != fx['z'][it]).sum()}"
        assert rel(s["phi"], fx["phi"][it]) < RTOL_PARAM
        assert rel(s["theta"], fx["theta"][it]) < RTOL_PARAM
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])
    e.close()


def test_lda_counts_bit_exact(g):
    fx = golden("lda_desk")
    e, s = lda_engine(g, fx)
    e.upload(s)
    K, V = int(fx["K"]), int(fx["V"])
    nkw, nmk = e.lda_counts()
    z, w, off = fx["z0"], fx["w"], fx["offsets"]
    want = np.zeros((K, V), dtype=np.int64)
    np.add.at(want, (z, w), 1)
    assert np.array_equal(nkw, want)
    docs = np.repeat(np.arange(len(off) - 1), np.diff(off))
    wm = np.zeros((len(off) - 1, K), dtype=np.int64)
    np.add.at(wm, (docs, z), 1)
    assert np.array_equal(nmk, wm)
    assert nkw.sum() == len(z)


def test_lda_graph_equals_direct_launch(g):
    fx = golden("lda_desk")
    e1, s1 = lda_engine(g, fx, graph=True)
    e2, s2 = lda_engine(g, fx, graph=False)
    for it in range(3):
        assert e1.sweep(s1, it) == e2.sweep(s2, it)
        assert np.array_equal(s1["z"], s2["z"]) and np.array_equal(s1["phi"], s2["phi"])


def test_lda_run_matches_stepwise(g):
    """run_device (one host sync for n sweeps) == n single sweeps, bitwise."""
    fx = golden("lda_desk")
    e1, s1 = lda_engine(g, fx)
    e2, s2 = lda_engine(g, fx)
    e1.upload(s1)
    lj, _ = e1.run_device(0, 4)
    e1.download(s1)
    ljs = [e2.sweep(s2, it) for it in range(4)]
    assert np.array_equal(lj, ljs)
    assert np.array_equal(s1["z"], s2["z"]) and np.array_equal(s1["theta"], s2["theta"])


def test_lda_observed_phi_never_written(g, restatement):
    """Clamped phi (bench.cpp:30-77 protocol): no phi block, phi untouched, z exact."""
    fx = golden("lda_desk")
    e, s = lda_engine(g, fx, observe=("phi",))
    phi0 = s["phi"].copy()
    K, V = int(fx["K"]), int(fx["V"])
    off, w = fx["offsets"], fx["w"]
    z, phi, theta = fx["z0"].copy(), fx["phi0"].copy(), fx["theta0"].copy()
    for it in range(3):
        lj = e.sweep(s, it)
        lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, int(fx["seed"]), it, observe_phi=True)
        assert np.array_equal(s["phi"], phi0)
        assert np.array_equal(s["z"], z)
        assert abs(lj - lj2) <= RTOL_LJ * abs(lj2)


def test_lda_bad_assignment_raises(g):
    fx = golden("lda_desk")
    e, s = lda_engine(g, fx)
    z = s["z"].copy()
    z[3] = int(fx["K"])  # outside the support
    s["z"] = z
    with pytest.raises(g.BnmcError):
        e.upload(s)


@pytest.mark.parametrize("K", [7, 300])
def test_lda_bound_store_transfers(g, K):
    """Engine::sweep on a bound store: the bytes moved per call (z up; z, theta, phi and
    the ring entry down), the caller's edits between calls are what the next sweep
    reads, and an out-of-range edit raises through the device check."""
    rs = np.random.default_rng(K)
    V, M, L = 50, 12, 30
    N = M * L
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    e = g.Engine("lda", hyper, g.RunConfig(seed=3))
    s = e.allocate()
    s["w"] = rs.integers(0, V, N)
    e.prior_init(s, 3)
    e.sweep(s, 0)  # binds
    e.sweep(s, 1)
    up, down = e.transfer_stats()
    assert up == N * 8
    assert down == N * 8 + M * K * 8 + K * V * 8 + 8 + 4
    # the caller's edit is what the next sweep reads: same result as a fresh engine
    z = s["z"].copy()
    z[::3] = (z[::3] + 1) % K
    s["z"] = z
    e2 = g.Engine("lda", hyper, g.RunConfig(seed=3))
    s2 = e2.allocate()
    for n in s.names:
        s2[n] = s[n].copy()
    lj = e.sweep(s, 2)
    lj2 = e2.sweep(s2, 2)
    assert lj == lj2 and np.array_equal(s["z"], s2["z"]) and np.array_equal(s["phi"], s2["phi"])
    bad = s["z"].copy()
    bad[5] = K
    s["z"] = bad
    with pytest.raises(g.BnmcError):
        e.sweep(s, 3)
    bad[5] = -1
    s["z"] = bad
    with pytest.raises(g.BnmcError):
        e.sweep(s, 3)
    e.close()
    e2.close()


@pytest.mark.parametrize("nccl", [False, True], ids=["single", "nccl-path"])
def test_lda_speculative_sweep_store(g, monkeypatch, nccl):
    """Repeated Engine::sweep calls on a bound store start from the device state while
    the store's z is uploaded (sweep_store speculation).  Results must equal the
    non-speculative path's call by call, including when the caller edits z between
    calls (the upload differs -> redo from it) or writes an invalid value (-> error)."""
    rs = np.random.default_rng(5)
    K, V, M, L = 20, 60, 16, 40
    N = M * L
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}

    def make():
        e = g.Engine("lda", hyper, g.RunConfig(seed=9))
        s = e.allocate()
        s["w"] = np.random.default_rng(1).integers(0, V, N)
        e.prior_init(s, 9)
        return e, s

    if nccl:  # the collective speculate / redo decisions, on a 1-rank communicator
        monkeypatch.setenv("BNMC_FORCE_NCCL", "1")
    e1, s1 = make()  # speculative (default)
    monkeypatch.setenv("BNMC_SPECULATE", "0")
    e2, s2 = make()
    monkeypatch.delenv("BNMC_SPECULATE")
    for it in range(8):
        if it in (4, 6):  # the caller edits the store between calls
            z = s1["z"].copy()
            z[rs.integers(0, N, 7)] = rs.integers(0, K, 7)
            s1["z"] = z
            s2["z"] = z.copy()
        lj1, lj2 = e1.sweep(s1, it), e2.sweep(s2, it)
        assert lj1 == lj2, it
        for n in ("z", "phi", "theta"):
            assert np.array_equal(s1[n], s2[n]), (it, n)
    bad = s1["z"].copy()
    bad[3] = K
    s1["z"] = bad
    with pytest.raises(g.BnmcError):
        e1.sweep(s1, 8)
    e1.close()
    e2.close()


def test_mh_bound_store_unchanged_skip(g, monkeypatch):
    """MH on a bound store skips the upload and the likelihood refresh when the store
    still holds the state last written back; results equal the always-upload path's
    call by call, including after the caller edits a weight."""
    rs = np.random.default_rng(2)
    N, K = 5000, 6
    x = rs.uniform(-1, 1, size=(N, K))
    y = (rs.random(N) < 0.5).astype(np.float64)
    hyper = {"N": N, "K": K, "l": -1.0, "u": 1.0}

    def make():
        e = g.Engine("logreg", hyper, g.RunConfig(seed=4, mh_scale=0.05))
        s = e.allocate()
        s["x"], s["y"] = x.ravel(), y
        e.prior_init(s, 4)
        return e, s

    e1, s1 = make()
    monkeypatch.setenv("BNMC_SPECULATE", "0")
    e2, s2 = make()
    monkeypatch.delenv("BNMC_SPECULATE")
    for it in range(10):
        if it == 6:
            for s in (s1, s2):
                w = s["w"].copy()
                w[1] += 0.25
                s["w"] = w
        acc1, acc2 = [], []
        lj1, lj2 = e1.sweep(s1, it, acc1), e2.sweep(s2, it, acc2)
        assert lj1 == lj2 and acc1 == acc2, it
        assert np.array_equal(s1["w"], s2["w"]) and np.array_equal(s1["b"], s2["b"]), it
    e1.close()
    e2.close()


def test_cpp_mirror_matches_python_engine(g, tmp_path):
    """include/bnmc_gpu.hpp driving the GPU path as a reference caller drives bnmc::Engine
    (prior_init, eval_log_joint, 5 x sweep, run with thin 2): every value equals the
    Python engine's over the same library."""
    import os
    import subprocess

    from conftest import ROOT

    K, V, M, L, seed = 6, 50, 8, 40, 17
    w = np.random.default_rng(3).integers(0, V, M * L).astype(np.int64)
    wp = tmp_path / "w.bin"
    w.tofile(wp)
    exe = tmp_path / "lda_engine_example"
    lib = os.path.join(ROOT, "paper_1312_3613_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "lda_engine_example.cpp"), "-L", lib, "-lbnmc_gpu",
                        f"-Wl,-rpath,{lib}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), str(wp), str(K), str(V), str(L), str(seed)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    got = {}
    for line in r.stdout.splitlines():
        parts = line.split()
        got[" ".join(parts[:-1])] = float(parts[-1])

    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": [L] * M}, g.RunConfig(seed=seed, thin=2))
    s = e.allocate()
    s["w"] = w
    e.prior_init(s, seed)
    assert got["prior"] == e.eval_log_joint(s)
    for i in range(5):
        assert got[f"sweep {i}"] == e.sweep(s, i), i
    tr = e.run(s, 4)
    for i, v in enumerate(tr["log_joint"]):
        assert got[f"run {i}"] == v, i
    assert got["map"] == tr["map_log_joint"]
    assert got["samples"] == len(tr["samples"]) == 2
    assert got["eval"] == e.eval_log_joint(s)
    assert got["z0"] == s["z"][0]
    e.close()


def _gen_lda(restatement, reference, M, V, K, L, seed):
    w, _, _ = reference.gen_lda(M, V, K, L, seed)
    off = np.arange(M + 1, dtype=np.int64) * L
    phi, theta, z = restatement.lda_prior_init(K, V, off, w, seed)
    return w, off, phi, theta, z


@pytest.mark.parametrize("cfg,env", [(("kos", 3430, 6906, 50, 136), {}), (("nips", 1500, 12419, 100, 1267), {})],
                         ids=["kos", "nips"])
def test_lda_full_size_one_sweep(g, restatement, reference, monkeypatch, cfg, env):
    """KOS / NIPS-shaped corpora: one sweep from the reference's prior_init
    state; z and the counts must be bit-exact (0 mismatches), floats within tolerance."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    name, M, V, K, L = cfg
    seed = 42
    w, off, phi, theta, z = _gen_lda(restatement, reference, M, V, K, L, seed)
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
    s = e.allocate()
    s["w"], s["z"], s["phi"], s["theta"] = w, z, phi, theta
    lj = e.sweep(s, 0)
    lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, seed, 0)
    mism = int((s["z"] != z).sum())
    assert mism == 0, f"{name}: {mism} z mismatches of {len(z)}"
    assert rel(s["phi"], phi) < RTOL_PARAM
    assert rel(s["theta"], theta) < RTOL_PARAM
    assert abs(lj - lj2) <= RTOL_LJ * abs(lj2)
    nkw, _ = e.lda_counts()
    want = np.zeros((K, V), dtype=np.int64)
    np.add.at(want, (z, w), 1)
    assert np.array_equal(nkw, want)


def test_lda_device_prior_init_matches_reference(g, restatement):
    fx = golden("lda_desk")
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    e, s = lda_engine(g, fx)
    e.prior_init(s, int(fx["seed"]))
    assert rel(s["phi"], fx["phi0"]) < RTOL_PARAM
    assert rel(s["theta"], fx["theta0"]) < RTOL_PARAM
    assert np.array_equal(s["z"], fx["z0"])


@pytest.mark.parametrize("V,K", [(12419, 100), (100000, 4), (2048, 3)], ids=["nips", "v1e5", "v2048"])
def test_lda_prior_init_long_rows(g, restatement, monkeypatch, V, K):
    """prior_init's phi rows (V gammas from one stream each, dist.cpp:193-200) drawn by the
    segmented walk (lda.cu dirichlet_rows): bitwise the thread-per-row draw, and the
    restatement (pinned to the reference) within tolerance; z exact."""
    M, L, seed = 24, 40, 11
    w = np.random.default_rng(seed).integers(0, V, M * L).astype(np.int64)
    off = np.arange(M + 1, dtype=np.int64) * L
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    got = {}
    for serial in ("1", "0"):
        monkeypatch.setenv("BNMC_PRIOR_SERIAL", serial)
        e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
        s = e.allocate()
        s["w"] = w
        e.prior_init(s, seed)
        got[serial] = (s["phi"].copy(), s["theta"].copy(), s["z"].copy())
        e.close()
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)
    phi, theta, z = restatement.lda_prior_init(K, V, off, w, seed)
    assert rel(got["0"][0], phi) < RTOL_PARAM
    assert rel(got["0"][1], theta) < RTOL_PARAM
    assert np.array_equal(got["0"][2], z)


@pytest.mark.parametrize("phi_conc", [0.05, 2.0], ids=["boost", "no-boost"])
def test_lda_generate_long_rows(g, monkeypatch, phi_conc):
    """lda_generate's true-phi rows (concentration 0.05 as gen.cpp:26-31, and 2.0: gammas
    without the shape < 1 boost, 3 counters per attempt) through the segmented walk: the
    corpus and the prior state equal the thread-per-row draw's."""
    K, V, M, L, seed = 6, 100000, 16, 64, 5
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    got = {}
    for serial in ("1", "0"):
        monkeypatch.setenv("BNMC_PRIOR_SERIAL", serial)
        e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
        e.lda_generate(seed, phi_conc=phi_conc)
        s = e.allocate()
        e.download(s)
        got[serial] = (e.lda_counts()[0].copy(), s["phi"].copy(), s["z"].copy())
        e.close()
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("K", [7, 1000, 2048], ids=["k7", "k1000", "k2048"])
def test_lda_doc_running_sums_equal_the_scan(g, monkeypatch, K):
    """prior_init's z and lda_generate's tokens pick topics by a binary search over each
    document's running sums (formed left to right in shared memory): the same picks as the
    reference's linear scan (draw_categorical, dist.cpp:183-191), bit for bit."""
    V, M, L, seed = 300, 12, 333, 8
    hyper = {"K": K, "V": V, "M": M, "N": [L + (m % 3) for m in range(M)]}
    got = {}
    for scan in ("1", "0"):
        monkeypatch.setenv("BNMC_DOC_SCAN", scan)
        e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
        e.lda_generate(seed)
        s = e.allocate()
        e.download(s)
        got[scan] = (e.lda_counts()[0].copy(), s["z"].copy(), s["theta"].copy())
        e.close()
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("K,V,block_docs", [(1000, 5000, 3), (300, 20000, 7), (150, 3000, 1), (1000, 100000, 0)],
                         ids=["k1000", "k300", "k150", "k1000-v1e5-default"])
def test_lda_word_major_zstep_equals_document_major(g, monkeypatch, K, V, block_docs):
    """The word-major z-step order (tokens sorted by (document block, word), the word's
    row resident, theta/S rows streamed) draws bitwise the document-major z: same
    products, sums and decisions (sampler.cpp:222-265); 3 sweeps, ragged and empty docs."""
    rng = np.random.default_rng(K + V)
    lens = rng.integers(0, 400, 40)
    lens[3] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    w = rng.integers(0, V, int(off[-1])).astype(np.int64)
    hyper = {"K": K, "V": V, "M": len(lens), "N": [int(x) for x in lens]}
    got = {}
    for wm in ("0", "1"):
        monkeypatch.setenv("BNMC_ZSTEP_WM", wm)
        if block_docs:
            monkeypatch.setenv("BNMC_WM_BLOCK_DOCS", str(block_docs))
        e = g.Engine("lda", hyper, g.RunConfig(seed=17))
        s = e.allocate()
        s["w"] = w
        e.prior_init(s, 17)
        ljs = [e.sweep(s, it) for it in range(3)]
        got[wm] = (ljs, s["z"].copy(), s["phi"].copy(), s["theta"].copy(), e.lda_counts()[0].copy())
        e.close()
    assert got["0"][0] == got["1"][0]
    for a, b in zip(got["0"][1:], got["1"][1:]):
        assert np.array_equal(a, b)


def test_lda_1b_word_major_equals_document_major_at_full_size(g, monkeypatch):
    """The 1B config itself (1e6 documents x 1000 tokens, K=1000, V=1e5; device generator +
    prior_init): two sweeps in the word-major order and in the document-major order give
    the same log-joints (bitwise) and the same topic-word counts."""
    K, V, M, L, seed = 1000, 100000, 1000000, 1000, 2024
    hyper = {"K": K, "V": V, "M": M, "N": [L] * M}
    got = {}
    for wm in ("1", "0"):
        monkeypatch.setenv("BNMC_ZSTEP_WM", wm)
        e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
        e.lda_generate(seed)
        lj, _ = e.run_device(0, 2)
        nkw, _ = e.lda_counts()
        got[wm] = (lj, nkw.sum(axis=1).copy(), nkw[:, :2000].copy())
        e.close()
    assert int(got["1"][1].sum()) == M * L
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("K,V,margin", [(100, 6000, None), (100, 6000, "1.0"), (300, 8000, None), (300, 8000, "1.0")],
                         ids=["k100", "k100-all-fallback", "k300", "k300-all-fallback"])
def test_lda_exact_weights_screen_equals_unscreened(g, monkeypatch, K, V, margin):
    """Exact-weights (log-space) mode: the fp32 screen + log-space fallback draws the
    topics of the unscreened log-space z-step (draw_from_log_weights, dist.cpp:202-215)
    over 3 sweeps; margin 1.0 sends every token through zfallback_log_kernel."""
    rng = np.random.default_rng(K)
    lens = rng.integers(50, 700, 300)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    w = rng.integers(0, V, int(off[-1])).astype(np.int64)
    hyper = {"K": K, "V": V, "M": len(lens), "N": [int(x) for x in lens]}
    got = {}
    for screen in ("0", "1"):
        monkeypatch.setenv("BNMC_ZSTEP_SCREEN", screen)
        if margin and screen == "1":
            monkeypatch.setenv("BNMC_SCREEN_MARGIN", margin)
        e = g.Engine("lda", hyper, g.RunConfig(seed=23, exact_weights=True))
        s = e.allocate()
        s["w"] = w
        e.prior_init(s, 23)
        ljs = [e.sweep(s, it) for it in range(3)]
        got[screen] = (ljs, s["z"].copy(), s["phi"].copy(), s["theta"].copy())
        e.close()
    assert np.array_equal(got["0"][1], got["1"][1])
    assert np.array_equal(got["0"][2], got["1"][2]) and np.array_equal(got["0"][3], got["1"][3])
    # (the w-factor: n (log g - log S) screened, n log(g / S) unscreened)
    for a, b in zip(got["0"][0], got["1"][0]):
        assert abs(a - b) <= RTOL_LJ * abs(b)


# ----------------------------------------------------------------------------------------
# GMM and MH
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "six-kernel"])
def test_gmm_sweeps_vs_reference(g, monkeypatch, fused):
    if not fused:
        monkeypatch.setenv("BNMC_GMM_FUSED", "0")
    fx = golden("gmm_small")
    hyper = {"N": int(fx["N"]), "K": 4}
    e = g.Engine("gmm", hyper, g.RunConfig(seed=int(fx["seed"])))
    s = e.allocate()
    s["x"], s["z"], s["pi"], s["mu"], s["sigma2"] = fx["x"], fx["z0"], fx["pi0"], fx["mu0"], fx["sigma20"]
    for it in range(len(fx["lj"])):
        lj = e.sweep(s, it)
        assert np.array_equal(s["z"], fx["z"][it])
        assert rel(s["pi"], fx["pi"][it]) < RTOL_PARAM
        assert rel(s["mu"], fx["mu"][it]) < RTOL_MU
        assert rel(s["sigma2"], fx["sigma2"][it]) < RTOL_MU
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])


def test_mh_linreg_vs_reference(g):
    fx = golden("mh_linreg")
    N, K = int(fx["N"]), int(fx["K"])
    e = g.Engine("regression", {"N": N, "K": K, "l": -1.0, "u": 1.0}, g.RunConfig(seed=int(fx["seed"])))
    s = e.allocate()
    s["x"], s["y"], s["w"], s["b"], s["tau"] = fx["x"], fx["y"], fx["w0"], [fx["b0"]], [fx["tau0"]]
    assert abs(e.eval_log_joint(s) - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"])
    for it in range(len(fx["lj"])):
        acc = []
        lj = e.sweep(s, it, acc)
        assert acc[0] == bool(fx["accepted"][it]), f"accept decision differs at step {it}"
        assert rel(s["w"], fx["w"][it]) < RTOL_PARAM
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])


def test_mh_logreg_vs_restatement(g, restatement):
    """Logistic MH: parity with the restated oracle (no reference model exists)."""
    rs = np.random.default_rng(5)
    N, K = 4000, 8
    x = rs.uniform(-1, 1, size=(N, K))
    wt = 0.3 * rs.normal(size=K)
    p = 1 / (1 + np.exp(-(x @ wt + 0.1)))
    y = (rs.uniform(size=N) < p).astype(np.float64)
    e = g.Engine("logreg", {"N": N, "K": K, "l": -1.0, "u": 1.0}, g.RunConfig(seed=3, mh_scale=0.05))
    s = e.allocate()
    s["x"], s["y"] = x.ravel(), y
    w, b = np.zeros(K), 0.0
    s["w"], s["b"] = w, [b]
    xs = np.ascontiguousarray(x.ravel())
    for it in range(20):
        acc = []
        lj = e.sweep(s, it, acc)
        b, _, lj2, acc2 = restatement.mh_step(xs, y, K, w, b, 0.0, 3, it, logistic=True, mh_scale=0.05)
        assert acc[0] == acc2
        assert rel(s["w"], w) < RTOL_PARAM
        assert abs(lj - lj2) <= RTOL_LJ * abs(lj2)


def test_lpp_vs_reference(g, reference):
    K, V, M, L = 6, 80, 12, 30
    rs = np.random.default_rng(1)
    phi = rs.dirichlet(np.ones(V), size=K)
    theta = rs.dirichlet(np.ones(K), size=M)
    w = rs.integers(0, V, M * L).astype(np.int64)
    off = np.arange(M + 1, dtype=np.int64) * L
    import ctypes
    out = ctypes.c_double()
    dp, ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
    pc, tc = np.ascontiguousarray(phi.ravel()), np.ascontiguousarray(theta.ravel())
    reference._check(reference.lib.bref_lpp(pc.ctypes.data_as(dp), tc.ctypes.data_as(dp), K, V,
                                            w.ctypes.data_as(ip), off.ctypes.data_as(ip), M, ctypes.byref(out)))
    got = g.log_predictive_probability(pc, tc, K, V, w, off)
    assert abs(got - out.value) <= 1e-10 * abs(out.value)


# ----------------------------------------------------------------------------------------
# z-step layouts: every screen / fallback instantiation against the restatement
# ----------------------------------------------------------------------------------------
def _ragged_corpus(restatement, K, V, M, seed):
    rs = np.random.default_rng(seed)
    lengths = rs.integers(0, 90, M)
    lengths[0] = 0          # an empty document
    lengths[1] = 700        # one document spanning several 512-token work units
    off = np.zeros(M + 1, dtype=np.int64)
    off[1:] = np.cumsum(lengths)
    # Zipf-like word frequencies (some words frequent: count-table contention)
    pw = 1.0 / np.arange(1, V + 1) ** 1.1
    w = rs.choice(V, size=int(off[-1]), p=pw / pw.sum()).astype(np.int64)
    phi, theta, z = restatement.lda_prior_init(K, V, off, w, seed)
    return off, w, phi, theta, z


LAYOUTS = [
    # (K, env): transposed screen (K <= 128, every round count), grouped screens, big K
    (1, {}), (5, {}), (32, {}), (33, {}), (64, {}), (100, {}), (128, {}),
    (129, {}), (200, {}), (256, {}), (300, {}), (512, {}), (513, {}), (1000, {}),
    (100, {"BNMC_ZSCREEN": "g4w8s"}), (100, {"BNMC_ZSCREEN": "g8w4r"}),
    (100, {"BNMC_ZSCREEN": "g16w4s"}), (100, {"BNMC_ZSCREEN": "g32w4r"}),
    (100, {"BNMC_ZSTEP_THETA": "smem"}),
    (100, {"BNMC_ZT_WU": "1"}), (33, {"BNMC_ZT_WU": "1", "BNMC_ZSTEP_THETA": "smem"}), (64, {"BNMC_ZT_WU": "0"}),
    # every token through the fp64 fallback queue
    (100, {"BNMC_SCREEN_MARGIN": "1.0"}), (1000, {"BNMC_SCREEN_MARGIN": "1.0"}),
    # screen off: the grouped fp64 kernel
    (100, {"BNMC_ZSTEP_SCREEN": "0"}), (1000, {"BNMC_ZSTEP_SCREEN": "0"}),
]


@pytest.mark.parametrize("K,V", [(600, 9000), (40, 140000)], ids=["K600-V9000", "K40-V140000"])
def test_lda_pool_multichunk_vs_restatement(g, restatement, K, V):
    """The warp-pool conjugate block with more than one shared-memory count chunk per
    warp (K V > 1024 cells per resident warp: 5.4 M / 5.6 M cells) -- chunk boundaries,
    the next-chunk prefetch, phi and theta cells in one range -- two sweeps bit-exact in z
    against the restatement."""
    M, seed = 30, 77
    off, w, phi, theta, z = _ragged_corpus(restatement, K, V, M, seed)
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": np.diff(off).tolist()}, g.RunConfig(seed=seed))
    s = e.allocate()
    s["w"], s["z"], s["phi"], s["theta"] = w, z, phi, theta
    for it in range(2):
        lj = e.sweep(s, it)
        lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, seed, it)
        assert int((s["z"] != z).sum()) == 0
        assert rel(s["phi"], phi) < RTOL_PARAM
        assert rel(s["theta"], theta) < RTOL_PARAM
        assert abs(lj - lj2) <= RTOL_LJ * abs(lj2)
    e.close()


@pytest.mark.parametrize("K,env", LAYOUTS, ids=[f"K{k}-" + "-".join(f"{a}={b}" for a, b in e.items()) for k, e in LAYOUTS])
def test_lda_layouts_vs_restatement(g, restatement, monkeypatch, K, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    V, M, seed = 400, 40, 11 + K
    off, w, phi, theta, z = _ragged_corpus(restatement, K, V, M, seed)
    hyper = {"K": K, "V": V, "M": M, "N": np.diff(off).tolist()}
    e = g.Engine("lda", hyper, g.RunConfig(seed=seed))
    s = e.allocate()
    s["w"], s["z"], s["phi"], s["theta"] = w, z, phi, theta
    for it in range(3):
        lj = e.sweep(s, it)
        lj2 = restatement.lda_sweep(K, V, off, w, z, phi, theta, seed, it)
        mism = int((s["z"] != z).sum())
        assert mism == 0, f"sweep {it}: {mism} z mismatches of {len(z)}"
        assert rel(s["phi"], phi) < RTOL_PARAM
        assert rel(s["theta"], theta) < RTOL_PARAM
        assert abs(lj - lj2) <= RTOL_LJ * abs(lj2)
    nkw, nmk = e.lda_counts()
    want = np.zeros((K, V), dtype=np.int64)
    np.add.at(want, (z, w), 1)
    assert np.array_equal(nkw, want)
    e.close()


# ----------------------------------------------------------------------------------------
# Engine::run with the device-resident trace (bnmc_gpu_run_trace)
# ----------------------------------------------------------------------------------------
def _stepwise_run(e, s, burnin, n, thin, names):
    """Engine::run (sampler.cpp:426-455) restated over single device sweeps."""
    lj, samples, map_lj, map_state = [], [], -np.inf, None
    for it in range(burnin + n):
        v = e.sweep(s, it)
        if it < burnin:
            continue
        k = it - burnin
        lj.append(v)
        if k % thin == 0:
            samples.append({x: s[x].copy() for x in names})
        if v > map_lj:
            map_lj, map_state = v, {x: s[x].copy() for x in names}
    return lj, samples, map_lj, map_state


@pytest.mark.parametrize("model", ["lda", "gmm", "regression"])
def test_run_trace_matches_stepwise(g, model):
    if model == "lda":
        fx = golden("lda_desk")
        mk = lambda: lda_engine(g, fx)  # noqa: E731
        names = ["phi", "theta", "z"]
    elif model == "gmm":
        fx = golden("gmm_small")

        def mk():
            e = g.Engine("gmm", {"N": int(fx["N"]), "K": 4}, g.RunConfig(seed=int(fx["seed"]), burnin=2, thin=3))
            s = e.allocate()
            s["x"], s["z"], s["pi"], s["mu"], s["sigma2"] = fx["x"], fx["z0"], fx["pi0"], fx["mu0"], fx["sigma20"]
            return e, s
        names = ["pi", "mu", "sigma2", "z"]
    else:
        fx = golden("mh_linreg")

        def mk():
            N, K = int(fx["N"]), int(fx["K"])
            e = g.Engine("regression", {"N": N, "K": K, "l": -1.0, "u": 1.0},
                         g.RunConfig(seed=int(fx["seed"]), burnin=2, thin=3))
            s = e.allocate()
            s["x"], s["y"], s["w"], s["b"], s["tau"] = fx["x"], fx["y"], fx["w0"], [fx["b0"]], [fx["tau0"]]
            return e, s
        names = ["w", "b", "tau"]
    burnin, n, thin = 2, 7, 3
    e1, s1 = mk()
    e1.cfg.burnin, e1.cfg.thin = burnin, thin
    tr = e1.run(s1, n)
    e2, s2 = mk()
    lj, samples, map_lj, map_state = _stepwise_run(e2, s2, burnin, n, thin, names)
    assert tr["log_joint"] == lj
    assert len(tr["samples"]) == len(samples) == 3
    for a, b in zip(tr["samples"], samples):
        for x in names:
            assert np.array_equal(a[x], b[x]), x
    assert tr["map_log_joint"] == map_lj
    for x in names:
        assert np.array_equal(tr["map_state"][x], map_state[x]), x
        assert np.array_equal(s1[x], s2[x]), x  # the store holds the final state
    assert len(tr["timing_ms"]) == n and all(t > 0 for t in tr["timing_ms"])


# ----------------------------------------------------------------------------------------
# the rest of the zoo: catmix, naivebayes, hmm (sequential scan), polyreg MH
# ----------------------------------------------------------------------------------------
ZOO = [("catmix_small", "catmix"), ("naivebayes_small", "naivebayes"), ("hmm_small", "hmm"),
       ("polyreg_small", "polyreg"), ("polyreg_gibbs", "polyreg"), ("regression_gibbs", "regression"),
       ("polyreg_mwg", "polyreg"), ("regression_mwg", "regression"),
       # the GammaPrecision conjugate kind (oracle/models/regprec.bn) under MH, Gibbs, MWG
       ("regprec_mh", "regprec"), ("regprec_gibbs", "regprec"), ("regprec_mwg", "regprec")]


def _zoo_engine(g, fx, model):
    import ast
    hyper = ast.literal_eval(str(fx["hyper"]))
    method = str(fx["method"]) if "method" in fx.files else ""
    cfg = g.RunConfig(seed=int(fx["seed"]), mh_scale=float(fx["mh_scale"]), method=method)
    e = g.Engine(model, hyper, cfg)
    s = e.allocate()
    for k in fx.files:
        if k.startswith("data_"):
            s[k[5:]] = fx[k]
    latent = [n for n in s.names if not s.observed[n]]
    return e, s, latent


@pytest.mark.parametrize("name,model", ZOO)
def test_zoo_prior_init_matches_reference(g, name, model):
    fx = golden(name)
    e, s, latent = _zoo_engine(g, fx, model)
    e.prior_init(s, int(fx["seed"]))
    for n in latent:
        if s[n].dtype == np.int64:
            assert np.array_equal(s[n], fx[n + "0"]), n
        else:
            assert rel(s[n], fx[n + "0"]) < RTOL_PARAM, n
    e.close()


@pytest.mark.parametrize("N,S", [(60000, 3), (40001, 16), (5000, 17)], ids=["s3", "s16", "s17-serial"])
def test_hmm_prior_chain_chunked(g, monkeypatch, N, S):
    """The HMM prior chain s[t] ~ Cat(T[s[t-1]]) (sampler.cpp:542-555) drawn as composed
    chunk maps equals the step-by-step chain (BNMC_PRIOR_SERIAL=1), bit for bit."""
    flips = np.random.default_rng(1).integers(0, 2, N).astype(np.int64)
    got = {}
    for serial in ("1", "0"):
        monkeypatch.setenv("BNMC_PRIOR_SERIAL", serial)
        e = g.Engine("hmm", {"N": N, "S": S}, g.RunConfig(seed=13))
        s = e.allocate()
        s["flips"] = flips
        e.prior_init(s, 13)
        got[serial] = (s["s"].copy(), s["T"].copy(), s["bias"].copy())
        e.close()
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)
    assert len(np.unique(got["0"][0])) > 1


@pytest.mark.parametrize("N,S", [(100000, 3), (30001, 16), (4000, 64)], ids=["s3", "s16", "s64"])
def test_hmm_chunked_scan_equals_the_sequential_scan(g, monkeypatch, N, S):
    """The HMM s-scan (each site sees the new s[t-1] and the old s[t+1], sampler.cpp:259-264)
    run as composed chunk maps equals the site-by-site scan (BNMC_HMM_SERIAL=1) bit for bit,
    sweep after sweep, with the log-joints."""
    flips = np.random.default_rng(2).integers(0, 2, N).astype(np.int64)
    got = {}
    for serial in ("1", "0"):
        monkeypatch.setenv("BNMC_HMM_SERIAL", serial)
        e = g.Engine("hmm", {"N": N, "S": S}, g.RunConfig(seed=21))
        s = e.allocate()
        s["flips"] = flips
        e.prior_init(s, 21)
        ljs, states = [], []
        for it in range(4):
            ljs.append(e.sweep(s, it))
            states.append(s["s"].copy())
        got[serial] = (ljs, states, s["T"].copy(), s["bias"].copy())
        e.close()
    assert got["1"][0] == got["0"][0]
    for a, b in zip(got["1"][1], got["0"][1]):
        assert np.array_equal(a, b)
    assert np.array_equal(got["1"][2], got["0"][2]) and np.array_equal(got["1"][3], got["0"][3])
    assert not np.array_equal(got["0"][1][0], got["0"][1][-1])


@pytest.mark.parametrize("name,model", ZOO)
def test_zoo_sweeps_vs_reference(g, name, model):
    fx = golden(name)
    e, s, latent = _zoo_engine(g, fx, model)
    for n in latent:
        s[n] = fx[n + "0"]
    assert abs(e.eval_log_joint(s) - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"])
    for it in range(len(fx["lj"])):
        acc = []
        lj = e.sweep(s, it, acc)
        if model in ("polyreg", "regression", "regprec"):  # the (last) MH block's decision
            assert acc[0] == bool(fx["accepted"][it]), f"accept decision differs at step {it}"
        for n in latent:
            if s[n].dtype == np.int64:
                assert np.array_equal(s[n], fx[n][it]), f"{n} differs at sweep {it}: {(s[n] != fx[n][it]).sum()}"
            else:
                assert rel(s[n], fx[n][it]) < RTOL_PARAM, (n, it, rel(s[n], fx[n][it]))
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it]), (it, lj, fx["lj"][it])
    e.close()


# ----------------------------------------------------------------------------------------
# the sharded code path (NCCL all-reduces inside the sweep's CUDA graph) on one GPU:
# BNMC_FORCE_NCCL=1 gives a 1-rank communicator, so every world > 1 branch runs
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["lda_desk", "lda_ragged"])
def test_lda_nccl_path_vs_reference(g, monkeypatch, name):
    monkeypatch.setenv("BNMC_FORCE_NCCL", "1")
    fx = golden(name)
    e, s = lda_engine(g, fx)
    assert abs(e.eval_log_joint(s) - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"])
    for it in range(len(fx["lj"])):
        lj = e.sweep(s, it)
        assert np.array_equal(s["z"], fx["z"][it])
        assert rel(s["phi"], fx["phi"][it]) < RTOL_PARAM
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])
    lj_dev, _ = e.run_device(len(fx["lj"]), 3)  # graph replays with the captured all-reduces
    assert np.all(np.isfinite(lj_dev))
    e.close()


def test_mh_nccl_path_vs_reference(g, monkeypatch):
    monkeypatch.setenv("BNMC_FORCE_NCCL", "1")
    fx = golden("mh_linreg")
    N, K = int(fx["N"]), int(fx["K"])
    e = g.Engine("regression", {"N": N, "K": K, "l": -1.0, "u": 1.0}, g.RunConfig(seed=int(fx["seed"])))
    s = e.allocate()
    s["x"], s["y"], s["w"], s["b"], s["tau"] = fx["x"], fx["y"], fx["w0"], [fx["b0"]], [fx["tau0"]]
    assert abs(e.eval_log_joint(s) - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"])
    for it in range(len(fx["lj"])):
        acc = []
        lj = e.sweep(s, it, acc)
        assert acc[0] == bool(fx["accepted"][it])
        assert abs(lj - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])
    e.close()


# ----------------------------------------------------------------------------------------
# checkpoint / resume and the binary corpus
# ----------------------------------------------------------------------------------------
def _resume_case(g, tmp_path, make, names, n_before=2, n_after=2):
    e1, s1 = make()
    for it in range(n_before):
        e1.sweep(s1, it)
    ck = str(tmp_path / "state.ckpt")
    e1.save_checkpoint(ck)
    for it in range(n_before, n_before + n_after):
        e1.sweep(s1, it)
    e2, s2 = make()
    e2.upload(s2)                       # observed data (and a stale latent state)
    assert e2.load_checkpoint(ck) == n_before
    e2.run_device(n_before, n_after)
    e2.download(s2)
    for x in names:
        assert np.array_equal(s1[x], s2[x]), x
    e1.close()
    e2.close()


def test_checkpoint_resume_lda(g, tmp_path):
    fx = golden("lda_desk")
    _resume_case(g, tmp_path, lambda: lda_engine(g, fx), ["z", "phi", "theta"])


def test_checkpoint_resume_gmm_mh_hmm(g, tmp_path):
    gm = golden("gmm_small")

    def mk_gmm():
        e = g.Engine("gmm", {"N": int(gm["N"]), "K": 4}, g.RunConfig(seed=int(gm["seed"])))
        s = e.allocate()
        s["x"], s["z"], s["pi"], s["mu"], s["sigma2"] = gm["x"], gm["z0"], gm["pi0"], gm["mu0"], gm["sigma20"]
        return e, s
    _resume_case(g, tmp_path, mk_gmm, ["z", "pi", "mu", "sigma2"])
    mh = golden("mh_linreg")

    def mk_mh():
        e = g.Engine("regression", {"N": int(mh["N"]), "K": int(mh["K"]), "l": -1.0, "u": 1.0},
                     g.RunConfig(seed=int(mh["seed"])))
        s = e.allocate()
        s["x"], s["y"], s["w"], s["b"], s["tau"] = mh["x"], mh["y"], mh["w0"], [mh["b0"]], [mh["tau0"]]
        return e, s
    _resume_case(g, tmp_path, mk_mh, ["w", "b", "tau"])
    hm = golden("hmm_small")

    def mk_hmm():
        e, s, latent = _zoo_engine(g, hm, "hmm")
        for n in latent:
            s[n] = hm[n + "0"]
        return e, s
    _resume_case(g, tmp_path, mk_hmm, ["T", "bias", "s"])


def test_checkpoint_rejects_other_seed(g, tmp_path):
    fx = golden("lda_desk")
    e1, s1 = lda_engine(g, fx)
    e1.sweep(s1, 0)
    ck = str(tmp_path / "a.ckpt")
    e1.save_checkpoint(ck)
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    e2 = g.Engine("lda", {"K": K, "V": V, "M": M, "N": np.diff(fx["offsets"]).tolist()}, g.RunConfig(seed=1))
    with pytest.raises(g.BnmcError):
        e2.load_checkpoint(ck)


def test_binary_corpus_device_workflow(g, tmp_path):
    """write_corpus -> bnmc_gpu_lda_load_corpus -> device prior_init -> sweeps: the same
    state as the reference's prior_init and sweeps (the 1B workflow, host never holds z)."""
    fx = golden("lda_desk")
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    path = str(tmp_path / "desk.bnc")
    g.write_corpus(path, fx["offsets"], fx["w"], V)
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": np.diff(fx["offsets"]).tolist()},
                 g.RunConfig(seed=int(fx["seed"])))
    e.lda_load_corpus(path)
    e.prior_init_device(int(fx["seed"]))
    s = e.allocate()
    e.download(s)
    assert np.array_equal(s["z"], fx["z0"])
    assert rel(s["phi"], fx["phi0"]) < RTOL_PARAM and rel(s["theta"], fx["theta0"]) < RTOL_PARAM
    lj, _ = e.run_device(0, len(fx["lj"]))
    e.download(s)
    assert np.array_equal(s["z"], fx["z"][-1])
    assert abs(lj[-1] - fx["lj"][-1]) <= RTOL_LJ * abs(fx["lj"][-1])
    bad = str(tmp_path / "bad.bnc")
    g.write_corpus(bad, fx["offsets"], np.full(len(fx["w"]), V + 3), V)
    with pytest.raises(g.BnmcError):
        e.lda_load_corpus(bad)


def test_lpp_curve_vs_restatement(g, restatement, reference):
    """lpp_curve (bench.cpp:30-77, the Fig. 3 protocol) on the device against the same
    protocol composed from the restatement: clamped phi, prior_init(seed + c) of theta
    and z, fit sweeps keeping the MAP state (strict >), log10 predictive probability."""
    K, V, Mh, L, seed, fit = 5, 60, 8, 20, 7, 4
    w_tr, _, _ = reference.gen_lda(30, V, K, 25, 3)
    phis = [restatement.lda_prior_init(K, V, np.arange(31, dtype=np.int64) * 25, w_tr, 100 + i)[0] for i in range(5)]
    rs = np.random.default_rng(4)
    hw = rs.integers(0, V, Mh * L).astype(np.int64)              # held-out documents (fit)
    hoff = np.arange(Mh + 1, dtype=np.int64) * L
    tw = rs.integers(0, V, Mh * 6).astype(np.int64)              # held-out test tokens
    toff = np.arange(Mh + 1, dtype=np.int64) * 6
    hyper = {"K": K, "V": V, "M": Mh, "N": [L] * Mh}
    got = g.lpp_curve(phis, [1.0] * 5, hyper, hw, (tw, toff), fit, seed)
    assert [p["samples"] for p in got] == [1, 2, 4, 5]
    for p in got:
        c = p["samples"]
        phi = phis[c - 1].copy()
        _, theta, z = restatement.lda_prior_init(K, V, hoff, hw, seed + c)
        best, best_theta = -np.inf, None
        for it in range(fit):
            lj = restatement.lda_sweep(K, V, hoff, hw, z, phi, theta, seed + c, it, observe_phi=True)
            if lj > best:
                best, best_theta = lj, theta.copy()
        want = restatement.lda_lpp(phi, best_theta, K, V, tw, toff)
        assert abs(p["lpp"] - want) <= 1e-10 * abs(want), (c, p["lpp"], want)
        assert p["seconds"] == c / 1000.0


# ----------------------------------------------------------------------------------------
# statistical checks (SURVEY.md 8c parity plan, step 3): posterior summaries over many
# sweeps -- the logistic likelihood has no reference model, so its MH chain is pinned by
# recovering a synthetic truth; GMM recovers its centres (acceptance crit. 4 pattern)
# ----------------------------------------------------------------------------------------
def test_logreg_posterior_recovers_truth(g):
    rs = np.random.default_rng(11)
    N, K = 20000, 4
    wt, bt = np.array([0.8, -0.5, 0.3, 0.0]), 0.2
    x = rs.uniform(-1, 1, size=(N, K))
    y = (rs.uniform(size=N) < 1 / (1 + np.exp(-(x @ wt + bt)))).astype(np.float64)
    cfg = g.RunConfig(seed=21, mh_scale=0.01, burnin=1500, thin=5)
    e = g.Engine("logreg", {"N": N, "K": K, "l": -1.0, "u": 1.0}, cfg)
    s = e.allocate()
    s["x"], s["y"] = x.ravel(), y
    e.prior_init(s, 21)
    tr = e.run(s, 6000)
    acc = np.mean(tr["accepted"])
    assert 0.05 < acc < 0.9, acc
    ws = np.array([smp["w"] for smp in tr["samples"]])
    bs = np.array([smp["b"][0] for smp in tr["samples"]])
    # posterior sd at N = 2e4 is ~0.03 per coefficient: 0.12 is ~4 sd
    assert np.max(np.abs(ws.mean(axis=0) - wt)) < 0.12, ws.mean(axis=0)
    assert abs(bs.mean() - bt) < 0.12, bs.mean()
    e.close()


def test_gmm_posterior_recovers_centres(g):
    rs = np.random.default_rng(12)
    N = 20000
    centres, sds = np.array([-6.0, -2.0, 2.0, 6.0]), np.array([0.5, 0.5, 0.5, 0.5])
    zt = rs.integers(0, 4, N)
    x = centres[zt] + sds[zt] * rs.normal(size=N)
    cfg = g.RunConfig(seed=22, burnin=800, thin=2)
    e = g.Engine("gmm", {"N": N, "K": 4}, cfg)
    s = e.allocate()
    s["x"] = x
    e.prior_init(s, 22)
    tr = e.run(s, 200)
    mus = np.sort(np.array([smp["mu"] for smp in tr["samples"]]), axis=1)
    s2 = np.array([smp["sigma2"] for smp in tr["samples"]])
    assert np.max(np.abs(mus.mean(axis=0) - centres)) < 0.05, mus.mean(axis=0)
    assert np.all(np.abs(np.sort(s2.mean(axis=0)) - 0.25) < 0.05), s2.mean(axis=0)
    e.close()


@pytest.mark.parametrize("name,model", [("hmm_small", "hmm"), ("catmix_small", "catmix"),
                                        ("naivebayes_small", "naivebayes"), ("regression_mwg", "regression")])
def test_zoo_run_trace_matches_stepwise(g, name, model):
    """Engine::run through bnmc_gpu_run_trace (device MAP tracking, thinned samples via the
    device snapshot slots on a copy stream) == stepwise sweeps, for the rest of the zoo."""
    fx = golden(name)
    burnin, n, thin = 1, 6, 2

    def mk():
        e, s, latent = _zoo_engine(g, fx, model)
        for v in latent:
            s[v] = fx[v + "0"]
        return e, s, latent

    e1, s1, latent = mk()
    e1.cfg.burnin, e1.cfg.thin = burnin, thin
    tr = e1.run(s1, n)
    e2, s2, _ = mk()
    lj, samples, map_lj, map_state = _stepwise_run(e2, s2, burnin, n, thin, latent)
    assert tr["log_joint"] == lj
    assert len(tr["samples"]) == len(samples) == 3
    for a, b in zip(tr["samples"], samples):
        for x in latent:
            assert np.array_equal(a[x], b[x]), x
    assert tr["map_log_joint"] == map_lj
    for x in latent:
        assert np.array_equal(tr["map_state"][x], map_state[x]), x
    e1.close()
    e2.close()


def test_lda_joint_known_answer(g):
    """The reference's lda_joint_oracle (tests/test_ir.cpp:148-177): the LDA log-joint of a
    tiny state written against the arrays directly -- Dirichlet(0.1) terms of every phi
    and theta row plus sum_t log theta[d_t, z_t] + log phi[z_t, w_t] -- against the
    device's eval_log_joint."""
    from math import lgamma, log

    K, V, lengths = 2, 3, [3, 4]
    rs = np.random.default_rng(7)
    phi = rs.dirichlet(np.ones(V), size=K)
    theta = rs.dirichlet(np.ones(K), size=len(lengths))
    N = sum(lengths)
    z = rs.integers(0, K, N)
    w = rs.integers(0, V, N)

    def dterm(x, a):
        return sum((a - 1.0) * log(xi) for xi in x) - len(x) * lgamma(a) + lgamma(a * len(x))

    want = sum(dterm(phi[k], 0.1) for k in range(K)) + sum(dterm(theta[m], 0.1) for m in range(len(lengths)))
    t = 0
    for m, L in enumerate(lengths):
        for _ in range(L):
            want += log(theta[m, z[t]]) + log(phi[z[t], w[t]])
            t += 1
    e = g.Engine("lda", {"K": K, "V": V, "M": len(lengths), "N": lengths}, g.RunConfig(seed=1))
    s = e.allocate()
    s["phi"], s["theta"], s["z"], s["w"] = phi.ravel(), theta.ravel(), z, w
    got = e.eval_log_joint(s)
    assert abs(got - want) <= 1e-12 * abs(want), (got, want)
    e.close()
