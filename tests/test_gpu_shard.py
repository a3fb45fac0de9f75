"""Sharded sweeps on ONE GPU: W ranks of a peer group (bnmc_gpu_group) in one process, one
host thread each, run the multi-GPU code path -- document / row shards with non-zero
token and document offsets (RNG keys, uploads, downloads, prior_init of a shard), the
per-sweep all-reduce of the topic-word counts (replacing the reference's
reduce_accumulate fold, executor.cpp:99-114), the log-joint pieces, the MH likelihood
sums and the collective bound-store speculation votes -- through libbnmc_gpu's own
peer-memory all-reduce kernel.

Contract: the gathered shards equal the unsharded chain -- z, counts and accept decisions
bit-exact, phi bitwise (every rank draws phi from the same all-reduced counts with the
same counter streams), theta <= 1e-12, the log-joint <= 1e-10 (its pieces are summed in a
different order).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

RTOL = 1e-12
RTOL_LJ = 1e-10


@pytest.fixture(scope="module")
def g():
    import paper_1312_3613_b200 as g

    g.lib()
    return g


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def on_ranks(fns):
    """Run one callable per rank concurrently (each rank's C-ABI calls on its own thread)."""
    with ThreadPoolExecutor(len(fns)) as ex:
        futs = [ex.submit(f) for f in fns]
        return [f.result(timeout=300) for f in futs]


class ShardedLda:
    def __init__(self, g, K, V, off, w, seed, W, exact=False):
        self.g, self.K, self.off, self.W = g, K, off, W
        self.group = g.PeerGroup(W)
        hyper = {"K": K, "V": V, "M": len(off) - 1, "N": np.diff(off).tolist()}
        self.eng, self.st, self.rng = [], [], []
        for r in range(W):
            e = g.Engine("lda", hyper, g.RunConfig(seed=seed, exact_weights=exact), rank=r, world_size=W,
                         group=self.group)
            s = e.allocate()
            s["w"] = w
            self.eng.append(e)
            self.st.append(s)
            b, en = g.partition(off, W, r)
            self.rng.append((b, en))

    def set_state(self, z, phi, theta):
        for s in self.st:
            s["z"], s["phi"], s["theta"] = z, phi, theta

    def sweep(self, it):
        return on_ranks([lambda r=r: self.eng[r].sweep(self.st[r], it) for r in range(self.W)])

    def gather(self):
        z = np.empty_like(self.st[0]["z"])
        th = np.empty_like(self.st[0]["theta"])
        for r, (b, e) in enumerate(self.rng):
            t0, t1 = self.off[b], self.off[e]
            z[t0:t1] = self.st[r]["z"][t0:t1]
            th[b * self.K:e * self.K] = self.st[r]["theta"][b * self.K:e * self.K]
        return z, th

    def close(self):
        for e in self.eng:
            e.close()
        self.group.close()


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("name", ["lda_desk", "lda_ragged"])
def test_sharded_lda_vs_reference_goldens(g, name, W):
    fx = golden(name)
    K, V = int(fx["K"]), int(fx["V"])
    sh = ShardedLda(g, K, V, fx["offsets"], fx["w"], int(fx["seed"]), W)
    assert all(b < e for b, e in sh.rng) or name == "lda_ragged"
    sh.set_state(fx["z0"], fx["phi0"], fx["theta0"])
    lj0 = on_ranks([lambda r=r: sh.eng[r].eval_log_joint(sh.st[r]) for r in range(W)])
    assert all(abs(v - fx["lj0"]) <= RTOL_LJ * abs(fx["lj0"]) for v in lj0)
    for it in range(len(fx["lj"])):
        ljs = sh.sweep(it)
        z, th = sh.gather()
        assert np.array_equal(z, fx["z"][it]), f"sweep {it}: {(z != fx['z'][it]).sum()} z mismatches"
        assert rel(th, fx["theta"][it]) < RTOL
        for r in range(W):  # every rank holds the full phi
            assert rel(sh.st[r]["phi"], fx["phi"][it]) < RTOL
            assert abs(ljs[r] - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])
    # the topic-word counts: all-reduced over the shards
    counts = on_ranks([lambda r=r: sh.eng[r].lda_counts() for r in range(W)])
    want = np.zeros((K, V), dtype=np.int64)
    np.add.at(want, (fx["z"][-1], fx["w"]), 1)
    for nkw, _ in counts:
        assert np.array_equal(nkw, want)
    sh.close()


def test_sharded_prior_init_matches_reference(g):
    """prior_init of a shard: theta rows and z keyed by GLOBAL document / token indices."""
    fx = golden("lda_desk")
    K, V = int(fx["K"]), int(fx["V"])
    sh = ShardedLda(g, K, V, fx["offsets"], fx["w"], int(fx["seed"]), 3)
    on_ranks([lambda r=r: sh.eng[r].prior_init(sh.st[r], int(fx["seed"])) for r in range(3)])
    z, th = sh.gather()
    assert np.array_equal(z, fx["z0"])
    assert rel(th, fx["theta0"]) < RTOL
    for r in range(3):
        assert rel(sh.st[r]["phi"], fx["phi0"]) < RTOL
    sh.close()


def _nips_like(restatement, M=300, V=4000, K=100, L=600, seed=5):
    rs = np.random.default_rng(seed)
    lengths = rs.integers(L // 2, 3 * L // 2, M)
    off = np.zeros(M + 1, dtype=np.int64)
    off[1:] = np.cumsum(lengths)
    pw = 1.0 / np.arange(1, V + 1) ** 1.05
    w = rs.choice(V, size=int(off[-1]), p=pw / pw.sum()).astype(np.int64)
    phi, theta, z = restatement.lda_prior_init(K, V, off, w, seed)
    return off, w, phi, theta, z


@pytest.mark.parametrize("W,exact", [(2, False), (4, False), (2, True)], ids=["W2", "W4", "W2-log-space"])
def test_sharded_equals_unsharded_on_a_large_corpus(g, restatement, W, exact):
    """A 180k-token ragged Zipf corpus at K = 100: W shards against one context, 3 sweeps."""
    K, V, seed = 100, 4000, 5
    off, w, phi, theta, z = _nips_like(restatement, V=V, K=K, seed=seed)
    hyper = {"K": K, "V": V, "M": len(off) - 1, "N": np.diff(off).tolist()}
    one = g.Engine("lda", hyper, g.RunConfig(seed=seed, exact_weights=exact))
    s1 = one.allocate()
    s1["w"], s1["z"], s1["phi"], s1["theta"] = w, z, phi, theta
    sh = ShardedLda(g, K, V, off, w, seed, W, exact=exact)
    sh.set_state(z, phi, theta)
    for it in range(3):
        lj1 = one.sweep(s1, it)
        ljs = sh.sweep(it)
        zg, thg = sh.gather()
        assert np.array_equal(zg, s1["z"]), f"sweep {it}: {(zg != s1['z']).sum()} z mismatches"
        assert np.array_equal(thg, s1["theta"])  # same draws from the same counts and streams
        for r in range(W):
            assert np.array_equal(sh.st[r]["phi"], s1["phi"])
            assert abs(ljs[r] - lj1) <= RTOL_LJ * abs(lj1)
    one.close()
    sh.close()


@pytest.mark.parametrize("K", [300, 1000])
def test_sharded_word_major_equals_unsharded_document_major(g, restatement, monkeypatch, K):
    """Word-major z-step order on W = 2 shards (each rank sorts its own tokens by
    (document block, word)) against one document-major context: z, theta, phi bitwise
    over 3 sweeps (a Zipf corpus, so frequent words span several kChunk units)."""
    V, seed, W = 3000, 9, 2
    off, w, phi, theta, z = _nips_like(restatement, M=120, V=V, K=K, L=500, seed=seed)
    hyper = {"K": K, "V": V, "M": len(off) - 1, "N": np.diff(off).tolist()}
    monkeypatch.setenv("BNMC_ZSTEP_WM", "0")
    one = g.Engine("lda", hyper, g.RunConfig(seed=seed))
    s1 = one.allocate()
    s1["w"], s1["z"], s1["phi"], s1["theta"] = w, z, phi, theta
    monkeypatch.setenv("BNMC_ZSTEP_WM", "1")
    monkeypatch.setenv("BNMC_WM_BLOCK_DOCS", "7")
    sh = ShardedLda(g, K, V, off, w, seed, W)
    sh.set_state(z, phi, theta)
    for it in range(3):
        lj1 = one.sweep(s1, it)
        ljs = sh.sweep(it)
        zg, thg = sh.gather()
        assert np.array_equal(zg, s1["z"]), f"sweep {it}: {(zg != s1['z']).sum()} z mismatches"
        assert np.array_equal(thg, s1["theta"])
        for r in range(W):
            assert np.array_equal(sh.st[r]["phi"], s1["phi"])
            assert abs(ljs[r] - lj1) <= RTOL_LJ * abs(lj1)
    one.close()
    sh.close()


def test_sharded_speculation_with_an_edit_on_one_rank(g, restatement):
    """Bound-store sweeps speculate collectively: a caller edit of z on ONE rank's shard
    must make every rank redo the sweep from the edited state (the vote is an all-reduce
    max), giving the unsharded engine's result for the same edit."""
    K, V, seed, W = 50, 2000, 9, 2
    off, w, phi, theta, z = _nips_like(restatement, M=120, V=V, K=K, L=300, seed=seed)
    hyper = {"K": K, "V": V, "M": len(off) - 1, "N": np.diff(off).tolist()}
    one = g.Engine("lda", hyper, g.RunConfig(seed=seed))
    s1 = one.allocate()
    s1["w"], s1["z"], s1["phi"], s1["theta"] = w, z, phi, theta
    sh = ShardedLda(g, K, V, off, w, seed, W)
    sh.set_state(z, phi, theta)
    b0, e0 = sh.rng[0]
    for it in range(5):
        if it == 3:  # the caller edits a few assignments of rank 0's documents only
            t0, t1 = off[b0], off[e0]
            idx = np.arange(t0, t1, 97)
            for s in (s1, sh.st[0]):
                zz = s["z"].copy()
                zz[idx] = (zz[idx] + 1) % K
                s["z"] = zz
        lj1 = one.sweep(s1, it)
        ljs = sh.sweep(it)
        zg, _ = sh.gather()
        assert np.array_equal(zg, s1["z"]), f"sweep {it}"
        assert all(abs(v - lj1) <= RTOL_LJ * abs(lj1) for v in ljs)
    one.close()
    sh.close()


def test_sharded_mh_rows_vs_reference(g):
    fx = golden("mh_linreg")
    N, K, W = int(fx["N"]), int(fx["K"]), 2
    grp = g.PeerGroup(W)
    eng, st = [], []
    for r in range(W):
        e = g.Engine("regression", {"N": N, "K": K, "l": -1.0, "u": 1.0}, g.RunConfig(seed=int(fx["seed"])),
                     rank=r, world_size=W, group=grp)
        s = e.allocate()
        s["x"], s["y"], s["w"], s["b"], s["tau"] = fx["x"], fx["y"], fx["w0"], [fx["b0"]], [fx["tau0"]]
        eng.append(e)
        st.append(s)
    for it in range(len(fx["lj"])):
        accs = [[] for _ in range(W)]
        ljs = on_ranks([lambda r=r: eng[r].sweep(st[r], it, accs[r]) for r in range(W)])
        for r in range(W):
            assert accs[r][0] == bool(fx["accepted"][it]), f"accept decision differs at step {it}"
            assert rel(st[r]["w"], fx["w"][it]) < RTOL
            assert abs(ljs[r] - fx["lj"][it]) <= RTOL_LJ * abs(fx["lj"][it])
    for e in eng:
        e.close()
    grp.close()


def test_group_misuse_is_reported(g):
    fx = golden("lda_desk")
    K, V = int(fx["K"]), int(fx["V"])
    hyper = {"K": K, "V": V, "M": int(fx["M"]), "N": np.diff(fx["offsets"]).tolist()}
    grp = g.PeerGroup(2)
    e0 = g.Engine("lda", hyper, g.RunConfig(seed=1), rank=0, world_size=2, group=grp)
    with pytest.raises(ValueError):
        g.Engine("lda", hyper, g.RunConfig(seed=1), rank=0, world_size=2, group=grp)  # rank taken
    with pytest.raises(ValueError):
        g.Engine("lda", hyper, g.RunConfig(seed=1), rank=1, world_size=3, group=grp)  # wrong world
    e0.close()
    grp.close()
