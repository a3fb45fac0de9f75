"""Host API semantics of the Engine mirrors (engine.py, bnmc_gpu.hpp) that the reference
defines by its borrow rules (sampler.hpp:43-44: the caller owns the ParamStore and lends
it per call; every call reads its current state)."""
import numpy as np
import pytest

from conftest import golden

RTOL_LJ = 1e-10


@pytest.fixture(scope="module")
def g():
    import paper_1312_3613_b200 as g

    g.lib()
    return g


def _lda(g, fx, **cfg):
    K, V, M = int(fx["K"]), int(fx["V"]), int(fx["M"])
    e = g.Engine("lda", {"K": K, "V": V, "M": M, "N": np.diff(fx["offsets"]).tolist()},
                 g.RunConfig(seed=int(fx["seed"]), **cfg))
    s = e.allocate()
    s["w"], s["z"], s["phi"], s["theta"] = fx["w"], fx["z0"], fx["phi0"], fx["theta0"]
    return e, s


# -- CPU: argument validation happens before any device call ---------------------------------
@pytest.mark.parametrize("model,hyper,var", [
    ("lda", {"K": 3, "V": 5, "M": 2, "N": [2, 2]}, "z"),
    ("lda", {"K": 3, "V": 5, "M": 2, "N": [2, 2]}, "theta"),
    ("gmm", {"K": 4, "N": 10}, "mu"),
    ("regression", {"K": 2, "N": 10}, "w"),
])
def test_observe_extra_outside_the_device_plans_is_refused(g, model, hyper, var):
    """A clamped variable the device sweep would keep resampling is refused (ValueError),
    never silently resampled (only LDA's phi -- the lpp protocol -- is clampable)."""
    with pytest.raises(ValueError, match="observe_extra"):
        g.Engine(model, hyper, g.RunConfig(observe_extra=[var]))


# -- GPU --------------------------------------------------------------------------------------
@pytest.mark.gpu
def test_eval_log_joint_and_run_read_the_callers_edits(g):
    """sweep(store) binds the store; a caller edit of z / theta afterwards must be seen by
    eval_log_joint(store) and run(store), exactly as by a fresh engine on the same store."""
    fx = golden("lda_desk")
    e, s = _lda(g, fx)
    e.sweep(s, 0)
    rs = np.random.default_rng(3)
    K = int(fx["K"])
    z = s["z"].copy()
    idx = rs.choice(z.size, 25, replace=False)
    z[idx] = (z[idx] + 1) % K
    s["z"] = z
    th = s["theta"].reshape(-1, K)
    th[0] = th[0][::-1]  # a permuted (still normalised) row
    s["theta"] = th.ravel()
    f, t = _lda(g, fx)
    t["z"], t["phi"], t["theta"] = s["z"], s["phi"], s["theta"]
    want = f.eval_log_joint(t)
    assert e.eval_log_joint(s) == want
    tr_e = e.run(s, 2)
    tr_f = f.run(t, 2)
    assert tr_e["log_joint"] == tr_f["log_joint"]
    assert np.array_equal(s["z"], t["z"])
    e.close()
    f.close()


@pytest.mark.gpu
def test_checkpoint_resume_through_a_store(g, tmp_path):
    """load_checkpoint(path, store): the restored state lands in the store, and
    sweep(store, it) continues the chain bit for bit."""
    fx = golden("lda_desk")
    e1, s1 = _lda(g, fx)
    for it in range(2):
        e1.sweep(s1, it)
    ck = str(tmp_path / "s.ckpt")
    e1.save_checkpoint(ck)
    lj1 = [e1.sweep(s1, it) for it in range(2, 5)]
    e2, s2 = _lda(g, fx)     # a fresh store: prior state, the same corpus
    assert e2.load_checkpoint(ck, s2) == 2
    lj2 = [e2.sweep(s2, it) for it in range(2, 5)]
    assert lj1 == lj2
    for x in ("z", "phi", "theta"):
        assert np.array_equal(s1[x], s2[x]), x
    e1.close()
    e2.close()


@pytest.mark.gpu
@pytest.mark.parametrize("change", ["exact_weights", "mh_scale"])
def test_checkpoint_rejects_other_configuration(g, tmp_path, change):
    fx = golden("lda_desk")
    e1, s1 = _lda(g, fx)
    e1.sweep(s1, 0)
    ck = str(tmp_path / "c.ckpt")
    e1.save_checkpoint(ck)
    e2, _ = _lda(g, fx, **({"exact_weights": True} if change == "exact_weights" else {"mh_scale": 0.25}))
    with pytest.raises(g.BnmcError, match="configuration"):
        e2.load_checkpoint(ck)
    e1.close()
    e2.close()


@pytest.mark.gpu
def test_observed_edit_needs_rebind(g):
    """Observed data is uploaded once per binding (the engine never writes it); an in-place
    edit of w is picked up after rebind(), giving the fresh-engine result."""
    fx = golden("lda_desk")
    e, s = _lda(g, fx)
    e.sweep(s, 0)
    V = int(fx["V"])
    w = s["w"].copy()
    w[:50] = (w[:50] + 7) % V
    s["w"][:] = w  # in place: the same array object the engine bound
    f, t = _lda(g, fx)
    t["w"], t["z"], t["phi"], t["theta"] = w, s["z"], s["phi"], s["theta"]
    e.rebind(s)
    assert e.sweep(s, 1) == f.sweep(t, 1)
    assert np.array_equal(s["z"], t["z"])
    e.close()
    f.close()


@pytest.mark.gpu
def test_store_already_page_locked_by_its_owner(g):
    """A store whose arrays are already pinned (torch pin_memory / cudaHostAlloc) binds: the
    engine's one-time page-locking skips them instead of failing."""
    import torch

    fx = golden("lda_desk")
    e, s = _lda(g, fx)
    for n in s.names:
        if not s.observed[n]:
            t = torch.empty(s.arrays[n].size, dtype=torch.from_numpy(s.arrays[n][:0]).dtype, pin_memory=True)
            a = t.numpy()
            a[:] = s.arrays[n]
            s.arrays[n] = a
    f, t2 = _lda(g, fx)
    for it in range(2):
        assert e.sweep(s, it) == f.sweep(t2, it)
        assert np.array_equal(s["z"], t2["z"])
    e.close()
    f.close()
