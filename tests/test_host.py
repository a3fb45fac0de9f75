"""CPU: the C-ABI library, the host mirror and the sharding logic (no GPU compute)."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bnmc_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(bnmc_gpu_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_1312_3613_b200 as g

    L = g.lib()  # loads libbnmc_gpu.so (built for sm_100a) without touching a device
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/bnmc_gpu.h but not exported"
    assert L.bnmc_gpu_abi_version() == g.engine.ABI_VERSION == 2
    out = subprocess.run(["nm", "-D", "--defined-only", g.engine.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_library_is_sm100a_code():
    import paper_1312_3613_b200 as g

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", g.engine.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    import torch

    import paper_1312_3613_b200 as g

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(g.BnmcError):
        g.Engine("lda", {"K": 2, "V": 3, "M": 1, "N": [2]})


def test_unsupported_model_rejected():
    import paper_1312_3613_b200 as g

    with pytest.raises(ValueError):
        g.Engine("nosuchmodel", {})
    with pytest.raises(ValueError):
        g.Engine("hmm", {"N": 4, "S": 2}, g.RunConfig(method="mh"))  # hmm.bn's plan is Gibbs
    with pytest.raises(ValueError):
        g.Engine("lda", {"K": 2, "V": 3, "M": 1, "N": [2]}, g.RunConfig(method="mh"))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_contiguous_balanced(world):
    import paper_1312_3613_b200 as g

    rs = np.random.default_rng(world)
    lengths = rs.integers(0, 50, 97)
    off = np.concatenate([[0], np.cumsum(lengths)])
    bounds = [g.partition(off, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == len(lengths)
    for (b0, e0), (b1, e1) in zip(bounds, bounds[1:]):
        assert e0 == b1 and b0 <= e0
    toks = [off[e] - off[b] for b, e in bounds]
    assert sum(toks) == off[-1]
    assert max(toks) - min(toks) <= 2 * lengths.max() + 1


def test_store_layout_mirrors_reference():
    import paper_1312_3613_b200 as g

    s = g.ParamStore("lda", {"K": 3, "V": 5, "M": 2, "N": [4, 1]})
    assert s.names == ["phi", "theta", "z", "w"]  # declaration order = reference var ids
    assert s["phi"].size == 15 and s["theta"].size == 6 and s["z"].size == 5
    assert s["z"].dtype == np.int64 and s["phi"].dtype == np.float64
    assert s.observed == {"phi": False, "theta": False, "z": False, "w": True}
    a = np.arange(5)
    s["z"] = a
    a[0] = 99
    assert s["z"][0] == 0  # the store owns its arrays
    with pytest.raises(g.BnmcError):
        s["z"] = np.arange(4)


def test_cpp_mirror_compiles():
    lib = os.path.join(ROOT, "paper_1312_3613_b200")
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "lda_sweep.cpp"), "-L", lib, "-lbnmc_gpu",
                        "-o", "/tmp/bnmc_lda_sweep_test"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c", HEADER],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    # the driver the GPU parity suite runs against the Python engine
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "lda_engine_example.cpp"), "-L", lib, "-lbnmc_gpu",
                        "-o", "/tmp/bnmc_lda_engine_example_test"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_bench_corpus_generator_shape():
    import bench

    w = bench.gen_lda_corpus(20, 300, 5, 17, 3)
    assert w.shape == (340,) and w.min() >= 0 and w.max() < 300
    assert np.array_equal(w, bench.gen_lda_corpus(20, 300, 5, 17, 3))


def test_store_view_cache_follows_the_arrays():
    """ParamStore._view is cached per array object and observed mask: replacing an array
    (through __setitem__ or .arrays) or flipping a mask rebuilds it, in-place writes do not
    need to (the pointers are unchanged)."""
    from paper_1312_3613_b200.engine import ParamStore

    s = ParamStore("gmm", {"N": 100, "K": 4})
    v1 = s._view()
    assert s._view() is v1
    s["z"][:] = 1  # in place: same buffer
    assert s._view() is v1
    s["z"] = np.zeros(100, dtype=np.int64)
    v2 = s._view()
    assert v2 is not v1 and v2.ival[3] is not None
    assert ctypes.addressof(v2.ival[3].contents) == s["z"].ctypes.data
    s.arrays["x"] = np.ones(100)
    v3 = s._view()
    assert v3 is not v2 and ctypes.addressof(v3.real[4].contents) == s["x"].ctypes.data
    s.observed["z"] = True
    assert s._view() is not v3


def test_bench_corpus_file_matches_engine_format(tmp_path):
    """bench.write_corpus_file (the reference arm's input) writes the bytes of
    engine.write_corpus (the library's .bnc format)."""
    import bench
    from paper_1312_3613_b200.engine import write_corpus

    w = bench.gen_lda_corpus(7, 50, 4, 9, 5)
    off = np.arange(8, dtype=np.int64) * 9
    bench.write_corpus_file(str(tmp_path / "a.bnc"), off, w, 50)
    write_corpus(str(tmp_path / "b.bnc"), off, w, 50)
    assert (tmp_path / "a.bnc").read_bytes() == (tmp_path / "b.bnc").read_bytes()


def test_bench_arms_share_config():
    """Both arms print shared_config(args, world): identical dicts per workload."""
    import argparse

    import bench

    for wl in bench.WORKLOADS:
        a = argparse.Namespace(workload=wl, seed=7)
        assert bench.shared_config(a, 1) == bench.shared_config(a, 1)
        assert "l2" in bench.shared_config(a, 2)


def test_reference_reads_the_bench_corpus(tmp_path):
    """oracle/_ref/ref_bench lda-file runs the reference on the corpus the GPU arm uses
    (first DOCS documents) and counts its sites."""
    import bench
    from oracle import REF_BENCH

    if not os.path.exists(REF_BENCH):
        pytest.skip("reference not built")
    w = bench.gen_lda_corpus(12, 200, 6, 30, 2)
    bench.write_corpus_file(str(tmp_path / "c.bnc"), np.arange(13, dtype=np.int64) * 30, w, 200)
    res, _ = bench.ref_bench(["lda-file", str(tmp_path / "c.bnc"), 6, 2, 1, 0, 2, 5], timeout=120)
    assert res["sites"] == 5 * 30 and len(res["ms"]) == 2
    x = bench.gmm_points(500, 3)
    x.tofile(str(tmp_path / "x.f64"))
    res, _ = bench.ref_bench(["gmm-file", str(tmp_path / "x.f64"), 3, 1, 0, 2], timeout=120)
    assert res["sites"] == 500


def test_bench_self_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself
    (torch.distributed.run, 127.0.0.1); with --impl reference rank 0 alone prints the
    line and rank 1 exits 0 without work -- the driver's reference-arm contract, here on
    the CPU with the GMM workload (its reference run takes ~1 s)."""
    import json

    from oracle import REF_BENCH

    if not os.path.exists(REF_BENCH):
        pytest.skip("reference not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--workload", "gmm", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
