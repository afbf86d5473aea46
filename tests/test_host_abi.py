"""C-ABI library on the CPU: it loads, exports every symbol the header
declares, and its host-side functions (visit order, generators, CSR builder)
match the reference.  No GPU compute is called here."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2301_09125_b200 as lp
from paper_2301_09125_b200 import _lib, graph as G
from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "labelprop_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == declared
    assert b"sm_100a" in L.lp_version()


def test_library_binary_targets_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_shuffled_indices_is_the_reference_permutation(golden_prng):
    for k in golden_prng.files:
        if k.startswith("shuffled/"):
            _, n, seed = k.split("/")
            assert np.array_equal(lp.shuffled_indices(int(n), int(seed)), golden_prng[k]), k


def test_prng_known_answers(golden_prng):
    assert lp.XorShift32(1).next() == 270369  # reference tests/test_prng.py:23-26
    assert lp.XorShift32(1).next_bounded(10) == 9  # :58-61
    from paper_2301_09125_b200.prng import mix_seed, xs32_next

    for seed, k, want in golden_prng["mix_seed"]:
        assert mix_seed(int(seed), int(k)) == int(want)
    for key in golden_prng.files:
        if key.startswith("xs32/"):
            x = int(key.split("/")[1])
            for want in golden_prng[key]:
                x = xs32_next(x)
                assert x == int(want)
    with pytest.raises(ValueError):
        lp.XorShift32(1).next_bounded(0)
    assert lp.XorShift32(0).state == 2463534242


def test_native_csr_builder_equals_preprocess():
    rng = np.random.default_rng(4)
    for trial in range(40):
        n = int(rng.integers(1, 400))
        k = int(rng.integers(0, 3000))
        u = rng.integers(0, n, k)
        v = rng.integers(0, n, k)
        a = G.undirected_csr(n, u, v)
        b = G.preprocess(G.from_arcs(n, u, v, np.ones(k)))
        assert G.graphs_equal(a, b) and a.total_weight == b.total_weight, trial
        c = G.undirected_csr_numpy(n, u, v)
        assert G.graphs_equal(a, c)


def test_native_builder_rejects_bad_pairs():
    with pytest.raises(ValueError):
        G.undirected_csr(3, [0, 5], [1, 2])


def test_rmat_generator_is_deterministic_and_skewed():
    s1, d1 = lp.synth.rmat_edges(12, seed=3)
    s2, d2 = lp.synth.rmat_edges(12, seed=3)
    assert np.array_equal(s1, s2) and np.array_equal(d1, d2)
    s3, _ = lp.synth.rmat_edges(12, seed=4)
    assert not np.array_equal(s1, s3)
    g = lp.rmat(12, seed=3)
    deg = np.diff(g.offsets)
    assert deg.max() > 20 * np.median(deg)  # power-law hubs
    G.check_symmetric(g)


def test_generators_produce_canonical_graphs():
    for g in (lp.planted_partition(2000, 20, seed=2), lp.road_grid(40, seed=1), lp.rmat(10, weighted=True)):
        G.check_symmetric(g)
        rows = np.repeat(np.arange(g.vertex_count), np.diff(g.offsets))
        # one self-loop per vertex, rows sorted by neighbour id
        assert int((rows == g.neighbors).sum()) == g.vertex_count
        for v in range(0, g.vertex_count, max(1, g.vertex_count // 50)):
            row = g.neighbors[g.offsets[v]:g.offsets[v + 1]]
            assert np.all(np.diff(row) > 0)
    gw = lp.rmat(10, weighted=True)
    w = gw.weights[gw.neighbors != np.repeat(np.arange(gw.vertex_count), np.diff(gw.offsets))]
    assert w.min() >= 1.0 and w.max() < 2.0
    assert np.array_equal(w.astype(np.float32).astype(np.float64), w)  # float32-exact


def test_no_gpu_means_loud_failure():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    g = lp.disjoint_cliques(2, 3)
    with pytest.raises(RuntimeError, match="CUDA|device"):
        lp.rak_detect(g, lp.RakParams(strict=True))


def test_graph_create_validates_arguments_before_touching_the_gpu():
    L = _lib.lib()
    h = C.c_void_p()
    off = np.array([0, 2, 1], dtype=np.int64)
    nbr = np.array([1, 0], dtype=np.int64)
    rc = L.lp_graph_create(2, 2, _lib.ptr(off), _lib.ptr(nbr), None, -1, C.byref(h))
    assert rc == _lib.LP_ERR_INVALID
    rc = L.lp_graph_create(-1, 0, None, None, None, -1, C.byref(h))
    assert rc == _lib.LP_ERR_INVALID
    assert b"negative" in L.lp_last_error()
