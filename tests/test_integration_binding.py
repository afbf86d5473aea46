"""INTEGRATION.md Option B: the ctypes binding a maintainer would paste into
the reference (``labelprop/_cuda.py``), kept verbatim in
tests/integration_cuda.py.  CPU: the document and the file agree.  GPU: the
binding, called the way the patched reference calls it, reproduces the
reference's own outputs (strict RAK: tests/golden/rak.npz, bit for bit) and
the oracle's COPRA / SLPA restatements."""

import importlib.util
import os
import re

import numpy as np
import pytest

from conftest import load_graph

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _binding_source():
    with open(os.path.join(HERE, "integration_cuda.py")) as f:
        return f.read()


def test_integration_doc_holds_the_tested_binding():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        doc = f.read()
    blocks = re.findall(r"```python\n(.*?)```", doc, flags=re.S)
    assert _binding_source() in blocks, "INTEGRATION.md Option B must hold tests/integration_cuda.py verbatim"


@pytest.fixture(scope="module")
def binding(gpu):
    from paper_2301_09125_b200 import _lib

    os.environ["LABELPROP_CUDA_LIB"] = _lib.LIB_PATH
    spec = importlib.util.spec_from_file_location("labelprop_cuda_binding", os.path.join(HERE, "integration_cuda.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.gpu
def test_binding_rak_matches_reference_goldens(binding, golden_rak):
    import paper_2301_09125_b200 as lp

    for name in ("cliques_8x6", "gnp_1000", "planted_4000", "rmat_12", "rmat_12_w", "ring_16x6", "grid_64"):
        g = load_graph(golden_rak, name)
        for seed in (1, 2, 3):
            for tol in (0.05, 1e-4):
                key = f"{name}/s/{seed}/{tol:g}"
                labels = np.arange(g.vertex_count, dtype=np.int64)
                order = lp.shuffled_indices(g.vertex_count, seed)
                it = binding.rak_cuda(g, labels, order, True, tol, 100, seed)
                assert it == int(golden_rak[f"{key}/iterations"]), key
                assert np.array_equal(labels, golden_rak[f"{key}/labels_per_iter"][-1]), key


@pytest.mark.gpu
def test_binding_copra_and_slpa_match_oracle(binding, golden_copra, golden_slpa, oracle):
    import paper_2301_09125_b200 as lp

    for name in ("ring_16x6", "gnp_1000", "planted_4000", "rmat_12"):
        g = load_graph(golden_copra, name)
        for K in (1, 4, 8):
            best, it, labs, bels, sizes = binding.copra_cuda(g, lp.CopraParams(max_labels=K, seed=1,
                                                                                max_iterations=30))
            obest, oit, olabs, obels, osizes = oracle.copra(g, max_labels=K, batches=0, tie=1, seed=1,
                                                            tolerance=0.01, max_iterations=30)
            assert it == oit and np.array_equal(best, obest) and np.array_equal(sizes, osizes), (name, K)
            for j in range(K):
                live = sizes > j
                assert np.array_equal(labs[live, j], olabs[live, j]) and np.array_equal(bels[live, j], obels[live, j])
    for name in ("cliques_8x6", "gnp_1000", "planted_4000", "rmat_12"):
        g = load_graph(golden_slpa, name)
        for T in (5, 12):
            labels, it, slots, filled = binding.slpa_cuda(g, lp.SlpaParams(memory_size=T, seed=3))
            want, oit, oslots, ofilled = oracle.slpa(g, memory_size=T, batches=0, tie=1, speaker_rng=1, seed=3,
                                                     tolerance=0.05)
            assert it == oit and np.array_equal(labels, want), (name, T)
            assert np.array_equal(slots[:, : it + 1], oslots[:, : it + 1]), (name, T)


@pytest.mark.gpu
def test_binding_errors_map_like_the_reference(binding):
    import paper_2301_09125_b200 as lp

    g = lp.ring_of_cliques(4, 5)
    labels = np.arange(g.vertex_count, dtype=np.int64)
    bad_order = np.zeros(g.vertex_count, dtype=np.int64)
    with pytest.raises(ValueError):
        binding.rak_cuda(g, labels, bad_order, True, 0.05, 10, 1)
