"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_golden python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (pure Python
+ numba; only the sequential kernels are used -- the parallel ones do not
compile under numba 0.65) and stores, for a set of
small seeded graphs, the reference's own outputs:

* prng.npz   -- xorshift32 streams, mix_seed values, shuffled_indices;
* rak.npz    -- per-iteration labels (a run with max_iterations = k gives
                the labels after sweep k, `tests/test_rak.py:45-56` prefix
                property) and iteration counts for strict and non-strict
                modes, several seeds and tolerances;
* copra.npz  -- best labels, label sets, belongings, sizes, iterations;
* slpa.npz   -- projected labels, memories, fill counts, iterations;
* modularity values for every final assignment.

Each graph's CSR is stored next to its outputs so the fixtures are
self-contained inputs for the oracle and the CUDA engine.  The fixtures are
committed; /root/reference is never read at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import labelprop as ref  # noqa: E402  (the reference)
from labelprop.copra import _detect_full as ref_copra_full  # noqa: E402
from labelprop.prng import mix_seed, shuffled_indices, xs32_next  # noqa: E402
from labelprop.slpa import _detect_full as ref_slpa_full  # noqa: E402

from paper_2301_09125_b200 import synth  # noqa: E402  (our generators, inputs only)


def rak_graphs():
    """Small graphs that cover the reference tests' shapes plus the
    benchmark generators at reduced size."""
    return {
        "cliques_8x6": ref.disjoint_cliques(8, 6),
        "cliques_2x4": ref.disjoint_cliques(2, 4),
        "ring_16x6": ref.ring_of_cliques(16, 6),
        "ring_8x5": ref.ring_of_cliques(8, 5),
        "gnp_400": ref.gnp(400, 0.02, seed=2),
        "gnp_1000": ref.gnp(1000, 0.01, seed=3),
        "gnp_3000": ref.gnp(3000, 0.005, seed=6),
        "star_50": ref.star(50),
        "path_100": ref.path(100),
        "isolated_12": ref.gnp(12, 0.0),
        "planted_4000": synth.planted_partition(4000, 40, seed=3),
        "rmat_12": synth.rmat(12, seed=5),
        "rmat_12_w": synth.rmat(12, seed=5, weighted=True),
        "grid_64": synth.road_grid(64, seed=2),
    }


def store_graph(out, name, g):
    out[f"{name}/offsets"] = np.asarray(g.offsets, dtype=np.int64)
    out[f"{name}/neighbors"] = np.asarray(g.neighbors, dtype=np.int32)
    out[f"{name}/weights"] = np.asarray(g.weights, dtype=np.float64)
    out[f"{name}/total_weight"] = np.float64(g.total_weight)


def make_prng():
    out = {}
    for seed in (1, 2, 12345, 0x80000000, 0xFFFFFFFF):
        x, seq = seed, []
        for _ in range(64):
            x = int(xs32_next(x))
            seq.append(x)
        out[f"xs32/{seed}"] = np.array(seq, dtype=np.uint32)
    ms = [[seed, k, int(mix_seed(seed, k))] for seed in (0, 1, 77, 0xFFFFFFFF) for k in (0, 1, 11, 4096, 0x4F524452)]
    out["mix_seed"] = np.array(ms, dtype=np.int64)
    for n, seed in ((1, 1), (2, 1), (10, 3), (1000, 5), (100_000, 1), (4096, 7)):
        out[f"shuffled/{n}/{seed}"] = shuffled_indices(n, seed)
    # worker_states and XorShift32 known answers (test_prng.py:23-26, :58-61)
    out["known/next1"] = np.array([ref.XorShift32(1).next()], dtype=np.int64)
    out["known/bounded10"] = np.array([ref.XorShift32(1).next_bounded(10)], dtype=np.int64)
    return out


def make_rak(graphs):
    out = {}
    for name, g in graphs.items():
        store_graph(out, name, g)
        for strict in (True, False):
            for seed in (1, 2, 3):
                for tol in (0.05, 1e-4):
                    p = ref.RakParams(strict=strict, seed=seed, tolerance=tol, max_iterations=100)
                    res = ref.rak_detect(g, p)
                    key = f"{name}/{'s' if strict else 'ns'}/{seed}/{tol:g}"
                    out[f"{key}/iterations"] = np.int64(res.iterations)
                    out[f"{key}/modularity"] = np.float64(res.modularity)
                    per = []
                    for k in range(1, res.iterations + 1):
                        rk = ref.rak_detect(g, ref.RakParams(strict=strict, seed=seed, tolerance=tol,
                                                             max_iterations=k))
                        per.append(rk.assignment)
                    per = np.stack(per) if per else np.zeros((0, g.vertex_count), np.int64)
                    assert np.array_equal(per[-1] if len(per) else np.arange(g.vertex_count),
                                          res.assignment)
                    out[f"{key}/labels_per_iter"] = per.astype(np.int32)
    return out


def make_copra(graphs):
    out = {}
    names = ["cliques_8x6", "ring_16x6", "gnp_400", "gnp_1000", "star_50", "path_100", "planted_4000",
             "rmat_12", "rmat_12_w"]
    for name in names:
        g = graphs[name]
        store_graph(out, name, g)
        for ml in (1, 4, 8):
            for seed in (1, 2):
                best, it, _, _, labs, bels, sizes = ref_copra_full(
                    g, ref.CopraParams(max_labels=ml, seed=seed, max_iterations=30))
                key = f"{name}/{ml}/{seed}"
                out[f"{key}/best"] = best.astype(np.int32)
                out[f"{key}/iterations"] = np.int64(it)
                out[f"{key}/labs"] = labs.astype(np.int32)
                out[f"{key}/bels"] = bels
                out[f"{key}/sizes"] = sizes.astype(np.int32)
                out[f"{key}/modularity"] = np.float64(ref.modularity(g, best))
    return out


def make_slpa(graphs):
    out = {}
    names = ["cliques_8x6", "ring_16x6", "gnp_400", "gnp_1000", "star_50", "isolated_12", "planted_4000",
             "rmat_12"]
    for name in names:
        g = graphs[name]
        store_graph(out, name, g)
        for strict in (True, False):
            for ms in (5, 12):
                seed = 3
                labels, it, _, slots, filled = ref_slpa_full(
                    g, ref.SlpaParams(memory_size=ms, strict=strict, seed=seed, tolerance=0.05))
                key = f"{name}/{'s' if strict else 'ns'}/{ms}/{seed}"
                out[f"{key}/labels"] = labels.astype(np.int32)
                out[f"{key}/iterations"] = np.int64(it)
                out[f"{key}/slots"] = slots.astype(np.int32)
                out[f"{key}/filled"] = filled.astype(np.int32)
                out[f"{key}/modularity"] = np.float64(ref.modularity(g, labels))
    return out


def main():
    graphs = rak_graphs()
    np.savez_compressed(os.path.join(HERE, "prng.npz"), **make_prng())
    np.savez_compressed(os.path.join(HERE, "rak.npz"), **make_rak(graphs))
    np.savez_compressed(os.path.join(HERE, "copra.npz"), **make_copra(graphs))
    np.savez_compressed(os.path.join(HERE, "slpa.npz"), **make_slpa(graphs))
    for f in ("prng.npz", "rak.npz", "copra.npz", "slpa.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
