"""The CPU oracle is pinned to the reference: its outputs equal the golden
fixtures produced by running the reference itself (tests/golden/make_golden.py).

CPU-only; these are the checks that make the oracle trustworthy as the GPU's
parity target."""

import numpy as np
import pytest

from conftest import load_graph


def _names(z):
    return sorted({k.split("/")[0] for k in z.files})


def test_shuffled_indices_match_reference(golden_prng, oracle):
    for k in golden_prng.files:
        if k.startswith("shuffled/"):
            _, n, seed = k.split("/")
            assert np.array_equal(oracle.shuffled_indices(int(n), int(seed)), golden_prng[k]), k


def test_xorshift_and_mix_seed_known_answers(golden_prng, oracle):
    L = oracle.lib()
    for k in golden_prng.files:
        if k.startswith("xs32/"):
            x = int(k.split("/")[1]) & 0xFFFFFFFF
            for want in golden_prng[k]:
                x = L.or_xs32_next(x)
                assert x == int(want)
    for seed, kk, want in golden_prng["mix_seed"]:
        assert L.or_mix_seed(int(seed) & 0xFFFFFFFF, int(kk)) == int(want)
    assert L.or_xs32_next(1) == 270369 == int(golden_prng["known/next1"][0])  # test_prng.py:23-26


@pytest.mark.parametrize("mode", ["s", "ns"])
def test_rak_sequential_equals_reference_every_iteration(golden_rak, oracle, mode):
    """batches = n reproduces rak._rak_seq label-for-label after every sweep,
    strict and non-strict (the latter with the reference's xorshift stream)."""
    tie = oracle.TIE_SCAN_FIRST if mode == "s" else oracle.TIE_XORSHIFT
    checked = 0
    for name in _names(golden_rak):
        g = load_graph(golden_rak, name)
        for seed in (1, 2, 3):
            for tol in (0.05, 1e-4):
                key = f"{name}/{mode}/{seed}/{tol:g}"
                lab, it, _, per = oracle.rak(g, batches=0, tie=tie, seed=seed, tolerance=tol,
                                             max_iterations=100, per_iteration=True)
                assert it == int(golden_rak[f"{key}/iterations"]), key
                assert np.array_equal(per, golden_rak[f"{key}/labels_per_iter"]), key
                checked += 1
    assert checked >= 80


def test_copra_equals_reference(golden_copra, oracle):
    for name in _names(golden_copra):
        g = load_graph(golden_copra, name)
        for ml in (1, 4, 8):
            for seed in (1, 2):
                key = f"{name}/{ml}/{seed}"
                best, it, labs, bels, sizes = oracle.copra(g, max_labels=ml, seed=seed, max_iterations=30)
                assert it == int(golden_copra[f"{key}/iterations"]), key
                assert np.array_equal(best, golden_copra[f"{key}/best"]), key
                assert np.array_equal(sizes, golden_copra[f"{key}/sizes"]), key
                assert np.array_equal(labs, golden_copra[f"{key}/labs"]), key
                assert np.array_equal(bels, golden_copra[f"{key}/bels"]), key


def test_slpa_equals_reference(golden_slpa, oracle):
    for name in _names(golden_slpa):
        g = load_graph(golden_slpa, name)
        for mode in ("s", "ns"):
            for ms in (5, 12):
                key = f"{name}/{mode}/{ms}/3"
                labels, it, slots, filled = oracle.slpa(
                    g, memory_size=ms, tie=oracle.TIE_SCAN_FIRST if mode == "s" else oracle.TIE_XORSHIFT,
                    seed=3, tolerance=0.05)
                assert it == int(golden_slpa[f"{key}/iterations"]), key
                assert np.array_equal(labels, golden_slpa[f"{key}/labels"]), key
                assert np.array_equal(slots, golden_slpa[f"{key}/slots"]), key
                assert np.array_equal(filled, golden_slpa[f"{key}/filled"]), key


def test_oracle_modularity_matches_reference_scores(golden_rak, oracle):
    for name in _names(golden_rak):
        g = load_graph(golden_rak, name)
        key = f"{name}/s/1/0.05"
        lab = golden_rak[f"{key}/labels_per_iter"][-1].astype(np.int64)
        assert oracle.modularity(g, lab) == pytest.approx(float(golden_rak[f"{key}/modularity"]), abs=1e-12)


def test_batched_extremes(golden_rak, oracle):
    """batches=1 is a Jacobi sweep: every vertex reads only sweep-start labels."""
    g = load_graph(golden_rak, "gnp_400")
    n = g.vertex_count
    lab1, it1, _ = oracle.rak(g, batches=1, tie=oracle.TIE_SCAN_FIRST, tolerance=1.0, max_iterations=1)
    # one Jacobi sweep by hand
    lab0 = np.arange(n)
    want = np.empty(n, np.int64)
    for v in range(n):
        row = g.neighbors[g.offsets[v]:g.offsets[v + 1]]
        seen, tally = [], {}
        for u in row:
            l = lab0[u]
            if l not in tally:
                seen.append(l)
                tally[l] = 0
            tally[l] += 1
        best = max(seen, key=lambda l: (tally[l], -seen.index(l)))
        want[v] = best
    assert it1 == 1 and np.array_equal(lab1, want)
