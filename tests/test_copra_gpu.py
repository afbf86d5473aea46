"""GPU parity for COPRA (copra.py), through the public API (copra_detect /
copra_run -> ctypes -> lp_copra_run).

Bars:
* every schedule (batches 0 = the reference's in-place index-order sweep,
  1 = synchronous, 7, 64) x k in {1, 2, 4, 8, 16}: best labels, label-set
  sizes, labels and float64 belongings (bitwise), iteration counts equal
  the oracle's restatement with the counter-hash fallback tie
  (``or_copra(tie=RANDOM)``), unit and float32-exact weights;
* the reference's behaviour tests (pkg/tests/test_copra.py:9-64).
"""

import numpy as np
import pytest

import paper_2301_09125_b200 as lp
from conftest import load_graph, partition_matches
from paper_2301_09125_b200.copra import copra_run

pytestmark = pytest.mark.gpu

TIE_RANDOM = 1


def _same_sets(labs, bels, sizes, olabs, obels, osizes):
    if not np.array_equal(sizes, osizes):
        return False
    K = labs.shape[1]
    mask = np.arange(K)[None, :] < sizes[:, None]
    return (np.array_equal(np.where(mask, labs, 0), np.where(mask, olabs, 0))
            and np.array_equal(np.where(mask, bels, 0.0).view(np.int64), np.where(mask, obels, 0.0).view(np.int64)))


@pytest.mark.parametrize("batches", [0, 1, 7, 64])
def test_copra_matches_oracle(gpu, golden_copra, oracle, batches):
    graphs = [(golden_copra, n) for n in sorted({k.split("/")[0] for k in golden_copra.files})]
    for z, name in graphs:
        g = load_graph(z, name)
        for K, seed, tol in ((1, 1, 0.01), (2, 2, 0.01), (4, 3, 1e-4), (8, 1, 0.01), (16, 5, 1e-4)):
            best, it, olabs, obels, osizes = oracle.copra(g, max_labels=K, batches=batches, tie=TIE_RANDOM, seed=seed,
                                                          tolerance=tol, max_iterations=15)
            p = lp.CopraParams(max_labels=K, seed=seed, tolerance=tol, max_iterations=15, batches=batches)
            gbest, git, labs, bels, sizes, _, _ = copra_run(g, p)
            key = (name, K, seed)
            assert git == it, key
            assert np.array_equal(gbest, best), key
            assert _same_sets(labs, bels, sizes, olabs, obels, osizes), key


def test_copra_big_rows_use_global_tables(gpu, oracle):
    # rows whose distinct labels overflow the per-warp table (hub of 3000 leaves + k = 8)
    g = lp.star(3000)
    best, it, olabs, obels, osizes = oracle.copra(g, max_labels=8, batches=0, tie=TIE_RANDOM, seed=2,
                                                  tolerance=1e-4, max_iterations=6)
    gbest, git, labs, bels, sizes, _, _ = copra_run(g, lp.CopraParams(max_labels=8, seed=2, tolerance=1e-4,
                                                                      max_iterations=6))
    assert git == it and np.array_equal(gbest, best)
    assert _same_sets(labs, bels, sizes, olabs, obels, osizes)
    r = lp.rmat(13, seed=4)
    for K in (1, 8):
        best, it, olabs, obels, osizes = oracle.copra(r, max_labels=K, batches=0, tie=TIE_RANDOM, seed=1,
                                                      tolerance=0.01, max_iterations=8)
        gbest, git, labs, bels, sizes, _, _ = copra_run(r, lp.CopraParams(max_labels=K, seed=1, max_iterations=8))
        assert git == it and np.array_equal(gbest, best), K
        assert _same_sets(labs, bels, sizes, olabs, obels, osizes), K


@pytest.mark.parametrize("long_row", ["0", "64"])
def test_copra_long_rows_take_the_team_path(gpu, oracle, monkeypatch, long_row):
    """Rows with more than LP_COPRA_LONG contributions (degree x k) skip the warp tiers for the
    16-warp team (one warp per hub row was the tail of every round): same sets either way."""
    from paper_2301_09125_b200 import _lib

    monkeypatch.setenv("LP_COPRA_LONG", long_row)
    for g in (lp.rmat(12, seed=6), lp.planted_partition(3000, 30, seed=3)):
        dg = _lib.DeviceGraph(g)  # fresh handle: reads the policy
        for K, batches in ((4, 0), (8, 16)):
            best, it, olabs, obels, osizes = oracle.copra(g, max_labels=K, batches=batches, tie=TIE_RANDOM, seed=3,
                                                          tolerance=0.01, max_iterations=8)
            p = lp.CopraParams(max_labels=K, seed=3, tolerance=0.01, max_iterations=8, batches=batches)
            gbest, git, labs, bels, sizes, _, _ = copra_run(g, p, device_graph=dg)
            assert git == it and np.array_equal(gbest, best), (long_row, K, batches)
            assert _same_sets(labs, bels, sizes, olabs, obels, osizes), (long_row, K, batches)
        dg.close()


def test_copra_reference_behaviour(gpu):
    """pkg/tests/test_copra.py:9-64."""
    tri = lp.disjoint_cliques(2, 3)
    assert partition_matches(lp.copra_detect(tri, lp.CopraParams(max_labels=1, seed=1)).assignment, 2, 3)
    r = lp.copra_detect(lp.gnp(1, 0.0), lp.CopraParams(seed=1))
    assert r.assignment.tolist() == [0] and r.iterations == 1
    eight = lp.disjoint_cliques(8, 6)
    for K in (1, 8):
        for seed in range(1, 11):
            assert partition_matches(lp.copra_detect(eight, lp.CopraParams(max_labels=K, seed=seed)).assignment,
                                     8, 6), (K, seed)
    g = lp.gnp(300, 0.03, seed=7)
    for K in (1, 4, 8):
        _, _, _, stats, labs, bels, sizes = lp.copra._detect_full(g, lp.CopraParams(max_labels=K, seed=3),
                                                                   check_invariants=True)
        assert stats[0] <= 1e-9 and stats[1] >= 1 and stats[2] <= K
        assert sizes.min() >= 1 and sizes.max() <= K
        for v in range(g.vertex_count):
            assert bels[v, : sizes[v]].sum() == pytest.approx(1.0, abs=1e-9)
            assert np.all(np.diff(labs[v, : sizes[v]]) > 0)
    g = lp.gnp(200, 0.05, seed=2)
    _, _, _, stats, _, _, sizes = lp.copra._detect_full(g, lp.CopraParams(max_labels=1, seed=5),
                                                         check_invariants=True)
    assert stats[1] == 1 and stats[2] == 1 and (sizes == 1).all()
    assert lp.copra_detect(g, lp.CopraParams(max_iterations=3, seed=1)).iterations <= 3
    with pytest.raises(ValueError, match="symmetric"):
        lp.copra_detect(lp.from_arcs(2, [0], [1], [1.0]))
    res = lp.copra_detect(lp.gnp(2000, 0.01, seed=9), lp.CopraParams(seed=1, max_iterations=30))
    assert res.assignment.min() >= 0 and res.assignment.max() < 2000


def test_copra_quality_vs_reference_fallback(gpu, oracle):
    """The counter-hash fallback tie vs the reference's xorshift draw: modularity
    and community counts of the projection stay close (R-MAT-14, k = 1, 4, 8)."""
    g = lp.rmat(14, seed=3)
    for K in (1, 4, 8):
        best, _, _, _, _ = oracle.copra(g, max_labels=K, batches=0, tie=3, seed=1, tolerance=0.01,
                                        max_iterations=20)
        ref_q = oracle.modularity(g, best)
        ours = lp.copra_detect(g, lp.CopraParams(max_labels=K, seed=1, max_iterations=20))
        assert abs(ours.modularity - ref_q) <= 0.02, (K, ours.modularity, ref_q)
        nc_ref, nc = len(np.unique(best)), len(np.unique(ours.assignment))
        assert abs(nc - nc_ref) <= 0.05 * nc_ref + 5, (K, nc, nc_ref)
