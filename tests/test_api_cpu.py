"""Host-side API contract (no GPU): parameter records and helpers keep the
reference's semantics (tests/test_rak.py:92-125, test_quality.py, test_graph.py)."""

import numpy as np
import pytest

import paper_2301_09125_b200 as lp
from paper_2301_09125_b200 import graph as G


class TestRakParams:
    def test_reference_defaults(self):
        p = lp.RakParams()
        assert (p.tolerance, p.strict, p.max_iterations, p.workers, p.seed) == (0.05, False, 100, 1, 1)
        assert p.batches == 0 and p.tie_rule == "random"
        assert lp.RakParams(strict=True).tie_rule == "scan-first"

    def test_validation(self):
        for bad in (dict(tolerance=0.0), dict(tolerance=1.5), dict(max_iterations=0), dict(workers=0),
                    dict(batches=-1), dict(tie="first"), dict(backend="cpu")):
            with pytest.raises(ValueError):
                lp.RakParams(**bad)


class TestChooseMaxLabel:
    """Known answers of the reference (tests/test_rak.py:92-113)."""

    def test_unique_max(self):
        assert lp.choose_max_label([5, 9], [2.0, 1.0], True, lp.XorShift32(1)) == 5
        assert lp.choose_max_label([5, 9], [2.0, 1.0], False, lp.XorShift32(1)) == 5

    def test_strict_first_in_scan_order(self):
        assert lp.choose_max_label([3, 7], [2.0, 2.0], True, lp.XorShift32(1)) == 3
        assert lp.choose_max_label([7, 3], [2.0, 2.0], True, lp.XorShift32(1)) == 7

    def test_non_strict_fair(self):
        rng = lp.XorShift32(42)
        picks = sum(lp.choose_max_label([3, 7], [2.0, 2.0], False, rng) == 3 for _ in range(10_000))
        assert abs(picks / 10_000 - 0.5) <= 0.02

    def test_duplicates_accumulate(self):
        assert lp.choose_max_label([4, 9, 4], [1.0, 1.5, 1.0], True, lp.XorShift32(1)) == 4

    def test_empty_rejected(self):
        with pytest.raises(ValueError):
            lp.choose_max_label([], [], True, lp.XorShift32(1))


class TestGraph:
    def test_from_arcs_merges_duplicates(self):
        g = G.from_arcs(3, [0, 0, 1], [1, 1, 2], [1.0, 2.0, 4.0])
        assert g.edge_count == 2 and g.weights.tolist() == [3.0, 4.0]

    def test_preprocess_idempotent_and_symmetric(self):
        raw = G.from_arcs(5, [0, 1, 2, 3, 3], [1, 2, 0, 4, 3], [2.0, 3.0, 1.0, 5.0, 7.0])
        g = G.preprocess(raw, unit_weights=False)
        G.check_symmetric(g)
        assert G.graphs_equal(g, G.preprocess(g, unit_weights=False))
        assert (np.diff(g.offsets) >= 1).all()

    def test_asymmetric_rejected(self):
        with pytest.raises(ValueError, match="symmetric"):
            G.check_symmetric(G.from_arcs(2, [0], [1], [1.0]))

    def test_degree_weights_count_loops_twice(self):
        g = lp.disjoint_cliques(1, 3)
        assert G.degree_weights(g).tolist() == [4.0, 4.0, 4.0]
        assert G.degree_weight(g, 0) == 4.0


class TestModularity:
    """Same scorer as the reference (quality.py); brute force check as in
    tests/test_quality.py:41-50."""

    def test_matches_brute_force(self):
        rng = np.random.default_rng(11)
        for trial in range(30):
            n = int(rng.integers(2, 60))
            g = lp.gnp(n, (0.05, 0.2, 0.5)[trial % 3], seed=int(rng.integers(1, 1 << 31)))
            lab = rng.integers(0, n, size=n)
            assert lp.modularity(g, lab) == pytest.approx(lp.brute_modularity(g, lab), abs=1e-9)

    def test_one_community_zero_and_two_triangles_half(self):
        g = lp.preprocess(lp.from_arcs(6, [0, 0, 1, 3, 3, 4], [1, 2, 2, 4, 5, 5], np.ones(6)), self_loops=False)
        assert lp.modularity(g, np.zeros(6, np.int64)) == pytest.approx(0.0, abs=1e-12)
        assert lp.modularity(g, np.array([0, 0, 0, 1, 1, 1])) == pytest.approx(0.5, abs=1e-12)

    def test_contract(self):
        g = lp.disjoint_cliques(2, 3)
        with pytest.raises(ValueError):
            lp.modularity(g, np.zeros(5, np.int64))
        with pytest.raises(ValueError):
            lp.modularity(g, np.full(6, 17))

    def test_oracle_scorer_agrees(self, oracle):
        g = lp.rmat(11, seed=3)
        lab = np.random.default_rng(0).integers(0, g.vertex_count, g.vertex_count)
        assert oracle.modularity(g, lab) == pytest.approx(lp.modularity(g, lab), abs=1e-12)


def test_empty_graph_needs_no_gpu():
    res = lp.rak_detect(lp.preprocess(lp.from_arcs(0, [], [], [])))
    assert res.iterations == 0 and res.assignment.size == 0


def test_reference_test_graphs_match_reference_fixtures(golden_rak):
    """Our ports of the reference's test generators rebuild the stored CSRs."""
    from conftest import load_graph

    for name, mk in (("cliques_8x6", lambda: lp.disjoint_cliques(8, 6)), ("ring_16x6", lambda: lp.ring_of_cliques(16, 6)),
                     ("gnp_400", lambda: lp.gnp(400, 0.02, seed=2)), ("gnp_3000", lambda: lp.gnp(3000, 0.005, seed=6)),
                     ("star_50", lambda: lp.star(50)), ("path_100", lambda: lp.path(100))):
        assert G.graphs_equal(mk(), load_graph(golden_rak, name)), name


def test_most_popular_label_reference_cases():
    # pkg/tests/test_slpa.py:82-96
    assert lp.most_popular_label([5, 5, 3]) == 5
    assert lp.most_popular_label([5, 3]) == 3
    assert lp.most_popular_label([7]) == 7
    with pytest.raises(ValueError):
        lp.most_popular_label([])


def test_slpa_params_validation():
    # slpa.py:42-48
    with pytest.raises(ValueError):
        lp.SlpaParams(memory_size=1)
    with pytest.raises(ValueError):
        lp.SlpaParams(tolerance=0.0)
    with pytest.raises(ValueError):
        lp.SlpaParams(workers=0)
    with pytest.raises(ValueError):
        lp.SlpaParams(batches=-1)
    assert lp.SlpaParams().tie_rule == "random" and lp.SlpaParams(strict=True).tie_rule == "scan-first"


def test_collect_and_threshold_reference_cases():
    # pkg/tests/test_copra.py:68-110
    labels, bels = lp.collect_and_threshold([10, 20], [0.6, 0.4], 4, lp.XorShift32(1))
    assert labels.tolist() == [10, 20] and bels.tolist() == pytest.approx([0.6, 0.4])
    labels, bels = lp.collect_and_threshold([1, 2, 3], [0.5, 0.3, 0.2], 4, lp.XorShift32(1))
    assert labels.tolist() == [1, 2] and bels.tolist() == pytest.approx([0.625, 0.375])
    seen = set()
    rng = lp.XorShift32(5)
    for _ in range(200):
        labels, bels = lp.collect_and_threshold([0, 1, 2, 3, 4], [0.2] * 5, 4, rng)
        assert labels.size == 1 and bels.tolist() == [1.0]
        seen.add(int(labels[0]))
    assert seen == {0, 1, 2, 3, 4}
    labels, bels = lp.collect_and_threshold([0, 2], [1.0, 1.0], 2, lp.XorShift32(1))
    assert labels.tolist() == [0, 2] and bels.tolist() == pytest.approx([0.5, 0.5])
    labels, _ = lp.collect_and_threshold([9, 1, 5], [0.4, 0.3, 0.3], 4, lp.XorShift32(1))
    assert labels.tolist() == sorted(labels.tolist())
    with pytest.raises(ValueError):
        lp.collect_and_threshold([], [], 4, lp.XorShift32(1))


def test_best_label_reference_cases():
    # pkg/tests/test_copra.py:113-126
    assert lp.best_label([7, 2], [0.6, 0.4]) == 7
    assert lp.best_label([7, 2], [0.5, 0.5]) == 2
    assert lp.best_label([3], [1.0]) == 3
    with pytest.raises(ValueError):
        lp.best_label([], [])


def test_copra_params_validation():
    # copra.py:42-50
    for bad in (dict(max_labels=0), dict(tolerance=0.0), dict(workers=0), dict(max_iterations=0), dict(batches=-1)):
        with pytest.raises(ValueError):
            lp.CopraParams(**bad)
    p = lp.CopraParams()
    assert (p.tolerance, p.max_labels, p.max_iterations, p.workers, p.seed) == (0.01, 8, 100, 1, 1)


def test_sweep_spec_and_csv_schema():
    """sweep.py keeps the reference harness's contract (labelprop/sweep.py:26-102):
    grid validation, combos per graph, the 11-column CSV row."""
    from paper_2301_09125_b200 import sweep

    assert lp.CSV_HEADER.split(",") == ["graph", "algorithm", "mode", "tolerance", "max_labels", "memory_size",
                                         "workers", "seed", "iterations", "elapsed_ms", "modularity"]
    with pytest.raises(ValueError):
        lp.SweepSpec("louvain")
    with pytest.raises(ValueError):
        lp.SweepSpec("rak", tolerances=())
    with pytest.raises(ValueError):
        lp.SweepSpec("rak", repetitions=0)
    assert lp.SweepSpec("rak", tolerances=(0.1, 0.05), workers=(1, 2), repetitions=3).combos_per_graph() == 24
    assert lp.SweepSpec("copra", tolerances=(0.01,), max_labels=(1, 4)).combos_per_graph() == 2
    assert lp.SweepSpec("slpa", memory_sizes=(4, 8), batches=(0, 1)).combos_per_graph() == 8
    pts = list(sweep.combos(lp.SweepSpec("copra", tolerances=(0.01,), max_labels=(1, 4))))
    assert [p["max_labels"] for p in pts] == [1, 4] and all(p["mode"] == "" for p in pts)
    r = lp.RunRecord("g", "copra", "", 0.01, 4, None, 1, 7, 3, 1.5, 0.25, batches=1, edges_scanned=3_000_000)
    assert r.csv_row() == "g,copra,,0.01,4,,1,7,3,1.500,0.250000000"
    assert r.csv_row(extended=True).endswith(",1,3000000,2.0000")
    assert len(r.csv_row(extended=True).split(",")) == len(sweep.CSV_HEADER_EXTENDED.split(","))


def test_cli_specs_and_info(tmp_path, capsys):
    """cli.py: generator specs, .npz CSR files, `info` (no GPU needed)."""
    from paper_2301_09125_b200 import cli

    g = cli.load_spec("planted:2000:20:3")
    assert G.graphs_equal(g, lp.planted_partition(2000, 20, seed=3))
    p = tmp_path / "g.npz"
    np.savez(p, offsets=g.offsets, neighbors=g.neighbors)
    assert G.graphs_equal(cli.load_spec(str(p)), g)
    with pytest.raises(ValueError):
        cli.load_spec("louvain:3")
    assert cli.main(["info", "rmat:10", str(p)]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "graph\tvertices\tedges\tavg_degree" and out[1].startswith("rmat:10\t1024\t")
    assert cli.main(["info", "bogus:1"]) == 2
