"""GPU parity for the RAK sweep, through the public API (rak_detect ->
ctypes -> liblabelprop_cuda.so).

Bars:
* batches = 0 (the reference's visit order), strict: labels bit-exact to the
  REFERENCE after every sweep and the same iteration count (golden fixtures
  produced by the reference itself);
* every schedule / tie rule: labels bit-exact to the oracle's restatement of
  the same schedule after every sweep;
* float weights in [1, 2) (float32-exact): bit-exact as well (exact 64-bit
  fixed-point sums).
"""

import numpy as np
import pytest

import paper_2301_09125_b200 as lp
from conftest import load_graph, partition_matches

pytestmark = pytest.mark.gpu

ORACLE_TIE = {"scan-first": 0, "random": 1, "min-label": 2}


def _names(z):
    return sorted({k.split("/")[0] for k in z.files})


def gpu_per_iteration(g, params, upto):
    out = []
    for k in range(1, upto + 1):
        p = lp.RakParams(**{**params.__dict__, "max_iterations": k})
        out.append(lp.rak_detect(g, p).assignment)
    return np.stack(out)


def test_exact_schedule_matches_reference_every_iteration(gpu, golden_rak):
    checked = 0
    for name in _names(golden_rak):
        g = load_graph(golden_rak, name)
        for seed in (1, 2, 3):
            for tol in (0.05, 1e-4):
                key = f"{name}/s/{seed}/{tol:g}"
                want_it = int(golden_rak[f"{key}/iterations"])
                want = golden_rak[f"{key}/labels_per_iter"]
                p = lp.RakParams(strict=True, seed=seed, tolerance=tol, max_iterations=100)
                res = lp.rak_detect(g, p)
                assert res.iterations == want_it, key
                assert np.array_equal(res.assignment, want[-1]), key
                assert res.modularity == pytest.approx(float(golden_rak[f"{key}/modularity"]), abs=1e-12)
                if tol == 0.05:
                    assert np.array_equal(gpu_per_iteration(g, p, want_it), want), key
                checked += 1
    assert checked == 6 * len(_names(golden_rak))


@pytest.mark.parametrize("tie", ["scan-first", "random", "min-label"])
@pytest.mark.parametrize("batches", [0, 1, 7, 64])
def test_schedules_match_oracle_every_iteration(gpu, golden_rak, oracle, tie, batches):
    for name in ("gnp_1000", "gnp_3000", "planted_4000", "rmat_12", "rmat_12_w", "ring_16x6", "grid_64", "star_50"):
        g = load_graph(golden_rak, name)
        for seed in (1, 5):
            want, it, changed, per = oracle.rak(g, batches=batches, tie=ORACLE_TIE[tie], seed=seed, tolerance=1e-4,
                                                max_iterations=12, per_iteration=True)
            p = lp.RakParams(seed=seed, tolerance=1e-4, max_iterations=12, batches=batches, tie=tie)
            res = lp.rak_detect(g, p, changed_history=True)
            assert res.iterations == it, (name, seed)
            assert np.array_equal(res.stats["changed"], changed), (name, seed)
            assert np.array_equal(res.assignment, want), (name, seed)
            assert np.array_equal(gpu_per_iteration(g, p, it), per), (name, seed)


def test_weighted_graph_uses_exact_fixed_point(gpu, golden_rak):
    g = load_graph(golden_rak, "rmat_12_w")
    info = lp._lib.device_graph(g).info()
    assert info["weight_mode"] == "fixed"


def test_non_strict_quality_close_to_reference(gpu, golden_rak):
    """Counter-RNG non-strict vs the reference's xorshift non-strict: the
    draws differ, so compare modularity (the reference's own seed spread is
    the yardstick on these small graphs)."""
    for name in ("gnp_3000", "planted_4000", "rmat_12"):
        g = load_graph(golden_rak, name)
        ref_q = [float(golden_rak[f"{name}/ns/{s}/0.05/modularity"]) for s in (1, 2, 3)]
        ours = [lp.rak_detect(g, lp.RakParams(strict=False, seed=s)).modularity for s in (1, 2, 3)]
        spread = max(ref_q) - min(ref_q)
        assert abs(np.mean(ours) - np.mean(ref_q)) <= max(0.02, 2 * spread), (name, ours, ref_q)


class TestReferenceBehaviour:
    """The reference's own RAK tests (tests/test_rak.py), run on the GPU."""

    def test_two_disjoint_four_cliques_strict(self, gpu):
        g = lp.disjoint_cliques(2, 4)
        assert partition_matches(lp.rak_detect(g, lp.RakParams(strict=True, seed=1)).assignment, 2, 4)

    def test_isolated_vertices_keep_their_labels(self, gpu):
        res = lp.rak_detect(lp.gnp(12, 0.0), lp.RakParams(strict=True, seed=1))
        assert np.array_equal(res.assignment, np.arange(12)) and res.iterations == 1

    def test_star_collapses_to_one_community(self, gpu):
        res = lp.rak_detect(lp.star(5), lp.RakParams(strict=True, seed=1))
        assert len(set(res.assignment.tolist())) == 1 and res.iterations <= 2

    def test_clique_recovery_all_modes_and_seeds(self, gpu):
        g = lp.disjoint_cliques(8, 6)
        for strict in (True, False):
            for seed in range(1, 11):
                res = lp.rak_detect(g, lp.RakParams(strict=strict, seed=seed))
                assert partition_matches(res.assignment, 8, 6), (strict, seed)

    def test_ring_of_cliques_not_degenerate(self, gpu):
        g = lp.ring_of_cliques(16, 6)
        for strict in (True, False):
            clean = sum(np.bincount(lp.rak_detect(g, lp.RakParams(strict=strict, seed=s)).assignment).max()
                        <= g.vertex_count / 2 for s in range(1, 21))
            assert clean >= 18

    def test_strict_is_deterministic(self, gpu):
        g = lp.gnp(500, 0.02, seed=5)
        a = lp.rak_detect(g, lp.RakParams(strict=True, seed=9)).assignment
        b = lp.rak_detect(g, lp.RakParams(strict=True, seed=9)).assignment
        assert a.tobytes() == b.tobytes()

    def test_tolerance_monotonic_and_prefix(self, gpu):
        for g in (lp.gnp(400, 0.02, seed=2), lp.ring_of_cliques(8, 5)):
            loose = lp.rak_detect(g, lp.RakParams(tolerance=0.1, strict=True, seed=4))
            tight = lp.rak_detect(g, lp.RakParams(tolerance=0.0001, strict=True, seed=4))
            assert tight.iterations >= loose.iterations
            replay = lp.rak_detect(g, lp.RakParams(tolerance=0.0001, strict=True, seed=4,
                                                   max_iterations=loose.iterations))
            assert np.array_equal(loose.assignment, replay.assignment)

    def test_asymmetric_graph_rejected(self, gpu):
        with pytest.raises(ValueError, match="symmetric"):
            lp.rak_detect(lp.from_arcs(2, [0], [1], [1.0]))

    def test_empty_graph(self, gpu):
        res = lp.rak_detect(lp.preprocess(lp.from_arcs(0, [], [], [])))
        assert res.iterations == 0 and res.assignment.size == 0

    def test_labels_stay_in_range(self, gpu):
        res = lp.rak_detect(lp.gnp(200, 0.05, seed=8), lp.RakParams(seed=3))
        assert res.assignment.min() >= 0 and res.assignment.max() < 200 and res.iterations <= 100


class TestEdgeCases:
    def test_graph_without_self_loops(self, gpu, oracle):
        """Degree-1 rows whose arc is not a self-loop must still move."""
        g = lp.preprocess(lp.from_arcs(6, [0, 1, 3, 4], [1, 2, 4, 5], np.ones(4)), self_loops=False)
        for batches in (0, 1):
            want, it, _ = oracle.rak(g, batches=batches, tie=0, tolerance=1e-4, max_iterations=10)
            res = lp.rak_detect(g, lp.RakParams(strict=True, tolerance=1e-4, max_iterations=10, batches=batches))
            assert np.array_equal(res.assignment, want) and res.iterations == it

    def test_custom_order_and_initial_labels(self, gpu, oracle):
        g = lp.gnp(800, 0.01, seed=4)
        rng = np.random.default_rng(0)
        order = rng.permutation(800)
        init = rng.integers(0, 800, 800)
        for batches in (0, 3):
            want, it, _ = oracle.rak(g, batches=batches, tie=0, order=order, labels=init, tolerance=1e-3,
                                     max_iterations=20)
            res = lp.rak_detect(g, lp.RakParams(strict=True, tolerance=1e-3, max_iterations=20, batches=batches),
                                order=order, labels=init)
            assert np.array_equal(res.assignment, want) and res.iterations == it

    def test_bad_order_and_labels_rejected(self, gpu):
        g = lp.gnp(50, 0.1, seed=1)
        with pytest.raises(ValueError):
            lp.rak_detect(g, order=np.zeros(50, dtype=np.int64))
        with pytest.raises(ValueError):
            lp.rak_detect(g, labels=np.full(50, 50))

    def test_single_vertex(self, gpu):
        res = lp.rak_detect(lp.gnp(1, 0.0), lp.RakParams(strict=True))
        assert res.assignment.tolist() == [0] and res.iterations == 1

    def test_hub_multipass_matches_oracle(self, gpu, oracle):
        """A hub whose distinct neighbour labels exceed one shared-memory
        table (forces the multi-pass partitioned tally and its overflow retry)."""
        n = 30_000
        hub_edges = np.arange(1, n)
        rng = np.random.default_rng(3)
        extra_u = rng.integers(1, n, 40_000)
        extra_v = rng.integers(1, n, 40_000)
        g = lp.undirected_csr(n, np.concatenate([np.zeros(n - 1, np.int64), extra_u]),
                              np.concatenate([hub_edges, extra_v]))
        for tie, otie in (("scan-first", 0), ("random", 1), ("min-label", 2)):
            for batches in (0, 1):
                want, it, _ = oracle.rak(g, batches=batches, tie=otie, tolerance=1e-4, max_iterations=6)
                res = lp.rak_detect(g, lp.RakParams(tie=tie, tolerance=1e-4, max_iterations=6, batches=batches))
                assert np.array_equal(res.assignment, want) and res.iterations == it, (tie, batches)


def test_gpu_modularity_matches_numpy(gpu, golden_rak):
    """quality.modularity_gpu (lp_modularity) vs the numpy restatement of
    quality.py:10-42: same value up to float64 summation order."""
    from paper_2301_09125_b200 import quality

    rng = np.random.default_rng(3)
    for name in ("gnp_1000", "planted_4000", "rmat_12", "rmat_12_w", "star_50", "grid_64", "isolated_12"):
        g = load_graph(golden_rak, name)
        n = g.vertex_count
        for lab in (np.arange(n), np.zeros(n, dtype=np.int64), rng.integers(0, max(1, n // 7), n),
                    lp.rak_detect(g, lp.RakParams(strict=True)).assignment):
            q_cpu = quality.modularity(g, lab)
            q_gpu = quality.modularity_gpu(g, lab)
            assert q_gpu == pytest.approx(q_cpu, abs=1e-12), name
    g = lp.rmat(16, seed=5)
    res = lp.rak_detect(g, lp.RakParams(strict=True))
    dg = lp._lib.device_graph(g)
    assert quality.modularity_gpu(g, None, device_graph=dg) == pytest.approx(quality.modularity(g, res.assignment),
                                                                             abs=1e-12)
    with pytest.raises(ValueError):
        quality.modularity_gpu(g, np.full(g.vertex_count, g.vertex_count))


def test_exact_schedule_full_size_rmat20(gpu, oracle):
    """The reference's in-place strict sweep on R-MAT-20 (1M vertices, 32M arcs):
    labels after the run and per-sweep changed counts bit-exact to the
    oracle's sequential restatement (which is pinned to the reference)."""
    g = lp.rmat(20, seed=1)
    want, it, changed = oracle.rak(g, batches=0, tie=0, seed=1, tolerance=0.05, max_iterations=20)
    res = lp.rak_detect(g, lp.RakParams(strict=True, seed=1, tolerance=0.05, max_iterations=20),
                        changed_history=True)
    assert res.iterations == it
    assert np.array_equal(res.stats["changed"], changed)
    assert np.array_equal(res.assignment, want)
    # and the synchronous / batched schedules against their restatements
    for batches, tie in ((1, 0), (64, 1)):
        want, it, changed = oracle.rak(g, batches=batches, tie=tie, seed=2, tolerance=0.05, max_iterations=20)
        res = lp.rak_detect(g, lp.RakParams(seed=2, tolerance=0.05, max_iterations=20, batches=batches,
                                            tie=["scan-first", "random"][tie]), changed_history=True)
        assert res.iterations == it and np.array_equal(res.assignment, want), batches


def test_exact_schedule_full_size_other_rules(gpu, oracle):
    """The reference visit order at scale for the other tie rules and weights
    (first rounds from ids, singleton two-pass tallies, hub partitions):
    non-strict and min-label on R-MAT-20, float32 weights (exact fixed point)
    on R-MAT-18 -- labels and per-sweep changed counts bit-exact to the oracle."""
    g = lp.rmat(20, seed=3)
    for tie in ("random", "min-label"):
        want, it, changed = oracle.rak(g, batches=0, tie=ORACLE_TIE[tie], seed=4, tolerance=0.05, max_iterations=20)
        res = lp.rak_detect(g, lp.RakParams(seed=4, tolerance=0.05, max_iterations=20, tie=tie), changed_history=True)
        assert res.iterations == it and np.array_equal(res.stats["changed"], changed), tie
        assert np.array_equal(res.assignment, want), tie
    gw = lp.rmat(18, seed=5, weighted=True)
    want, it, changed = oracle.rak(gw, batches=0, tie=0, seed=1, tolerance=0.05, max_iterations=20)
    res = lp.rak_detect(gw, lp.RakParams(strict=True, seed=1, tolerance=0.05, max_iterations=20), changed_history=True)
    assert res.iterations == it and np.array_equal(res.stats["changed"], changed)
    assert np.array_equal(res.assignment, want)


def test_malformed_csr_rejected_on_upload(gpu):
    from paper_2301_09125_b200 import _lib

    off = np.array([0, 2, 1, 3], dtype=np.int64)  # decreasing
    nbr = np.array([0, 1, 2], dtype=np.int64)
    g = lp.Graph(3, 3, off, nbr, np.ones(3), 3.0)
    with pytest.raises(ValueError, match="non-decreasing"):
        _lib.DeviceGraph(g)
    g = lp.Graph(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 7]), np.ones(3), 3.0)
    with pytest.raises(ValueError, match="neighbor ids"):
        _lib.DeviceGraph(g)


@pytest.mark.parametrize("env", [
    {"LP_DENSE_FRAC": "1.01"},                    # always marks + frontier rounds
    {"LP_DENSE_FRAC": "0.0"},                     # always full rounds
    {"LP_CARRY_FRAC": "1.0"},                     # carry the frontier across every sweep
    {"LP_MARGIN": "0"},                           # no margin skipping
    {"LP_FIRST_ROUND": "0", "LP_SWEEP_FRONTIER": "0"},
    {"LP_WAVES": "4"},                            # dense waves
    {"LP_ID_SINGLE": "0"},                        # no first-sweep singleton labels
    {"LP_FIRST_ROUND": "0"},                      # singleton labels in a full first round (all weight 1)
    {"LP_CAP_ROUTE": "1", "LP_WARP0_MAXD": "512"},  # capacity / degree routing
    {"LP_REG_EST": "32", "LP_PUSH_DIV": "50"},    # register tables up to 32 labels, pulled sweep marks
    {"LP_MID_MAX": "0"},                          # no thread-per-row mid-degree kernel
    {"LP_MARK_BITMAP": "0"},                      # marks always queued by scanning
    {"LP_ID_SINGLE_W": "0", "LP_ID_SINGLE_RANDOM": "0"},  # singletons for unit weights / scan ties only
    {"LP_TWO_TEAM_W": "0"},                       # weighted team rows insert every label
    {"LP_MID_HASH": "0"},                         # mid-degree rows by O(d^2) compares
    {"LP_HUB_BUCKET": "1", "LP_FIRST_EST_MIN": "16", "LP_FIRST_EST_DIV": "64"},  # hub buckets, low estimates
    {"LP_FIRST_CHAIN": "0"},                      # plain first-arc first round in exact schedules
    {"LP_FUSE_MAXD": "0"},                        # every row through the phase-1 buffer
    {"LP_FUSE_MAXD": "-1"},                       # every row gathers its own labels (fused)
    {"LP_FUSE_MAXD": "64", "LP_L2_PERSIST": "0"},  # small and mid rows fused; no L2 window
    {"LP_SWEEP_FRONTIER": "0"},                   # no frontier across sweeps (random ties too)
    {"LP_LOOP_ROWS": "0"},                        # no frontier loop: every round through the class kernels
    {"LP_LOOP_ROWS": "1000000", "LP_LOOP_MAX_QUEUE": "1000000"},  # the loop takes every frontier it can
    {"LP_LOOP_DENSE_ARCS": "0"},                  # frontier loop for tails only (no dense rounds in it)
    {"LP_LOOP_ROWS": "1000000", "LP_LOOP_BLOCKS": "1", "LP_DENSE_FRAC": "1.01"},  # one block per SM, long loops
])
def test_engine_policies_keep_exactness(gpu, oracle, env, monkeypatch):
    """Every scheduling policy of the engine (chosen per handle from the
    environment) must reach the same fixed point: bit-exact to the oracle."""
    from paper_2301_09125_b200 import _lib

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for g in (lp.rmat(14, seed=3), lp.planted_partition(6000, 60, seed=2),
              lp.synth.with_edge_weights(lp.rmat(12, seed=4), seed=1)):
        dg = _lib.DeviceGraph(g)  # fresh handle: reads the policy
        for batches, tie in ((0, "scan-first"), (0, "random"), (1, "scan-first"), (16, "min-label")):
            want, it, changed = oracle.rak(g, batches=batches, tie=ORACLE_TIE[tie], seed=2, tolerance=1e-3,
                                           max_iterations=15)
            p = lp.RakParams(seed=2, tolerance=1e-3, max_iterations=15, batches=batches, tie=tie)
            out, git, st, gch = lp.rak_labels(g, p, device_graph=dg)
            assert git == it and np.array_equal(gch, changed), (env, batches, tie)
            assert np.array_equal(out, want), (env, batches, tie)
        dg.close()


def test_gpu_graph_builders_match_host(gpu, monkeypatch):
    """lp_gen_rmat_csr / lp_csr_build_undirected_gpu build the same arrays as
    the host builder (which tests/test_host_abi.py pins to the reference's
    preprocess(from_arcs(...)))."""
    import ctypes as C

    from paper_2301_09125_b200 import _lib, synth

    monkeypatch.setenv("LP_BUILD_GPU", "0")
    host = synth.rmat(14, seed=7)
    monkeypatch.setenv("LP_BUILD_GPU", "1")
    dev = synth.rmat(14, seed=7)
    assert np.array_equal(host.offsets, dev.offsets) and np.array_equal(host.neighbors, dev.neighbors)
    rng = np.random.default_rng(5)
    n = 3000
    u = rng.integers(0, n, 40000)
    v = rng.integers(0, n, 40000)
    v[:500] = u[:500]  # self pairs
    u[500:900] = u[900:1300]  # duplicates
    v[500:900] = v[900:1300]
    want = lp.undirected_csr(n, u, v)
    off = np.empty(n + 1, dtype=np.int64)
    nbr = np.empty(2 * u.size + n, dtype=np.int64)
    m = C.c_int64(0)
    _lib.check(_lib.lib().lp_csr_build_undirected_gpu(n, u.size, u.astype(np.int64), v.astype(np.int64), -1, off, nbr,
                                                      nbr.size, C.byref(m)))
    assert m.value == want.edge_count
    assert np.array_equal(off, want.offsets) and np.array_equal(nbr[: m.value], want.neighbors)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().lp_csr_build_undirected_gpu(10, 1, np.array([0]), np.array([11]), -1,
                                                          np.empty(11, np.int64), np.empty(12, np.int64), 12,
                                                          C.byref(m)))


def test_sweep_runs_the_cuda_detectors(gpu):
    """run_sweep (sweep.py, the reference harness's interface) streams one record
    per grid point with the detectors' own results."""
    g = lp.planted_partition(3000, 30, seed=4)
    spec = lp.SweepSpec("rak", tolerances=(0.05,), modes=("strict",), batches=(0, 1), repetitions=2, seed=3)
    recs = list(lp.run_sweep(spec, [("planted", g)]))
    assert len(recs) == spec.combos_per_graph() == 4
    for r in recs:
        want = lp.rak_detect(g, lp.RakParams(tolerance=0.05, strict=True, seed=r.seed, batches=r.batches))
        assert r.iterations == want.iterations and abs(r.modularity - want.modularity) < 1e-12
        assert r.edges_scanned == g.edge_count * r.iterations and r.gteps > 0
    crec = list(lp.run_sweep(lp.SweepSpec("copra", tolerances=(0.01,), max_labels=(2,)), [("planted", g)]))
    srec = list(lp.run_sweep(lp.SweepSpec("slpa", memory_sizes=(8,), modes=("strict",)), [("planted", g)]))
    assert len(crec) == 1 and len(srec) == 1 and crec[0].iterations >= 1 and srec[0].iterations >= 1


def test_cli_detect_and_sweep(gpu, tmp_path, capsys):
    """`python -m paper_2301_09125_b200 detect / sweep` (cli.py) on the CUDA detectors."""
    from paper_2301_09125_b200 import cli

    out = tmp_path / "labels.tsv"
    assert cli.main(["detect", "--graph", "planted:3000:30:4", "--algorithm", "rak", "--strict", "--seed", "3",
                     "--output", str(out)]) == 0
    got = np.loadtxt(out, dtype=np.int64)
    want = lp.rak_detect(lp.planted_partition(3000, 30, seed=4), lp.RakParams(strict=True, seed=3))
    assert np.array_equal(got[:, 0], np.arange(3000)) and np.array_equal(got[:, 1], want.assignment)
    assert "iterations=%d" % want.iterations in capsys.readouterr().err
    assert cli.main(["sweep", "--algorithm", "slpa", "--graph", "planted:3000:30:4", "--memory-sizes", "8",
                     "--modes", "strict", "--batches-grid", "0,1", "--extended"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].endswith(",batches,edges_scanned,gteps") and len(lines) == 3


def test_graph_stays_picklable_and_device_copy_releasable(gpu):
    """the device copy is cached outside the Graph (the reference's
    Graph pickles and deep-copies; so must ours after a detection)."""
    import copy
    import pickle

    g = lp.ring_of_cliques(6, 5)
    first = lp.rak_detect(g, lp.RakParams(strict=True, seed=2))
    g2 = pickle.loads(pickle.dumps(g))
    assert lp.graphs_equal(g, g2) and lp.graphs_equal(g, copy.deepcopy(g))
    assert np.array_equal(lp.rak_detect(g2, lp.RakParams(strict=True, seed=2)).assignment, first.assignment)
    assert lp.release_device_graph(g) is True
    assert lp.release_device_graph(g) is False
    again = lp.rak_detect(g, lp.RakParams(strict=True, seed=2))  # re-uploads
    assert np.array_equal(again.assignment, first.assignment)


def _float_weighted(g, seed=3):
    """Same graph with float64 weights in [1, 2) that are not float32-exact
    (both arc directions equal): the device's kFloat path."""
    from paper_2301_09125_b200 import synth

    gw = synth.with_edge_weights(g, seed=seed)
    rows = np.repeat(np.arange(g.vertex_count), np.diff(g.offsets))
    cols = np.asarray(g.neighbors)
    lo, hi = np.minimum(rows, cols), np.maximum(rows, cols)
    jitter = ((lo * 2654435761 + hi * 40503) % 1000003) / 1000003.0 * 2.0**-30
    w = np.where(rows == cols, 1.0, gw.weights + jitter)
    total = float(w.sum() + w[rows == cols].sum())
    return lp.Graph(g.vertex_count, g.edge_count, g.offsets, g.neighbors, w, total)


@pytest.mark.parametrize("batches", [0, 1])
def test_float_weights_deterministic_and_close_to_reference(gpu, oracle, batches):
    """Weights that are not float32-exact: tallied in float64 on the
    device, so strict runs are deterministic; the reference sums the exact
    float64 weights (rak.py:105) while the device rounds each weight to
    float32 first, so parity is statistical: |dQ| <= 1e-3, communities
    within 1% (the north star's bar for float weights)."""
    g = _float_weighted(lp.rmat(15, seed=4))
    assert lp._lib.device_graph(g).info()["weight_mode"] == "float"
    p = lp.RakParams(strict=True, seed=1, tolerance=0.05, max_iterations=20, batches=batches)
    a, b = lp.rak_detect(g, p), lp.rak_detect(g, p)
    assert np.array_equal(a.assignment, b.assignment) and a.iterations == b.iterations
    want, it, _ = oracle.rak(g, batches=batches, tie=0, seed=1, tolerance=0.05, max_iterations=20)
    q_ref = oracle.modularity(g, want)
    n_ref, n = len(np.unique(want)), len(np.unique(a.assignment))
    assert abs(a.modularity - q_ref) <= 1e-3, (a.modularity, q_ref)
    assert abs(n - n_ref) <= 0.01 * n_ref, (n, n_ref)
