"""Parity at the BASELINE.json configs at full size ("next" 1).

Each test runs the public API on the GPU and the CPU oracle
(oracle/lp_oracle.c, pinned to the reference's own outputs by
tests/test_oracle_golden.py) on the same seeded graph:

* deterministic modes (strict scan-first ties, unit or float32-exact weights,
  every schedule): labels, per-sweep changed counts and iteration count
  bit-exact -- R-MAT-22 unit and float32 U[1,2), planted n=100k, grid 4096^2,
  COPRA R-MAT-20 k = 1/4/8/16 (with the counter-hash fallback tie) and SLPA
  planted-1M T = 10/20/50 (counter-RNG speakers);
* stochastic modes against the reference's own xorshift draws (which no
  parallel schedule can replay; the oracle's TIE_XORSHIFT / speaker_rng=0
  paths): the north star's bar, |dQ| <= 1e-3 and community count within 1%
  (QTOL / NTOL below), with the reference's seed-to-seed spread printed
  beside every comparison.

The oracle runs on the host's cores in a thread pool (ctypes releases the
GIL) while the GPU works.
"""

import concurrent.futures as cf
import os

import numpy as np
import pytest

import paper_2301_09125_b200 as lp
from paper_2301_09125_b200 import synth
from paper_2301_09125_b200.copra import copra_run
from paper_2301_09125_b200.slpa import slpa_run

pytestmark = pytest.mark.gpu

QTOL = 1e-3  # north star: final modularity within 1e-3 of the reference's
NTOL = 0.01  # and the number of communities within 1%

SCAN_FIRST, RANDOM, XORSHIFT = 0, 1, 3


@pytest.fixture(scope="module")
def pool():
    with cf.ThreadPoolExecutor(max_workers=max(2, (os.cpu_count() or 2) - 1)) as ex:
        yield ex


@pytest.fixture(scope="module")
def rmat22():
    return synth.rmat(22, seed=1)


def ncom(labels):
    return int(np.unique(labels).size)


def _rak_exact(g, oracle, pool, strict=True, batches=0, seed=1, tol=0.05, max_it=20):
    job = pool.submit(oracle.rak, g, batches=batches, tie=SCAN_FIRST if strict else RANDOM, seed=seed,
                      tolerance=tol, max_iterations=max_it)
    res = lp.rak_detect(g, lp.RakParams(strict=strict, seed=seed, tolerance=tol, max_iterations=max_it,
                                        batches=batches), changed_history=True)
    want, it, changed = job.result()
    assert res.iterations == it
    assert np.array_equal(res.stats["changed"], changed)
    assert np.array_equal(res.assignment, want)
    return res


def _stochastic_close(name, g, ours_labels, ours_q, oracle_runs):
    """oracle_runs: {seed: labels} of the reference's draws; seed 1 is the
    comparison, the others give the reference's own spread (printed)."""
    from oracle import oracle as O

    qs = {s: O.modularity(g, lab) for s, lab in oracle_runs.items()}
    ns = {s: ncom(lab) for s, lab in oracle_runs.items()}
    q_ref, n_ref = qs[1], ns[1]
    n = ncom(ours_labels)
    print(f"\n[{name}] ours Q={ours_q:.6f} ncom={n}; reference seed 1 Q={q_ref:.6f} ncom={n_ref}; "
          f"reference seed spread Q {min(qs.values()):.6f}..{max(qs.values()):.6f} "
          f"ncom {min(ns.values())}..{max(ns.values())} (seeds {sorted(qs)})")
    assert abs(ours_q - q_ref) <= QTOL, (name, ours_q, q_ref)
    assert abs(n - n_ref) <= NTOL * n_ref, (name, n, n_ref)


# --------------------------------------------------------------------------
# RAK, deterministic: bit-exact at full size
# --------------------------------------------------------------------------

def test_rmat22_unit_strict_exact(gpu, oracle, pool, rmat22):
    """BASELINE configs[1], the bench graph: the reference's deterministic
    mode (strict, sequential sweep in the seeded visit order)."""
    _rak_exact(rmat22, oracle, pool)


def test_rmat22_unit_synchronous(gpu, oracle, pool, rmat22):
    _rak_exact(rmat22, oracle, pool, batches=1)


def test_rmat22_float32_weights_strict_exact(gpu, oracle, pool, rmat22):
    """configs[1] second run: float32 U[1,2) weights per undirected edge
    (float32-exact, so the device's fixed-point sums equal the reference's
    float64 sums and ties break identically)."""
    g = synth.with_edge_weights(rmat22, seed=1001)
    assert lp._lib.device_graph(g).info()["weight_mode"] == "fixed"
    _rak_exact(g, oracle, pool)


@pytest.mark.parametrize("batches", [0, 1])
def test_planted_100k_strict(gpu, oracle, pool, batches):
    g = synth.planted_partition(100_000, 1_000, seed=1)
    _rak_exact(g, oracle, pool, batches=batches)


def test_grid_4096_strict(gpu, oracle, pool):
    g = synth.road_grid(4096, seed=1)
    _rak_exact(g, oracle, pool, max_it=50)


# --------------------------------------------------------------------------
# RAK, non-strict: counter-hash ties bit-exact; vs the reference's draws by
# modularity and community count
# --------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["planted_100k", "rmat22"])
def test_nonstrict_vs_reference_draws(gpu, oracle, pool, rmat22, name):
    g = rmat22 if name == "rmat22" else synth.planted_partition(100_000, 1_000, seed=1)
    jobs = {s: pool.submit(oracle.rak, g, batches=0, tie=XORSHIFT, seed=s, tolerance=0.05, max_iterations=20)
            for s in (1, 2, 3)}
    res = _rak_exact(g, oracle, pool, strict=False)
    _stochastic_close(f"RAK non-strict {name}", g, res.assignment, res.modularity,
                      {s: j.result()[0] for s, j in jobs.items()})


# --------------------------------------------------------------------------
# COPRA R-MAT-20, k = 1/4/8/16 (BASELINE configs[3])
# --------------------------------------------------------------------------

@pytest.fixture(scope="module")
def rmat20():
    return synth.rmat(20, seed=1)


@pytest.mark.parametrize("k", [1, 4, 8, 16])
def test_copra_rmat20(gpu, oracle, pool, rmat20, k):
    g = rmat20
    same = pool.submit(oracle.copra, g, max_labels=k, batches=0, tie=RANDOM, seed=1, tolerance=0.01,
                       max_iterations=20)
    ref = {s: pool.submit(oracle.copra, g, max_labels=k, batches=0, tie=XORSHIFT, seed=s, tolerance=0.01,
                          max_iterations=20) for s in (1, 2, 3)}
    p = lp.CopraParams(max_labels=k, seed=1, max_iterations=20)
    gbest, git, labs, bels, sizes, _, _ = copra_run(g, p)
    best, it, olabs, obels, osizes = same.result()
    assert git == it
    assert np.array_equal(gbest, best)
    assert np.array_equal(sizes, osizes)
    for j in range(k):
        live = sizes > j
        assert np.array_equal(labs[live, j], olabs[live, j])
        assert np.array_equal(bels[live, j], obels[live, j])
    from oracle import oracle as O

    _stochastic_close(f"COPRA R-MAT-20 k={k}", g, gbest, O.modularity(g, gbest),
                      {s: j.result()[0] for s, j in ref.items()})


# --------------------------------------------------------------------------
# SLPA planted n=1M, T = 10/20/50 (BASELINE configs[4])
# --------------------------------------------------------------------------

@pytest.fixture(scope="module")
def planted1m():
    return synth.planted_partition(1_000_000, 10_000, seed=1)


@pytest.mark.parametrize("T", [10, 20, 50])
def test_slpa_planted_1m(gpu, oracle, pool, planted1m, T):
    g = planted1m
    same = pool.submit(oracle.slpa, g, memory_size=T, batches=0, tie=RANDOM, speaker_rng=1, seed=1,
                       tolerance=0.05)
    ref = {s: pool.submit(oracle.slpa, g, memory_size=T, batches=0, tie=XORSHIFT, speaker_rng=0, seed=s,
                          tolerance=0.05) for s in (1, 2, 3)}
    labels, git, gslots, gfilled, _, _ = slpa_run(g, lp.SlpaParams(memory_size=T, seed=1))
    want, it, slots, filled = same.result()
    assert git == it
    assert np.array_equal(gfilled, filled)
    assert np.array_equal(gslots[:, : it + 1], slots[:, : it + 1])
    assert np.array_equal(labels, want)
    from oracle import oracle as O

    _stochastic_close(f"SLPA planted-1M T={T}", g, labels, O.modularity(g, labels),
                      {s: j.result()[0] for s, j in ref.items()})
