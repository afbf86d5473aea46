#!/usr/bin/env python
"""bench.py -- RAK GTEPS on R-MAT scale 22 on B200 (BASELINE.json configs[1]).

One "step" = one full RAK detection (rak_detect semantics: labels = ids,
sweeps until changed <= tolerance * n or max_iterations) on the seeded
R-MAT-22 graph.  value = dense-equivalent GTEPS = edge_count x sweeps /
device time (edge_count includes the n self-loops),
aggregated over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config rmat22|rmat22w|planted|grid] [--non-strict]
                    [--batches B] [--no-configs] [--no-parity]

The line also carries
  parity      -- the timed run's labels, per-sweep changed counts and
                 iteration count against the CPU oracle's restatement of the
                 same schedule (oracle/lp_oracle.c, pinned to the reference's
                 own outputs), and modularity / community count against it;
  modes       -- the synchronous schedule and non-strict ties on the same
                 graph, each with its parity;
  configs     -- the other BASELINE RAK configs (R-MAT-22 float32 weights,
                 planted n=100k strict and non-strict, 4096^2 grid): device
                 time, GTEPS, step roofline fraction and parity;
  cpu_baseline-- the reference's deterministic mode (rak_detect(strict,
                 workers=1) = the sequential sweep, restated in C) on one
                 host core, on the same graph.

--impl reference times the reference's CPU path on all host cores: the
OpenMP C port of rak._rak_par (oracle/lp_oracle.c; the Python reference
cannot travel to the GPU box), on a graph built by the oracle's own
generators (oracle/graphs.py -- the product library is never loaded), with
the CSR conversion and the visit order prepared outside the timed region as
the reference does (rak.py:171-172).

Multi-GPU (torchrun): replicas only -- each rank runs the full detection on
its own copy of the graph, no collective on the data path;
value = all ranks' edges / max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "rmat22": dict(desc="R-MAT scale 22, edge factor 16, (a,b,c,d)=(.57,.19,.19,.05), unit weights",
                   tolerance=0.05, max_iterations=20),
    "rmat22w": dict(desc="R-MAT scale 22, float32 weights U[1,2) per undirected edge",
                    tolerance=0.05, max_iterations=20),
    "planted": dict(desc="planted partition n=100000, 1000 communities x 100, 16 intra + 4 random",
                    tolerance=0.05, max_iterations=20),
    "grid": dict(desc="4096x4096 grid, 4-neighbour, 10% edges dropped, 2% diagonal shortcuts",
                 tolerance=0.05, max_iterations=50),
}

METRIC = "RAK GTEPS on R-MAT-22 (dense-equivalent: edge_count x sweeps / time)"

# oracle tie codes (oracle/oracle.py)
OR_SCAN_FIRST, OR_RANDOM, OR_XORSHIFT = 0, 1, 3


def make_graph(name: str, host_only: bool = False):
    """The config's graph: the product generators (GPU / native builders) for
    our arm, the oracle's independent generators for the reference arm (the
    same arrays; tests/test_oracle_graphs.py)."""
    if host_only:
        from oracle import graphs as OG

        if name not in OG.BENCH_GRAPHS:
            raise SystemExit(f"unknown config {name}")
        return OG.BENCH_GRAPHS[name]()
    from paper_2301_09125_b200 import synth

    if name == "rmat22":
        return synth.rmat(22, seed=1)
    if name == "rmat22w":
        return synth.rmat(22, seed=1, weighted=True)
    if name == "planted":
        return synth.planted_partition(100_000, 1_000, seed=1)
    if name == "grid":
        return synth.road_grid(4096, seed=1)
    raise SystemExit(f"unknown config {name}")


def bench_config(args, g, world: int) -> dict:
    """The `config` object: identical in both arms."""
    cfg = CONFIGS[args.config]
    return {"workload": args.config, "desc": cfg["desc"],
            "mode": "non-strict" if args.non_strict else "strict",
            "schedule": "reference visit order (sequential sweep)" if args.batches == 0 else f"{args.batches} batches",
            "tolerance": cfg["tolerance"], "max_iterations": cfg["max_iterations"], "seed": args.seed,
            "vertices": int(g.vertex_count), "arcs": int(g.edge_count),
            "l2": ("inputs larger than L2 (int32 CSR %.0f MB vs 126 MB L2)" if 4 * g.edge_count > 126e6 else
                   "inputs fit in L2 (int32 CSR %.0f MB vs 126 MB L2); no flush") % (4 * g.edge_count / 1e6),
            "parallelism": f"replicas x{world}"}


def algorithmic_bytes(vertices: int, arcs: int, weighted: bool) -> int:
    """per vertex 4 B row offset + 4 B own-label read + 4 B
    label write; per arc 4 B neighbour index + 4 B neighbour-label gather
    (+ 4 B weight)."""
    return 12 * vertices + (12 if weighted else 8) * arcs


def kernel_table(per, weighted):
    """Per-kernel totals over the timed steps, with each kernel's own
    algorithmic bytes: phase-1 gather = 4 B index + 4 B neighbour-label
    gather + 4 B label store per arc; tally kernels = 4 B label (+4 B weight)
    per arc + 12 B per vertex (row offset, own label read, label write)."""
    from paper_2301_09125_b200 import _lib

    out = {}
    fused = all(p.get("flags", 0) & _lib.STATS_FUSED for p in per)
    # fused rounds: the tally kernels read the neighbour index and gather its
    # label (SURVEY §8 d4's per-arc bytes); two-phase: they read lbuf
    per_arc = (8 if fused else 4) + (4 if weighted else 0)
    for b, name in enumerate(_lib.BIN_NAMES):
        ms = sum(p["bin_ms"][b] for p in per)
        if ms <= 0:
            continue
        arcs = sum(p["bin_arcs"][b] for p in per)
        verts = sum(p["bin_vertices"][b] for p in per)
        out[f"tally_{name}"] = {"ms": ms, "launches": sum(p["bin_launches"][b] for p in per),
                                "bytes": per_arc * arcs + 12 * verts,
                                "model": "(%s%s per arc) + 12 B per vertex" % (
                                    "4 B index + 4 B neighbour-label gather" if fused else "4 B label",
                                    " + 4 B weight" if weighted else "")}
    gms = sum(p["gather_ms"] for p in per)
    if gms > 0:
        out["k_gather"] = {"ms": gms, "launches": sum(p["gather_launches"] for p in per),
                           "bytes": 12 * sum(p["arcs_gathered"] for p in per),
                           "model": "12 B per gathered arc (index + neighbour label + label store)"}
    rms = sum(p["aux_ms"] for p in per)
    if rms > 0:
        out["k_route"] = {"ms": rms, "launches": 1, "bytes": 0, "model": "routing"}
    return out


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def reduce_max(x: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (device-timed values are
    combined this way: the job is as slow as its slowest rank)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gteps(arcs_per_rank: int, ms_max: float, world: int) -> float:
    """Replicas: every rank processes `arcs_per_rank` arcs; whole-job GTEPS
    is all ranks' arcs over the max-over-ranks time."""
    return world * arcs_per_rank / (ms_max / 1e3) / 1e9


def ncom(labels) -> int:
    return int(np.unique(labels).size)


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def product_library_loaded() -> bool:
    """Whether this process mapped liblabelprop_cuda.so (the reference arm
    must not)."""
    try:
        with open("/proc/self/maps") as f:
            return any("liblabelprop_cuda" in line for line in f)
    except OSError:
        return False


def run_reference(args, world, rank):
    """The reference's CPU path on all host cores: the OpenMP port of
    rak._rak_par (chunks of 1024 positions of the seeded order, per-thread
    tallies; rak.py:119-158), plus one run of its deterministic mode
    (workers=1, the sequential _rak_seq) on one core.  Rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = CONFIGS[args.config]
    g = make_graph(args.config, host_only=True)
    prep = O.prepare(g)  # CSR conversion outside the clock, as rak.py:171-172
    order = O.shuffled_indices(g.vertex_count, args.seed)
    threads = os.cpu_count() or 1
    strict = not args.non_strict
    kw = dict(strict=strict, seed=args.seed, tolerance=cfg["tolerance"], max_iterations=cfg["max_iterations"],
              threads=threads, order=order)
    for _ in range(args.warmup):
        O.rak_par(prep, **kw)
    arcs, it = 0, 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        lab, it = O.rak_par(prep, **kw)
        arcs += g.edge_count * it
    dt = time.perf_counter() - t0
    gteps = arcs / dt / 1e9
    q_par = O.modularity(prep, lab)
    # the deterministic mode (rak_detect(strict=True, workers=1)): one core
    t1 = time.perf_counter()
    slab, sit, _ = O.rak(prep, batches=0, tie=OR_SCAN_FIRST if strict else OR_XORSHIFT, seed=args.seed,
                         tolerance=cfg["tolerance"], max_iterations=cfg["max_iterations"], order=order)
    st = time.perf_counter() - t1
    model = cpu_model()
    line = {
        "impl": "reference",
        "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 tally / int64 labels", "data": "synthetic",
        "config": bench_config(args, g, world),
        "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": threads, "kind": "port", "cpu": model,
                         "sample": f"{args.steps} full RAK detections ({it} sweeps each) of rak._rak_par restated in C "
                                   f"(OpenMP, {threads} threads, 1024-position chunks); CSR and order prepared "
                                   f"outside the timed region"},
        "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations": int(it), "modularity": q_par, "communities": ncom(lab),
        "sequential": {"value": g.edge_count * sit / st / 1e9, "unit": "GTEPS", "cores": 1, "cpu": model,
                       "ms_per_run": st * 1e3, "iterations": int(sit),
                       "what": "the reference's deterministic mode (rak_detect strict, workers=1 = _rak_seq, "
                               "rak.py:87-116) restated in C, one core, one detection",
                       "modularity": O.modularity(prep, slab), "communities": ncom(slab)},
        "graph": "built by oracle/graphs.py",
        "product_library_loaded": product_library_loaded(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _oracle_tie(tie_rule: str) -> int:
    return {"scan-first": OR_SCAN_FIRST, "random": OR_RANDOM, "min-label": 2}[tie_rule]


class Detector:
    """One uploaded graph + a way to run and read back a detection."""

    def __init__(self, g, local):
        from paper_2301_09125_b200 import _lib

        self.g = g
        self.L = _lib.lib()
        self._lib = _lib
        self.dg = _lib.DeviceGraph(g, device=local)

    def run(self, opts, stats=None, changed=None):
        """One detection through the C-ABI (lp_rak_run: labels = ids, the
        seeded order; final labels downloaded after the timed sweeps)."""
        st = stats if stats is not None else self._lib.RunStats()
        self.out = np.empty(self.g.vertex_count, dtype=np.int64)
        self._lib.check(self.L.lp_rak_run(self.dg.handle, C.byref(opts), None, None, self._lib.ptr(self.out),
                                          self._lib.ptr(changed), C.byref(st)))
        return st

    def labels(self):
        return self.out

    def modularity(self):
        from paper_2301_09125_b200 import quality

        return quality.modularity_gpu(self.g, None, device_graph=self.dg)

    def close(self):
        self.dg.close()


def timed_runs(det, params, runs: int):
    """Warm once, then `runs` detections; device ms per run from the
    library's CUDA events (inputs resident).  Returns a result record with
    the last run's labels and changed counts."""
    import paper_2301_09125_b200 as lp

    o = lp.rak._opts(params)
    det.run(o)
    tms, it = 0.0, 0
    changed = np.zeros(params.max_iterations, dtype=np.int64)
    for _ in range(runs):
        st = det.run(o, changed=changed)
        tms += st.kernel_ms
        it = int(st.iterations)
    return {"ms": tms / runs, "iterations": it, "changed": changed[:it].copy(), "labels": det.labels(),
            "q": det.modularity(), "rounds": int(st.rounds)}


def parity_jobs(pool, prep, order, params, rec):
    """Oracle runs checking one of our results: the same schedule and tie
    rule (bit-exact), plus, for non-strict ties, the reference's own
    xorshift draws (modularity within 1e-3, communities within 1%)."""
    from oracle import oracle as O

    kw = dict(batches=params.batches, seed=params.seed, tolerance=params.tolerance,
              max_iterations=params.max_iterations, order=order)
    jobs = {"same": pool.submit(O.rak, prep, tie=_oracle_tie(params.tie_rule), **kw)}
    if params.tie_rule == "random":
        jobs["xorshift"] = pool.submit(O.rak, prep, tie=OR_XORSHIFT, **kw)
    return jobs


def parity_record(prep, rec, jobs):
    from oracle import oracle as O

    lab, it, ch = jobs["same"].result()
    q_ref = O.modularity(prep, lab)
    out = {"labels_equal_oracle": bool(np.array_equal(rec["labels"], lab)),
           "iterations_equal": int(it) == rec["iterations"],
           "changed_equal": bool(np.array_equal(np.asarray(ch), rec["changed"])),
           "q_ours": rec["q"], "q_ref": q_ref, "ncom_ours": ncom(rec["labels"]), "ncom_ref": ncom(lab),
           "oracle": "oracle/lp_oracle.c or_rak, same schedule and tie rule"}
    if "xorshift" in jobs:
        xl, xit, _ = jobs["xorshift"].result()
        qx, nx = O.modularity(prep, xl), ncom(xl)
        out["reference_rng"] = {"q_ref": qx, "ncom_ref": nx, "dq": abs(rec["q"] - qx),
                                "ncom_rel": abs(ncom(rec["labels"]) - nx) / max(nx, 1),
                                "within_1e-3_and_1pct": abs(rec["q"] - qx) <= 1e-3
                                and abs(ncom(rec["labels"]) - nx) <= 0.01 * nx,
                                "what": "the reference's own non-strict draws (xorshift stream in visit order, "
                                        "rak.py:71-83) restated in C: no parallel schedule can replay them, so "
                                        "modularity / community count are compared"}
    return out


def run_ours(args, world, rank, local):
    import paper_2301_09125_b200 as lp
    from oracle import oracle as O
    from paper_2301_09125_b200 import _lib

    cfg = CONFIGS[args.config]
    weighted = args.config.endswith("w")
    t_gen = time.perf_counter()
    g = make_graph(args.config)
    t_gen = time.perf_counter() - t_gen
    params = lp.RakParams(strict=not args.non_strict, seed=args.seed, tolerance=cfg["tolerance"],
                          max_iterations=cfg["max_iterations"], batches=args.batches)
    det = Detector(g, local)
    dg = det.dg
    opts = lp.rak._opts(params)
    # per-launch CUDA events (the roofline's kernel times) cost ~0.6 ms per
    # detection: the K timed steps run without them, K more steps with them
    opts_ev = lp.rak._opts(params)
    opts_ev.flags |= _lib.RAK_PROFILE
    L = _lib.lib()

    def one(stats, o=opts):
        _lib.check(L.lp_rak_run_resident(dg.handle, C.byref(o), None, C.byref(stats)))

    for _ in range(max(args.warmup, 1)):
        one(_lib.RunStats())

    import torch

    torch.cuda.set_device(local)
    stream = torch.cuda.ExternalStream(dg.stream, device=torch.device("cuda", local))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    per = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            st = _lib.RunStats()
            one(st)
            per.append(st.as_dict())
        ev1.record(stream)
        torch.cuda.synchronize()
    dt_ms = reduce_max(ev0.elapsed_time(ev1), world, device=f"cuda:{local}")
    arcs_dense = sum(p["arcs_dense"] for p in per)
    value = whole_job_gteps(arcs_dense, dt_ms, world)
    per_t = per
    if not args.no_kernel_events:
        # the same K steps again with per-launch events: kernel times for the roofline
        per = []
        for _ in range(args.steps):
            st = _lib.RunStats()
            one(st, opts_ev)
            per.append(st.as_dict())
        torch.cuda.synchronize()

    # roofline of the dominant kernel (per-launch averages over the timed region)
    kernels = kernel_table(per, weighted)
    if not kernels:  # --no-kernel-events
        kernels = {"none": {"ms": 1e-9, "launches": 1, "bytes": 0, "model": "no per-launch events"}}
    top = max(kernels, key=lambda k: kernels[k]["ms"])
    kt = kernels[top]
    bytes_per_launch = kt["bytes"] / max(kt["launches"], 1)
    ms_per_launch = kt["ms"] / max(kt["launches"], 1)
    achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(args.config, {}).get(top)
        except Exception:
            traffic = None
    # whole-step roofline: SURVEY §8 d4 bytes of the dense sweeps / device time
    sweep_bytes = sum(algorithmic_bytes(g.vertex_count, g.edge_count, weighted) * p["iterations"] for p in per_t)
    total_kernel_ms = sum(k["ms"] for k in kernels.values())
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": top, "bytes_per_launch": bytes_per_launch, "ms_per_launch": ms_per_launch,
        "bytes_model": kt["model"], "peak_source": peak_src, "frac_of_8TBs": achieved / 8000.0,
        "step_achieved_gbs": sweep_bytes / (dt_ms / 1e3) / 1e9,
        "step_frac": sweep_bytes / (dt_ms / 1e3) / 1e9 / peak,
        "step_bytes_model": "SURVEY §8 d4: (12 n + %d m) bytes per sweep x sweeps" % (12 if weighted else 8),
        "kernel_share": {k: v["ms"] / max(total_kernel_ms, 1e-9) for k, v in kernels.items()},
    }

    # the main run's result (untimed): labels + per-sweep changed counts
    main = timed_runs(det, params, 1)
    main["ms"] = dt_ms / args.steps

    # the other schedules / tie rules on the same graph (device time, inputs resident)
    mode_recs = {}
    if not args.no_modes:
        for name, kw in (("synchronous_strict", dict(batches=1, strict=True)),
                         ("exact_nonstrict", dict(batches=0, strict=False))):
            mp = lp.RakParams(seed=args.seed, tolerance=cfg["tolerance"], max_iterations=cfg["max_iterations"], **kw)
            mode_recs[name] = (mp, timed_runs(det, mp, 3))
    det.close()

    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32 labels / u32 counts" if not weighted else "int32 labels / u64 fixed-point sums",
        "data": "synthetic",
        "config": bench_config(args, g, world),
        "iterations": per_t[-1]["iterations"], "rounds": per_t[-1]["rounds"],
        "arcs_scanned_per_step": per[-1]["arcs_scanned"], "arcs_dense_per_step": per_t[-1]["arcs_dense"],
        "gpu_launches": int(sum(p["launches"] for p in per_t)),
        "kernel_events": "kernel times (roofline) from K more steps run with per-launch CUDA events on the "
                          "library's streams right after the timed region (the events cost ~0.6 ms per step)",
        "roofline": roofline,
        "modularity": main["q"],
        "graph_gen_s": t_gen,
        "clocks": clk.summary(),
    }

    # the other BASELINE configs: device time, roofline fraction, parity
    extra = []
    if world == 1 and args.config == "rmat22" and not args.no_configs:
        for name, strict in (("rmat22w", True), ("planted", True), ("planted", False), ("grid", True)):
            c = CONFIGS[name]
            eg = make_graph(name)
            ep = lp.RakParams(strict=strict, seed=args.seed, tolerance=c["tolerance"],
                              max_iterations=c["max_iterations"])
            edet = Detector(eg, local)
            rec = timed_runs(edet, ep, 3)
            edet.close()
            extra.append((name + ("" if strict else "_nonstrict"), eg, ep, rec))

    # CPU side: the reference's deterministic mode on one core (timed alone),
    # then every parity check in parallel (the oracle releases the GIL)
    parity_on = rank == 0 and not args.no_parity
    if parity_on or (rank == 0 and world == 1 and not args.no_cpu_baseline):
        prep = O.prepare(g)
        order = O.shuffled_indices(g.vertex_count, args.seed)
        threads = os.cpu_count() or 1
        with cf.ThreadPoolExecutor(max_workers=max(1, threads // 2)) as pool:
            if world == 1 and not args.no_cpu_baseline:
                t0 = time.perf_counter()
                slab, sit, sch = O.rak(prep, batches=0, tie=OR_SCAN_FIRST if params.strict else OR_XORSHIFT,
                                       seed=args.seed, tolerance=cfg["tolerance"],
                                       max_iterations=cfg["max_iterations"], order=order)
                sdt = time.perf_counter() - t0
                line["cpu_baseline"] = {
                    "value": g.edge_count * sit / sdt / 1e9, "unit": "GTEPS", "cores": 1, "kind": "port",
                    "cpu": cpu_model(),
                    "sample": f"1 full detection ({sit} sweeps, {sdt:.2f} s) in the reference's deterministic mode "
                              f"(rak_detect strict, workers=1 = _rak_seq, rak.py:87-116) restated in C, one core, "
                              f"same graph and visit order",
                    "modularity": O.modularity(prep, slab), "communities": ncom(slab)}
            if parity_on:
                jobs = parity_jobs(pool, prep, order, params, main)
                mjobs = {k: parity_jobs(pool, prep, order, mp, rec) for k, (mp, rec) in mode_recs.items()}
                eprep = {}
                ejobs = {}
                for name, eg, ep, rec in extra:
                    eprep[name] = O.prepare(eg)
                    eorder = O.shuffled_indices(eg.vertex_count, ep.seed)
                    ejobs[name] = parity_jobs(pool, eprep[name], eorder, ep, rec)
                line["parity"] = parity_record(prep, main, jobs)
                line["modes"] = {}
                for k, (mp, rec) in mode_recs.items():
                    line["modes"][k] = {"gteps": g.edge_count * rec["iterations"] / (rec["ms"] * 1e-3) / 1e9,
                                        "ms_per_run": rec["ms"], "iterations": rec["iterations"],
                                        "rounds": rec["rounds"], "modularity": rec["q"],
                                        "step_frac": algorithmic_bytes(g.vertex_count, g.edge_count, weighted)
                                        * rec["iterations"] / (rec["ms"] * 1e-3) / 1e9 / peak,
                                        "parity": parity_record(prep, rec, mjobs[k])}
                line["configs"] = {}
                for name, eg, ep, rec in extra:
                    w = name.startswith("rmat22w")
                    line["configs"][name] = {
                        "gteps": eg.edge_count * rec["iterations"] / (rec["ms"] * 1e-3) / 1e9,
                        "ms_per_run": rec["ms"], "iterations": rec["iterations"], "rounds": rec["rounds"],
                        "vertices": eg.vertex_count, "arcs": eg.edge_count,
                        "mode": "strict" if ep.strict else "non-strict",
                        "step_frac": algorithmic_bytes(eg.vertex_count, eg.edge_count, w) * rec["iterations"]
                        / (rec["ms"] * 1e-3) / 1e9 / peak,
                        "parity": parity_record(eprep[name], rec, ejobs[name])}
    extra = None

    if not args.no_e2e:
        line["e2e"] = e2e(args, g, params, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)


def e2e(args, g, params, world, local):
    """Same metric through the public API with host buffers: each step
    uploads the CSR from pinned host memory into a fresh device graph,
    detects, and downloads the labels."""
    import paper_2301_09125_b200 as lp
    from paper_2301_09125_b200 import _lib

    L = _lib.lib()
    arrays = [np.ascontiguousarray(g.offsets), np.ascontiguousarray(g.neighbors)]
    weighted = not np.all(g.weights == 1.0)
    if weighted:
        arrays.append(np.ascontiguousarray(g.weights))
    for a in arrays:
        _lib.check(L.lp_host_register(_lib.ptr(a), a.nbytes))
    h2d = sum(a.nbytes for a in arrays)
    d2h = 8 * g.vertex_count
    arcs = 0
    steps = max(1, min(args.steps, args.e2e_steps))
    try:
        # warm-up (first plan build, allocator)
        fresh = lp.Graph(g.vertex_count, g.edge_count, arrays[0], arrays[1], g.weights, g.total_weight)
        dg = _lib.DeviceGraph(fresh, device=local, unit=not weighted)
        lp.rak_labels(fresh, params, device_graph=dg)
        dg.close()
        import torch

        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            fresh = lp.Graph(g.vertex_count, g.edge_count, arrays[0], arrays[1], g.weights, g.total_weight)
            dg = _lib.DeviceGraph(fresh, device=local, unit=not weighted)
            labels, it, st, _ = lp.rak_labels(fresh, params, device_graph=dg)
            dg.close()
            arcs += g.edge_count * it
        dt = reduce_max(time.perf_counter() - t0, world, device=f"cuda:{local}")
    finally:
        for a in arrays:
            L.lp_host_unregister(_lib.ptr(a))
    return {"value": whole_job_gteps(arcs, dt * 1e3, world), "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt / steps * 1e3, "steps": steps,
            "what": "rak_labels() on a freshly uploaded graph each step: CSR H2D from pinned host memory "
                    "(int64 offsets/neighbours as the reference's Graph holds them), plan build, sweeps, "
                    "int64 labels D2H"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="rmat22")
    ap.add_argument("--non-strict", action="store_true")
    ap.add_argument("--batches", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity checks")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--no-modes", action="store_true", help="skip the secondary schedule / tie-rule timings")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="time the steps without per-launch events (no kernel roofline)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
