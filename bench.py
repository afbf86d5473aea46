#!/usr/bin/env python
"""bench.py -- RAK GTEPS on R-MAT scale 22 on B200 (BASELINE.json configs[1]).

One "step" = one full RAK detection (rak_detect semantics: labels = ids,
sweeps until changed <= tolerance * n or max_iterations) on the seeded
R-MAT-22 graph.  value = dense-equivalent GTEPS = edge_count x sweeps /
device time (edge_count includes the n self-loops),
aggregated over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config rmat22|rmat22w|planted|grid] [--non-strict]
                    [--batches B]

--impl reference times the reference's CPU path restated in C (the OpenMP
port of rak._rak_par in oracle/lp_oracle.c; the Python reference cannot
travel to the GPU box) on all host cores, same graph / metric / unit.

Multi-GPU (torchrun): replicas only -- each rank runs the full detection on
its own copy of the graph, no collective on the data path;
value = all ranks' edges / max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
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


def make_graph(name: str):
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
    for b, name in enumerate(_lib.BIN_NAMES):
        ms = sum(p["bin_ms"][b] for p in per)
        if ms <= 0:
            continue
        arcs = sum(p["bin_arcs"][b] for p in per)
        verts = sum(p["bin_vertices"][b] for p in per)
        out[f"tally_{name}"] = {"ms": ms, "launches": sum(p["bin_launches"][b] for p in per),
                                "bytes": (8 if weighted else 4) * arcs + 12 * verts,
                                "model": "(4 B label%s per arc) + 12 B per vertex" % (" + 4 B weight" if weighted else "")}
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


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

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


def run_reference(args, world, rank):
    """CPU arm: OpenMP port of the reference's _rak_par on all host cores."""
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = CONFIGS[args.config]
    g = make_graph(args.config)
    threads = os.cpu_count() or 1
    strict = not args.non_strict
    for _ in range(args.warmup):
        O.rak_par(g, strict=strict, seed=args.seed, tolerance=cfg["tolerance"], max_iterations=cfg["max_iterations"],
                  threads=threads)
    arcs = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        lab, it = O.rak_par(g, strict=strict, seed=args.seed, tolerance=cfg["tolerance"],
                            max_iterations=cfg["max_iterations"], threads=threads)
        arcs += g.edge_count * it
    dt = time.perf_counter() - t0
    gteps = arcs / dt / 1e9
    line = {
        "impl": "reference",
        "metric": "RAK GTEPS on R-MAT-22 (dense-equivalent: edge_count x sweeps / time)",
        "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 tally / int64 labels", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "mode": "strict" if strict else "non-strict",
                   "tolerance": cfg["tolerance"], "max_iterations": cfg["max_iterations"],
                   "vertices": g.vertex_count, "arcs": g.edge_count},
        "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full RAK detections (rak._rak_par restated in C, OpenMP, "
                                   f"{threads} threads, chunk 1024)"},
        "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations": int(it),
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import paper_2301_09125_b200 as lp
    from paper_2301_09125_b200 import _lib

    cfg = CONFIGS[args.config]
    weighted = args.config.endswith("w")
    t_gen = time.perf_counter()
    g = make_graph(args.config)
    t_gen = time.perf_counter() - t_gen
    params = lp.RakParams(strict=not args.non_strict, seed=args.seed, tolerance=cfg["tolerance"],
                          max_iterations=cfg["max_iterations"], batches=args.batches)
    dg = _lib.DeviceGraph(g, device=local)
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
    sweep_bytes = sum(algorithmic_bytes(g.vertex_count, g.edge_count, weighted) * p["iterations"] for p in per)
    total_kernel_ms = sum(k["ms"] for k in kernels.values())
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": top, "bytes_per_launch": bytes_per_launch, "ms_per_launch": ms_per_launch,
        "bytes_model": kt["model"], "peak_source": peak_src, "frac_of_8TBs": achieved / 8000.0,
        "step_achieved_gbs": sweep_bytes / (dt_ms / 1e3) / 1e9,
        "step_frac": sweep_bytes / (dt_ms / 1e3) / 1e9 / peak,
        "kernel_share": {k: v["ms"] / max(total_kernel_ms, 1e-9) for k, v in kernels.items()},
    }

    # modularity of the final labels (untimed, the reference's parity metric), on the device
    from paper_2301_09125_b200 import quality

    q_ours = quality.modularity_gpu(g, None, device_graph=dg)

    # the other schedules / tie rules on the same graph (device time, inputs resident)
    modes = {}
    if not args.no_modes:
        for name, kw in (("synchronous_strict", dict(batches=1, strict=True)),
                         ("exact_nonstrict", dict(batches=0, strict=False))):
            mp = lp.RakParams(seed=args.seed, tolerance=cfg["tolerance"], max_iterations=cfg["max_iterations"], **kw)
            mo = lp.rak._opts(mp)
            st = _lib.RunStats()
            _lib.check(L.lp_rak_run_resident(dg.handle, C.byref(mo), None, C.byref(st)))  # warm
            tms, arcs_m = 0.0, 0
            for _ in range(3):
                st = _lib.RunStats()
                _lib.check(L.lp_rak_run_resident(dg.handle, C.byref(mo), None, C.byref(st)))
                tms += st.kernel_ms
                arcs_m += g.edge_count * st.iterations
            modes[name] = {"gteps": arcs_m / (tms * 1e-3) / 1e9, "ms_per_run": tms / 3, "iterations": int(st.iterations),
                           "modularity": quality.modularity_gpu(g, None, device_graph=dg)}

    line = {
        "metric": "RAK GTEPS on R-MAT-22 (dense-equivalent: edge_count x sweeps / time)",
        "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32 labels / u32 counts" if not weighted else "int32 labels / u64 fixed-point sums",
        "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"],
                   "mode": "strict (scan-first ties)" if not args.non_strict else "non-strict (counter-RNG ties)",
                   "schedule": "reference visit order (exact async)" if args.batches == 0 else f"{args.batches} batches",
                   "tolerance": cfg["tolerance"], "max_iterations": cfg["max_iterations"],
                   "vertices": g.vertex_count, "arcs": g.edge_count,
                   "l2": "inputs larger than L2 (int32 CSR %.0f MB vs 126 MB L2)" % (4 * g.edge_count / 1e6),
                   "parallelism": f"replicas x{world}"},
        "iterations": per_t[-1]["iterations"], "rounds": per_t[-1]["rounds"],
        "arcs_scanned_per_step": per[-1]["arcs_scanned"], "arcs_dense_per_step": per_t[-1]["arcs_dense"],
        "gpu_launches": int(sum(p["launches"] for p in per_t)),
        "kernel_events": "kernel times (roofline) from K more steps run with per-launch CUDA events on the "
                          "library's streams right after the timed region (the events cost ~0.6 ms per step)",
        "roofline": roofline,
        "modularity": q_ours,
        "modes": modes,
        "graph_gen_s": t_gen,
    }

    if not args.no_e2e:
        line["e2e"] = e2e(args, g, params, world, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, g, cfg)
        line["cpu_baseline"]["modularity"] = line["cpu_baseline"].pop("_q")
    line["clocks"] = clk.summary()
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
    return {"value": whole_job_gteps(arcs, dt * 1e3, world), "unit": "GTEPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt / steps * 1e3, "steps": steps,
            "what": "rak_labels() on a freshly uploaded graph each step: CSR H2D from pinned host memory "
                    "(int64 offsets/neighbours as the reference's Graph holds them), plan build, sweeps, "
                    "int64 labels D2H"}


def cpu_baseline(args, g, cfg):
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    lab, it = O.rak_par(g, strict=not args.non_strict, seed=args.seed, tolerance=cfg["tolerance"],
                        max_iterations=cfg["max_iterations"], threads=threads)
    dt = time.perf_counter() - t0
    return {"value": g.edge_count * it / dt / 1e9, "unit": "GTEPS", "cores": threads, "kind": "port",
            "sample": f"1 full RAK detection ({it} sweeps) on the same graph, rak._rak_par restated in C "
                      f"(OpenMP, {threads} threads, 1024-vertex chunks), {dt:.2f} s",
            "_q": O.modularity(g, lab)}


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
