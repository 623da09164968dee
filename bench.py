#!/usr/bin/env python3
"""Benchmark of the DF hot path (BASELINE.json metric) — one JSON line on rank 0.

Default workload = configs[1], the config the metric is quoted on: 65,536
independent coupled walls x 256 nodes, fp64, 1e5 steps per run (one implicit
starting step + 99,999 Dufort-Frankel steps, the run() convention
building.cpp:311-323).  A bench "step" is one such full run from the
initial state (restored from a device snapshot: inputs resident in HBM).
Weak scaling: every rank marches its own 65,536 walls, no data-path
collective; `value` = all ranks' node-updates / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config cfg0|cfg1|cfg2|cfg3|cfg4|cfg5] [--run-steps S]

--config selects the other BASELINE configs (supplementary lines): cfg0 the
single nonlinear wall (replicas at N>1), cfg2 fp32 + variable dt (weak),
cfg3 the zone ring and cfg4 the long domain (strong scaling through
shard.py's deep-halo decomposition at N>1).
--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the unmodified reference library compiled from its sources, or
the C restatement where that is absent) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DF node-updates/sec (fp64) and % of min(HBM,FP64) roofline, 1/2/4/8 B200"
UNIT = "node-updates/s"

# per config: algorithmic flop and HBM bytes per node-update,
# the bound, the dominant kernel and how the work divides over ranks
CONFIGS = {
    "cfg0": dict(flop=21, bytes=0, bound="fp64 (one SM: latency-bound single wall)",
                 kernel="df_analytic_fused", scaling="replicas", dtype="f64", run_steps=100_000),
    "cfg1": dict(flop=14, bytes=0, bound="fp64", kernel="df_coupled_fused_f64", scaling="weak", dtype="f64",
                 run_steps=100_000),
    "cfg2": dict(flop=14, bytes=0, bound="fp32", kernel="df_coupled_fused_f32", scaling="weak", dtype="f32",
                 run_steps=100_000),
    # cfg3 runs K6 (k_ring_split.cuh: zone air + wall cones in launches of 8 steps, then
    # every wall in registers for 16 steps): per zone and walls launch 64 B x 768 nodes
    # (walls) + 2 x 4 layers x 80 B x 6 walls x 72/56 (cone tails, halo copies included)
    # + 4 x (144 + 80) B x 6 walls (stub: tails read, compact tails written) + 256 B (air
    # series), over 768 x 16 updates = 4.86 B/update — so its bound is SURVEY §8(d)'s:
    # FP64 (14.1 flop/update), with the HBM fraction of its own traffic beside (the walls
    # kernel alone: 64 B per node + 256 B per zone over 16 steps = 4.02 B/update);
    # --ring-depth 1 (8 steps per walls launch): 8.40 B/update; K4r (--ring-kernel 1,
    # k_ring_reg.cuh: B = 4 zones per block, S = 8 steps per launch):
    # (64 B x 3072 owned + 32 B x 756 halo nodes) / (3072 x 8) = 8.98 B/update; K5
    # (--ring-kernel 3, k_ring_pipe.cuh: B = 3, S = 12, halo trimmed to the cone):
    # (64 B x 2304 + 32 B x 864) / (2304 x 12) = 6.33 B/update
    "cfg3": dict(flop=14.1, bytes=4.86, bound="fp64", kernel="ring_walls", scaling="strong", dtype="f64",
                 run_steps=80_000, bytes_by_kernel={"ring_pipe": 6.33, "ring_reg": 8.98, "ring_walls": 4.02}),
    # cfg4 runs the temporally blocked K3w (k_dv_warp.cuh: 256-node windows, 8 steps
    # per launch, (32 x 256 + 32 x 240) / (240 x 8) = 8.27 B/update), so min(HBM,
    # FP64) is the FP64 side; sharded (N>1) every slab runs K3w too
    "cfg4": dict(flop=33, bytes=8.27, bound="fp64", kernel="df_analytic_tiled", scaling="strong", dtype="f64",
                 run_steps=10_000),
    # beyond BASELINE's five: load-bearing material walls,
    # k_material_step: 2 strict evaluations x 82 flop (exp/log/pow/div = 1, the
    # §8(d) convention) + ~41 flop of df_step_nonlinear rows per update, 48 B
    "cfg5": dict(flop=205, bytes=48, bound="fp64", kernel="material_step", scaling="weak", dtype="f64",
                 run_steps=1_000),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="cfg1", choices=sorted(CONFIGS))
    p.add_argument("--run-steps", type=int, default=0, help="time steps per run incl. the start (0: config default)")
    p.add_argument("--walls", type=int, default=65536)
    p.add_argument("--nodes", type=int, default=256)
    p.add_argument("--zones", type=int, default=8192)
    p.add_argument("--long-nodes", type=int, default=1 << 26)
    p.add_argument("--material-walls", type=int, default=16384)
    p.add_argument("--halo", type=int, default=0, help="shard halo depth (0: config default)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ring-kernel", type=int, default=0, help="cfg3: 0 auto (K6), 1 K4r, 2 K4, 3 K5, 4 K6 (A/B runs)")
    p.add_argument("--material-exact", action="store_true",
                   help="cfg5: the parity material evaluation (hyg_crmath.cuh) instead of the default fast one")
    p.add_argument("--ring-depth", type=int, default=0,
                   help="cfg3, K6: cone launches (8 steps each) per walls launch, 1..3 (0: library default) (A/B runs)")
    p.add_argument("--tiled-load", type=int, default=0,
                   help="cfg4: 0 TMA tiles (k_dv_tiled_tma), 1 per-lane cp.async (k_dv_tiled_stream) (A/B runs)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-sharded", action="store_true",
                   help="skip the strong-scaling block (cfg4 x-slabs, cfg3 zone blocks) of the default cfg1 line")
    a = p.parse_args()
    if not a.run_steps:
        a.run_steps = CONFIGS[a.config]["run_steps"]
    return a


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Clocks:
    """SM clock / throttle-reason sampling during the timed region (the
    B200_PROFILING.md clocks line).  In-process NVML queries every 200 ms
    (cheap ioctls; a polling nvidia-smi child takes driver locks that stall
    launch-heavy paths), nvidia-smi -lms as the fallback.  Started before the
    warm-up; samples are filtered to the region's wall-clock window."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop_flag = threading.Event()
        self.source = "none"

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksThrottleReasonHwSlowdown, N.nvmlClocksThrottleReasonHwThermalSlowdown,
                    N.nvmlClocksThrottleReasonSwThermalSlowdown, N.nvmlClocksThrottleReasonSwPowerCap]
            smax = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

            def once():
                try:
                    sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
                    r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.rows.append((time.time(), [sm, smax, pw] + [bool(r & b) for b in bits]))
                except Exception:
                    pass

            def poll():
                while not self.stop_flag.is_set():
                    once()
                    self.stop_flag.wait(0.2)

            self.once = once

            self.nvml = N
            self.source = "nvml"
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                try:
                    self.rows.append((time.time(), [float(parts[0]), float(parts[1]),
                                                    float(parts[2]) if parts[2].replace(".", "").isdigit() else 0.0]
                                      + [p.lower().startswith("active") for p in parts[3:]]))
                except ValueError:
                    pass

    def mark(self, which: str):
        # one sample right inside each end of the window, so a timed region shorter than
        # the polling period (configs[0]: tens of milliseconds) still carries its clocks
        once = getattr(self, "once", None)
        if which == "t_start":
            setattr(self, which, time.time())
            if once:
                once()
        else:
            if once:
                once()
            setattr(self, which, time.time())

    def stop(self) -> dict:
        self.stop_flag.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.source == "none":
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"]}
        self.t.join(timeout=2)
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_end", 1e30)
        rows = [r for (ts, r) in self.rows if t0 <= ts <= t1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": self.source}
        sm = [r[0] for r in rows]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[3 + i]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": rows[0][1], "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[2] for r in rows), "source": self.source}


def make_workload(args, rank, world):
    from paper_1703_10119_b200 import workloads
    c = args.config
    if c == "cfg1":
        return workloads.batched_walls(n_walls=args.walls, n_nodes=args.nodes, nsteps=args.run_steps, seed=1 + rank)
    if c == "cfg2":
        return workloads.batched_walls(n_walls=args.walls, n_nodes=args.nodes, nsteps=args.run_steps, seed=1 + rank,
                                       precision="f32", variable_dt=True)
    if c == "cfg0":
        return workloads.single_wall_d(nsteps=args.run_steps)
    if c == "cfg3":
        return workloads.zone_ring(n_zones=args.zones, nsteps=args.run_steps)
    if c == "cfg5":
        return workloads.material_walls(n_walls=args.material_walls, n_nodes=101, nsteps=args.run_steps,
                                        seed=5 + rank)
    return workloads.long_domain(n_nodes=args.long_nodes, nsteps=args.run_steps)


def workload_config(args, world):
    """The `config` block of both arms, from the arguments alone (the reference
    arm never builds the GPU arm's Workload)."""
    c = CONFIGS[args.config]
    cfg = args.config
    boot = {"cfg0": "explicit", "cfg4": "none"}.get(cfg, "implicit")
    name, notes, nodes, walls, zones = {
        "cfg0": ("cfg0_single_wall_d", "N=101, tau=24.0", 101, 1, 0),
        "cfg1": ("cfg1_batched_fp64", f"{args.walls} walls x {args.nodes} nodes, seed 1", args.nodes, args.walls, 0),
        "cfg2": ("cfg2_batched_fp32_vardt", f"{args.walls} walls x {args.nodes} nodes, seed 1", args.nodes,
                 args.walls, 0),
        "cfg3": ("cfg3_zone_ring", f"{args.zones} zones x 6 walls x 128", 128, 6 * args.zones, args.zones),
        "cfg4": ("cfg4_long_domain", f"N={args.long_nodes}, seed 4", args.long_nodes, 1, 0),
        "cfg5": ("material_walls", f"{args.material_walls} material walls x 101", 101, args.material_walls, 0),
    }[cfg]
    cells = nodes * walls
    d = {"workload": f"{name}: {notes}, {args.run_steps} steps per run "
                     f"(start: {boot}{'' if boot == 'none' else ', counted as step 1'})",
         "config_index": int(cfg[-1]), "nodes": nodes, "walls": walls, "zones": zones,
         "steps_per_run": args.run_steps, "dt": 1e-3, "state_bytes": cells * 32,
         "l2": ("inputs larger than L2" if cells * 32 > 126e6 else
                "working set L2/on-chip resident (single wall); no L2 flush between runs"),
         "parallelism": {"weak": f"walls sharded per rank (weak), {world} rank(s), no collective on the data path",
                         "replicas": f"{world} independent replica(s)",
                         "strong": f"{'deep-halo shards (shard.py)' if world > 1 else 'one GPU'}, {world} rank(s)"}
         [c["scaling"]]}
    if cfg == "cfg2":
        n, dt = args.run_steps, 1e-3
        sched = [(10_000, dt), (10_000, 2 * dt), (10_000, 4 * dt), (10_000, 8 * dt), (n - 40_000, 16 * dt)]
        d["dt_schedule"] = [(k, x) for k, x in sched if k > 0]
    return d


def run_steps_of(w):
    """[(nsteps, dt)] for advance() after the start step."""
    if w.dt_schedule:
        out, first = [], True
        for n, d in w.dt_schedule:
            out.append((n - 1 if first and w.boot != "none" else n, d))
            first = False
        return out
    return [(w.nsteps - (0 if w.boot == "none" else 1), w.model.dt)]


# ---------------------------------------------------------------------------------
REF_BENCH = ROOT / "oracle" / "_ref" / "ref_bench"


def ref_bench(args, steps: int, warmup: int, threads: int) -> dict:
    """The reference's own CPU path on the host cores: oracle/_ref/ref_bench,
    a program linked from the unmodified reference sources that builds the
    config's workload through the reference's API and times its stepping
    functions (DF, and the Euler-implicit path beside it).  Runs as a child
    process: nothing of this package is imported, linked or loaded there."""
    if not REF_BENCH.exists():
        raise FileNotFoundError(f"{REF_BENCH} is missing (built from /root/reference by `make -C oracle refbench`)")
    cmd = [str(REF_BENCH), "--config", args.config, "--steps", str(steps), "--warmup", str(warmup),
           "--threads", str(threads), "--walls", str(args.walls),
           "--nodes", str(128 if args.config == "cfg3" else args.nodes),
           "--zones", str(args.zones), "--long-nodes", str(args.long_nodes),
           "--material-walls", str(args.material_walls)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3600)
    if r.returncode != 0:
        raise RuntimeError(f"ref_bench rc={r.returncode}: {r.stderr[-400:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_baseline_of(rb: dict, warmup: int) -> dict:
    df = rb["df"]
    out = {"value": statistics.median(df["rates"][warmup:]), "unit": UNIT, "cores": df["cores"],
           "kind": df["kind"], "sample": f"{df['sample']}; {df['path']}",
           "host_threads": rb["threads"], "effective_cores": rb["effective_cores"]}
    imp = rb.get("implicit")
    if imp:
        out.update(implicit_value=statistics.median(imp["rates"][warmup:]), implicit_kind=imp["kind"],
                   implicit_cores=imp["cores"], implicit_sample=f"{imp['sample']}; {imp['path']}")
    if "serial_step_explicit" in rb:
        out["serial_step_explicit_value"] = rb["serial_step_explicit"]
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    try:
        rb = ref_bench(args, args.steps, args.warmup, threads)
    except Exception as e:     # the compiled reference did not travel with the snapshot
        print(json.dumps({"impl": "reference", "unavailable": str(e).splitlines()[0]}), flush=True)
        return 0
    cpu = cpu_baseline_of(rb, args.warmup)
    value = cpu["value"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(rb["df"]["secs"][args.warmup:]),
            "higher_is_better": True, "scaling": "strong" if CONFIGS[args.config]["scaling"] == "strong" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": workload_config(args, 1), "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "each step = one bounded sample of the workload through the reference's own stepping "
                    "functions (oracle/_ref/ref_bench, linked from the unmodified reference sources)"}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------
class Runner:
    """One rank's engine for the selected config: a Context, or a shard of one."""

    def __init__(self, args, w, rank, world, local):
        from paper_1703_10119_b200 import Context, shard
        self.w, self.args = w, args
        cfg = CONFIGS[args.config]
        w.model.device = local
        self.shard = None
        if cfg["scaling"] == "strong" and world > 1:
            comm = shard.Comm()          # the NCCL group: halos device to device over NVLink
            if args.config == "cfg4":
                self.shard = shard.LongDomainShard(w.model, w.init, comm, Context, halo=args.halo or 64)
            else:
                self.shard = shard.ZoneRingShard(w.model, w.init, comm, Context, walls_per_zone=6,
                                                 halo=args.halo or 8)
            self.ctx = self.shard.engine
            self.updates = w.cells / world
        else:
            self.ctx = Context(w.model)
            if args.ring_kernel:
                self.ctx.set_tuning("ring_kernel", args.ring_kernel)
            if args.material_exact:
                self.ctx.set_tuning("material_exact", 1)
            if args.tiled_load:
                self.ctx.set_tuning("tiled_load", args.tiled_load)
            if args.ring_depth:
                self.ctx.set_tuning("ring_depth", args.ring_depth)
            for ch, (first, tab) in w.tables.items():
                self.ctx.set_channel_table(ch, first, tab)
            self.ctx.set_state(**w.init)
            self.updates = w.cells
        self.ctx.snapshot()

    def run(self):
        self.ctx.restore()
        w = self.w
        if self.shard is not None:
            if w.boot != "none":
                self.shard.bootstrap(w.boot)
            for n, d in run_steps_of(w):
                self.shard.advance(n)
            return
        if w.boot != "none":
            self.ctx.bootstrap(w.boot)
        for n, d in run_steps_of(w):
            self.ctx.advance(n, d)


def measure_sharded(args, name, rank, world, local, barrier, max_over_ranks):
    """`name` (cfg4: x-slabs with 64-node halos; cfg3: zone blocks with 24-zone halos)
    divided over the job's GPUs — the configs that communicate — as full-length runs:
    device time (CUDA events on the engine's stream, max over ranks) and, per halo
    interval, the exchange and compute time of the shards.  At N = 1 the undivided
    run, so the lines of a 1/2/4/8 SCALE run give the strong-scaling efficiency."""
    import copy
    import torch
    a = copy.copy(args)
    a.config, a.run_steps = name, CONFIGS[name]["run_steps"]
    a.halo = args.halo or {"cfg4": 64, "cfg3": 24}[name]
    a.ring_kernel = a.ring_depth = a.tiled_load = 0
    a.material_exact = False
    w = make_workload(a, 0, world)
    R = Runner(a, w, rank, world, local)
    ctx = R.ctx
    try:
        R.run()                                   # warm-up
        ctx.synchronize()
        if R.shard is not None:
            R.shard.timer.reset()
        runs = 2
        barrier()
        torch.cuda.synchronize()
        ctx.record(0)
        for _ in range(runs):
            R.run()
        ctx.record(1)
        ctx.synchronize()
        barrier()
        ms = max_over_ranks(ctx.elapsed_ms(0, 1))
        out = {"value": float(w.cells) * w.nsteps * runs / (ms * 1e-3), "unit": UNIT, "ms_per_run": ms / runs,
               "n_gpus": world, "scaling": "strong", "steps_per_run": w.nsteps,
               "workload": workload_config(a, world)["workload"]}
        if R.shard is not None:
            t = R.shard.timer.totals()
            n = max(1, t["intervals"])
            out["halo"] = a.halo
            out["per_interval_us"] = {"exchange": 1e3 * max_over_ranks(t["exchange"]) / n,
                                      "compute": 1e3 * max_over_ranks(t["compute"]) / n,
                                      "intervals": t["intervals"],
                                      "overlapped": bool(getattr(R.shard, "overlap", False))}
        return out
    finally:
        ctx.close()


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    cfg = CONFIGS[args.config]
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        import datetime
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=600))
    from paper_1703_10119_b200 import api

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = make_workload(args, rank if cfg["scaling"] != "strong" else 0, world)
    peak64 = api.probe_fp64_peak(local)
    peak32 = api.probe_fp32_peak(local) if cfg["bound"] == "fp32" else None
    R = Runner(args, w, rank, world, local)
    ctx = R.ctx

    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        R.run()
    ctx.synchronize()
    clocks.mark("t_start")
    launches0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    ctx.record(0)
    for _ in range(args.steps):
        R.run()
    ctx.record(1)
    ctx.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ctx.elapsed_ms(0, 1)
    clocks.mark("t_end")
    clk = clocks.stop()
    launches = ctx.launches - launches0
    ms_max = max_over_ranks(ms)
    total_updates = float(w.cells if cfg["scaling"] == "strong" else w.cells * world) * w.nsteps * args.steps
    value = total_updates / (ms_max * 1e-3)

    # dominant kernel: CUDA events around every launch on the launching stream (one extra run)
    ctx.reset_kernel_stats()
    ctx.profiling(True)
    R.run()
    ctx.synchronize()
    ctx.profiling(False)
    stats = ctx.kernel_stats()
    top = max(stats, key=lambda s: s["ms"])
    kernel_rate = top["node_updates"] / (top["ms"] * 1e-3) if top["node_updates"] else 0.0
    share = top["ms"] / sum(s["ms"] for s in stats)
    bytes_per_update = cfg.get("bytes_by_kernel", {}).get(top["name"], cfg["bytes"])
    extra = {}
    if cfg["bound"] == "hbm":
        achieved = kernel_rate * bytes_per_update / 1e9
        # the same kernel against SURVEY §8(d)'s FP64 roofline (its own convention)
        extra = {"fp64_achieved_tflops": kernel_rate * cfg["flop"] / 1e12, "fp64_peak_tflops": peak64,
                 "fp64_frac": kernel_rate * cfg["flop"] / 1e12 / peak64}
        peak, unit, peak_src = 6458.4, "GB/s", "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
        try:
            peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        except Exception:
            peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    elif cfg["bound"] == "fp32":
        achieved, peak, unit = kernel_rate * cfg["flop"] / 1e12, peak32, "TFLOP/s"
        peak_src = "FFMA probe measured in this run"
    else:
        achieved, peak, unit = kernel_rate * cfg["flop"] / 1e12, peak64, "TFLOP/s"
        peak_src = ("DFMA probe measured in this run (MEASURED_PEAKS.json has no FP64 figure); "
                    "nominal 148 SM x 64 x 2 x 1.965 GHz = 37.2")
        if bytes_per_update:
            # the same kernel against the HBM roofline of its own algorithmic traffic
            try:
                hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
            except Exception:
                hbm = 6650.0
            extra = {"hbm_achieved_gbs": kernel_rate * bytes_per_update / 1e9, "hbm_peak_gbs": hbm,
                     "hbm_frac": kernel_rate * bytes_per_update / 1e9 / hbm}
        if args.config == "cfg0":
            peak = peak64 / 148.0
            peak_src = "one SM's share of the DFMA probe (a single wall is one dependency chain per step)"

    e2e = None
    if not args.no_e2e and R.shard is None:
        host = {k: np.ascontiguousarray(v) for k, v in w.init.items()}
        out = {k: np.empty_like(host[k]) for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        pinned = list(host.values()) + list(out.values())
        lib = api.load_library()
        for a in pinned:
            lib.hyg_host_register(a.ctypes.data, a.nbytes)
        e2e_steps = max(1, min(args.steps, 3))
        barrier()
        ctx.synchronize()
        ctx.record(2)
        for _ in range(e2e_steps):
            ctx.set_state(**host)
            if w.boot != "none":
                ctx.bootstrap(w.boot)
            for n, d in run_steps_of(w):
                ctx.advance(n, d)
            ctx.get_state(out)
        ctx.record(3)
        ms_e2e = max_over_ranks(ctx.elapsed_ms(2, 3))
        for a in pinned:
            lib.hyg_host_unregister(a.ctypes.data)
        b = 4 * w.cells * 8 + 2 * len(w.model.zones) * 8 * ("zone_u" in host)
        e2e = {"value": float(w.cells) * w.nsteps * e2e_steps * world / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": b, "d2h_bytes_per_step": b,
               "path": "Context.set_state -> bootstrap -> advance -> get_state (hyg_* C ABI), pinned host buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_of(ref_bench(args, 2, 1, len(os.sched_getaffinity(0))), 1)
        except Exception as e:
            cpu = {"unavailable": str(e).splitlines()[0]}

    traffic = None
    tf = ROOT / "profiles" / f"{top['name']}_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if R.shard is None:
        ctx.close()
    sharded = None
    if args.config == "cfg1" and not args.no_sharded:
        # the configs that communicate, measured on the same N GPUs (the driver's
        # SCALE run then sees their strong scaling); failures are reported, not fatal
        sharded = {}
        for name in ("cfg4", "cfg3"):
            try:
                sharded[name] = measure_sharded(args, name, rank, world, local, barrier, max_over_ranks)
            except Exception as e:          # noqa: BLE001 — reported in the line
                sharded[name] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong" if cfg["scaling"] == "strong" else "weak", "vs_baseline": None,
                "dtype": cfg["dtype"], "data": "synthetic (seeded)", "config": workload_config(args, world),
                "roofline": {"bound": cfg["bound"], "achieved": achieved, "peak": peak, "unit": unit,
                             "frac": achieved / peak if peak else None, "traffic": traffic,
                             "kernel": top["name"], "kernel_share_of_step": share,
                             "flop_per_update": cfg["flop"], "bytes_per_update": bytes_per_update,
                             "peak_source": peak_src, "kernel_node_updates_per_s": kernel_rate, **extra},
                "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu}
        if sharded is not None:
            line["sharded"] = sharded
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
