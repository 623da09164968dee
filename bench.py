#!/usr/bin/env python3
"""Benchmark of the DF hot path (BASELINE.json metric) — one JSON line on rank 0.

Workload (configs[1], the config the metric is quoted on): 65,536 independent
coupled walls x 256 nodes, fp64, 1e5 steps per run (one implicit starting
step + 99,999 Dufort–Frankel steps, the run() convention building.cpp:311-323).
A bench "step" is one such full run from the initial state.  Weak scaling:
every rank marches its own 65,536 walls (seeded per rank), no data-path
collective; `value` = all ranks' node-updates / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--run-steps S] [--walls B]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the unmodified reference library compiled from its sources, or
the C restatement when that is absent) on the host cores with all threads.
"""
from __future__ import annotations

import argparse
import json
import math
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
FLOP_PER_UPDATE = 14      # SURVEY.md §8d convention for cfg1 (add/mul 1, FMA 2)
BYTES_PER_UPDATE_HBM = 0  # whole profile register-resident inside a launch


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--run-steps", type=int, default=100_000, help="time steps per run (incl. the start)")
    p.add_argument("--walls", type=int, default=65536)
    p.add_argument("--nodes", type=int, default=256)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.time(), parts))

    def mark(self, which: str):
        setattr(self, which, time.time())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_end", 1e30)
        rows = [r for (ts, r) in self.rows if t0 <= ts <= t1 and r[0].replace(".", "").isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


def make_workload(args, rank):
    from paper_1703_10119_b200 import workloads
    return workloads.batched_walls(n_walls=args.walls, n_nodes=args.nodes, nsteps=args.run_steps, seed=1 + rank)


def workload_config(args, world):
    return {"workload": f"cfg1_batched_fp64: {args.walls} walls x {args.nodes} nodes per GPU, "
                        f"{args.run_steps} steps per run (1 implicit start + {args.run_steps - 1} DF), dt*=1e-3",
            "walls_per_gpu": args.walls, "nodes": args.nodes, "steps_per_run": args.run_steps,
            "state_bytes_per_gpu": args.walls * args.nodes * 32,
            "l2": "inputs larger than L2 (state 537 MB per GPU at the default size)",
            "parallelism": f"walls sharded per rank (weak), {world} rank(s), no collective on the data path"}


# ---------------------------------------------------------------------------------
def cpu_reference_rate(w, nsteps, threads, implicit=False):
    """Time the reference CPU DF path (or its Euler-implicit path) on w for nsteps."""
    import oracle as O
    from paper_1703_10119_b200 import workloads
    impl = "ref" if O.ref_lib() is not None else "oracle"
    dt = w.model.dt
    times = workloads.accumulate_times(np.full(nsteps + 1, dt))
    tab = O.forcing_table(w.model, times, 0, w.tables)
    wb = O.WallBatch(w.model, w.init, tab)
    t0 = time.perf_counter()
    if implicit:
        O.march_implicit(impl, wb, nsteps, dt, nthreads=threads)
    else:
        O.march(impl, wb, nsteps, dt, threads)
    sec = time.perf_counter() - t0
    return w.cells * nsteps / sec, sec, ("reference" if impl == "ref" else "port")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    w = make_workload(args, 0)
    # bounded sample per step: all walls, a few steps (each step a few seconds of CPU work)
    sample_steps = max(1, int(4e8 // w.cells))
    for _ in range(args.warmup):
        cpu_reference_rate(w, max(1, sample_steps // 4), threads)
    rates, secs = [], []
    kind = "port"
    for _ in range(args.steps):
        r, s, kind = cpu_reference_rate(w, sample_steps, threads)
        rates.append(r)
        secs.append(s)
    value = statistics.median(rates)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": workload_config(args, 1), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"all {w.model.n_walls} walls x {sample_steps} DF steps per bench step "
                                       f"(df_step_coupled, wall.cpp:144-194, threads split walls)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_1703_10119_b200 import Context, api

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = make_workload(args, rank)
    w.model.device = local
    fp64_peak = api.probe_fp64_peak(local)
    ctx = Context(w.model)
    for ch, (first, tab) in w.tables.items():
        ctx.set_channel_table(ch, first, tab)
    ctx.set_state(**w.init)
    ctx.snapshot()                      # inputs resident in HBM; each run restores them
    nsteps = w.nsteps

    def one_run():
        ctx.restore()
        ctx.bootstrap(w.boot)
        ctx.advance(nsteps - 1)

    # the sampler starts before the warm-up: nvidia-smi start-up stalls the
    # device briefly and must not fall inside the timed region
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        one_run()
    ctx.synchronize()
    clocks.mark("t_start")
    launches0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    ctx.record(0)
    for _ in range(args.steps):
        one_run()
    ctx.record(1)
    ctx.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ctx.elapsed_ms(0, 1)
    clocks.mark("t_end")
    clk = clocks.stop()
    launches = ctx.launches - launches0
    ms_max = max_over_ranks(ms)
    updates = float(w.cells) * nsteps * args.steps * world
    value = updates / (ms_max * 1e-3)

    # dominant kernel: per-launch CUDA events on the launching stream (one extra run)
    ctx.reset_kernel_stats()
    ctx.profiling(True)
    one_run()
    ctx.synchronize()
    ctx.profiling(False)
    stats = ctx.kernel_stats()
    top = max(stats, key=lambda s: s["ms"])
    kernel_rate = top["node_updates"] / (top["ms"] * 1e-3)
    achieved_tf = kernel_rate * FLOP_PER_UPDATE / 1e12
    share = top["ms"] / sum(s["ms"] for s in stats)

    # e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        host = {k: np.ascontiguousarray(v) for k, v in w.init.items()}
        out = {k: np.empty_like(host[k]) for k in ("u_prev", "u_curr", "v_prev", "v_curr")}
        pinned = list(host.values()) + list(out.values())
        for a in pinned:
            api.load_library().hyg_host_register(a.ctypes.data, a.nbytes)
        e2e_steps = max(1, min(args.steps, 3))
        barrier()
        ctx.synchronize()
        ctx.record(2)
        for _ in range(e2e_steps):
            ctx.set_state(**host)
            ctx.bootstrap(w.boot)
            ctx.advance(nsteps - 1)
            ctx.get_state(out)
        ctx.record(3)
        ms_e2e = max_over_ranks(ctx.elapsed_ms(2, 3))
        for a in pinned:
            api.load_library().hyg_host_unregister(a.ctypes.data)
        b = 4 * w.cells * 8
        e2e = {"value": float(w.cells) * nsteps * e2e_steps * world / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": b, "d2h_bytes_per_step": b,
               "path": "Context.set_state -> bootstrap -> advance -> get_state (hyg_* C ABI), pinned host buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        sample = max(1, int(4e8 // w.cells))
        r, sec, kind = cpu_reference_rate(w, sample, threads)
        ri, seci, _ = cpu_reference_rate(w, max(1, sample // 4), threads, implicit=True)
        cpu = {"value": r, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"all {w.model.n_walls} walls x {sample} DF steps ({sec:.1f} s)",
               "implicit_value": ri,
               "implicit_sample": f"all walls x {max(1, sample // 4)} Euler-implicit steps ({seci:.1f} s)"}

    traffic = None
    tf = ROOT / "profiles" / "k1_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
                "config": workload_config(args, world),
                "roofline": {"bound": "fp64", "achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": achieved_tf / fp64_peak, "traffic": traffic,
                             "kernel": top["name"], "kernel_share_of_step": share,
                             "flop_per_update": FLOP_PER_UPDATE,
                             "peak_source": "DFMA probe measured in this run (MEASURED_PEAKS.json has no FP64 figure); "
                                            "nominal 148 SM x 64 x 2 x 1.965 GHz = 37.2",
                             "kernel_node_updates_per_s": kernel_rate},
                "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
