#!/usr/bin/env python
"""bench.py -- cpRRTC planning on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], the metric's own config): the
7-DoF Panda-like arm (arm7) in the table scene, end effector kept upright on
the plane z = 0.60 with a locked orientation (0,1,0,0), tau_task 0.01, W = 16
waypoints per motion; start/goal pairs from the reference's own generate_pair
(tests/golden/pairs.npz, pair_seed 300+k).

A step = plan Q queries one after another, each with the whole GPU (one
persistent-kernel launch per query).  value = median planning time of the
solved queries on the device (inputs resident): the planner's own clock
(globaltimer) from the init kernel's start to the last team leaving the
query, when the results are complete -- the single-query graph records no
CUDA events ("Teardown after the solve"; r2s and earlier: events
from the H2D copy to the results); e2e = the same median through the public
plan() call (host buffers in, H2D + D2H inside the timed region); success
rate beside it.  The L2 is flushed (256 MiB write) before every query.

Every N also reports ``throughput``: BASELINE configs[4], 1024 independent
constrained queries per GPU per step in one persistent launch (weak scaling:
N x 1024 queries per step over N GPUs, no collective -- queries shard), as
whole-job queries/s from the max-over-ranks device time, and end to end.

N = 1 adds (rank 0): CC checks/s of the collision kernel on a 999-box shelf
(the BASELINE's "CC checks/s"), the NN scan's streaming bandwidth, configs[0],
[2] and [3], the projection ablation, the reference's FP64 revalidate_path pass
rate over the GPU's paths, and the reference planner itself (oracle/_ref, the
stock maniplan install, compiled backend) timed on the host cores on every
config: ``cpu_baseline`` (configs[1]), ``other_configs.*.cpu_reference``,
``throughput.cpu_reference`` (configs[4] on all cores) and
``cpu_cc_checks_per_s``.  The configs[1] GPU and CPU trial records are written
in the reference's records.csv / cdf_*.csv formats (``--records-dir``).

--impl reference runs the reference planner on the host cores over the same
queries, one process per core.  --gpus N > 1 without torchrun relaunches itself
under torch.distributed.run, one rank per GPU.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

METRIC = "median planning time (ms) + success rate, constrained Panda; CC checks/s"
WORKLOAD = ("configs[1] constrained Panda: arm7 + table, plane z=0.60 + fixed orientation (0,1,0,0), "
            "tau 0.01, W=16")
N_PAIRS = 100
BATCH = 1024
# algorithmic FP32 flop per work unit (counted from the
# reference formulas): projection stage 1 with plane+orientation (m=4) / plane
# (m=1), FK + world spheres of arm7, one sphere-primitive check, one NN node.
FLOP_STAGE1_M4 = 1750.0
FLOP_STAGE1_M1 = 1240.0
FLOP_FK_ARM7 = 1195.0
FLOP_CHECK = 11.0
FLOP_NN7 = 20.0
BYTES_NN7 = 28.0


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clocks_setting"}

    def __init__(self, device):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        rs = [n for b, n in self.NAMES.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": rs, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workloads (shared by both arms)
# ---------------------------------------------------------------------------

def query_index(step, j, Q, world, rank):
    """Weak scaling: rank r plans queries [r*Q, (r+1)*Q) of step's global
    block of world*Q queries (pair index modulo the 100 pairs)."""
    return (step * Q * world + rank * Q + j) % N_PAIRS


def query_seed(step, k):
    return (step * 7919 + k) * 10_000


def headline_config(args, world):
    """The config dict both arms print (same queries, seeds and budgets)."""
    return {"workload": WORKLOAD, "pairs": "reference generate_pair, pair_seed 300..399 (tests/golden/pairs.npz)",
            "seed_offset": "(step*7919 + pair)*10000", "queries_per_step_per_gpu": args.queries,
            "max_iterations": args.max_iterations, "time_budget_ms": args.budget_ms,
            "parallelism": f"replicas x{world} (independent queries per GPU)"}


def workload():
    import fixtures as fx
    return (fx.robot("arm7"), fx.scene("table"), fx.spec("upright"),
            fx.pairs()["upright_start"], fx.pairs()["upright_goal"])


def batch_arrays(step):
    """configs[4]: 1024 table-plane queries (constrained100's table_plane,
    pair_seed 0..1023), seed_offset (step*1024 + i)*10000."""
    import fixtures as fx
    prs = fx.pairs()
    seeds = (np.arange(BATCH, dtype=np.int64) + step * BATCH) * 10_000
    return prs["table_plane_start"][:BATCH], prs["table_plane_goal"][:BATCH], seeds


def _cfg_problems(name):
    """(label, [(model, scene, spec, start, goal, params_kw)]) for the other
    BASELINE configs; pairs come from the reference's generate_pair."""
    import fixtures as fx
    prs = fx.pairs()
    arm7, arm8d = fx.robot("arm7"), fx.robot("arm8_dense")
    out = []
    if name == "configs[0]":
        for sd in range(10):
            sc = fx.scene(f"rand10_s{sd}")
            for i in range(len(prs[f"rand10_s{sd}_seed"]))[:2]:
                out.append((arm7, sc, None, prs[f"rand10_s{sd}_start"][i], prs[f"rand10_s{sd}_goal"][i],
                            dict(width=32)))
        return "unconstrained arm7, 10-primitive random scenes (5 boxes + 5 spheres), W=32", out
    if name.startswith("configs[2]"):
        sc = fx.scene(name.split(":")[1])
        for key, m, spn in (("shelf_arm7", arm7, None), ("shelf_arm8", fx.robot("arm8"), None),
                            ("shelf_sweep", arm7, "plane55")):
            for i in range(len(prs[f"{key}_seed"])):
                sp = None if spn is None else fx.spec(spn)
                out.append((m, sc, sp, prs[f"{key}_start"][i], prs[f"{key}_goal"][i], dict(width=16)))
        return (f"shelf suite problems (reference data/suites/shelf.yaml) in the shelf densified to "
                f"{sc.primitive_count} boxes: arm7 / arm8 reaches + arm7 plane sweep, W=16"), out
    if name == "configs[3]":
        sp = fx.spec("table_line_8")
        for i in range(min(20, len(prs["dense8_line_seed"]))):
            out.append((arm8d, fx.scene("table"), sp, prs["dense8_line_start"][i],
                        prs["dense8_line_goal"][i], dict(width=16)))
        return "8-DoF arm8 with 36 collision spheres / 96 self pairs, table, line constraint, W=16", out
    raise KeyError(name)


# ---------------------------------------------------------------------------
# distributed plumbing (control plane only: the queries shard, no collective)
# ---------------------------------------------------------------------------

def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("CPRRTC_BENCH_ONE_GPU") == "1":
        # test mode only (exercises the N > 1 code path on a one-GPU box):
        # every rank plans on cuda:0; such a run is not a scaling measurement
        local = 0
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def gather(world, obj):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def _visible_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _relaunch(args):
    """--gpus N > 1 outside torchrun: one rank per GPU under
    torch.distributed.run (the driver's own launch form)."""
    have = _visible_gpus()
    if have < args.gpus and os.environ.get("CPRRTC_BENCH_ONE_GPU") != "1":
        sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible")
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args, world, rank, local):
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
    model, scene, spec, starts, goals = workload()
    opt = DeviceOptions(device=local, teams=args.teams, cc_broadphase=args.cc_broadphase)
    Q = args.queries

    def problem(step, j):
        k = query_index(step, j, Q, world, rank)
        return k, PlanProblem(model, scene, spec, starts[k], goals[k],
                              PlanParams(width=16, max_iterations=args.max_iterations,
                                         time_budget_ms=args.budget_ms, seed_offset=query_seed(step, k)),
                              name=f"upright#{k}")

    ctx = prepare(problem(0, 0)[1], opt)
    recs = []

    def one_step(step, timed):
        for j in range(Q):
            k, p = problem(step, j)
            ctx.flush_l2()
            t0 = time.perf_counter()
            r = plan(p, opt)
            wall = (time.perf_counter() - t0) * 1e3
            tot, kern = ctx.last_timing()
            if timed:
                st = r.stats
                recs.append(dict(k=k, step=step, seed=p.params.seed_offset, solved=r.solved, status=r.status,
                                 device_ms=tot, kernel_ms=kern, wall_ms=wall, stage1=st.stage1_evals,
                                 fk=st.cc_fk_evals, checks=st.cc_performed, possible=st.cc_possible,
                                 nn=st.nn_nodes, iterations=st.iterations, pfail=st.projection_failures,
                                 path=len(r.path) if r.solved else 0, result=r, problem=p))

    for s in range(args.warmup):
        one_step(s, False)
    barrier(world)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        step_ms = []
        for s in range(args.steps):
            t0 = time.perf_counter()
            one_step(args.warmup + s, True)
            step_ms.append((time.perf_counter() - t0) * 1e3)
    barrier(world)
    launches = ctx.launches - launches0

    keep = [{k: v for k, v in r.items() if k not in ("result", "problem")} for r in recs]
    all_recs = sum(gather(world, keep), [])
    max_step = float(max(gather(world, float(np.mean(step_ms)))))
    solved = [r for r in all_recs if r["solved"]]
    import fixtures as fx
    feas = fx.upright_feasible()
    rf = [r for r in all_recs if feas[r["k"]]]
    med = lambda xs: float(np.median(xs)) if xs else None   # noqa: E731
    pct = lambda xs, q: float(np.percentile(xs, q)) if xs else None   # noqa: E731

    # roofline of the dominant kernel (cp_plan_kernel) over the SOLVED queries
    # (the headline's population): algorithmic FP32 work from the device's own
    # counters / the kernel's event-timed duration.  Unsolved queries run the
    # whole time budget on an infeasible pair; they are reported beside it.
    flops = sum(r["stage1"] * FLOP_STAGE1_M4 + r["fk"] * FLOP_FK_ARM7 + r["checks"] * FLOP_CHECK
                + r["nn"] * FLOP_NN7 for r in solved)
    kern_s = sum(r["kernel_ms"] for r in solved) * 1e-3
    kern_all = sum(r["kernel_ms"] for r in all_recs) * 1e-3
    sms = 148
    try:
        sms = int(subprocess.run(["nvidia-smi", "--query-gpu=multiprocessor_count", "--format=csv,noheader"],
                                 capture_output=True, text=True, timeout=10).stdout.split()[0])
    except Exception:
        pass
    clocks = clk.summary()
    max_mhz = clocks.get("sm_max_mhz") or 1965
    fp32_peak = sms * 128 * 2 * max_mhz * 1e6 / 1e12     # nominal FMA TFLOP/s
    achieved = flops / kern_s / 1e12 if kern_s > 0 else 0.0
    solved_dev = [r["device_ms"] for r in solved]
    line = {
        "metric": METRIC,
        "value": med(solved_dev),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_step,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic queries from the reference's generate_pair (pair_seed 300..399); "
                "robot/scene/constraint are the reference's arm7 / table / upright-EE plane",
        "config": headline_config(args, world),
        "device_options": {"teams": args.teams or "auto", "cc_broadphase": args.cc_broadphase},
        "l2": "flushed (256 MiB write) before every query",
        "value_clock": "planner globaltimer, init kernel start -> last team out of the query (results complete)",
        "success_rate": len(solved) / max(1, len(all_recs)),
        "success_rate_feasible": sum(r["solved"] for r in rf) / max(1, len(rf)),
        "feasible_note": "14 of the 100 pairs are unsolved by the reference planner too (3 seeds x 20 s, "
                         "tests/golden/upright_feasibility.json; DESIGN.md section 10 for the GPU's long-budget "
                         "sweep of them)",
        "queries": len(all_recs),
        "p10_ms": pct(solved_dev, 10),
        "p90_ms": pct(solved_dev, 90),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": med([r["wall_ms"] for r in solved]), "unit": "ms",
                "h2d_bytes_per_step": Q * (2 * 7 * 8 + 8),
                "d2h_bytes_per_step": int(Q * (64 + 8 * 12) + sum(r["path"] for r in recs) * 28
                                          // max(1, args.steps))},
        "roofline": {"bound": "fp32", "kernel": "cp_plan_kernel", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                     "population": f"{len(solved)} solved queries (the headline's); "
                                   f"{len(all_recs) - len(solved)} unsolved queries ran the full budget and "
                                   f"took {100 * (1 - kern_s / kern_all) if kern_all else 0:.2f} % of the "
                                   "kernel time",
                     "peak_source": f"nominal FP32 FMA ({sms} SM x 128 lanes x 2 x {max_mhz} MHz); "
                                    "MEASURED_PEAKS.json has no FP32 entry",
                     "traffic": _ncu_traffic("cp_plan_kernel"),
                     "work": "stage1 x 1750 + cc_fk x 1195 + checks x 11 + nn_nodes x 20 flop"},
        "unsolved_rate": 1 - len(solved) / max(1, len(all_recs)),
    }
    if rank == 0:
        line["e2e_back_to_back"] = back_to_back(ctx, recs, opt)
    line["throughput"] = throughput(args, world, rank, local, line)
    if rank == 0 and world == 1 and not args.no_extras:
        line.update(extras(args, local, line))
        line["other_configs"] = other_configs(args, local)
        line["ablation_projection"] = ablation_projection(args, local)
    if rank == 0 and world == 1:
        line["revalidate_ref_pass_rate"] = revalidate_ref(recs)
        if not args.no_cpu:
            cpu_arms(args, line, recs)
    return line


def back_to_back(ctx, recs, opt):
    """The timed region's solved queries (same pairs, same seeds) again, plan()
    called back to back with no L2 flush in between: the previous call's
    cp_reset_kernel (the NaN refill behind the results event) lands on this
    call, as it would in a serving loop."""
    from paper_2505_06791_b200.planner import plan
    walls, devs, flushed = [], [], []
    for r in recs:
        if not r["solved"]:
            continue
        t0 = time.perf_counter()
        plan(r["problem"], opt)
        walls.append((time.perf_counter() - t0) * 1e3)
        devs.append(ctx.last_timing()[0])
        flushed.append(r["wall_ms"])
    return {"value": float(np.median(walls)) if walls else None, "unit": "ms",
            "device_ms": float(np.median(devs)) if devs else None, "queries": len(walls),
            "same_queries_flushed_ms": float(np.median(flushed)) if flushed else None,
            "note": "median plan() wall over the timed region's solved queries replayed consecutively, "
                    "no L2 flush (the previous call's reset kernel included)"}


def throughput(args, world, rank, local, line):
    """configs[4]: every rank plans its own 1024 queries per step in one
    persistent launch (plan_many, the columnar public API); queries/s from the
    max-over-ranks device time per step (CUDA events), and end to end (wall)."""
    import fixtures as fx
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, plan_many
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prm = PlanParams(width=16, max_iterations=300)
    opt = DeviceOptions(device=local)
    ctx = kernels.context(m, local)
    for w in range(max(3, args.warmup)):
        s, g, seeds = batch_arrays(w)
        plan_many(m, sc, sp, s, g, seeds, prm, opt)
    dev, wall, solved, kern, flops, ccall = [], [], 0, [], 0.0, []
    for step in range(args.steps):
        s, g, seeds = batch_arrays(100 + step)
        barrier(world)
        t0 = time.perf_counter()
        r = plan_many(m, sc, sp, s, g, seeds, prm, opt)
        w = (time.perf_counter() - t0) * 1e3
        tot, kms = ctx.last_timing()
        both = gather(world, (tot, w))
        dev.append(max(b[0] for b in both))
        wall.append(max(b[1] for b in both))
        solved += int(r.solved.sum())
        kern.append(kms)
        ccall.append(r.wall_ms)
        st = r.stats.astype(np.float64).sum(axis=0)
        flops += st[8] * FLOP_STAGE1_M1 + st[9] * FLOP_FK_ARM7 + st[5] * FLOP_CHECK + st[10] * FLOP_NN7
    # the same batches as a stream: two in flight per GPU (PlanStream), so a
    # batch's slowest queries overlap the next batch's start; end to end
    # (wall, max over ranks) from the first submit to the last result
    from paper_2505_06791_b200.planner import PlanStream
    stream = PlanStream(m, sc, sp, prm, opt, depth=2)
    for w in range(2):
        stream.result(stream.submit(*batch_arrays(w)))
    barrier(world)
    t0 = time.perf_counter()
    tickets = [stream.submit(*batch_arrays(100 + step)) for step in range(min(2, args.steps))]
    psolved = 0
    for step in range(args.steps):
        r = stream.result(tickets[step])
        psolved += int(r.solved.sum())
        if step + 2 < args.steps:
            tickets.append(stream.submit(*batch_arrays(100 + step + 2)))
    pwall = max(gather(world, (time.perf_counter() - t0) * 1e3))
    psolved = sum(gather(world, psolved))
    solved_all = sum(gather(world, solved))
    total = world * BATCH * args.steps
    peak = line["roofline"]["peak"]
    bach = flops / (sum(kern) * 1e-3) / 1e12
    return {"metric": "configs[4] batched constrained queries/s (whole job)", "unit": "queries/s",
            "value": total / (sum(dev) * 1e-3), "higher_is_better": True, "scaling": "weak",
            "e2e": {"value": total / (sum(wall) * 1e-3), "unit": "queries/s",
                    "h2d_bytes_per_step": BATCH * (2 * 7 * 8 + 8),
                    "d2h_bytes_per_step": BATCH * (64 + 8 * 12)},
            "pipelined": {"e2e_queries_per_s": total / (pwall * 1e-3), "ms_per_step_wall": pwall / args.steps,
                          "success_rate": psolved / total,
                          "how": "the same steps' batches through PlanStream (two batches in flight per GPU: a batch's "
                                 "slowest queries overlap the next one's start), wall clock from the first submit "
                                 "to the last result, max over ranks"},
            "ms_per_step_device": float(np.mean(dev)), "ms_per_step_wall": float(np.mean(wall)),
            "ms_per_step_c_call_rank0": float(np.mean(ccall)),
            "kernel_ms_per_step_rank0": float(np.mean(kern)), "success_rate": solved_all / total,
            "config": f"configs[4]: {BATCH} arm7 table-plane (z=0.60, tau 0.01) queries per GPU per step, W=16, "
                      "max_iterations 300 each, one persistent launch per GPU (plan_many), "
                      f"{world} GPU(s), no collective",
            "roofline": {"bound": "fp32", "kernel": "cp_plan_kernel (batch, every resident team, rank 0)",
                         "achieved": bach, "peak": peak, "unit": "TFLOP/s", "frac": bach / peak,
                         "work": "stage1 x 1240 (m=1) + cc_fk x 1195 + checks x 11 + nn_nodes x 20 flop"}}


def extras(args, local, line):
    """CC checks/s (BASELINE metric) and the NN streaming roofline."""
    import fixtures as fx
    from paper_2505_06791_b200 import kernels
    model = fx.robot("arm7")
    out = {}
    # -- CC throughput: 999-box shelf, W=16, flag off (every check performed)
    sc = fx.scene("shelf_x111")
    # 16384 motions x 16 waypoints = 8192 warps: several resident waves on 148 SMs
    B, W = 16384, 16
    wps = cc_motions(model, B, W, device=local)
    kernels.validate_batch(model, sc, wps[:64], False, device=local)
    best = None
    for _ in range(3):
        r = kernels.validate_batch(model, sc, wps, False, device=local)
        if best is None or r["kernel_ms"] < best["kernel_ms"]:
            best = r
    checks = int(best["gpu_checks"].sum())
    on = kernels.validate_batch(model, sc, wps, True, device=local)
    poss = int(on["possible"].sum())
    s_off = best["kernel_ms"] * 1e-3
    cc_flops = checks * FLOP_CHECK + B * W * FLOP_FK_ARM7
    peak = line["roofline"]["peak"]
    out["cc_checks_per_s"] = checks / s_off
    out["cc_effective_checks_per_s_flag_on"] = poss / (on["kernel_ms"] * 1e-3)
    # the same motions through the clustered broad phase: reference checks
    # resolved per second (possible / time) and the checks it evaluated
    bp = None
    for _ in range(3):
        r = kernels.validate_batch(model, sc, wps, True, device=local, broadphase=True)
        if bp is None or r["kernel_ms"] < bp["kernel_ms"]:
            bp = r
    assert (bp["valid"] == on["valid"]).mean() > 0.99
    out["cc_broadphase"] = {"effective_checks_per_s": poss / (bp["kernel_ms"] * 1e-3),
                            "checks_evaluated_frac": float(bp["performed"].sum()) / poss,
                            "kernel_ms": bp["kernel_ms"], "flag": "on",
                            "kernel": f"cp_validate_cull_kernel (999 boxes, {B} motions x {W})"}
    out["roofline_cc"] = {"bound": "fp32", "kernel": f"cp_validate_kernel (999 boxes, {B} motions x {W})",
                          "achieved": cc_flops / s_off / 1e12, "peak": peak, "unit": "TFLOP/s",
                          "frac": cc_flops / s_off / 1e12 / peak, "traffic": _ncu_traffic("cp_validate_kernel"),
                          "kernel_ms": best["kernel_ms"]}
    # -- NN scan streaming: 2368 distinct trees of 16384 nodes (1.1 GB > L2)
    T, N = 2368, 16384
    rng = np.random.default_rng(0)
    nodes = rng.uniform(-2.0, 2.0, size=(T, N, 7))
    qq = rng.uniform(-2.0, 2.0, size=(T, 7))
    kernels.nearest_trees(model, nodes[:4], qq[:4], device=local)
    ms = min(kernels.nearest_trees(model, nodes, qq, device=local)[1] for _ in range(3))
    gbs = T * N * BYTES_NN7 / (ms * 1e-3) / 1e9
    hbm = _measured_hbm()
    out["roofline_nn"] = {"bound": "hbm", "kernel": f"cp_nearest_kernel ({T} trees x {N} nodes, SoA float4)",
                          "achieved": gbs, "peak": hbm[0], "unit": "GB/s", "frac": gbs / hbm[0],
                          "peak_source": hbm[1], "traffic": _ncu_traffic("cp_nearest_kernel"),
                          "algorithmic_bytes": T * N * BYTES_NN7, "kernel_ms": ms}
    return out


def cc_motions(model, B, W, device=0):
    """B straight motions of W waypoints between Halton samples (seed 12345)."""
    from paper_2505_06791_b200 import kernels
    qs = kernels.halton_batch(model, 2 * B, 1, 12345, device=device)
    t = np.linspace(0, 1, W)[None, :, None]
    return qs[0::2][:, None, :] * (1 - t) + qs[1::2][:, None, :] * t


def ablation_projection(args, local):
    """The paper's projection ablation (parallel vs the
    sequential "naive" projector) on the headline workload: 30 feasible
    upright pairs x 2 seeds per mode, device median time and success."""
    import fixtures as fx
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
    model, scene, spec, starts, goals = workload()
    feas = np.nonzero(fx.upright_feasible())[0][:30]
    opt = DeviceOptions(device=local)
    out = {}
    for mode in ("parallel", "naive", "literal-gap"):
        times, ok, n = [], 0, 0
        for k in feas:
            for seed in range(2):
                p = PlanProblem(model, scene, spec, starts[k], goals[k],
                                PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0,
                                           seed_offset=int(k) * 10_000 + seed, projection_mode=mode))
                ctx = prepare(p, opt)
                ctx.flush_l2()
                r = plan(p, opt)
                n += 1
                if r.solved:
                    ok += 1
                    times.append(ctx.last_timing()[0])
        out[mode] = {"median_ms": float(np.median(times)) if times else None, "success_rate": ok / n,
                     "queries": n}
    out["workload"] = "configs[1] upright Panda, 30 feasible pairs x 2 seeds, W=16"
    return out


OTHER = ("configs[0]", "configs[2]:shelf_x11", "configs[2]:shelf_x111", "configs[3]")


def other_configs(args, local):
    """Median device planning time + success for configs[0], [2], [3]
    (three seeds per query)."""
    import fixtures as fx
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
    res = {}
    for name in OTHER:
        label, probs = _cfg_problems(name)
        # configs[2] ablations: early-exit flag on/off x broad phase (auto: on
        # whenever the scene has obstacles) / the reference's lockstep check order
        variants = ((("on", -1, ""), ("off", -1, " (cc flag off)"), ("on", 0, " (lockstep order)"),
                     ("off", 0, " (lockstep order, cc flag off)"))
                    if name.startswith("configs[2]") else (("on", -1, ""),))
        feas = fx.dense8_feasible() if name == "configs[3]" else None
        for flag, bp, suffix in variants:
            tflag = []
            nfeas = sfeas = 0
            opt = DeviceOptions(device=local, cc_broadphase=bp)
            for qi, (m, sc, sp, s, g, kw) in enumerate(probs):
                for seed in range(3):
                    p = PlanProblem(m, sc, sp, s, g, PlanParams(max_iterations=10**6, time_budget_ms=2000.0,
                                                                seed_offset=seed * 10_000, flag_mode=flag, **kw))
                    ctx = prepare(p, opt)
                    ctx.flush_l2()
                    r = plan(p, opt)
                    if r.solved:
                        tflag.append(ctx.last_timing()[0])
                    if feas is not None and feas[qi]:
                        nfeas += 1
                        sfeas += r.solved
            res[name + suffix] = {"workload": label, "median_ms": float(np.median(tflag)) if tflag else None,
                                  "queries": len(probs) * 3, "success_rate": len(tflag) / (len(probs) * 3)}
            if feas is not None:
                res[name + suffix]["success_rate_feasible"] = sfeas / max(1, nfeas)
                res[name + suffix]["feasible_note"] = (
                    f"{int((~feas).sum())} of the {len(feas)} pairs are unsolved by the reference planner too "
                    "(3 seeds x 20 s, tests/golden/dense8_feasibility.json)")
    return res


def revalidate_ref(recs):
    """The reference's own FP64 revalidate_path (oracle/_ref, planner.py:508-523)
    over every solved GPU path of the timed region: re-derives each edge in FP64
    from the FP32 tree nodes (stricter than reproducing the certified motion)."""
    import refpkg
    if not refpkg.available():
        return None
    M = refpkg.load("compiled")
    cache = {}
    ok = n = 0
    for r in recs:
        if r["solved"]:
            n += 1
            ok += bool(M.revalidate_path(r["result"], refpkg.to_ref_problem(M, r["problem"], cache)))
    return {"value": ok / max(1, n), "paths": n, "checker": "maniplan.revalidate_path, compiled FP64 backend"}


# ---------------------------------------------------------------------------
# the reference planner on the host cores (oracle/_ref: stock maniplan build)
# ---------------------------------------------------------------------------

_W: dict = {}


def _worker_ref():
    if "M" not in _W:
        import refpkg
        _W["M"] = refpkg.load("compiled")
        _W["cache"] = {}
    return _W["M"], _W["cache"]


def _ref_plan_job(job):
    """One reference plan() in a worker process (one core): job = (kind,
    index, seed_offset, params overrides) -> (solved, wall_ms, status, stats)."""
    import refpkg
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem
    M, cache = _worker_ref()
    kind, i, seed, kw = job
    if kind == "configs[1]":
        model, scene, spec, starts, goals = workload()
        prob = PlanProblem(model, scene, spec, starts[i], goals[i], PlanParams(seed_offset=seed, **kw))
    elif kind == "configs[4]":
        import fixtures as fx
        prs = fx.pairs()
        prob = PlanProblem(fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane"),
                           prs["table_plane_start"][i], prs["table_plane_goal"][i], PlanParams(seed_offset=seed, **kw))
    else:
        m, sc, sp, s, g, pkw = _cfg_problems(kind)[1][i]
        prob = PlanProblem(m, sc, sp, s, g, PlanParams(seed_offset=seed, **{**pkw, **kw}))
    rp = refpkg.to_ref_problem(M, prob, cache)
    t0 = time.perf_counter()
    r = M.plan(rp)
    wall = (time.perf_counter() - t0) * 1e3
    st = r.stats
    return (r.solved, wall, r.status, (st.iterations, st.projection_failures, st.cc_performed, st.cc_possible))


def _ref_cc_job(job):
    """The reference's validate_waypoints (compiled backend) on a pre-packed
    999-box shelf, flag off, on one core: (checks performed, seconds)."""
    import fixtures as fx
    M, _ = _worker_ref()
    from maniplan._kernels import _compiled
    import refpkg
    B, W = job
    model = refpkg.to_ref_robot(M, fx.robot("arm7"))
    robot = model.packed
    scene = refpkg.to_ref_scene(M, fx.scene("shelf_x111")).packed()
    # the first B motions of the GPU's CC workload (cc_motions: Halton samples
    # from index 1 at seed_offset 12345, the reference's own HaltonState)
    hs = M.HaltonState(model.n, seed_offset=12345)
    q = np.array([hs.next_sample(model.limits) for _ in range(2 * B)])
    t = np.linspace(0, 1, W)[None, :, None]
    mot = np.ascontiguousarray(q[0::2][:, None, :] * (1 - t) + q[1::2][:, None, :] * t)
    _compiled.validate_waypoints(mot[0], robot, scene, False)
    done = 0
    t0 = time.perf_counter()
    for k in range(B):
        done += _compiled.validate_waypoints(mot[k], robot, scene, False)[1]
    return done, time.perf_counter() - t0


def _pool(cores):
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    return ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"))


def cpu_arms(args, line, recs):
    """The reference planner beside every config, on this box's host cores:
    one query per process (single-core latencies, run concurrently on the
    cores), configs[4] as queries/s over all cores, CC checks/s on one core.
    Also writes the configs[1] GPU + CPU trial records (reference formats)."""
    import refpkg
    if not refpkg.available():
        line["cpu_baseline"] = {"value": None, "unavailable": "oracle/_ref not built"}
        return
    cores = os.cpu_count() or 1
    n = args.cpu_queries
    budget = args.budget_ms
    head = [(r["k"], r["seed"]) for r in recs[:n]]
    t_all = time.perf_counter()
    with _pool(cores) as ex:
        list(ex.map(_ref_plan_job, [("configs[1]", 0, 0, dict(width=16, max_iterations=50, time_budget_ms=50.0))]
                    * cores))
        # configs[1]: the first n timed GPU queries (same pair, same seed)
        kw1 = dict(width=16, max_iterations=args.max_iterations, time_budget_ms=budget)
        t0 = time.perf_counter()
        res1 = list(ex.map(_ref_plan_job, [("configs[1]", k, s, kw1) for k, s in head]))
        el1 = time.perf_counter() - t0
        solved1 = [w for ok, w, *_ in res1 if ok]
        import fixtures as fx
        feas = fx.upright_feasible()
        nf = sum(bool(feas[k]) for k, _ in head)
        sf = sum(ok for (ok, *_), (k, _) in zip(res1, head) if feas[k])
        line["cpu_baseline"] = {
            "value": float(np.median(solved1)) if solved1 else None, "unit": "ms",
            "success_rate": len(solved1) / max(1, n), "success_rate_feasible": sf / max(1, nf),
            "cores": 1, "kind": "reference",
            "sample": f"the first {n} timed GPU queries (same pair, same seed_offset, same budget "
                      f"{budget:.0f} ms), reference plan() one query per process on one core, {cores} processes "
                      f"concurrently ({el1:.1f} s)",
            "build": "stock pip install of /root/reference/pkg (only _compiled.pyx compiled, "
                     "MANIPLAN_KERNELS=compiled)"}
        # the other configs: >= 20 samples each (a query x seed grid)
        for name in OTHER:
            label, probs = _cfg_problems(name)
            jobs = [(name, qi, seed * 10_000, dict(max_iterations=10**6, time_budget_ms=budget))
                    for seed in range(max(1, -(-20 // len(probs)))) for qi in range(len(probs))][:max(20, len(probs))]
            t0 = time.perf_counter()
            rr = list(ex.map(_ref_plan_job, jobs))
            ok = [w for s, w, *_ in rr if s]
            line.setdefault("other_configs", {}).setdefault(name, {})["cpu_reference"] = {
                "median_ms": float(np.median(ok)) if ok else None, "success_rate": len(ok) / len(jobs),
                "samples": len(jobs), "cores": 1,
                "sample": f"{len(jobs)} (pair, seed) samples, one query per process on one core, budget "
                          f"{budget:.0f} ms ({time.perf_counter() - t0:.1f} s)"}
        # configs[4]: 1024 queries over every host core
        kw4 = dict(width=16, max_iterations=300)
        _, _, seeds = batch_arrays(100)
        jobs = [("configs[4]", i, int(seeds[i]), kw4) for i in range(BATCH)]
        t0 = time.perf_counter()
        rr = list(ex.map(_ref_plan_job, jobs, chunksize=8))
        el = time.perf_counter() - t0
        line["throughput"]["cpu_reference"] = {
            "value": BATCH / el, "unit": "queries/s", "cores": cores, "success_rate": sum(r[0] for r in rr) / BATCH,
            "sample": f"the {BATCH} configs[4] queries of the first timed step, reference plan() on {cores} "
                      f"processes ({el:.1f} s)"}
        # CC checks/s: validate_waypoints on one core
        done, secs = ex.submit(_ref_cc_job, (args.cpu_cc_motions, 16)).result()
        line["cpu_cc_checks_per_s"] = {"value": done / secs, "unit": "checks/s", "cores": 1,
                                       "sample": f"the first {args.cpu_cc_motions} of the GPU's motions x 16 waypoints "
                                                 "vs the 999-box shelf, flag off, "
                                                 f"reference _compiled.validate_waypoints ({secs:.1f} s)"}
    line["cpu_arms_s"] = time.perf_counter() - t_all
    write_trial_records(args, line, recs, head, res1)


def write_trial_records(args, line, recs, head, res1):
    """configs[1] trial records of both arms in the reference's formats:
    records.csv (problem = "<arm>:upright#<pair>") + cdf_*.csv per arm."""
    from paper_2505_06791_b200 import harness as H
    gpu = [H.TrialRecord(f"b200:upright#{r['k']}", r["step"], "parallel", "on", 1, r["seed"], r["status"],
                         r["wall_ms"], r["iterations"], r["pfail"], r["checks"], r["possible"]) for r in recs]
    cpu = [H.TrialRecord(f"reference:upright#{k}", 0, "parallel", "on", 1, s, st, w, it, pf, cp, cq)
           for (k, s), (_, w, st, (it, pf, cp, cq)) in zip(head, res1)]
    out = args.records_dir
    os.makedirs(out, exist_ok=True)
    H.write_records(gpu + cpu, os.path.join(out, "records.csv"))
    cdfs = H.write_cdfs(gpu, os.path.join(out, "b200")) + H.write_cdfs(cpu, os.path.join(out, "reference"))
    line["records"] = {"dir": os.path.relpath(out, ROOT), "csv": "records.csv",
                       "cdfs": [os.path.relpath(p, out) for p in cdfs],
                       "summary": {"b200": H.summarize(gpu), "reference": H.summarize(cpu)},
                       "note": "GPU wall_ms = plan() end to end; reference wall_ms = its plan() on one core"}


def _ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the newest
    committed ncu --set full summary (profiles/r*_traffic.json, written by
    tools/summarize_profiles.py from the capture of the same kernel), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))   # r1 < r1b < ... < r2
    for f in reversed(files):
        try:
            with open(f) as fh:
                d = json.load(fh)
            if kernel in d:
                return float(d[kernel]["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


def _measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args, world, rank):
    if rank != 0:
        return None
    import refpkg
    if not refpkg.available():
        return {"impl": "reference", "unavailable": "oracle/_ref not built (oracle/build_ref.sh)"}
    cores = os.cpu_count() or 1
    Q = args.queries
    steps, all_res = [], []
    kw = dict(width=16, max_iterations=args.max_iterations, time_budget_ms=args.budget_ms)
    with _pool(cores) as ex:
        list(ex.map(_ref_plan_job, [("configs[1]", 0, 0, dict(width=16, max_iterations=50, time_budget_ms=50.0))]
                    * cores))
        for s in range(args.warmup + args.steps):
            jobs = []
            for j in range(Q):
                k = query_index(s, j, Q, world, 0)
                jobs.append(("configs[1]", k, query_seed(s, k), kw))
            t0 = time.perf_counter()
            res = list(ex.map(_ref_plan_job, jobs))
            if s >= args.warmup:
                steps.append((time.perf_counter() - t0) * 1e3)
                all_res += res
    solved = [w for ok, w, *_ in all_res if ok]
    med = float(np.median(solved)) if solved else None
    return {"metric": METRIC, "value": med, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.mean(steps)), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "same synthetic queries",
            "config": headline_config(args, world),
            "impl": "reference", "success_rate": len(solved) / max(1, len(all_res)),
            "cpu_baseline": {"value": med, "unit": "ms", "cores": cores, "kind": "reference",
                             "sample": f"{len(all_res)} queries (the B200 arm's pairs and seeds), one reference "
                                       f"plan() per process, {cores} processes",
                             "build": "stock pip install of /root/reference/pkg (only _compiled.pyx compiled, "
                                      "MANIPLAN_KERNELS=compiled)"},
            "e2e": {"value": med, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--queries", type=int, default=25, help="queries per step per GPU")
    ap.add_argument("--teams", type=int, default=_env_int("CPRRTC_TEAMS", 0))
    ap.add_argument("--max-iterations", type=int, default=1_000_000)
    ap.add_argument("--cc-broadphase", type=int, default=-1,
                    help="planner CC: 1 clustered broad phase, 0 reference lockstep order, -1 auto")
    ap.add_argument("--budget-ms", type=float, default=2000.0)
    ap.add_argument("--cpu-queries", type=int, default=100,
                    help="reference configs[1] sample: the first K timed GPU queries")
    ap.add_argument("--cpu-cc-motions", type=int, default=2000)
    ap.add_argument("--records-dir", default=os.path.join(ROOT, "bench_records"))
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)
    if os.environ.get("CPRRTC_BENCH_ONE_GPU") == "1":
        print("bench.py: CPRRTC_BENCH_ONE_GPU=1 -- every rank on cuda:0 (code-path test, not a measurement)",
              file=sys.stderr)
    world, rank, local = dist_setup()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        line = run_reference(args, world, rank)
    else:
        if world > 1 and _visible_gpus() <= local and os.environ.get("CPRRTC_BENCH_ONE_GPU") != "1":
            sys.exit(f"bench.py: rank {rank} needs cuda:{local}, {_visible_gpus()} device(s) visible")
        line = run_b200(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
