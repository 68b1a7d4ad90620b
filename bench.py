#!/usr/bin/env python
"""bench.py -- cpRRTC planning on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): 7-DoF Panda-like arm (arm7), table scene,
end effector kept upright on the plane z = 0.60 with a locked orientation
(0,1,0,0), tau_task 0.01, W = 16 waypoints per motion; start/goal pairs from
the reference's own generate_pair (tests/golden/pairs.npz, pair_seed 300+k).

A step = plan Q queries one after another, each with the whole GPU (one
persistent-kernel launch per query).  value = median planning time of the
solved queries (device time, inputs resident: CUDA events after the H2D copy
to after path extraction); e2e = the same median through the public
plan() call (host buffers in, H2D + D2H inside the timed region); success
rate beside it.  The L2 is flushed (256 MiB write) before every query.

Also measured on the same run: CC checks/s of the collision kernel on a
999-box shelf (BASELINE "CC checks/s"), the NN scan's streaming bandwidth,
and the 1024-query batched throughput (configs[4]).

--impl reference runs the reference planner (oracle/_ref: maniplan compiled
from the reference's own sources; else the C oracle port) on the host cores
over the same queries.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

METRIC = "median planning time (ms) + success rate, constrained Panda; CC checks/s"
N_PAIRS = 100
# algorithmic FP32 flop per work unit (counted from the
# reference formulas): projection stage 1 with plane+orientation (m=4), FK +
# world spheres of arm7, one sphere-primitive check, one NN node (3n-1).
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


def query_index(step, j, Q, world, rank):
    """Weak scaling: rank r plans queries [r*Q, (r+1)*Q) of step's global
    block of world*Q queries (pair index modulo the 100 pairs)."""
    return (step * Q * world + rank * Q + j) % N_PAIRS


def merge_ranks(world, recs, step_ms):
    """Gather per-rank query records and step times (rank-0 summary: median
    over every query of every rank, max step time over ranks)."""
    all_recs = sum(gather(world, recs), [])
    all_steps = gather(world, float(np.mean(step_ms)) if step_ms else 0.0)
    return all_recs, float(max(all_steps))


def workload():
    import fixtures as fx
    return (fx.robot("arm7"), fx.scene("table"), fx.spec("upright"),
            fx.pairs()["upright_start"], fx.pairs()["upright_goal"])


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")   # control plane only: no data-path collective
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


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args, world, rank, local):
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
    model, scene, spec, starts, goals = workload()
    opt = DeviceOptions(device=local, teams=args.teams, cc_broadphase=args.cc_broadphase)
    Q = args.queries

    def problem(step, j):
        k = query_index(step, j, Q, world, rank)
        seed = (step * 7919 + k) * 10_000
        return PlanProblem(model, scene, spec, starts[k], goals[k],
                           PlanParams(width=16, max_iterations=args.max_iterations,
                                      time_budget_ms=args.budget_ms, seed_offset=seed))

    ctx = prepare(problem(0, 0), opt)
    launches0 = None
    recs = []

    def one_step(step, timed):
        nonlocal launches0
        for j in range(Q):
            p = problem(step, j)
            ctx.flush_l2()
            t0 = time.perf_counter()
            r = plan(p, opt)
            wall = (time.perf_counter() - t0) * 1e3
            tot, kern = ctx.last_timing()
            if timed:
                st = r.stats
                k = query_index(step, j, Q, world, rank)
                recs.append(dict(k=k, solved=r.solved, device_ms=tot, kernel_ms=kern, wall_ms=wall,
                                 stage1=st.stage1_evals, fk=st.cc_fk_evals, checks=st.cc_performed,
                                 nn=st.nn_nodes, path=len(r.path) if r.solved else 0))

    for s in range(args.warmup):
        one_step(s, False)
    barrier(world)
    launches0 = ctx.launches
    t_start = time.perf_counter()
    with ClockSampler(local) as clk:
        step_ms = []
        for s in range(args.steps):
            t0 = time.perf_counter()
            one_step(args.warmup + s, True)
            step_ms.append((time.perf_counter() - t0) * 1e3)
    barrier(world)
    wall_total = time.perf_counter() - t_start
    launches = ctx.launches - launches0

    all_recs, max_step = merge_ranks(world, recs, step_ms)
    solved = [r for r in all_recs if r["solved"]]
    succ = len(solved) / max(1, len(all_recs))
    import fixtures as fx
    feas = fx.upright_feasible()
    rf = [r for r in all_recs if feas[r["k"]]]
    succ_f = sum(r["solved"] for r in rf) / max(1, len(rf))
    med_dev = float(np.median([r["device_ms"] for r in solved])) if solved else None
    med_wall = float(np.median([r["wall_ms"] for r in solved])) if solved else None
    p10 = float(np.percentile([r["device_ms"] for r in solved], 10)) if solved else None
    p90 = float(np.percentile([r["device_ms"] for r in solved], 90)) if solved else None

    # roofline of the dominant kernel (cp_plan_kernel): algorithmic FP32 work
    # from the device's own work counters / its event-timed duration
    flops = sum(r["stage1"] * FLOP_STAGE1_M4 + r["fk"] * FLOP_FK_ARM7 + r["checks"] * FLOP_CHECK
                + r["nn"] * FLOP_NN7 for r in all_recs)
    kern_s = sum(r["kernel_ms"] for r in all_recs) * 1e-3
    import ctypes
    sms = 148
    try:
        from paper_2505_06791_b200 import _lib  # noqa: F401
        import subprocess
        sms = int(subprocess.run(["nvidia-smi", "--query-gpu=multiprocessor_count", "--format=csv,noheader"],
                                 capture_output=True, text=True, timeout=10).stdout.split()[0])
    except Exception:
        pass
    clocks = clk.summary()
    max_mhz = clocks.get("sm_max_mhz") or 1965
    fp32_peak = sms * 128 * 2 * max_mhz * 1e6 / 1e12     # nominal FMA TFLOP/s
    achieved = flops / kern_s / 1e12 if kern_s > 0 else 0.0
    line = {
        "metric": METRIC,
        "value": med_dev,
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
        "config": {"workload": "configs[1] constrained Panda: arm7 + table, plane z=0.60 + fixed "
                               "orientation (0,1,0,0), tau 0.01, W=16",
                   "queries_per_step_per_gpu": Q, "max_iterations": args.max_iterations,
                   "time_budget_ms": args.budget_ms, "teams": args.teams or "auto",
                   "l2": "flushed (256 MiB write) before every query",
                   "parallelism": f"replicas x{world} (independent queries per GPU)"},
        "success_rate": succ,
        "success_rate_feasible": succ_f,
        "feasible_note": "14 of the 100 pairs are unsolved by the reference planner too (3 seeds x 20 s, "
                         "tests/golden/upright_feasibility.json): infeasible, disconnected manifold",
        "queries": len(all_recs),
        "p10_ms": p10,
        "p90_ms": p90,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": med_wall, "unit": "ms",
                "h2d_bytes_per_step": Q * (2 * 7 * 8 + 8),
                "d2h_bytes_per_step": int(Q * (64 + 8 * 12) + sum(r["path"] for r in recs) * 28 // max(1, args.steps))},
        "roofline": {"bound": "fp32", "kernel": "cp_plan_kernel", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                     "peak_source": f"nominal FP32 FMA ({sms} SM x 128 lanes x 2 x {max_mhz} MHz); "
                                    "MEASURED_PEAKS.json has no FP32 entry",
                     "traffic": _ncu_traffic("cp_plan_kernel"),
                     "work": "stage1 x 1750 + cc_fk x 1195 + checks x 11 + nn_nodes x 20 flop"},
    }
    if rank == 0 and not args.no_extras:
        line.update(extras(args, local, model, line))
        line["other_configs"] = other_configs(args, local)
        line["ablation_projection"] = ablation_projection(args, local)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args)
    return line


def extras(args, local, model, line):
    """CC checks/s (BASELINE metric), NN streaming roofline, batched queries."""
    import fixtures as fx
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan_batch
    out = {}
    # -- CC throughput: 999-box shelf, W=16, flag off (every check performed)
    sc = fx.scene("shelf_x111")
    # 16384 motions x 16 waypoints = 8192 warps: several resident waves on 148 SMs
    B, W = 16384, 16
    qs = kernels.halton_batch(model, 2 * B, 1, 12345, device=local)
    t = np.linspace(0, 1, W)[None, :, None]
    wps = qs[0::2][:, None, :] * (1 - t) + qs[1::2][:, None, :] * t
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
    # -- NN scan streaming: 4736 distinct trees of 16384 nodes (2.2 GB > L2)
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
    # -- batched queries (configs[4]): 1024 table-plane queries in one launch
    m, sc2, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prs = fx.pairs()
    probs = [PlanProblem(m, sc2, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                         PlanParams(width=16, max_iterations=300, seed_offset=i * 10_000))
             for i in range(1024)]
    opt = DeviceOptions(device=local)
    from paper_2505_06791_b200.planner import prepare
    bctx = prepare(probs[0], opt)
    plan_batch(probs[:8], opt)
    best, best_res, best_kms = None, None, None
    for _ in range(3):
        t0 = time.perf_counter()
        res = plan_batch(probs, opt)
        dt = time.perf_counter() - t0
        if best is None or dt < best:
            best, best_res, best_kms = dt, res, bctx.last_timing()[1]
    dt, res = best, best_res
    # the same kernel at full occupancy (throughput mode): algorithmic FP32
    # work of the batch (plane constraint: m = 1 stage-1 cost) / kernel time
    bflops = sum(r.stats.stage1_evals * FLOP_STAGE1_M1 + r.stats.cc_fk_evals * FLOP_FK_ARM7
                 + r.stats.cc_performed * FLOP_CHECK + r.stats.nn_nodes * FLOP_NN7 for r in res)
    bach = bflops / (best_kms * 1e-3) / 1e12
    out["batch_1024"] = {"queries_per_s": 1024 / dt, "wall_ms": dt * 1e3,
                         "success_rate": sum(r.solved for r in res) / 1024,
                         "config": "configs[4]: 1024 arm7 table-plane (z=0.60, tau 0.01) queries, W=16, "
                                   "max_iterations 300 each, one persistent launch",
                         "roofline": {"bound": "fp32", "kernel": "cp_plan_kernel (batch, every resident team)",
                                      "achieved": bach, "peak": line["roofline"]["peak"], "unit": "TFLOP/s",
                                      "frac": bach / line["roofline"]["peak"], "kernel_ms": best_kms,
                                      "work": "stage1 x 1240 (m=1) + cc_fk x 1195 + checks x 11 + nn_nodes x 20 flop"}}
    return out


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


def other_configs(args, local):
    """Median device planning time + success for configs[0], [2], [3] (a few
    queries each, three seeds per query), with the CPU reference beside it."""
    import fixtures as fx
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
    res = {}
    for name in ("configs[0]", "configs[2]:shelf_x11", "configs[2]:shelf_x111", "configs[3]"):
        label, probs = _cfg_problems(name)
        times, solved, total = [], 0, 0
        # configs[2] ablations: early-exit flag on/off x broad phase (auto: on
        # from 32 primitives) / the reference's lockstep check order
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
                    total += 1
                    if r.solved:
                        solved += 1
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
        if not args.no_cpu:
            cpu = []
            ok = 0
            for (m, sc, sp, s, g, kw) in probs[: max(2, min(5, len(probs)))]:
                r = _cpu_generic(m, sc, sp, s, g, kw, budget=args.cpu_budget_ms)
                ok += r[0]
                if r[0]:
                    cpu.append(r[1])
            res[name]["cpu_reference_median_ms"] = float(np.median(cpu)) if cpu else None
            res[name]["cpu_reference_success"] = f"{ok}/{max(2, min(5, len(probs)))} (1 core, budget {args.cpu_budget_ms:.0f} ms)"
    return res


def _cpu_generic(model, scene, spec, s, g, kw, budget):
    from oracle import oracle as orc
    t0 = time.perf_counter()
    r = orc.plan(model.packed, scene.packed(), None if spec is None else spec.packed, s, g,
                 max_iterations=10**6, time_budget_ms=budget, **kw)
    return r["status"] == "Solved", (time.perf_counter() - t0) * 1e3


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
# CPU reference (oracle/_ref compiled maniplan, else the C oracle port)
# ---------------------------------------------------------------------------

def _ref_available():
    return os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "maniplan"))


def _cpu_job(job):
    """One reference plan() in a worker process; returns (solved, wall_ms)."""
    k, seed, budget = job
    model, scene, spec, starts, goals = workload()
    if _ref_available():
        os.environ["MANIPLAN_KERNELS"] = "compiled"
        sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
        import maniplan as M
        from maniplan.constraints import ConstraintSpec, PlaneConstraint
        from maniplan.geometry import Aabb, Scene
        from maniplan.kinematics import Joint, LinkSphere, RobotModel
        key = "_ref_objs"
        objs = globals().get(key)
        if objs is None:
            rm = RobotModel(joints=tuple(Joint(j.jtype, j.axis, j.origin_xyz, j.origin_rpy, j.lo, j.hi, j.name)
                                         for j in model.joints),
                            link_spheres=tuple(LinkSphere(s.link, s.center, s.radius) for s in model.link_spheres),
                            ee_link=model.ee_link, self_collision_pairs=model.self_collision_pairs)
            from maniplan.geometry import Sphere as RS
            rs = Scene(boxes=tuple(Aabb(b.min, b.max) for b in scene.boxes),
                       spheres=tuple(RS(s.center, s.radius) for s in scene.spheres))
            rsp = ConstraintSpec(PlaneConstraint(spec.position.normal, spec.position.offset),
                                 fixed_orientation=spec.fixed_orientation,
                                 angular_weight=spec.angular_weight, tau_task=spec.tau_task)
            objs = globals()[key] = (rm, rs, rsp)
        rm, rs, rsp = objs
        prob = M.PlanProblem(rm, rs, rsp, starts[k], goals[k],
                             M.PlanParams(width=16, max_iterations=10**6, time_budget_ms=budget,
                                          seed_offset=seed))
        t0 = time.perf_counter()
        r = M.plan(prob)
        return r.solved, (time.perf_counter() - t0) * 1e3
    from oracle import oracle as orc
    t0 = time.perf_counter()
    r = orc.plan(model.packed, scene.packed(), spec.packed, starts[k], goals[k], width=16,
                 max_iterations=10**6, time_budget_ms=budget, seed_offset=seed)
    return r["status"] == "Solved", (time.perf_counter() - t0) * 1e3


def cpu_baseline(args):
    """Bounded CPU sample on one host core (rank 0, N=1)."""
    n = args.cpu_queries
    jobs = [(k % N_PAIRS, k * 10_000, args.cpu_budget_ms) for k in range(n)]
    t0 = time.perf_counter()
    res = [_cpu_job(j) for j in jobs]
    el = time.perf_counter() - t0
    solved = [w for ok, w in res if ok]
    import fixtures as fx
    feas = fx.upright_feasible()
    nf = sum(bool(feas[j[0]]) for j in jobs)
    sf = sum(ok for (ok, _), j in zip(res, jobs) if feas[j[0]])
    return {"value": float(np.median(solved)) if solved else None, "unit": "ms",
            "success_rate": len(solved) / n, "success_rate_feasible": sf / max(1, nf), "cores": 1,
            "kind": "reference" if _ref_available() else "port",
            "sample": f"{n} of the same upright-table queries, one core, time budget "
                      f"{args.cpu_budget_ms:.0f} ms each ({el:.1f} s total)"}


def run_reference(args, world, rank):
    if rank != 0:
        return None
    from concurrent.futures import ProcessPoolExecutor
    cores = os.cpu_count() or 1
    Q = args.queries
    steps = []
    all_res = []
    with ProcessPoolExecutor(max_workers=cores) as ex:
        list(ex.map(_cpu_job, [(0, 0, 100.0)] * cores))
        for s in range(args.warmup + args.steps):
            jobs = [((s * Q + j) % N_PAIRS, (s * 7919 + (s * Q + j) % N_PAIRS) * 10_000, args.cpu_budget_ms)
                    for j in range(Q)]
            t0 = time.perf_counter()
            res = list(ex.map(_cpu_job, jobs))
            if s >= args.warmup:
                steps.append((time.perf_counter() - t0) * 1e3)
                all_res += res
    solved = [w for ok, w in all_res if ok]
    med = float(np.median(solved)) if solved else None
    kind = "reference" if _ref_available() else "port"
    return {"metric": METRIC, "value": med, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.mean(steps)), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "same synthetic queries",
            "config": {"workload": "configs[1] constrained Panda (arm7, table, upright EE, W=16)",
                       "queries_per_step": Q, "time_budget_ms": args.cpu_budget_ms},
            "impl": "reference", "success_rate": len(solved) / max(1, len(all_res)),
            "cpu_baseline": {"value": med, "unit": "ms", "cores": cores, "kind": kind,
                             "sample": f"{len(all_res)} queries, one process per core, "
                                       f"budget {args.cpu_budget_ms:.0f} ms each"},
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
    ap.add_argument("--cpu-queries", type=int, default=20)
    ap.add_argument("--cpu-budget-ms", type=float, default=2000.0)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        line = run_reference(args, world, rank)
    else:
        line = run_b200(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
