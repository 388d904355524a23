#!/usr/bin/env python
"""bench.py -- throughput of the B200 hot path of tsnnls' block principal
pivoting NNLS solver (BASELINE.json metric: NNLS solves/s and pivot
iterations/s, FP64; fraction of the FP64-tensor / HBM roofline).

One step = one pass of the whole hot path over
one synthetic problem already resident in HBM: ingest (validation, CSC), Gram
A^T A and A^T b, the pivot loop (decide/exchange, gather+Cholesky+solves,
dual update, zeroing), the final LSQR and the KKT report, x left in HBM.

Default workload (N = 1): BASELINE.json configs[1], a single 2000 x 1000 CSR
problem with 5% N(0,1) nonzeros (quantized to 2^-12), b = A x0 + 0.01 noise.
Under torchrun (N > 1) every rank solves its own independent problem (seed +
rank): the single-problem path does not shard ("replicas", weak scaling).
--config 4 runs the batched config (65536 problems of 128 x 64; problems
sharded over ranks, no communication).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
only reference this paper-derived build has) on the host cores, rank 0 only.
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
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "NNLS solves/s and pivot iterations/s (FP64); % of FP64-TC / HBM roofline"
L2_FLUSH_BYTES = 256 << 20
HBM_FALLBACK_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--batch", type=int, default=65536, help="config 4: total problems (all ranks)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard-gram", action="store_true",
                    help="single problem: row-shard A^T A over the ranks + one NCCL all-reduce "
                         "(strong scaling) instead of one independent problem per rank")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_desc(cfg, batch=None):
    import nnls_gen as g
    c = g.CONFIGS[cfg]
    if cfg == 4:
        return (f"config4: {batch} independent NNLS, each {c['m']}x{c['n']} CSR {c['density']:.0%} "
                "N(0,1) (2^-12 grid), b = A x0 + 0.01 N(0,1)")
    rhs = "b = A x* (x* 40% zeros)" if c["rhs"] == "degenerate" else "b = A x0 + 0.01 N(0,1)"
    return (f"config{cfg}: single NNLS {c['m']}x{c['n']} CSR {c['density']:.1%} N(0,1) "
            f"(2^-12 grid), {rhs}")


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle reasons
    during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index, period=0.02):
        self.period = period
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hdl, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hdl, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self.t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"
    if os.path.exists(path):
        try:
            hbm = float(json.load(open(path))["hbm_gbs"])
            src = "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            pass
    fp64, fsrc = 37.139, "profiles/r01_microbench_fp64.json dmma_tflops (measured, this pool)"
    mb = os.path.join(ROOT, "profiles", "r01_microbench_fp64.json")
    if os.path.exists(mb):
        try:
            fp64 = float(json.load(open(mb))["dmma_tflops"])
        except Exception:
            pass
    return hbm, src, fp64, fsrc


def load_traffic():
    """DRAM bytes per launch from committed `ncu --set full` captures, keyed by
    config then phase (profiles/ncu_traffic.json); absent -> null."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except Exception:
            return {}
    return {}


# ------------------------------------------------- algorithmic work models
# (DESIGN.md §"Roofline": bytes a step must move / flops it must do; avoided
#  dense work is not counted)
def phase_work(phase, prob, traces, lsqr_itns, nnzF_list):
    m, n, nnz = prob.m, prob.n, prob.nnz
    if phase == "gram":       # read CSR+CSC+b, write full G (n*n) and c
        return "hbm", float(2 * 12 * nnz + 4 * (m + n) + 8 * m + 8 * n * n + 8 * n)
    if phase == "chol_factor":
        fl = 0.0
        for tr in traces:
            for t in tr:
                f = t["f"]
                fl += f ** 3 / 3.0 + f * f  # Cholesky f^3/3 + bordered forward row
        return "tensor", fl
    if phase == "chol_solve":
        return "hbm", float(sum(8 * t["f"] * (t["f"] + 1) / 2 for tr in traces for t in tr))
    if phase == "dual":
        return "hbm", float(sum(8 * t["f"] * (n - t["f"]) + 8 * (t["f"] + 2 * n) for tr in traces for t in tr))
    if phase == "decide":
        return "hbm", float(sum((len(tr) + 1) * (n * 17 + 8 * n) for tr in traces))
    if phase == "lsqr":
        by = 0.0
        for itn, nzf, tr in zip(lsqr_itns, nnzF_list, traces):
            f = tr[-1]["f"] if tr else 0
            by += itn * (2 * 12 * nzf + 8 * (3 * m + 6 * f)) + 2 * 12 * nnz + 8 * (2 * m + 2 * n)
        return "hbm", by
    if phase in ("validate", "csc"):
        return "hbm", float(len(traces) * (12 * nnz + 4 * m) * (1 if phase == "validate" else 3))
    return "hbm", 0.0


# ----------------------------------------------------------------- ours
def run_ours(args):
    import torch

    import nnls_gen as g
    import paper_cs_0408029_b200 as P

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    hbm_gbs, hbm_src, fp64_tf, fp64_src = load_peaks()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    cfg = args.config
    batched = cfg == 4
    if batched:
        per = args.batch // world
        start = rank * per
        B = g.make_batch(seed=args.seed, start=start, count=per)
        host = dict(nnz_off=B.nnz_off, rowptr=B.rowptr, colind=B.colind, vals=B.vals, b=B.b)
        solver = P.BatchedSolver(stream=stream)
        units_per_step = per
    elif args.shard_gram:
        from paper_cs_0408029_b200.dist import allreduce_gram, row_shards
        prob = g.make_problem(cfg, seed=args.seed)          # the same problem on every rank
        host = dict(rowptr=prob.rowptr, colind=prob.colind, vals=prob.vals, b=prob.b)
        r0, r1 = row_shards(prob.m, world)[rank]
        solver = P.ShardSolver(prob.m, prob.n, prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1,
                               stream=stream, trace=1)
        units_per_step = 1
    else:
        prob = g.make_problem(cfg, seed=args.seed + rank)
        host = dict(rowptr=prob.rowptr, colind=prob.colind, vals=prob.vals, b=prob.b)
        solver = P.Solver(stream=stream, trace=1)
        units_per_step = 1
    devt = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in host.items()}
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in host.items()}
    nx = (B.count * B.n) if batched else prob.n
    x_dev = torch.empty(nx, dtype=torch.float64, device=dev)
    x_pin = torch.empty(nx, dtype=torch.float64).pin_memory()

    def step(inputs, x_out):
        if args.shard_gram and not batched:
            solver.load_shard(prob.m, prob.n, inputs["rowptr"], inputs["colind"], inputs["vals"], inputs["b"],
                              r0, r1)
            if world > 1:
                allreduce_gram(solver)
            else:
                solver.finalize()
            _, info = solver.solve(x_out=x_out)
            return info
        if batched:
            if not inputs["b"].is_cuda:
                # host buffers: the pipelined load + solve (chunk k+1 copies in
                # and chunk k-1 copies out while chunk k solves)
                solver.run(B.count, B.m, B.n, inputs["nnz_off"], inputs["rowptr"], inputs["colind"],
                           inputs["vals"], inputs["b"], x_out=x_out, want_info=False)
                return None
            solver.load(B.count, B.m, B.n, inputs["nnz_off"], inputs["rowptr"], inputs["colind"],
                        inputs["vals"], inputs["b"])
            solver.solve(x_out=x_out, want_info=False)
            return None
        solver.load(prob.m, prob.n, inputs["rowptr"], inputs["colind"], inputs["vals"], inputs["b"])
        _, info = solver.solve(x_out=x_out)
        return info

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]

    def timed_pass(inputs, x_out, collect):
        infos, traces = [], []
        total_ms = 0.0
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()                      # evict L2 (256 MiB > 126 MB L2) between steps
            e0, e1 = ev[k]
            e0.record(stream)
            info = step(inputs, x_out)
            e1.record(stream)
            if collect and not batched:
                infos.append(info)
                traces.append(solver.trace())
        torch.cuda.synchronize(dev)
        for e0, e1 in ev:
            total_ms += e0.elapsed_time(e1)
        return total_ms, infos, traces

    # warm-up
    for _ in range(args.warmup):
        step(devt, x_dev)
    torch.cuda.synchronize(dev)

    # ---- device-resident timed pass (value): the production path (the pivot
    #      loop runs inside one CUDA graph with a device-side WHILE node)
    P.timing_enable(solver.h, False)  # resets the launch counters
    barrier()
    with ClockSampler(local) as clk:
        total_ms, infos, traces = timed_pass(devt, x_dev, collect=True)
    barrier()
    launches_timed = P.timing_read(solver.h)
    t_max = total_ms
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    # ---- instrumented pass (same K steps): per-phase CUDA events on the
    #      library's stream (host-driven pivot loop, so each kernel is bracketed)
    P.timing_enable(solver.h, True)
    barrier()
    instr_ms, _, _ = timed_pass(devt, x_dev, collect=False)
    barrier()
    phases = P.timing_read(solver.h)
    P.timing_enable(solver.h, False)

    # ---- end-to-end pass through the public API with HOST buffers (value e2e)
    e2e_ms = None
    if not args.no_e2e:
        for _ in range(2):
            step(pinned, x_pin)
        barrier()
        e2e_ms, _, _ = timed_pass(pinned, x_pin, collect=False)
        barrier()
        if dist is not None:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())

    shard = args.shard_gram and not batched
    units = units_per_step * args.steps * (1 if shard else world)
    value = units / (t_max / 1e3)
    out = {"metric": METRIC, "value": round(value, 3), "unit": "solves/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 5),
           "higher_is_better": True, "scaling": "strong" if shard else "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)", "impl": "ours"}
    if not batched:
        iters = sum(i["iterations"] for i in infos) * (1 if shard else world)
        out["pivot_iterations_per_s"] = round(iters / (t_max / 1e3), 3)
        out["per_solve"] = {"iterations": infos[0]["iterations"], "free_count": infos[0]["free_count"],
                            "lsqr_iterations": infos[0]["lsqr_iterations"], "status": infos[0]["status"]}
    out["config"] = {"workload": workload_desc(cfg, args.batch), "config_index": cfg,
                     "seed": args.seed, "l2": "flushed between timed steps (256 MiB write, outside events)",
                     "parallelism": ("problems sharded over ranks, no communication" if batched
                                     else ("A^T A row-sharded over ranks + NCCL all-reduce of [G|c]"
                                           if shard else "replicas: one independent problem per GPU"))}
    if batched:
        out["config"].update(m=B.m, n=B.n, problems_per_gpu=B.count)
    else:
        out["config"].update(m=prob.m, n=prob.n, nnz=prob.nnz)

    # ---- phases, dominant kernel, roofline
    kernel_phases = ["validate", "csc", "gram", "init", "decide", "chol_factor", "chol_solve", "dual",
                     "lsqr", "batched"]
    out["gpu_launches"] = int(sum(launches_timed[p][1] for p in kernel_phases))
    out["phase_timing"] = {"pass": "instrumented (host-driven loop, CUDA events per phase)",
                           "ms_per_step": round(instr_ms / args.steps, 5)}
    out["phase_ms_per_step"] = {p: round(phases[p][0] / args.steps, 5) for p in P.PHASES if phases[p][1] or phases[p][0]}
    dom = max(kernel_phases, key=lambda p: phases[p][0])
    traffic = load_traffic()
    if batched:
        # per problem: CSR + b in, x + info out (G, factor, vectors stay on chip)
        nzp = int(B.nnz_off[1] - B.nnz_off[0])
        bytes_per = 12 * nzp + 4 * (B.m + 1) + 8 * B.m + 8 * B.n + B.n + 8 * 8 + 5 * 8
        bound, work = "hbm", float(bytes_per * B.count * args.steps)
    else:
        nnzF = []
        rp = prob.rowptr
        for _ in infos:
            mask = solver.free_set()
            nnzF.append(int(mask[prob.colind].sum()))
        bound, work = phase_work(dom, prob, traces, [i["lsqr_iterations"] for i in infos], nnzF)
    dom_s = phases[dom][0] / 1e3
    if bound == "tensor":
        achieved = work / dom_s / 1e12
        peak, unit, psrc = fp64_tf, "TFLOP/s", fp64_src
    else:
        achieved = work / dom_s / 1e9
        peak, unit, psrc = hbm_gbs, "GB/s", hbm_src
    launches = max(1, phases[dom][1])
    out["roofline"] = {"kernel": dom, "bound": bound, "achieved": round(achieved, 4), "peak": peak,
                       "unit": unit, "frac": round(achieved / peak, 6), "peak_source": psrc,
                       "algorithmic_per_launch": work / launches,
                       "avg_launch_ms": round(phases[dom][0] / launches, 5),
                       "share_of_step": round(phases[dom][0] / max(instr_ms, 1e-9), 4),
                       "traffic": traffic.get("config%d" % args.config, {}).get(dom, {}).get("dram_bytes_per_launch")}
    if e2e_ms is not None:
        h2d = sum(int(v.nbytes) for v in host.values())
        out["e2e"] = {"value": round(units / (e2e_ms / 1e3), 3), "unit": "solves/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(nx * 8),
                      "path": ("BatchedSolver.run(pinned host CSR,b; x_out=pinned host): chunked copy/compute pipeline"
                               if batched else "Solver.load(pinned host CSR,b) + Solver.solve(x_out=pinned host)")}
    out["clocks"] = clk.summary()

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, budget=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------ oracle (CPU)
def cpu_baseline(args, cfg, budget):
    import nnls_gen as g
    import oracle as O
    if cfg == 4:
        count = 2048
        B = g.make_batch(seed=args.seed, start=0, count=count)
        t0 = time.perf_counter()
        out = O.solve_batched(B, threads=0)
        dt = time.perf_counter() - t0
        return {"value": round(count / dt, 3), "unit": "solves/s", "cores": out["threads"],
                "kind": "oracle", "sample": f"{count} config-4 problems (OpenMP over problems)",
                "seconds": round(dt, 3)}
    prob = g.make_problem(cfg, seed=args.seed)
    done, t0 = 0, time.perf_counter()
    iters = 0
    while True:
        r = O.solve(prob)
        done += 1
        iters += r["iterations"]
        if time.perf_counter() - t0 > budget or done >= 1000:
            break
    dt = time.perf_counter() - t0
    return {"value": round(done / dt, 4), "unit": "solves/s", "cores": 1, "kind": "oracle",
            "sample": f"{done} full oracle solves of the config-{cfg} problem (single thread)",
            "pivot_iterations_per_s": round(iters / dt, 4), "seconds": round(dt, 3)}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import nnls_gen as g
    import oracle as O
    cfg = args.config
    if cfg == 4:
        count = 1024
        B = g.make_batch(seed=args.seed, start=0, count=count)
        for _ in range(args.warmup):
            O.solve_batched(B, threads=0)
        t0 = time.perf_counter()
        threads = 1
        for _ in range(args.steps):
            threads = O.solve_batched(B, threads=0)["threads"]
        dt = time.perf_counter() - t0
        value = count * args.steps / dt
        sample = f"{count} config-4 problems per step (OpenMP over problems)"
        cores = threads
    else:
        prob = g.make_problem(cfg, seed=args.seed)
        for _ in range(args.warmup):
            O.solve(prob)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            O.solve(prob)
        dt = time.perf_counter() - t0
        value = args.steps / dt
        sample = f"one full oracle solve of the config-{cfg} problem per step (single thread)"
        cores = 1
    out = {"metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE config shapes)", "impl": "reference",
           "config": {"workload": workload_desc(cfg, args.batch), "config_index": cfg, "seed": args.seed},
           "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
