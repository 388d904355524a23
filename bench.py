#!/usr/bin/env python
"""bench.py -- throughput of the B200 hot path of tsnnls' block principal
pivoting NNLS solver (BASELINE.json metric: NNLS solves/s and pivot
iterations/s, FP64; fraction of the FP64-tensor / HBM roofline).

One step = one pass of the whole hot path over
one synthetic problem already resident in HBM: ingest (validation, CSC), Gram
A^T A and A^T b, the pivot loop (decide/exchange, gather+Cholesky+solves,
dual update, zeroing), the final LSQR and the KKT report, x left in HBM.

Default workload: BASELINE.json configs[2], the largest single-GPU
configuration -- one 40000 x 8000 CSR problem with 0.5% N(0,1) nonzeros
(quantized to 2^-12), b = A x0 + 0.01 noise; the Cholesky of |F| ~ 4000 and
the HBM kernels carry §8(d)'s targets there.  The same line carries configs
1, 3 and 4 (the batched 65536 x (128x64) config) under "other_configs".

Multi-GPU (`--gpus N`, re-launched through torchrun when WORLD_SIZE is
unset): config 2 forms A^T A row-sharded over the ranks (each rank uploads
only its row block; the packed partial Grams are reduced to rank 0 with one
NCCL reduce; rank 0 runs the pivot loop: strong scaling), and the config-4
batch is sharded over the ranks with no communication ("config4_sharded").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
only reference this paper-derived build has) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "NNLS solves/s and pivot iterations/s (FP64); % of FP64-TC / HBM roofline"
L2_FLUSH_BYTES = 256 << 20
HBM_FALLBACK_GBS = 6650.0
REF_BUDGET_S = 150.0   # reference arm: timed oracle work per run (a bounded sample)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--batch", type=int, default=65536, help="config 4: total problems (all ranks)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs / alternatives")
    ap.add_argument("--reduce", choices=["reduce", "allreduce"], default="reduce",
                    help="N>1 config 2: collective for the packed partial Grams")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_torchrun(args):
    """--gpus N > 1 without a torchrun environment: start N ranks here."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def workload_desc(cfg, batch=None):
    import nnls_gen as g
    c = g.CONFIGS[cfg]
    if cfg == 4:
        return (f"config4: {batch} independent NNLS, each {c['m']}x{c['n']} CSR {c['density']:.0%} "
                "N(0,1) (2^-12 grid), b = A x0 + 0.01 N(0,1)")
    rhs = "b = A x* (x* 40% zeros)" if c["rhs"] == "degenerate" else "b = A x0 + 0.01 N(0,1)"
    return (f"config{cfg}: single NNLS {c['m']}x{c['n']} CSR {c['density']:.1%} N(0,1) "
            f"(2^-12 grid), {rhs}")


def config_dict(cfg, args, world):
    """The `config` object -- identical in both arms (--impl ours / reference)."""
    import nnls_gen as g
    c = g.CONFIGS[cfg]
    d = {"workload": workload_desc(cfg, args.batch), "config_index": cfg, "seed": args.seed,
         "m": c["m"], "n": c["n"], "density": c["density"],
         "l2": "flushed between timed steps (256 MiB write, outside the events)"}
    if cfg == 4:
        d.update(problems=args.batch, parallelism="problems sharded over ranks, no communication")
    elif world > 1 and cfg == 2:
        d["parallelism"] = (f"A^T A row-sharded over {world} ranks (packed partial Grams, NCCL {args.reduce} "
                            "to rank 0); pivot loop on rank 0")
    elif world > 1:
        d["parallelism"] = "replicas: one independent problem per GPU"
    else:
        d["parallelism"] = "one GPU"
    return d


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle reasons
    during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index, period=0.01):
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
    fp64, fsrc = 37.139, "profiles/r01_microbench_fp64.json dmma_tflops (DMMA 8x8x4 peak measured on this pool)"
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
# (bytes a step must move / flops it must do)
def chol_flops(f, q=0):
    """Executed Cholesky flops of the bordered (f+1) x (f+1) factorization when
    the leading q columns of the previous factor are reused: the left-looking
    column j costs 2 j (f - j) flops, of which the kept columns only redo the
    rows below q, 2 j (f - q): sum = (f^3 - q^3)/3; plus the bordered
    (forward-substitution) row, f^2 - q^2.  q = 0: the method's f^3/3 + f^2."""
    return (f ** 3 - q ** 3) / 3.0 + (f * f - q * q)


def phase_work(phase, prob, traces, lsqr_itns, nnzF_list):
    m, n, nnz = prob.m, prob.n, prob.nnz
    if phase == "gram":       # read CSR+CSC+b, write full G (n*n) and c; once per solve
        return "hbm", float(len(traces) * (2 * 12 * nnz + 4 * (m + n) + 8 * m + 8 * n * n + 8 * n))
    if phase == "chol_factor":
        return "tensor", float(sum(chol_flops(t["f"], t.get("kept", 0)) for tr in traces for t in tr))
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


KERNEL_PHASES = ["validate", "csc", "gram", "init", "decide", "chol_factor", "chol_solve", "dual", "lsqr",
                 "batched"]


# ----------------------------------------------------------------- ours
class Ctx:
    def __init__(self, args):
        import torch
        self.torch = torch
        self.args = args
        self.world, self.rank, self.local = dist_env()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=self.dev)
        self.peaks = load_peaks()

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v):
        if self.dist is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, step, steps, inputs, x_out, after=None):
        """K steps, each bracketed by CUDA events on the library's stream, L2
        flushed before each (outside the events).  Returns total device ms."""
        torch = self.torch
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            with torch.cuda.stream(self.stream):
                self.flush.zero_()
            ev[k][0].record(self.stream)
            step(inputs, x_out)
            ev[k][1].record(self.stream)
            if after is not None:
                after()
        torch.cuda.synchronize(self.dev)
        return sum(a.elapsed_time(b) for a, b in ev)


def measure_single(C, cfg, steps, warmup, shard=False, with_e2e=True, full_fact=True, trace=True, raw=False,
                   **solver_kw):
    """Single problem (configs 0-3).  shard (N > 1, config 2): row-sharded Gram
    + reduce to rank 0, the loop on rank 0."""
    import nnls_gen as g
    import paper_cs_0408029_b200 as P
    torch, args = C.torch, C.args
    world, rank = C.world, C.rank
    prob = g.make_problem(cfg, seed=args.seed + (0 if shard else rank), raw=raw)
    host = dict(rowptr=prob.rowptr, colind=prob.colind, vals=prob.vals, b=prob.b)
    if shard:
        from paper_cs_0408029_b200.dist import reduce_gram, row_block, row_shards
        r0, r1 = row_shards(prob.m, world)[rank]
        if rank == 0:
            solver = P.ShardSolver(prob.m, prob.n, prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1,
                                   stream=C.stream, trace=1)
        else:  # only this rank's row block travels to its GPU
            rp, ci, v, bb = row_block(prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
            host = dict(rowptr=rp, colind=ci, vals=v, b=bb)
            solver = P.BlockSolver(stream=C.stream).load_block(r1 - r0, prob.n, rp, ci, v, bb)
    else:
        solver = P.Solver(stream=C.stream, trace=1 if trace else 0, **solver_kw)
    devt = {k: torch.from_numpy(np.ascontiguousarray(v)).to(C.dev) for k, v in host.items()}
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in host.items()}
    x_dev = torch.empty(prob.n, dtype=torch.float64, device=C.dev)
    x_pin = torch.empty(prob.n, dtype=torch.float64).pin_memory()
    infos = []
    mode = [args.reduce]

    def step(inp, x_out):
        if shard:
            if rank == 0:
                solver.load_shard(prob.m, prob.n, inp["rowptr"], inp["colind"], inp["vals"], inp["b"], r0, r1)
            else:
                solver.load_block(r1 - r0, prob.n, inp["rowptr"], inp["colind"], inp["vals"], inp["b"])
            reduce_gram(solver, mode[0], 0, stream=C.stream)
            if rank == 0:
                infos.append(solver.solve(x_out=x_out)[1])
            return
        solver.load(prob.m, prob.n, inp["rowptr"], inp["colind"], inp["vals"], inp["b"])
        infos.append(solver.solve(x_out=x_out)[1])

    for _ in range(warmup):
        step(devt, x_dev)
    torch.cuda.synchronize(C.dev)
    # ---- value pass: the production path (pivot loop inside one CUDA graph)
    P.timing_enable(solver.h, False)  # resets the launch counters
    infos.clear()
    C.barrier()
    with ClockSampler(C.local) as clk:
        total = C.timed(step, steps, devt, x_dev)
    C.barrier()
    launches = P.timing_read(solver.h)
    t_max = C.max_over_ranks(total)
    res = {"ms_per_step": t_max / steps, "value": steps / (t_max / 1e3), "clocks": clk.summary(),
           "gpu_launches": int(sum(launches[p][1] for p in KERNEL_PHASES))}
    if shard and world > 1 and not args.no_extra:
        other = "allreduce" if args.reduce == "reduce" else "reduce"
        mode[0] = other
        C.barrier()
        alt = C.max_over_ranks(C.timed(step, steps, devt, x_dev))
        mode[0] = args.reduce
        res["alternative_collective"] = {"collective": other, "ms_per_step": round(alt / steps, 5),
                                         "value": round(steps / (alt / 1e3), 3)}
    if rank == 0:
        info = infos[0]
        trace = solver.trace()
        res["pivot_iterations_per_s"] = info["iterations"] * steps / (t_max / 1e3)
        res["per_solve"] = {k: info[k] for k in ("iterations", "free_count", "lsqr_iterations", "status",
                                                 "single_exchanges", "kappa", "refined")}
        res["per_solve"]["trace"] = [{"k": t["k"], "branch": t["branch"], "f": t["f"], "kept": t["kept"]}
                                     for t in trace]
    # ---- instrumented pass: per-phase CUDA events (host-driven pivot loop)
    P.timing_enable(solver.h, True)
    C.barrier()
    instr = C.timed(step, steps, devt, x_dev)
    C.barrier()
    phases = P.timing_read(solver.h)
    P.timing_enable(solver.h, False)
    res["phase_timing"] = {"pass": "instrumented (host-driven loop, CUDA events per phase)",
                           "ms_per_step": round(instr / steps, 5)}
    res["phase_ms_per_step"] = {p: round(phases[p][0] / steps, 5) for p in P.PHASES
                                if phases[p][1] or phases[p][0]}
    if rank == 0:
        hbm, hsrc, fp64, fsrc = C.peaks
        dom = max(KERNEL_PHASES, key=lambda p: phases[p][0])
        mask = solver.free_set()
        nnzF = int(mask[prob.colind].sum())
        traces = [trace] * steps
        bound, work = phase_work(dom, prob, traces, [info["lsqr_iterations"]] * steps, [nnzF] * steps)
        nl = max(1, phases[dom][1])
        dom_s = phases[dom][0] / 1e3
        tensor = bound == "tensor"
        achieved = work / dom_s / (1e12 if tensor else 1e9)
        peak = fp64 if tensor else hbm
        res["roofline"] = {
            "kernel": dom, "bound": bound, "achieved": round(achieved, 4), "peak": peak,
            "unit": "TFLOP/s" if tensor else "GB/s", "frac": round(achieved / peak, 6),
            "peak_source": fsrc if tensor else hsrc,
            "algorithmic_per_launch": work / nl, "avg_launch_ms": round(phases[dom][0] / nl, 5),
            "launches_per_step": nl / steps, "share_of_step": round(phases[dom][0] / max(instr, 1e-9), 4),
            "traffic": load_traffic().get("config%d" % cfg, {}).get(dom, {}).get("dram_bytes_per_launch"),
            "work_model": ("executed Cholesky flops: sum over launches of (f^3 - q^3)/3 + f^2 - q^2, q = factor "
                           "prefix reused from the previous pivot iteration (trace 'kept')" if tensor else
                           "algorithmic bytes (DESIGN.md §8)")}
        # every kernel's rate against its own roofline (DESIGN.md §8 work models)
        per = {}
        for p in ("gram", "chol_factor", "chol_solve", "dual", "lsqr", "decide"):
            if not phases[p][1]:
                continue
            b, w = phase_work(p, prob, traces, [info["lsqr_iterations"]] * steps, [nnzF] * steps)
            s = phases[p][0] / 1e3
            a = w / s / (1e12 if b == "tensor" else 1e9)
            per[p] = {"bound": b, "achieved": round(a, 3), "frac": round(a / (fp64 if b == "tensor" else hbm), 4),
                      "avg_launch_ms": round(phases[p][0] / phases[p][1], 5)}
        res["kernel_rooflines"] = per
    # ---- full factorizations (no prefix reuse): the FP64-TC target of §8(d)
    if rank == 0 and full_fact and not shard:
        os.environ["NNLS_NO_REUSE"] = "1"
        try:
            s2 = P.Solver(stream=C.stream, trace=1)
        finally:
            del os.environ["NNLS_NO_REUSE"]
        s2.load(prob.m, prob.n, devt["rowptr"], devt["colind"], devt["vals"], devt["b"])
        s2.solve(x_out=x_dev)
        P.timing_enable(s2.h, True)
        nrep = max(2, min(steps, 5))
        for _ in range(nrep):
            with torch.cuda.stream(C.stream):
                C.flush.zero_()
            s2.solve(x_out=x_dev)
        torch.cuda.synchronize(C.dev)
        ph2 = P.timing_read(s2.h)
        tr2 = s2.trace()
        fl = sum(chol_flops(t["f"]) for t in tr2) * nrep
        ms = ph2["chol_factor"][0]
        fp64 = C.peaks[2]
        res["full_factorization"] = {
            "f": [t["f"] for t in tr2], "launches": ph2["chol_factor"][1],
            "avg_launch_ms": round(ms / max(1, ph2["chol_factor"][1]), 5),
            "tflops": round(fl / (ms / 1e3) / 1e12, 4), "frac": round(fl / (ms / 1e3) / 1e12 / fp64, 4),
            "note": "NNLS_NO_REUSE handle: every pivot iteration factors (A^T A)_FF from scratch; "
                    "flops f^3/3 + f^2 per launch"}
        s2.close()
    # ---- end-to-end through the public API with HOST buffers
    if with_e2e:
        for _ in range(2):
            step(pinned, x_pin)
        C.barrier()
        e2e = C.max_over_ranks(C.timed(step, steps, pinned, x_pin))
        h2d = sum(int(v.nbytes) for v in host.values())
        res["e2e"] = {"value": round(steps / (e2e / 1e3), 3), "unit": "solves/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": int(prob.n * 8) if rank == 0 else 0,
                      "path": "Solver.load(pinned host CSR, b) + Solver.solve(x_out=pinned host)"}
    res["_prob"] = prob
    solver.close()
    return res


def measure_batched(C, steps, warmup, with_e2e=True):
    import nnls_gen as g
    import paper_cs_0408029_b200 as P
    from paper_cs_0408029_b200.dist import batch_shard
    torch, args = C.torch, C.args
    start, per = batch_shard(args.batch, C.world, C.rank)
    B = g.make_batch(seed=args.seed, start=start, count=per)
    host = dict(nnz_off=B.nnz_off, rowptr=B.rowptr, colind=B.colind, vals=B.vals, b=B.b)
    solver = P.BatchedSolver(stream=C.stream)
    devt = {k: torch.from_numpy(np.ascontiguousarray(v)).to(C.dev) for k, v in host.items()}
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in host.items()}
    x_dev = torch.empty(B.count * B.n, dtype=torch.float64, device=C.dev)
    x_pin = torch.empty(B.count * B.n, dtype=torch.float64).pin_memory()

    def step(inp, x_out):
        if not inp["b"].is_cuda:  # host buffers: the pipelined load + solve
            solver.run(B.count, B.m, B.n, inp["nnz_off"], inp["rowptr"], inp["colind"], inp["vals"], inp["b"],
                       x_out=x_out, want_info=False)
            return
        solver.load(B.count, B.m, B.n, inp["nnz_off"], inp["rowptr"], inp["colind"], inp["vals"], inp["b"])
        solver.solve(x_out=x_out, want_info=False)

    for _ in range(warmup):
        step(devt, x_dev)
    torch.cuda.synchronize(C.dev)
    P.timing_enable(solver.h, False)
    C.barrier()
    with ClockSampler(C.local) as clk:
        total = C.timed(step, steps, devt, x_dev)
    C.barrier()
    launches = P.timing_read(solver.h)
    t_max = C.max_over_ranks(total)
    res = {"ms_per_step": t_max / steps, "value": args.batch * steps / (t_max / 1e3), "clocks": clk.summary(),
           "gpu_launches": int(sum(launches[p][1] for p in KERNEL_PHASES)), "problems_per_gpu": per}
    out = solver.solve(x_out=x_dev, want_info=True)
    its = float(out["info"]["iterations"].sum())
    if C.dist is not None:  # pivot iterations of all ranks' problems
        t = torch.tensor([its], dtype=torch.float64, device=C.dev)
        C.dist.all_reduce(t)
        its = float(t.item())
    res["pivot_iterations_per_s"] = its * steps / (t_max / 1e3)
    P.timing_enable(solver.h, True)
    C.barrier()
    instr = C.timed(step, steps, devt, x_dev)
    C.barrier()
    phases = P.timing_read(solver.h)
    P.timing_enable(solver.h, False)
    res["phase_ms_per_step"] = {p: round(phases[p][0] / steps, 5) for p in P.PHASES if phases[p][1] or phases[p][0]}
    dom = max(KERNEL_PHASES, key=lambda p: phases[p][0])
    nzp = float(B.nnz_off[-1] - B.nnz_off[0]) / B.count
    bytes_per = 12 * nzp + 4 * (B.m + 1) + 8 * B.m + 8 * B.n + B.n + 8 * 8 + 5 * 8
    hbm, hsrc, fp64, fsrc = C.peaks
    nl = max(1, phases[dom][1])
    work = bytes_per * B.count * steps
    achieved = work / (phases[dom][0] / 1e3) / 1e9
    res["roofline"] = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 4), "peak": hbm, "unit": "GB/s",
                       "frac": round(achieved / hbm, 6), "peak_source": hsrc,
                       "algorithmic_per_launch": work / nl, "avg_launch_ms": round(phases[dom][0] / nl, 5),
                       "share_of_step": round(phases[dom][0] / max(instr, 1e-9), 4),
                       "traffic": load_traffic().get("config4", {}).get(dom, {}).get("dram_bytes_per_launch"),
                       "work_model": "per problem: CSR + b in, x + info out (G, factor, vectors stay on chip)"}
    if with_e2e:
        for _ in range(2):
            step(pinned, x_pin)
        C.barrier()
        e2e = C.max_over_ranks(C.timed(step, steps, pinned, x_pin))
        res["e2e"] = {"value": round(args.batch * steps / (e2e / 1e3), 3), "unit": "solves/s",
                      "h2d_bytes_per_step": sum(int(v.nbytes) for v in host.values()),
                      "d2h_bytes_per_step": int(B.count * B.n * 8),
                      "path": "BatchedSolver.run(pinned host CSR, b; x_out=pinned host): chunked copy/compute pipeline"}
    res["_batch"] = B
    solver.close()
    return res


def round_res(r):
    out = {}
    for k, v in r.items():
        if k.startswith("_"):
            continue
        out[k] = round(v, 5) if isinstance(v, float) else v
    return out


def run_ours(args):
    C = Ctx(args)
    world, rank = C.world, C.rank
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    cfg = args.config
    if cfg == 4:
        res = measure_batched(C, args.steps, args.warmup, with_e2e=not args.no_e2e)
        args._batch = res.get("_batch")
    else:
        res = measure_single(C, cfg, args.steps, args.warmup, shard=(world > 1 and cfg == 2),
                             with_e2e=not args.no_e2e)
    shard = world > 1 and cfg == 2
    out = {"metric": METRIC, "value": round(res["value"], 3), "unit": "solves/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 5),
           "higher_is_better": True,
           "scaling": "strong" if (shard or cfg == 4) else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)",
           "impl": "ours", "config": config_dict(cfg, args, world)}
    for k, v in round_res(res).items():
        if k not in ("value", "ms_per_step"):
            out[k] = v
    # ---- the other BASELINE configs (N = 1) / the sharded batch (N > 1)
    if not args.no_extra:
        extra = {}
        if world == 1:
            for c2 in [c for c in (1, 3, 4, 2) if c != cfg]:
                if c2 == 4:
                    r = measure_batched(C, max(3, args.steps // 4), 3, with_e2e=not args.no_e2e)
                else:
                    r = measure_single(C, c2, args.steps, 3, with_e2e=not args.no_e2e, full_fact=False)
                extra[f"config{c2}"] = {k: v for k, v in round_res(r).items()
                                        if k in ("value", "ms_per_step", "pivot_iterations_per_s", "e2e",
                                                 "roofline", "per_solve", "phase_ms_per_step", "problems_per_gpu",
                                                 "full_factorization")}
                extra[f"config{c2}"]["workload"] = workload_desc(c2, args.batch)
                if "per_solve" in extra[f"config{c2}"]:
                    extra[f"config{c2}"]["per_solve"].pop("trace", None)
        if world == 1 and cfg != 4:
            # NEXT-2: the adaptive final step (condition estimate of the final
            # (A^T A)_FF, LSQR only when kappa 2^-52 > 1e-8) on the same problem
            r = measure_single(C, cfg, args.steps, 3, with_e2e=False, full_fact=False, lsqr_mode=3)
            extra["adaptive_lsqr_mode3"] = {k: v for k, v in round_res(r).items()
                                            if k in ("value", "ms_per_step", "phase_ms_per_step", "per_solve")}
            extra["adaptive_lsqr_mode3"]["per_solve"].pop("trace", None)
            extra["adaptive_lsqr_mode3"]["workload"] = workload_desc(cfg, args.batch) + ", lsqr_mode 3"
            # the unquantized variant: A^T A and A^T b are not exact in FP64, so
            # the Gram takes the ordered (oracle summation order) path
            r = measure_single(C, cfg, args.steps, 3, with_e2e=False, full_fact=False, raw=True)
            extra["raw_inputs"] = {k: v for k, v in round_res(r).items()
                                   if k in ("value", "ms_per_step", "phase_ms_per_step", "per_solve",
                                            "kernel_rooflines")}
            extra["raw_inputs"]["per_solve"].pop("trace", None)
            extra["raw_inputs"]["workload"] = (workload_desc(cfg, args.batch).replace("(2^-12 grid)", "(raw)")
                                               + ", unquantized values (ordered Gram path)")
        elif cfg != 4:
            r = measure_batched(C, max(3, args.steps // 4), 3, with_e2e=False)
            extra["config4_sharded"] = {k: v for k, v in round_res(r).items()
                                        if k in ("value", "ms_per_step", "pivot_iterations_per_s", "roofline",
                                                 "problems_per_gpu")}
            extra["config4_sharded"]["workload"] = workload_desc(4, args.batch) + f", {world} ranks"
        out["other_configs"] = extra
    # ---- CPU oracle baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, budget=args.cpu_seconds, batch=getattr(args, "_batch", None))
    if rank == 0:
        print(json.dumps(out), flush=True)
    if C.dist is not None:
        C.dist.barrier()
        C.dist.destroy_process_group()


# ------------------------------------------------------------ oracle (CPU)
def cpu_baseline(args, cfg, budget, batch=None):
    import nnls_gen as g
    import oracle as O
    if cfg == 4:
        # the oracle on 1 core and on all cores, each on a slice of the same
        # batch sized to ~budget/2 seconds of CPU work (a 256-problem probe first)
        B = batch if batch is not None else g.make_batch(seed=args.seed, start=0, count=16384)
        out = {}
        for label, thr in (("1core", 1), ("all", 0)):
            probe = g.make_batch(seed=args.seed, start=0, count=256)
            t1 = time.perf_counter()
            O.solve_batched(probe, threads=thr)
            rate = 256 / (time.perf_counter() - t1)
            cnt = int(min(B.count, max(256, rate * budget / 2)))
            sub = B if cnt == B.count else g.make_batch(seed=args.seed, start=0, count=cnt)
            t1 = time.perf_counter()
            used = O.solve_batched(sub, threads=thr)["threads"]
            dt = time.perf_counter() - t1
            out[label] = (cnt / dt, used, cnt, dt)
        v, used, done, dt = out["all"]
        return {"value": round(v, 3), "unit": "solves/s", "cores": used, "kind": "oracle",
                "sample": f"{done} config-4 problems (OpenMP over problems, {used} threads)",
                "seconds": round(dt, 3), "one_core": {"value": round(out["1core"][0], 3), "cores": 1,
                                                      "sample": f"{out['1core'][2]} problems",
                                                      "seconds": round(out["1core"][3], 3)}}
    prob = g.make_problem(cfg, seed=args.seed)
    done, t0, iters = 0, time.perf_counter(), 0
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
    """The CPU oracle on the host cores, as it stands, on this arm's workload;
    each step is one full solve (config 4: a fixed sample of the batch).  The
    run is bounded: timed steps stop once REF_BUDGET_S of oracle work is spent
    (config 2: one solve is ~25-40 s), so `steps` reports those actually timed."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import nnls_gen as g
    import oracle as O
    cfg = args.config
    if cfg == 4:
        count = 2048
        B = g.make_batch(seed=args.seed, start=0, count=count)
        work = lambda: O.solve_batched(B, threads=0)["threads"]  # noqa: E731
        sample = f"{count} config-4 problems per step (OpenMP over problems)"
        units = count
    else:
        prob = g.make_problem(cfg, seed=args.seed)
        work = lambda: (O.solve(prob), 1)[1]  # noqa: E731
        sample = f"one full oracle solve of the config-{cfg} problem per step (single thread)"
        units = 1
    t_w0 = time.perf_counter()
    cores, warm = 1, 0
    for i in range(args.warmup):
        cores = work()
        warm += 1
        if time.perf_counter() - t_w0 > REF_BUDGET_S / 5:   # one warm-up is enough for a slow solve
            break
    done, t0 = 0, time.perf_counter()
    while done < args.steps:
        cores = work()
        done += 1
        if time.perf_counter() - t0 > REF_BUDGET_S:
            break
    dt = time.perf_counter() - t0
    value = units * done / dt
    if done < args.steps or warm < args.warmup:
        sample += (f"; {done} of the {args.steps} requested steps timed after {warm} warm-up(s) "
                   f"(bounded at {REF_BUDGET_S:.0f} s of oracle work)")
    out = {"metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
           "steps": done, "warmup": warm, "ms_per_step": round(dt * 1e3 / done, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE config shapes)", "impl": "reference",
           "config": config_dict(cfg, args, world),
           "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
