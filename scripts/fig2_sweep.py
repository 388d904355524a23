#!/usr/bin/env python
"""NEXT-1: the paper's timing workloads (PAPER.md P:553-560,
Fig. 2: n x (n-10) sprandn-like matrices, density 1 and 0.01) on the B200
path, the CPU oracle beside them, and the dense Gram's FP64 tensor rate.

* solves/s per size: device-resident CSR + b -> x (load + Gram + pivot loop +
  LSQR), CUDA events, L2 flushed between steps; the oracle (single thread) on
  a bounded sample.
* dense Gram (the DMMA SYRK of gram_dense.cu) on a large dense problem: its
  executed flops m n^2 (both triangles of the DMMA tiles) / time vs the
  measured DMMA peak, and the row-sharding crossover of SURVEY.md §8(e): one
  GPU forms G in t_1; with P GPUs each forms its 1/P row block in ~t_1/P and
  the packed partials are reduced to rank 0 (4 n^2 (P-1)/P bytes at ~900 GB/s
  per NVLink 5 direction -- a model; this sandbox has one GPU).

    python scripts/fig2_sweep.py [--out profiles/r02_fig2_sweep.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nnls_gen as g  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_fig2_sweep.json"))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--oracle-seconds", type=float, default=3.0)
    args = ap.parse_args()
    import torch

    import oracle as O
    import paper_cs_0408029_b200 as P
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    rows = []
    for d, sizes in ((1.0, [100, 200, 300, 500, 700, 1000]), (0.01, [800, 1000, 1200, 1420])):
        for n in sizes:
            prob = g.make_fig2(n, d, seed=0)
            dv = {k: torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).to(dev)
                  for k in ("rowptr", "colind", "vals", "b")}
            S = P.Solver(stream=stream)
            x = torch.empty(prob.n, dtype=torch.float64, device=dev)

            def step():
                S.load(prob.m, prob.n, dv["rowptr"], dv["colind"], dv["vals"], dv["b"])
                return S.solve(x_out=x)[1]
            for _ in range(3):
                info = step()
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(args.reps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            ms = tot / args.reps
            t0, k = time.perf_counter(), 0
            while True:
                O.solve(prob)
                k += 1
                if time.perf_counter() - t0 > args.oracle_seconds:
                    break
            oms = (time.perf_counter() - t0) * 1e3 / k
            rec = {"density": d, "n": n, "m": prob.m, "cols": prob.n, "nnz": prob.nnz, "gpu_ms": round(ms, 4),
                   "gpu_solves_per_s": round(1e3 / ms, 2), "oracle_ms_1core": round(oms, 3),
                   "iterations": info["iterations"], "free": info["free_count"]}
            rows.append(rec)
            print(rec)
            S.close()
    # large dense Gram: the DMMA SYRK rate
    dense = []
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_microbench_fp64.json")))["dmma_tflops"]
    for m, n in ((8192, 4096), (16384, 8000)):
        # fully dense, entries N(0,1) on the 2^-12 grid and b on the same grid
        # (every Gram / A^T b partial sum exact -> the dense DMMA path)
        rng = np.random.default_rng([m, n])
        vals = np.clip(np.round(rng.standard_normal(m * n) * 4096), -8 * 4096, 8 * 4096) / 4096
        vals[vals == 0] = 1.0 / 4096
        prob = g.Problem(m, n, (np.arange(m + 1, dtype=np.int64) * n).astype(np.int32),
                         np.tile(np.arange(n, dtype=np.int32), m), vals,
                         np.round(rng.standard_normal(m) * 4096) / 4096, np.zeros(n), "dense", 0)
        dv = {k: torch.from_numpy(np.ascontiguousarray(getattr(prob, k))).to(dev) for k in ("rowptr", "colind", "vals", "b")}
        S = P.Solver(stream=stream)
        S.load(m, n, dv["rowptr"], dv["colind"], dv["vals"], dv["b"])
        P.timing_enable(S.h, True)
        reps = 3
        for _ in range(reps):
            S.load(m, n, dv["rowptr"], dv["colind"], dv["vals"], dv["b"])
        torch.cuda.synchronize()
        ph = P.timing_read(S.h)
        P.timing_enable(S.h, False)
        gms = ph["gram"][0] / reps
        ntc = (n + 63) // 64
        fl_exec = 2.0 * m * (64 * ntc) * (64 * ntc + 64) / 2 * 1.0  # lower tiles incl. diagonal, full 64x64 DMMA
        fl_alg = float(m) * n * n                                 # P:117 "n^2 m"
        tf = fl_alg / (gms / 1e3) / 1e12
        packed = 8.0 * n * (n + 1) / 2
        row = {"m": m, "n": n, "gram_ms": round(gms, 3), "alg_tflops": round(tf, 3), "frac_of_dmma_peak": round(tf / fp64, 4),
               "executed_tflops": round(fl_exec / (gms / 1e3) / 1e12, 3), "peak_tflops": fp64,
               "crossover_model": {f"P{p}": {"gram_ms": round(gms / p, 3),
                                             "reduce_ms_at_900GBps": round(packed * (p - 1) / p / 900e9 * 1e3, 3),
                                             "total_ms": round(gms / p + packed * (p - 1) / p / 900e9 * 1e3, 3)}
                                   for p in (1, 2, 4, 8)}}
        dense.append(row)
        print(row)
        S.close()
    out = {"what": "Fig. 2 workloads (n x (n-10), density 1 / 0.01) on one B200 + the dense DMMA Gram rate",
           "sweep": rows, "dense_gram": dense}
    json.dump(out, open(args.out, "w"), indent=1)
    print("->", args.out)


if __name__ == "__main__":
    main()
