#!/usr/bin/env python
"""Fused-gate sweep (BASELINE.json configs[2]): one Haar k-qubit gate,
k = 1..6, at several placements on an n = 32 complex64 state (32 GiB), on one
B200.  Reports per (k, placement) the median and best pass time and the
achieved HBM GB/s (2 x state bytes / pass time) against MEASURED_PEAKS.json.

    python bench_sweep.py [--n 32] [--dtype c64] [--reps 20] [--ks 1,2,3,4,5,6]

Pass times are CUDA events on the library's stream around each apply (the
state is > L2, so no flush is needed).  One JSON line per (k, placement) plus
a summary line.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ks", default="1,2,3,4,5,6")
    ap.add_argument("--placements", default="low,high,spread,random0,random1,random2")
    args = ap.parse_args()
    import torch
    from paper_2111_06868_b200 import build
    build.build()
    import paper_2111_06868_b200 as hq
    from hq_inputs import haar_sweep_gate
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    n = args.n
    es = 8 if args.dtype == "c64" else 16
    from hq_inputs.states import random_state_torch
    # dense random-normal state (config [2]): every amplitude non-zero, so the
    # tensor cores see generic operand activity (a |0>-derived state is mostly
    # zeros and draws less power under the 1 kW cap)
    psi_t = random_state_torch(n, "cuda", seed=32, dtype=args.dtype)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    s = hq.hq_state_create_from_buffers(n, args.dtype, psi_t.data_ptr(), stream.cuda_stream)
    nbytes = 2 * es * 2 ** n
    summary = {}
    for k in [int(x) for x in args.ks.split(",")]:
        for pl in args.placements.split(","):
            if pl.startswith("b:") and pl.count("-") + 1 != k:
                continue
            g = haar_sweep_gate(n, k, pl, 2000 + k)
            for _ in range(args.warmup):
                hq.hq_apply_matrix(s, g.U, g.qubits)
            ts = []
            for _ in range(args.reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                hq.hq_apply_matrix(s, g.U, g.qubits)
                b.record(stream)
                ts.append((a, b))
            torch.cuda.synchronize()
            ms = [a.elapsed_time(b) for a, b in ts]
            med, best = statistics.median(ms), min(ms)
            gbs = nbytes / (med * 1e-3) / 1e9
            rec = {"k": k, "placement": pl, "qubits": list(g.qubits),
                   "phys_bits": sorted(n - 1 - q for q in g.qubits), "median_ms": med,
                   "best_ms": best, "gbs": gbs, "frac": gbs / peak}
            print(json.dumps(rec), flush=True)
            summary.setdefault(k, []).append(gbs)
    out = {"summary": {k: {"min_gbs": min(v), "median_gbs": statistics.median(v),
                           "min_frac": min(v) / peak} for k, v in summary.items()},
           "n": n, "dtype": args.dtype, "peak_gbs": peak}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
