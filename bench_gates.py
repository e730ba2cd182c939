#!/usr/bin/env python
"""Per-pass profile of a fused benchmark circuit: times every fused gate of
the circuit (CUDA events on the library stream) and prints its physical target
bits, kernel path and achieved HBM GB/s, sorted by time.  Used to find which
placements dominate the circuit wall time.

    python bench_gates.py [--n 34] [--cycles 20] [--seed 3000] [--kmax 6] [--reps 2]
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
    ap.add_argument("--n", type=int, default=34)
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--seed", type=int, default=3000)
    ap.add_argument("--kmax", type=int, default=6)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--dtype", default="c64")
    a = ap.parse_args()
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import sycamore_circuit
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    fused = hq.hq_fuse(sycamore_circuit(a.n, a.cycles, a.seed), a.kmax, blocks=True)
    s = hq.hq_state_create(a.n, a.dtype, 1)
    st = torch.cuda.Stream()
    hq.hq_state_set_stream(s, st.cuda_stream)
    hq.hq_state_init_basis(s, 0)
    es = 8 if a.dtype == "c64" else 16
    nbytes = 2 * es * 2 ** a.n
    times = {i: [] for i in range(len(fused))}
    for rep in range(a.reps + 1):
        evs = []
        for i, (q, U) in enumerate(fused):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            hq.hq_apply_matrix(s, U, q)
            e1.record(st)
            evs.append((i, e0, e1))
        torch.cuda.synchronize()
        if rep > 0:
            for i, e0, e1 in evs:
                times[i].append(e0.elapsed_time(e1))
    rows = []
    total = 0.0
    for i, (q, U) in enumerate(fused):
        ms = statistics.median(times[i])
        total += ms
        rows.append((ms, i, sorted(a.n - 1 - x for x in q)))
    rows.sort(reverse=True)
    for ms, i, bits in rows:
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"gate": i, "k": len(bits), "bits": bits, "ms": round(ms, 3),
                          "gbs": round(gbs), "frac": round(gbs / peak, 3)}))
    print(json.dumps({"total_ms": total, "passes": len(fused),
                      "circuit_gbs": len(fused) * nbytes / (total * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
