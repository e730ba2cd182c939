#!/usr/bin/env python
"""Row f3 measurement: trajectory throughput (shots/s) on a noisy
Sycamore-style circuit, one shot per state against batched shots.

    python bench_traj.py [--n 12] [--cycles 8] [--p 0.01] [--shots 4096] [--batch 1,256,4096]

Noise: a depolarizing channel after every single-qubit gate of the first
`noisy` qubits (the paper's Fig. 1 channel).  Prints one JSON line
per batch size: shots/s, ms per shot, the mean <Z> of qubit 0 (the
observable), and the state-update GB/s of the passes it ran.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=12)
    ap.add_argument("--cycles", type=int, default=8)
    ap.add_argument("--p", type=float, default=0.01)
    ap.add_argument("--noisy", type=int, default=4)
    ap.add_argument("--shots", type=int, default=4096)
    ap.add_argument("--batch", default="1,256,4096")
    ap.add_argument("--max-unbatched", type=int, default=512)
    a = ap.parse_args()
    import numpy as np
    import torch
    from hq_inputs import sycamore_circuit, X, Y, Z
    from paper_2111_06868_b200.trajectories import Channel, sample_trajectories
    n = a.n
    s4 = np.sqrt(a.p / 4)
    depol = [np.sqrt(1 - 3 * a.p / 4) * np.eye(2), s4 * X, s4 * Y, s4 * Z]
    ops, nch = [], 0
    for g in sycamore_circuit(n, a.cycles, 6000):
        ops.append(g)
        if len(g.qubits) == 1 and g.qubits[0] < a.noisy:
            ops.append(Channel(g.qubits, depol))
            nch += 1
    for b in [int(x) for x in a.batch.split(",")]:
        shots = min(a.shots, a.max_unbatched) if b == 1 else a.shots
        sample_trajectories(n, ops, min(shots, 2 * b), observe=[0], seed=1, batch=b)     # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sample_trajectories(n, ops, shots, observe=[0], seed=1, batch=b)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        z = float((res["rho"][0, 0] - res["rho"][1, 1]).real)
        print(json.dumps({"metric": "trajectory shots/s", "value": shots / dt, "unit": "shots/s",
                          "batch": b, "shots": shots, "ms_per_shot": 1e3 * dt / shots, "mean_Z0": z,
                          "config": {"n": n, "cycles": a.cycles, "channels_per_shot": nch, "p_depol": a.p,
                                     "gates": len(ops) - nch}}), flush=True)


if __name__ == "__main__":
    main()
