#!/usr/bin/env python
"""Row f2 measurement: noisy Sycamore-style circuit on an N-qubit density
matrix by doubling ("a super circuit becomes a regular
circuit"): every gate U becomes U (x) conj(U) on (qubits, qubits + N) and every
noise channel its superoperator sum_m K_m (x) conj(K_m); the resulting
2N-qubit gate list goes through the same fusion planner, layout planner and
apply kernels as a pure-state circuit.

    python bench_dm.py [--N 15] [--cycles 10] [--p 0.01] [--kmax 6] [--steps 3]

Prints one JSON line: state-update GB/s of the 2N-qubit vec(rho) passes, the
circuit time, and tr(rho) after the run.
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
    ap.add_argument("--N", type=int, default=15)
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--p", type=float, default=0.01)
    ap.add_argument("--kmax", type=int, default=6)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--fuse", default="blocks", choices=["blocks", "c7"],
                    help="planner: hq_fuse_blocks (default) or the C7 greedy hq_fuse")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import sycamore_circuit, Gate, X, Y
    N = a.N
    pure = sycamore_circuit(N, a.cycles, 5000)
    s4 = np.sqrt(a.p / 4)
    depol = [np.sqrt(1 - 3 * a.p / 4) * np.eye(2), s4 * X, s4 * Y, s4 * np.diag([1, -1]).astype(complex)]
    S1 = hq.hq_dm_superop(depol)
    # super circuit -> regular 2N-qubit circuit (depolarising noise after each single-qubit layer)
    gates = []
    for g in pure:
        k = len(g.qubits)
        gates.append(Gate("S", tuple(g.qubits) + tuple(q + N for q in g.qubits), np.kron(g.U, g.U.conj())))
        if k == 1:
            q = g.qubits[0]
            gates.append(Gate("D", (q, q + N), S1))
    t0 = time.perf_counter()
    fused = hq.hq_fuse(gates, a.kmax, blocks=a.fuse == "blocks")
    layout, _, _ = hq.hq_plan_layout(2 * N, 0, fused, a.dtype)
    plan_ms = (time.perf_counter() - t0) * 1e3
    s = hq.hq_state_create(2 * N, a.dtype, 1)
    st = torch.cuda.Stream()
    hq.hq_state_set_stream(s, st.cuda_stream)
    hq.hq_state_set_layout(s, layout)
    c = hq.hq_circuit_create(s, fused)
    es = 8 if a.dtype == "c64" else 16
    ms = []
    for i in range(a.steps + 2):
        hq.hq_state_init_basis(s, 0)             # rho = |0><0|
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hq.hq_circuit_run(s, c)
        e1.record(st)
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    t = sum(ms) / len(ms)
    tr = hq.hq_dm_trace(s)
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    gbs = len(fused) * 2 * es * 4 ** N / (t * 1e-3) / 1e9
    print(json.dumps({"metric": "state-update GB/s (density matrix by doubling)", "value": gbs,
                      "unit": "GB/s", "frac_of_hbm": gbs / peak, "ms_per_circuit": t,
                      "config": {"N": N, "vec_qubits": 2 * N, "cycles": a.cycles, "p_depol": a.p,
                                 "kmax": a.kmax, "pure_gates": len(pure), "super_gates": len(gates),
                                 "passes": len(fused), "fusion": a.fuse, "dtype": a.dtype},
                      "plan_ms": plan_ms, "trace": [tr.real, tr.imag]}))


if __name__ == "__main__":
    main()
