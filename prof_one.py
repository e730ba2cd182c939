#!/usr/bin/env python
"""Small driver for ncu captures: apply one Haar k-qubit gate `reps` times at a
named placement on an n-qubit state (same inputs as bench_sweep.py).

    python prof_one.py --n 30 --k 6 --placement high --reps 3 [--dtype c64]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--k", type=int, default=6)
    ap.add_argument("--placement", default="high")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtype", default="c64")
    a = ap.parse_args()
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import haar_sweep_gate
    from hq_inputs.states import random_state_torch
    psi_t = random_state_torch(a.n, "cuda", seed=32, dtype=a.dtype)     # dense state (see bench_sweep.py)
    torch.cuda.synchronize()
    s = hq.hq_state_create_from_buffers(a.n, a.dtype, psi_t.data_ptr(), None)
    g = haar_sweep_gate(a.n, a.k, a.placement, 2000 + a.k)
    for _ in range(a.reps):
        hq.hq_apply_matrix(s, g.U, g.qubits)
    hq.hq_sync(s)
    print("ok", a.n, a.k, a.placement, hq.hq_norm(s))


if __name__ == "__main__":
    main()
