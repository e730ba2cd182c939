#!/usr/bin/env python
"""Library baseline for the k = 6 pass: the same contraction as a cuBLAS
complex64 GEMM through torch.matmul, at the two placements where it is a
plain GEMM without a gather (targets = the 6 lowest bits: psi as a
(2^(n-6), 64) row-major matrix times U^T; targets = the 6 highest bits: U
times psi as a (64, 2^(n-6)) matrix), out of place, against this library's
in-place pass on the same placement and a dense state.  CUDA events, median
of `reps` after warm-up; fp32 (no TF32) and TF32-allowed matmul.  Not a
product path; it puts the hand-written kernel next to the library call a
user would otherwise write.

Also the general placement through torch.tensordot (the paper's einsum
engine idea), which adds two transposing copies to the GEMM.

    python tools/cublas_baseline.py [--n 32] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps, stream):
    import torch
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import haar_unitary
    from hq_inputs.states import random_state_torch
    n, k = a.n, 6
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    nbytes = 2 * 8 * 2 ** n
    U = haar_unitary(k, np.random.default_rng(7))
    Ut = torch.tensor(U, dtype=torch.complex64, device="cuda")
    psi = random_state_torch(n, "cuda", seed=32)
    out = torch.empty_like(psi)
    st = torch.cuda.current_stream()
    s = hq.hq_state_create_from_buffers(n, "c64", psi.data_ptr(), st.cuda_stream)
    rows = []
    for placement, qubits in (("low", list(range(n - k, n))), ("high", list(range(k)))):
        # qubit q <-> index bit n-1-q: qubits n-6..n-1 are bits 5..0 (low), qubits 0..5 bits n-1..n-6 (high)
        ours = timed(lambda: hq.hq_apply_matrix(s, U, qubits), a.reps, st)
        if placement == "low":
            A = psi.view(2 ** (n - k), 2 ** k)
            O = out.view(2 ** (n - k), 2 ** k)
            gemm = lambda: torch.matmul(A, Ut.T, out=O)
        else:
            A = psi.view(2 ** k, 2 ** (n - k))
            O = out.view(2 ** k, 2 ** (n - k))
            gemm = lambda: torch.matmul(Ut, A, out=O)
        res = {"placement": placement, "n": n, "k": k, "hq_ms": ours, "hq_frac_of_hbm": nbytes / (ours * 1e-3) / 1e9 / peak}
        for tf32 in (False, True):
            torch.backends.cuda.matmul.allow_tf32 = tf32
            ms = timed(gemm, a.reps, st)
            res["cublas_%s_ms" % ("tf32" if tf32 else "fp32")] = ms
        torch.backends.cuda.matmul.allow_tf32 = False
        res["speedup_vs_cublas_fp32"] = res["cublas_fp32_ms"] / ours
        rows.append(res)
        print(json.dumps(res), flush=True)
    # a general placement as the paper's tensordot engine would do it in
    # PyTorch: move the target axes last, one GEMM, move them back
    # (two transposing copies + the GEMM)
    qubits = [2, 9, 15, 20, 26, n - 2]
    ours = timed(lambda: hq.hq_apply_matrix(s, U, qubits), a.reps, st)
    T = psi.view(*([2] * n))
    Uk = Ut.view(*([2] * (2 * k)))

    def tensordot():
        r = torch.tensordot(T, Uk, dims=(qubits, list(range(k, 2 * k))))   # target axes appended last
        return torch.movedim(r, list(range(n - k, n)), qubits).contiguous()

    res = {"placement": "spread %s" % qubits, "n": n, "k": k, "hq_ms": ours,
           "hq_frac_of_hbm": nbytes / (ours * 1e-3) / 1e9 / peak}
    for tf32 in (False, True):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        res["torch_tensordot_%s_ms" % ("tf32" if tf32 else "fp32")] = timed(tensordot, a.reps, st)
    torch.backends.cuda.matmul.allow_tf32 = False
    res["speedup_vs_tensordot_fp32"] = res["torch_tensordot_fp32_ms"] / ours
    print(json.dumps(res), flush=True)
    s.close()


if __name__ == "__main__":
    main()
