#!/usr/bin/env python
"""Rows f3/f4 state operations on a dense n-qubit complex64 state: wall time
per call (each synchronises), median of `reps`: hq_norm, hq_probabilities
(1, 4 and 10 qubits, low and high bits), hq_reduced_dm (1 and 2 qubits),
hq_project."""
import os, sys, json, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2111_06868_b200 as hq
from hq_inputs.states import random_state_torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = 5
psi = random_state_torch(n, "cuda", seed=3)
torch.cuda.synchronize()
s = hq.hq_state_create_from_buffers(n, "c64", psi.data_ptr(), torch.cuda.current_stream().cuda_stream)


def t(fn):
    fn()
    ms = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ms.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ms)


state_gb = 8 * 2 ** n / 1e9
rows = {"norm": t(lambda: hq.hq_norm(s))}
for nq, where in ((1, "high"), (1, "low"), (4, "high"), (4, "low"), (10, "high")):
    qs = list(range(nq)) if where == "high" else list(range(n - nq, n))
    rows["probabilities_%d_%s" % (nq, where)] = t(lambda: hq.hq_probabilities(s, qs))
for k in (1, 2):
    rows["reduced_dm_%d" % k] = t(lambda: hq.hq_reduced_dm(s, list(range(k))))
rows["measure_1"] = t(lambda: hq.hq_measure(s, [0], 0.3))
rows["probabilities_1_high_after"] = t(lambda: hq.hq_probabilities(s, [0]))
rows["project_1_keep"] = t(lambda: hq.hq_project(s, [0], [0], renormalize=True))
rows["project_1_renorm"] = t(lambda: hq.hq_project(s, [n - 1], [0], renormalize=True))
rows["init_tokens_plus"] = t(lambda: hq.hq_state_init_tokens(s, "+"))
K = [np.sqrt(0.9) * np.eye(2), np.sqrt(0.1) * np.array([[0, 1], [1, 0]], dtype=complex)]
rows["kraus_sample_1"] = t(lambda: hq.hq_kraus_sample(s, K, [3], 0.4))
print(json.dumps({"n": n, "ms": rows, "read_gbs": {k: state_gb / (v * 1e-3) for k, v in rows.items()}}))
