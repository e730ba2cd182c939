#!/usr/bin/env python
"""hq_norm on a dense n-qubit complex64 state: wall time per call (it
synchronises), median of `reps`, and the read rate it implies."""
import os, sys, json, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_06868_b200 as hq
from hq_inputs.states import random_state_torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 34
reps = 10
psi = random_state_torch(n, "cuda", seed=3)
torch.cuda.synchronize()
s = hq.hq_state_create_from_buffers(n, "c64", psi.data_ptr(), torch.cuda.current_stream().cuda_stream)
hq.hq_norm(s)
ms = []
for _ in range(reps):
    t = time.perf_counter()
    v = hq.hq_norm(s)
    ms.append((time.perf_counter() - t) * 1e3)
m = statistics.median(ms)
print(json.dumps({"n": n, "norm": v, "ms": m, "read_gbs": 8 * 2 ** n / (m * 1e-3) / 1e9}))
