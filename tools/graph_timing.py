#!/usr/bin/env python
"""Small-n circuit timing with and without the CUDA-graph replay of
hq_circuit_run (profiling on disables the graph)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_06868_b200 as hq
from hq_inputs import sycamore_circuit

for n, cyc in ((12, 10), (16, 14), (20, 16), (24, 20)):
    fused = hq.hq_fuse(sycamore_circuit(n, cyc, 0), 6)
    s = hq.hq_state_create(n, "c64", 1)
    st = torch.cuda.Stream()
    hq.hq_state_set_stream(s, st.cuda_stream)
    c = hq.hq_circuit_create(s, fused)
    for graph in (False, True):
        hq.hq_profile_enable(s, not graph)
        for _ in range(3):
            hq.hq_state_init_basis(s, 0); hq.hq_circuit_run(s, c)
        hq.hq_sync(s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a.record(st)
        for _ in range(reps):
            hq.hq_circuit_run(s, c)
        b.record(st)
        torch.cuda.synchronize()
        hq.hq_kernel_times(s)
        print("n=%d passes=%d graph=%s: %.3f ms per circuit" % (n, len(fused), graph, a.elapsed_time(b) / reps), flush=True)
