#!/usr/bin/env python
"""Small-n compiled circuits: time per hq_circuit_run (CUDA events over 50
back-to-back runs) for n = 4..12 Sycamore-style circuits fused to k <= 6.
The runtime picks the shared-memory whole-circuit kernel for n_local <= 10 and
the per-pass kernels in a CUDA graph above (the round-2 A/B that set this rule
used an experiment switch since removed: 8q 16.5 vs 28.7 us, 10q 45 vs 55 us,
12q 132 vs 237 us in favour of the selected path)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_06868_b200 as hq
from hq_inputs import sycamore_circuit

for dtype in ("c64", "c128"):
    for n in (4, 6, 8, 10, 11, 12):
        fused = hq.hq_fuse(sycamore_circuit(n, 10, 0), min(6, n))
        s = hq.hq_state_create(n, dtype, 1)
        st = torch.cuda.Stream()
        hq.hq_state_set_stream(s, st.cuda_stream)
        hq.hq_state_init_basis(s, 0)
        c = hq.hq_circuit_create(s, fused)
        for _ in range(5):
            hq.hq_circuit_run(s, c)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(50):
            hq.hq_circuit_run(s, c)
        b.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"dtype": dtype, "n": n, "passes": len(fused), "us_per_circuit": a.elapsed_time(b) * 1e3 / 50}), flush=True)
