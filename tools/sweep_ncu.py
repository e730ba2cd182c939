#!/usr/bin/env python
"""One pass per k = 1..6 at a placement (default 'spread') on an n = 32
complex64 DENSE random-normal state (BASELINE configs[2]; tensor-core and FMA
power depend on operand activity, so a |0>-derived, mostly-zero state would
flatter them), for an ncu metrics capture of every kernel family: tensor-pipe
and FMA-pipe use and DRAM bytes per k.

    ncu --metrics ... python tools/sweep_ncu.py [n] [placement]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2111_06868_b200 as hq  # noqa: E402
from hq_inputs import haar_sweep_gate  # noqa: E402
from hq_inputs.states import random_state_torch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
placement = sys.argv[2] if len(sys.argv) > 2 else "spread"
psi_t = random_state_torch(n, "cuda", seed=32, dtype="c64")
torch.cuda.synchronize()
s = hq.hq_state_create_from_buffers(n, "c64", psi_t.data_ptr(), None)
for k in range(1, 7):
    g = haar_sweep_gate(n, k, placement, 2000 + k)
    hq.hq_apply_matrix(s, g.U, g.qubits)
hq.hq_sync(s)
print("ok", hq.hq_norm(s))
