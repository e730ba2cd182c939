#!/usr/bin/env python
"""One pass per k = 1..6 at the 'spread' placement on n = 32 (complex64), for
an ncu metrics capture of every kernel family (tensor-pipe / FMA-pipe use per
k, BASELINE configs[2])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_06868_b200 as hq
from hq_inputs import haar_sweep_gate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
s = hq.hq_state_create(n, "c64", 1)
hq.hq_state_init_basis(s, 0)
hq.hq_norm(s)
for k in range(1, 7):
    g = haar_sweep_gate(n, k, "spread", 2000 + k)
    hq.hq_apply_matrix(s, g.U, g.qubits)
hq.hq_sync(s)
print("ok")
