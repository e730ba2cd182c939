#!/usr/bin/env python
"""Long-circuit accuracy of the tensor-core passes (no assertion): P Haar
k = 5, 6 passes at random placements on a 20-qubit complex64 state against the
fp64 oracle, ||psi - psi_ref||_2 every 80 passes (tests/test_gpu_accuracy.py
asserts the 320-pass case).

    python tools/accuracy_long.py [P]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from hq_inputs import random_circuit, random_state
import paper_2111_06868_b200 as hq

npass = int(sys.argv[1]) if len(sys.argv) > 1 else 960
n = 20
gates = random_circuit(n, npass, 9320, kmax=6, kmin=5)
psi0 = random_state(n, 93)
s = hq.hq_state_create(n, "c64", 1)
hq.hq_set_amplitudes(s, psi0)
want = psi0.copy()
errs = {}
for i0 in range(0, npass, 80):
    chunk = gates[i0:i0 + 80]
    hq.hq_apply_circuit(s, chunk)
    for g in chunk:
        want = O.apply_gate(want, g.U, g.qubits)
    errs[i0 + len(chunk)] = float(np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - want))
print(json.dumps({"n": n, "passes": npass, "error_after": errs, "norm": hq.hq_norm(s)}))
