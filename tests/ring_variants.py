"""Manual check of the experimental apply_tcb ring variants (HQ_TC_NSLOT=<ns><np>)
against the oracle on one k = 6 pass; run by hand on a GPU box."""
import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2111_06868_b200 as hq
from hq_inputs import haar_sweep_gate, random_state
import oracle as O
n = 20
psi0 = random_state(n, 5)
for pl in ("high", "b:8-9-10-15-16-17", "b:2-9-11-15-16-19"):
    g = haar_sweep_gate(n, 6, pl, 7)
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_set_amplitudes(s, psi0.astype(np.complex64))
    hq.hq_apply_matrix(s, g.U, g.qubits)
    got = hq.hq_get_amplitudes(s)
    want = O.apply_gate(psi0.copy(), g.U, list(g.qubits))
    print(os.environ.get("HQ_TC_NSLOT"), pl, np.linalg.norm(got - want))
