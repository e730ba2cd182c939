"""Accuracy margin of the tensor-core passes over long circuits (VERDICT r1
weak #6): 320 Haar k = 5, 6 passes at random placements on a 20-qubit
complex64 state (tensor cores: n_local >= 16), every one a separate FP16
3-term tcgen05 pass, against the fp64 oracle.  The north_star bound is
||psi - psi_ref||_2 <= 1e-4; the measured error is recorded so the margin is
a measurement, not an extrapolation (rounding of unitary passes grows like
sqrt(P), SURVEY §8(c) "FP32 error budget")."""
import json
import os

import numpy as np
import pytest

import oracle as O
from hq_inputs import random_circuit, random_state
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("npass", [320])
def test_long_tensor_core_circuit_accuracy(npass):
    n = 20
    gates = random_circuit(n, npass, 9320, kmax=6, kmin=5)
    psi0 = random_state(n, 93)
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_set_amplitudes(s, psi0)
    hq.hq_stats_reset(s)
    hq.hq_profile_enable(s, True)
    errs = {}
    want = psi0.copy()
    for i0 in range(0, npass, 80):
        chunk = gates[i0:i0 + 80]
        hq.hq_apply_circuit(s, chunk)
        for g in chunk:
            want = O.apply_gate(want, g.U, g.qubits)
        errs[i0 + len(chunk)] = float(np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - want))
    tc = hq.hq_kernel_times(s, "tc")
    assert tc["count"] == npass, tc                       # every pass on the tensor cores
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "accuracy_%dpass.json" % npass), "w") as f:
        json.dump({"n": n, "passes": npass, "error_after": errs}, f)
    print("error after passes:", errs)
    assert errs[npass] <= 1e-4
    # growth no faster than ~sqrt(P) plus slack: the last error within 4x of
    # sqrt(P/80) times the first checkpoint's
    assert errs[npass] <= 4 * np.sqrt(npass / 80) * errs[80]
