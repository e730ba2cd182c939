#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): one pass of every apply kernel family at 17-20 qubits, the 12q
configs[0] circuit through the compiled-circuit path, and a virtual-shard
circuit with remaps and folded packs.  Each result is checked against the
oracle so a sanitizer run also fails loudly on wrong numbers.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2111_06868_b200 as hq  # noqa: E402
from hq_inputs import haar_sweep_gate, random_state, sycamore_circuit  # noqa: E402


def main():
    n = 17
    psi0 = random_state(n, 1)
    cases = [(6, "spread"), (6, "low"), (5, "spread"), (5, "low"), (6, "b:1-2-3-7-8-9"), (6, "b:0-3-7-9-12-15"),
             (4, "spread"), (4, "low"), (2, "random0"), (1, "high")]
    for k, pl in cases:
        g = haar_sweep_gate(n, k, pl, 3000 + k)
        s = hq.hq_state_create(n, "c64", 1)
        hq.hq_set_amplitudes(s, psi0)
        hq.hq_apply_matrix(s, g.U, g.qubits)
        err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.apply_gate(psi0.copy(), g.U, g.qubits))
        assert err < 2e-6, (k, pl, err)
        print("k=%d %s err=%.2e" % (k, pl, err), flush=True)
    gates = sycamore_circuit(12, 10, 0)
    for dtype, kmax in (("c64", 6), ("c128", 4)):
        s = hq.hq_state_create(12, dtype, 1)
        hq.hq_state_init_basis(s, 0)
        c = hq.hq_circuit_create(s, hq.hq_fuse(gates, kmax))
        hq.hq_circuit_run(s, c)
        err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.simulate(12, gates))
        assert err < 1e-4, err
        print("12q %s kmax=%d err=%.2e" % (dtype, kmax, err), flush=True)
    n = 18
    gates = sycamore_circuit(n, 8, 9)
    fused = hq.hq_fuse(gates, 6, blocks=True)
    s = hq.hq_state_create_virtual(n, "c64", 4)
    pi0, _, _ = hq.hq_plan_layout(n, 2, fused)
    hq.hq_state_set_layout(s, pi0)
    hq.hq_state_init_basis(s, 0)
    hq.hq_apply_circuit(s, fused)
    st = hq.hq_stats_get(s)
    err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.simulate(n, gates))
    assert err < 1e-4, err
    print("18q on 4 virtual shards: remaps=%d packs=%d err=%.2e" % (st["remaps"], st["packs"], err), flush=True)
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
