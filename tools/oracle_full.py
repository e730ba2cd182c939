#!/usr/bin/env python
"""The fp64 oracle on a whole BASELINE circuit, unfused, on the host cores
(SURVEY §8(d) "Oracle timing": configs[0] and [1] in full where the complex128
state fits host RAM).  Prints one JSON line; used once per round on the GPU
box, not by the default bench.

    python tools/oracle_full.py --n 30 --cycles 20 --seed 1000 [--threads T]
"""
import argparse
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1000)
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    import oracle as O
    from hq_inputs import sycamore_circuit
    if a.threads:
        O.set_threads(a.threads)
    gates = sycamore_circuit(a.n, a.cycles, a.seed)
    t0 = time.perf_counter()
    psi = O.init_basis(a.n, 0)
    t1 = time.perf_counter()
    for g in gates:
        O.apply_gate(psi, g.U, g.qubits)
    t2 = time.perf_counter()
    nrm = O.norm(psi)
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    print(json.dumps({"n": a.n, "cycles": a.cycles, "seed": a.seed, "gates": len(gates),
                      "seconds": t2 - t1, "init_seconds": t1 - t0, "threads": O.max_threads(),
                      "norm": nrm, "cpu": cpu or platform.processor(),
                      "state_gib_c128": 16 * 2 ** a.n / 2 ** 30}), flush=True)


if __name__ == "__main__":
    main()
