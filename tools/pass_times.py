#!/usr/bin/env python
"""Per-pass device times of the bench circuit (34q d20, k <= 6, planned layout):
one CUDA-event pair around every fused pass, repeated `--rounds` times back to
back so the GPU reaches its sustained (power-capped) clock.  Prints one JSON
line per pass of the last round: k, physical target bits, ms, GB/s.

    python tools/pass_times.py [--n 34] [--rounds 3] [--kmax 6]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=34)
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--seed", type=int, default=3000)
    ap.add_argument("--kmax", type=int, default=6)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--c7", action="store_true", help="plain C7 fusion instead of hq_fuse_blocks")
    a = ap.parse_args()
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import sycamore_circuit
    n = a.n
    fused = hq.hq_fuse(sycamore_circuit(n, a.cycles, a.seed), a.kmax, blocks=not a.c7)
    layout = hq.hq_plan_layout(n, 0, fused, "c64")[0]
    s = hq.hq_state_create(n, "c64", 1)
    st = torch.cuda.Stream()
    hq.hq_state_set_stream(s, st.cuda_stream)
    hq.hq_state_set_layout(s, layout)
    hq.hq_state_init_basis(s, 0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in fused]
    for r in range(a.rounds):
        for (q, U), (e0, e1) in zip(fused, ev):
            e0.record(st)
            hq.hq_apply_matrix(s, U, q)
            e1.record(st)
        torch.cuda.synchronize()
    tot = 0.0
    for (q, U), (e0, e1) in zip(fused, ev):
        ms = e0.elapsed_time(e1)
        tot += ms
        print(json.dumps({"k": len(q), "bits": sorted(layout[x] for x in q), "ms": round(ms, 3),
                          "gbs": round(2 * 8 * 2 ** n / ms / 1e6, 1)}))
    print(json.dumps({"total_ms": tot, "passes": len(fused)}))


if __name__ == "__main__":
    main()
