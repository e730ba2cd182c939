#!/usr/bin/env python
"""Remap cost on virtual shards (one B200): the same distributed circuit run
with separate exchanges (HQ_REMAP_EXCHANGE: each remap is a device-to-device
copy pass of 7/8 of every shard after the apply pass) and with fused remaps
(HQ_REMAP_FUSED: the apply pass before each remap writes every element
straight into its destination shard's buffer).  CUDA events on the state's
stream around the whole circuit; per-kernel times from the library's
per-launch events.  The difference is the remap time the fusion hides behind
the pass.

    python tools/remap_timeline.py [--n 30] [--G 8] [--cycles 20] [--kmax 6]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--kmax", type=int, default=6)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2111_06868_b200 as hq
    from hq_inputs import sycamore_circuit
    gates = sycamore_circuit(a.n, a.cycles, 1000 + a.n)
    fused = hq.hq_fuse(gates, a.kmax, blocks=True)
    m = a.G.bit_length() - 1
    pi0, _, _ = hq.hq_plan_layout(a.n, m, fused)
    res = {"n": a.n, "G": a.G, "kmax": a.kmax, "passes": len(fused)}
    amps = {}
    for mode in ("exchange", "fused"):
        s = hq.hq_state_create_virtual(a.n, "c64", a.G)
        hq.hq_state_set_remap_mode(s, mode)
        hq.hq_state_set_layout(s, pi0)
        c = hq.hq_circuit_create(s, fused)
        info = hq.hq_circuit_info(c)
        times = []
        for rep in range(a.reps + 1):
            hq.hq_state_init_basis(s, 0)
            hq.hq_sync(s)
            hq.hq_stats_reset(s)
            hq.hq_profile_enable(s, rep > 0)
            hq.hq_kernel_times(s)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            hq.hq_circuit_run(s, c)
            hq.hq_sync(s)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                kt = hq.hq_kernel_times(s)
                times.append({"circuit_ms": e0.elapsed_time(e1), "apply_kernels_ms": kt["total_ms"]})
        st = hq.hq_stats_get(s)
        res[mode] = {"remaps": info["remaps"], "remaps_fused": st["remaps_fused"], "packs": st["packs"],
                     "circuit_ms": min(t["circuit_ms"] for t in times),
                     "apply_kernels_ms": min(t["apply_kernels_ms"] for t in times),
                     "norm": hq.hq_norm(s)}
        res[mode]["remap_and_other_ms"] = res[mode]["circuit_ms"] - res[mode]["apply_kernels_ms"]
        amps[mode] = hq.hq_get_amplitudes(s, 0, 1 << 16)
        s.close()
    import numpy as np
    res["fused_equals_exchange_first_65536"] = bool(np.array_equal(amps["exchange"], amps["fused"]))
    res["hidden_ms"] = res["exchange"]["circuit_ms"] - res["fused"]["circuit_ms"]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
