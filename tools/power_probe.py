#!/usr/bin/env python
"""Sustained behaviour of one pass type: apply the same k-qubit gate `reps`
times back to back on an n-qubit c64 state while NVML samples the SM clock,
power and throttle reasons every 50 ms.  One JSON line per case with the mean
pass time (last half of the reps, after the clock settles), GB/s, median SM
clock and mean power over that window.

    python tools/power_probe.py [--n 34] [--reps 40] [--cases 6:b:16-17-18-22-23-24,2:b:3-20,4:b:8-12-20-28]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=34)
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--cases", default="6:b:16-17-18-22-23-24,5:b:16-17-18-22-23,4:b:8-12-20-28,2:b:3-20,1:b:20")
    a = ap.parse_args()
    import numpy as np
    import torch
    import pynvml
    import paper_2111_06868_b200 as hq
    from hq_inputs import haar_sweep_gate
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    from hq_inputs.states import random_state_torch
    psi_t = random_state_torch(a.n, "cuda", seed=32)        # dense state: generic operand activity
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    s = hq.hq_state_create_from_buffers(a.n, "c64", psi_t.data_ptr(), st.cuda_stream)
    for case in a.cases.split(","):
        k, pl = case.split(":", 1)
        g = haar_sweep_gate(a.n, int(k), pl, seed=7)
        samples, stop = [], threading.Event()

        def sampler():
            while not stop.is_set():
                samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
                time.sleep(0.05)

        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
        th = threading.Thread(target=sampler)
        th.start()
        t_start = time.perf_counter()
        for e0, e1 in ev:
            e0.record(st)
            hq.hq_apply_matrix(s, g.U, g.qubits)
            e1.record(st)
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        stop.set()
        th.join()
        ms = [e0.elapsed_time(e1) for e0, e1 in ev]
        half = ms[len(ms) // 2:]
        t_mid = t_start + (t_end - t_start) / 2
        win = [x for x in samples if x[0] >= t_mid]
        clk = sorted(x[1] for x in win)
        print(json.dumps({"k": int(k), "placement": pl, "ms": sum(half) / len(half),
                          "gbs": 2 * 8 * 2 ** a.n / (sum(half) / len(half)) / 1e6,
                          "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                          "power_w_mean": sum(x[2] for x in win) / max(len(win), 1),
                          "reasons": sorted({x[3] for x in win})}), flush=True)


if __name__ == "__main__":
    main()
