#!/usr/bin/env python
"""Benchmark: state-update GB/s and circuit wall time for a Sycamore-style
random circuit through the C ABI (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 34q] [--kmax 4]
    python bench.py --impl reference ...      # the fp64 CPU oracle arm

A "step" is one pass of the whole hot path over one synthetic circuit:
fused gate list (planned before the timed region, reported as plan_ms) ->
every apply pass and remap on the device -> norm.  The state (2^n complex64)
is initialised to |0> before each step, outside the per-step events.

value  = passes * 2 * (state bytes) / circuit time (whole job, all GPUs),
         device-timed with CUDA events on the library's stream, max over ranks.
e2e    = the same metric through the public API with host inputs: per step
         hq_fuse(host gates) + hq_apply_circuit (matrices copied H2D) +
         hq_norm (D2H), host wall clock.
For N>1 the same circuit is strong-scaled: the state is sharded on the top
log2 N qubits and remaps run as NCCL all-to-all exchanges.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, cycles, seed, default kmax, BASELINE configs index)
    "12q": (12, 10, 0, 6, 0),
    "30q": (30, 20, 1000, 2, 1),
    "34q": (34, 20, 3000, 6, 3),
    "36q": (36, 24, 4000, 6, 4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hq", choices=["hq", "reference"])
    ap.add_argument("--config", default="34q", choices=sorted(CONFIGS))
    ap.add_argument("--kmax", type=int, default=None)
    ap.add_argument("--fuse", default="merged", choices=["merged", "c7"],
                    help="planner: hq_fuse_merged (default) or the plain C7 greedy hq_fuse")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-layout", action="store_true",
                    help="keep the default qubit layout instead of hq_plan_layout's")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(cfg, kmax, path, bytes_per_launch):
    """DRAM traffic per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_traffic.json): the capture's measured
    dram__bytes_read.sum + dram__bytes_write.sum per algorithmic byte, times
    this launch's algorithmic bytes (the capture runs the same kernel on a
    smaller state so that ncu can save/restore it for replay)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d[path]
        return e["ratio"] * bytes_per_launch, e["source"]
    except Exception:
        return None, None


# ------------------------------------------------------------------ oracle arm
def oracle_sample(n_full, cycles, seed, kmax, seconds=15.0, n_sample=None, merged=True):
    """Time the fp64 oracle (as it stands) on a bounded sample of the same
    workload: the first unfused gates of the same generator's circuit at a
    smaller n (c128 state must fit host RAM), extrapolated per gate by
    2^(n_full - n_sample).  Returns (value in the GPU arm's unit, info)."""
    import numpy as np
    import oracle as O
    from hq_inputs import sycamore_circuit
    gates_full = sycamore_circuit(n_full, cycles, seed)
    # the pass count of the unit, from the oracle's own reading of the planner
    # (C7, plus the merging reading when the GPU arm uses hq_fuse_merged)
    groups = O.compress(gates_full, kmax)
    P = len(O.merge_groups(gates_full, groups, kmax)) if merged else len(groups)
    if n_sample is None:
        n_sample = min(n_full, 26)
    gates_s = sycamore_circuit(n_sample, cycles, seed)
    psi = O.init_basis(n_sample, 0)
    t0 = time.perf_counter()
    done = 0
    for g in gates_s:
        O.apply_gate(psi, g.U, g.qubits)
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    per_gate = dt / done * 2 ** (n_full - n_sample)
    T_full = per_gate * len(gates_full)
    work = P * 2 * 8 * 2 ** n_full          # same algorithmic bytes as the GPU arm (c64)
    value = work / T_full / 1e9
    info = {"sample": "first %d of %d unfused gates of the same generator's circuit at n=%d "
                      "(c128, %.1f s), extrapolated x2^%d per gate to the %d-gate n=%d circuit"
                      % (done, len(gates_s), n_sample, dt, n_full - n_sample, len(gates_full), n_full),
            "extrapolated_circuit_s": T_full, "cores": O.max_threads()}
    return value, info


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    n, cycles, seed, kdef, cidx = CONFIGS[args.config]
    kmax = args.kmax or kdef
    vals = []
    info = None
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    for i in range(args.warmup + args.steps):
        v, info = oracle_sample(n, cycles, seed, kmax, seconds=per_step, merged=args.fuse == "merged")
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": "state-update GB/s", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": info["extrapolated_circuit_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s Sycamore-style d%d random circuit (BASELINE configs[%d]), "
                               "oracle unfused fp64" % (args.config, cycles, cidx),
                   "n": n, "cycles": cycles, "seed": seed, "kmax": kmax},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def run_hq(args):
    import numpy as np
    import torch
    world, rank, local = dist_env()
    n_gpus = args.gpus
    if world != n_gpus:
        raise SystemExit("--gpus %d but WORLD_SIZE=%d" % (n_gpus, world))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2111_06868_b200 import build as hqbuild
    if rank == 0:
        hqbuild.build()
    if world > 1:
        dist.barrier()
    import paper_2111_06868_b200 as hq
    from hq_inputs import sycamore_circuit, circuit_sha256

    n, cycles, seed, kdef, cidx = CONFIGS[args.config]
    kmax = args.kmax or kdef
    gates = sycamore_circuit(n, cycles, seed)
    t0 = time.perf_counter()
    merged = args.fuse == "merged"
    fused = hq.hq_fuse(gates, kmax, merged=merged)
    plan_ms = (time.perf_counter() - t0) * 1e3
    es = 8 if args.dtype == "c64" else 16

    # PyTorch owns the device memory and the stream (plumbing); the library
    # only borrows them: this rank's shard and, for world > 1, its receive buffer
    nid = [None]
    if world > 1:
        nid = [hq.hq_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
    m_bits = world.bit_length() - 1
    cdt = torch.complex64 if args.dtype == "c64" else torch.complex128
    psi_t = torch.empty(2 ** (n - m_bits), dtype=cdt, device="cuda:%d" % local)
    buf_t = torch.empty_like(psi_t) if world > 1 else None
    stream = torch.cuda.Stream(device=local)
    state = hq.hq_state_create_rank_from_buffers(n, args.dtype, world, rank, psi_t.data_ptr(),
                                                 buf_t.data_ptr() if buf_t is not None else None,
                                                 stream.cuda_stream, nid[0])
    layout = None
    if world == 1 and not args.no_layout:
        t0 = time.perf_counter()
        layout, cost0, cost1 = hq.hq_plan_layout(n, 0, fused, args.dtype)
        plan_ms += (time.perf_counter() - t0) * 1e3
        hq.hq_state_set_layout(state, layout)
    circ = hq.hq_circuit_create(state, fused)
    info = hq.hq_circuit_info(circ)
    P, R = info["passes"], info["remaps"]
    state_bytes = es * 2 ** n                     # whole job
    work_bytes = P * 2 * state_bytes              # algorithmic HBM bytes per step (all ranks)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # ---- warmup
    for _ in range(args.warmup):
        hq.hq_state_init_basis(state, 0)      # also restores the canonical qubit layout
        hq.hq_circuit_run(state, circ)
    hq.hq_sync(state)

    # ---- timed region
    clocks = ClockSampler(local)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    hq.hq_stats_reset(state)
    hq.hq_profile_enable(state, True)
    hq.hq_kernel_times(state)
    barrier()
    clocks.start()
    for i in range(args.steps):
        hq.hq_state_init_basis(state, 0)
        with torch.cuda.stream(stream):
            starts[i].record(stream)
        hq.hq_circuit_run(state, circ)
        with torch.cuda.stream(stream):
            ends[i].record(stream)
    barrier()
    clk = clocks.stop()
    hq.hq_profile_enable(state, False)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kt_paths = {p: hq.hq_kernel_times(state, p) for p in ("tc", "simt", "generic")}
    stats = hq.hq_stats_get(state)
    nrm = hq.hq_norm(state)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        l = torch.tensor([stats["kernel_launches"]], device="cuda", dtype=torch.float64)
        dist.all_reduce(l)
        launches = int(l.item())
    else:
        launches = int(stats["kernel_launches"])
    ms_per_step = total_ms / args.steps
    value = work_bytes / (ms_per_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (largest share of apply time)
    peak, peak_src = peaks()
    dom = max(kt_paths, key=lambda p: kt_paths[p]["total_ms"])
    kt = kt_paths[dom]
    avg_ms = kt["total_ms"] / max(kt["count"], 1)
    bytes_per_launch = kt["bytes"] / max(kt["count"], 1)
    achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9
    traffic, traffic_src = traffic_from_profiles(args.config, kmax, dom, bytes_per_launch)
    names = {"tc": "apply_tcb / apply_tcL(b) (tcgen05, TMA bulk-copy producers, 3-term split products)", "simt": "apply_reg (SIMT FFMA2)",
             "generic": "apply_gen (generic SIMT)"}
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": names[dom], "launches": kt["count"],
            "avg_launch_ms": avg_ms, "algorithmic_bytes_per_launch": bytes_per_launch,
            "share_of_step": kt["total_ms"] / max(total_ms, 1e-9) if world == 1 else None,
            "other_kernels": {p: {"launches": v["count"], "total_ms": v["total_ms"]}
                              for p, v in kt_paths.items() if p != dom and v["count"]},
            "peak_source": peak_src}

    # ---- e2e through the public API with host inputs
    e2e_ms = []
    h2d = sum(es * (4 ** len(q)) for q, _ in fused)
    for i in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        barrier()
        t0 = time.perf_counter()
        hq.hq_state_init_basis(state, 0)
        fz = hq.hq_fuse(gates, kmax, merged=merged)
        if layout is not None:
            hq.hq_state_set_layout(state, hq.hq_plan_layout(n, 0, fz, args.dtype)[0])
            hq.hq_state_init_basis(state, 0)
        hq.hq_apply_circuit(state, fz)
        nv = hq.hq_norm(state)           # D2H of the result, synchronises
        barrier()
        if i > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e = None
    if e2e_ms:
        e2e_t = statistics.mean(e2e_ms)
        if world > 1:
            t = torch.tensor([e2e_t], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = float(t.item())
        e2e = {"value": work_bytes / (e2e_t * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * 148 * 16,
               "ms_per_step": e2e_t,
               "api": "hq_fuse + hq_plan_layout + hq_state_set_layout + hq_state_init_basis + "
                      "hq_apply_circuit + hq_norm"}

    line = {
        "metric": "state-update GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": "%s Sycamore-style d%d random circuit, fused k<=%d (BASELINE configs[%d])"
                               % (args.config, cycles, kmax, cidx),
                   "n": n, "cycles": cycles, "seed": seed, "kmax": kmax, "gates": len(gates),
                   "passes": P, "remaps": R, "circuit_sha256": circuit_sha256(gates),
                   "state_gib": state_bytes / 2 ** 30,
                   "l2": "no flush: state %.0f GiB >> 126 MB L2" % (state_bytes / 2 ** 30),
                   "parallelism": "sv-shard%d" % world,
                   "layout": "hq_plan_layout" if layout is not None else "default",
                   "fusion": "hq_fuse_merged (C7 groups + convex merging)" if merged else "hq_fuse (C7)"},
        "circuit_wall_s": ms_per_step / 1e3,
        "per_gpu_gbs": value / world,
        "frac_of_hbm_per_gpu": value / world / peak,
        "plan_ms": plan_ms,
        "norm_after": nrm,
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, inf = oracle_sample(n, cycles, seed, kmax, seconds=15.0, merged=merged)
        line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": inf["cores"], "kind": "oracle",
                                "sample": inf["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_hq(args)


if __name__ == "__main__":
    sys.exit(main())
