#!/usr/bin/env python
"""Benchmark: state-update GB/s and circuit wall time for a Sycamore-style
random circuit through the C ABI (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 34q] [--kmax 4]
    python bench.py --impl reference ...      # the fp64 CPU oracle arm

A "step" is one pass of the whole hot path over one synthetic circuit: every
fused apply pass and every remap of the compiled circuit (hq_circuit_run), on
the device.  The fused gate list and the layout are planned before the timed
region (reported as plan_ms); the state (2^n complex64) is initialised to |0>
before each step, outside the per-step CUDA events; the norm is read once
after the timed region (norm_after).

value  = passes * 2 * (state bytes) / circuit time (whole job, all GPUs),
         device-timed with CUDA events on the library's stream, max over ranks.
e2e    = the same metric through the public API with host inputs: per step
         hq_fuse(host gates) + layout + hq_apply_circuit (matrices copied H2D)
         + hq_norm (the step's result read back to the host), host wall
         clock; the H2D/D2H byte counts are the library's own (hq_stats).
         Only the norm comes back: the 128 GiB state is never copied out.
sweep  = (N=1) the fused-gate sweep of BASELINE configs[2] on the bench's own
         dense state: one Haar k-qubit gate per k=1..6 at the low / spread /
         random0 placements, median of 5 passes, as a fraction of the HBM peak.
other_configs = (N=1, 34q) BASELINE configs[0] (12q d10) and configs[1] (30q
         d20, 2-qubit fused gates) on their own buffers, circuit time.
The planner is hq_fuse_blocks (--fuse c7 for the paper's greedy rule).
For N>1 the same circuit is strong-scaled: the state is sharded on the top
log2 N qubits and remaps run fused into the preceding apply pass (peer writes
over NVLink, CUDA IPC) or as NCCL exchanges; the line then carries a parity
object computed through that transport (mirror circuit C.C^dagger distance
from |0>, pin P9; reversible circuit |x> -> |f(x)> bit-exact, P10).
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
    ap.add_argument("--fuse", default="blocks", choices=["blocks", "c7"],
                    help="planner: hq_fuse_blocks (default) or the plain C7 greedy hq_fuse")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the configs[0] / configs[1] circuits appended to the N=1 line")
    ap.add_argument("--sweep-reps", type=int, default=5,
                    help="N=1: passes per fused-gate sweep cell on the bench state (0: no sweep)")
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
# Fused pass count P of the GPU arm's plan per (config, kmax, planner).  Both
# arms express their time in the same unit, P * 2 * (c64 state bytes) / T, so
# the driver's ratio of the two values is the ratio of circuit times.  The GPU
# arm checks its own P against this table (unit_passes_match); the 34q entry
# is pinned by tests/test_abi_cpu.py::test_fuse_blocks_bench_circuits.
UNIT_PASSES = {
    ("12q", 2, "blocks"): 43, ("12q", 4, "blocks"): 10, ("12q", 5, "blocks"): 9, ("12q", 6, "blocks"): 7,
    ("12q", 2, "c7"): 43, ("12q", 4, "c7"): 16, ("12q", 5, "c7"): 17, ("12q", 6, "c7"): 15,
    ("30q", 2, "blocks"): 245, ("30q", 4, "blocks"): 70, ("30q", 5, "blocks"): 49, ("30q", 6, "blocks"): 33,
    ("30q", 2, "c7"): 245, ("30q", 4, "c7"): 101, ("30q", 5, "c7"): 100, ("30q", 6, "c7"): 67,
    ("34q", 2, "blocks"): 280, ("34q", 4, "blocks"): 79, ("34q", 5, "blocks"): 59, ("34q", 6, "blocks"): 36,
    ("34q", 2, "c7"): 280, ("34q", 4, "c7"): 116, ("34q", 5, "c7"): 115, ("34q", 6, "c7"): 80,
    ("36q", 2, "blocks"): 360, ("36q", 4, "blocks"): 100, ("36q", 5, "blocks"): 79, ("36q", 6, "blocks"): 42,
    ("36q", 2, "c7"): 360, ("36q", 4, "c7"): 144, ("36q", 5, "c7"): 144, ("36q", 6, "c7"): 96,
}
ORACLE_SAMPLE_N = 26     # the oracle's c128 state at n=26 is 1 GiB; the full 725-gate circuit takes ~15 s


class OracleRun:
    """The fp64 oracle (as it stands, all host threads) on the same
    generator's circuit at n_sample qubits, gate by gate from |0>; run(m)
    applies the next m gates and returns their wall time."""

    def __init__(self, n_sample, cycles, seed):
        import oracle as O
        from hq_inputs import sycamore_circuit
        self.O = O
        self.gates = sycamore_circuit(n_sample, cycles, seed)
        self.psi = O.init_basis(n_sample, 0)
        self.next = 0

    def run(self, m):
        hi = min(self.next + m, len(self.gates))
        t0 = time.perf_counter()
        for g in self.gates[self.next:hi]:
            self.O.apply_gate(self.psi, g.U, g.qubits)
        dt = time.perf_counter() - t0
        done, self.next = hi - self.next, hi
        return dt, done


def oracle_unit_value(n_full, cycles, seed, P, seconds, gates_timed, n_sample=ORACLE_SAMPLE_N):
    """The oracle's time per unfused gate at n_sample, extrapolated x2^(n_full -
    n_sample) per gate to the n_full circuit, in the GPU arm's unit."""
    from hq_inputs import sycamore_circuit
    n_gates_full = len(sycamore_circuit(n_full, cycles, seed))
    per_gate = seconds / max(gates_timed, 1) * 2 ** (n_full - n_sample)
    T_full = per_gate * n_gates_full
    return P * 2 * 8 * 2 ** n_full / T_full / 1e9, T_full


def oracle_full_circuit(n, cycles, seed, threads=None):
    """The whole unfused circuit through the oracle (configs[0] size), wall time."""
    import oracle as O
    from hq_inputs import sycamore_circuit
    gates = sycamore_circuit(n, cycles, seed)
    old = O.max_threads()
    if threads:
        O.set_threads(threads)
    try:
        t0 = time.perf_counter()
        O.simulate(n, gates)
        return time.perf_counter() - t0, len(gates)
    finally:
        O.set_threads(old)


def cpu_baseline_block(config, kmax, fusion):
    """cpu_baseline of the N=1 GPU line: the oracle on the complete 26-qubit
    circuit of the same generator (~15 s, extrapolated per gate to the bench
    circuit, the same sample the reference arm times), plus the full
    configs[0] circuit (12q d10) on all host threads and on one thread
    (SURVEY §8(d) "Oracle timing")."""
    import oracle as O
    n, cycles, seed, _, _ = CONFIGS[config]
    P = UNIT_PASSES[(config, kmax, fusion)]
    n_s = min(n, ORACLE_SAMPLE_N)
    run = OracleRun(n_s, cycles, seed)
    sec, done = run.run(len(run.gates))
    value, T_full = oracle_unit_value(n, cycles, seed, P, sec, done, n_s)
    t12, g12 = oracle_full_circuit(12, 10, 0)
    t12_1, _ = oracle_full_circuit(12, 10, 0, threads=1)
    return {"value": value, "unit": "GB/s", "cores": O.max_threads(), "kind": "oracle",
            "sample": "all %d unfused gates of the same generator's circuit at n=%d (c128, %.1f s), "
                      "extrapolated x2^%d per gate to the n=%d circuit (%.0f s), in the GPU arm's unit "
                      "(P=%d passes x 2 x c64 state bytes / time)" % (done, n_s, sec, n - n_s, n, T_full, P),
            "extrapolated_circuit_s": T_full,
            "config0_full_circuit": {"workload": "12q d10 seed 0 (BASELINE configs[0]), %d unfused gates, fp64"
                                                 % g12,
                                     "seconds_all_threads": t12, "threads": O.max_threads(),
                                     "seconds_1_thread": t12_1}}


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands on the host cores.  The
    K timed steps together run the complete 26-qubit circuit of the bench's
    generator once (step i = the i-th contiguous slice of its gates; the
    same ~15 s sample as the GPU line's cpu_baseline); the W warm-up steps
    run one gate each.  Value = the extrapolated rate in the GPU arm's unit."""
    import oracle as O
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    n, cycles, seed, kdef, cidx = CONFIGS[args.config]
    kmax = args.kmax or kdef
    P = UNIT_PASSES[(args.config, kmax, args.fuse)]
    n_s = min(n, ORACLE_SAMPLE_N)
    warm = OracleRun(n_s, cycles, seed)
    for i in range(args.warmup):
        warm.run(1)
    del warm
    run = OracleRun(n_s, cycles, seed)
    ng_s = len(run.gates)
    K = max(args.steps, 1)
    bounds = [round(i * ng_s / K) for i in range(K + 1)]
    sec, done = 0.0, 0
    for i in range(K):
        t, g = run.run(bounds[i + 1] - bounds[i])
        sec += t
        done += g
    value, T_full = oracle_unit_value(n, cycles, seed, P, sec, done, n_s)
    sample = ("all %d unfused gates of the same generator's circuit at n=%d (c128, %.1f s) in %d timed slices, "
              "extrapolated x2^%d per gate to the n=%d circuit" % (done, n_s, sec, K, n - n_s, n))
    line = {
        "impl": "reference", "metric": "state-update GB/s", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": T_full * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s Sycamore-style d%d random circuit (BASELINE configs[%d]), "
                               "oracle unfused fp64; ms_per_step = the extrapolated full-circuit time"
                               % (args.config, cycles, cidx),
                   "n": n, "cycles": cycles, "seed": seed, "kmax": kmax, "unit_passes": P},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": O.max_threads(), "kind": "oracle",
                         "sample": sample},
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
    blocks = args.fuse == "blocks"
    fused = hq.hq_fuse(gates, kmax, blocks=blocks)
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
    if not args.no_layout:
        # the same planned layout on every rank: local bits by the pass cost
        # model, and (world > 1) the first global set outside the schedule's
        # first segment, so that segment needs no remap
        t0 = time.perf_counter()
        layout, cost0, cost1 = hq.hq_plan_layout(n, m_bits, fused, args.dtype)
        plan_ms += (time.perf_counter() - t0) * 1e3
        hq.hq_state_set_layout(state, layout)
    fused_ok = hq.hq_state_set_remap_mode(state, "fused+gather") if world > 1 else False
    circ = hq.hq_circuit_create(state, fused)
    info = hq.hq_circuit_info(circ)
    P, R = info["passes"], info["remaps"]
    standalone_permutes = info["permutes"]
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
    e2e_ms, e2e_h2d, e2e_d2h = [], [], []
    for i in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        barrier()
        st0 = hq.hq_stats_get(state)
        t0 = time.perf_counter()
        hq.hq_state_init_basis(state, 0)
        fz = hq.hq_fuse(gates, kmax, blocks=blocks)
        if layout is not None:
            hq.hq_state_set_layout(state, hq.hq_plan_layout(n, m_bits, fz, args.dtype)[0])
            hq.hq_state_init_basis(state, 0)
        hq.hq_apply_circuit(state, fz)
        nv = hq.hq_norm(state)           # D2H of the result, synchronises
        barrier()
        if i > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
            st1 = hq.hq_stats_get(state)
            e2e_h2d.append(st1["h2d_bytes"] - st0["h2d_bytes"])
            e2e_d2h.append(st1["d2h_bytes"] - st0["d2h_bytes"])
    e2e = None
    if e2e_ms:
        e2e_t = statistics.mean(e2e_ms)
        if world > 1:
            t = torch.tensor([e2e_t], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = float(t.item())
        e2e = {"value": work_bytes / (e2e_t * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(max(e2e_h2d)), "d2h_bytes_per_step": int(max(e2e_d2h)),
               "bytes_counted_by": "hq_stats h2d_bytes / d2h_bytes (every host<->device copy the library makes, "
                                   "this rank)",
               "ms_per_step": e2e_t,
               "readback": "the norm only (fp64 partial sums); the %.0f GiB state stays on the device"
                           % (state_bytes / 2 ** 30),
               "api": "hq_fuse + hq_plan_layout + hq_state_set_layout + hq_state_init_basis + "
                      "hq_apply_circuit + hq_norm"}

    # ---- N>1: correctness through the real transport (pins P9, P10)
    parity = None
    if world > 1:
        parity = remap_parity(hq, state, n, gates, kmax, blocks, world, rank, dist, torch)

    # ---- N=1: fused-gate sweep (BASELINE configs[2]) on this dense state
    sweep = None
    if world == 1 and args.sweep_reps > 0:
        sweep = run_sweep(hq, torch, psi_t, stream, n, args.dtype, args.sweep_reps)
    others = None
    if world == 1 and args.config == "34q" and args.dtype == "c64" and not args.no_other_configs:
        others = run_other_configs(hq, torch, stream)

    line = {
        "metric": "state-update GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": "%s Sycamore-style d%d random circuit, fused k<=%d (BASELINE configs[%d])"
                               % (args.config, cycles, kmax, cidx),
                   "n": n, "cycles": cycles, "seed": seed, "kmax": kmax, "gates": len(gates),
                   "passes": P, "remaps": R, "standalone_permutes": standalone_permutes,
                   "circuit_sha256": circuit_sha256(gates),
                   "unit_passes_match": UNIT_PASSES.get((args.config, kmax, args.fuse)) == P,
                   "state_gib": state_bytes / 2 ** 30,
                   "l2": "no flush: state %.0f GiB >> 126 MB L2" % (state_bytes / 2 ** 30),
                   "parallelism": "sv-shard%d" % world,
                   "layout": "hq_plan_layout" if layout is not None else "default",
                   "fusion": "hq_fuse_blocks (frontier block planner)" if blocks else "hq_fuse (C7)"},
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
    if parity is not None:
        line["parity"] = parity
    if world > 1:
        line["remaps_fused_per_step"] = stats["remaps_fused"] / max(args.steps, 1)
        line["remap_transport"] = ("fused into the apply pass (peer writes over NVLink, CUDA IPC); "
                                   "isolated global accesses as pair gathers" if fused_ok
                                   else "NCCL grouped send/recv")
        line["gathers_per_step"] = stats["gathers"] / max(args.steps, 1)
    if sweep is not None:
        line["sweep"] = sweep
    if others is not None:
        line["other_configs"] = others
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_block(args.config, kmax, args.fuse)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def reversible_image(n, gates, x):
    """f(x) of a permutation circuit by host bit operations (pin P10's
    definition): the target bits of the index are the column c of each gate
    (qubits[0] = MSB), the row r with U[r][c] = 1 replaces them."""
    import numpy as np
    y = int(x)
    for g in gates:
        k = len(g.qubits)
        c = 0
        for j, q in enumerate(g.qubits):
            c |= ((y >> (n - 1 - q)) & 1) << (k - 1 - j)
        r = int(np.flatnonzero(np.abs(np.asarray(g.U)[:, c]) > 0.5)[0])
        for j, q in enumerate(g.qubits):
            b = n - 1 - q
            y = (y & ~(1 << b)) | (((r >> (k - 1 - j)) & 1) << b)
    return y


def remap_parity(hq, state, n, gates, kmax, blocks, world, rank, dist, torch):
    """Correctness of the sharded path through the NCCL remaps, at full size:
    mirror circuit C.C^dagger from |0> (pin P9: returns to |0>; distance
    ||psi - |0>||_2 = sqrt(||psi||^2 - 2 Re psi_0 + 1) <= 1e-4 in complex64)
    and a reversible circuit of permutation gates on every qubit from a basis
    state |x> (pin P10: exactly |f(x)>, compared with ==)."""
    import numpy as np
    from hq_inputs import Gate, reversible_circuit

    def amp(i):        # amplitude i, owned by one rank; the others contribute 0
        a = np.zeros(1, dtype=np.complex64)
        hq.hq_get_amplitudes(state, i, 1, a)
        owner = 1.0 if a[0] != 0 else 0.0
        t = torch.tensor([float(a[0].real), float(a[0].imag), owner], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return complex(t[0].item(), t[1].item()), t[2].item()

    out = {}
    mirror = list(gates) + [Gate(g.name + "^dag", g.qubits, np.conj(np.asarray(g.U)).T) for g in reversed(gates)]
    fz = hq.hq_fuse(mirror, kmax, blocks=blocks)
    c = hq.hq_circuit_create(state, fz)
    info = hq.hq_circuit_info(c)
    s_begin = hq.hq_stats_get(state)
    hq.hq_state_init_basis(state, 0)
    hq.hq_circuit_run(state, c)
    nrm = hq.hq_norm(state)
    a0, _ = amp(0)
    dist_ = float(np.sqrt(max(nrm ** 2 - 2 * a0.real + 1, 0.0)))
    out["mirror_dist"] = dist_
    out["mirror_ok"] = dist_ <= 1e-4
    out["mirror_passes"], out["mirror_remaps"] = info["passes"], info["remaps"]
    del c
    rev = reversible_circuit(n, 4 * n, 4242, kmax=3)
    x = int.from_bytes(np.random.default_rng(4243).bytes(8), "little") & ((1 << n) - 1)
    y = reversible_image(n, rev, x)
    fz = hq.hq_fuse(rev, kmax, blocks=blocks)
    st0 = hq.hq_stats_get(state)
    hq.hq_state_init_basis(state, x)
    hq.hq_apply_circuit(state, fz)
    st1 = hq.hq_stats_get(state)
    ay, owners = amp(y)
    nrm = hq.hq_norm(state)
    out["reversible_exact"] = bool(ay == 1.0 and owners == 1.0 and nrm == 1.0)
    out["reversible_remaps"] = st1["remaps"] - st0["remaps"]
    s_end = hq.hq_stats_get(state)
    fused = s_end["remaps_fused"] - s_begin["remaps_fused"]
    total = s_end["remaps"] - s_begin["remaps"]
    out["remaps_fused"], out["remaps_total"] = fused, total
    out["transport"] = ("%d of %d remaps fused into the apply pass (peer writes), the rest NCCL grouped "
                        "send/recv, between %d ranks" % (fused, total, world))
    return out


def run_sweep(hq, torch, psi_t, stream, n, dtype, reps, ks=(1, 2, 3, 4, 5, 6),
              placements=("low", "spread", "random0")):
    """BASELINE configs[2] on the bench's own buffer: the dense state the
    circuit left (a default-layout view of the same memory), one Haar k-qubit
    gate per (k, placement), 1 warm-up + `reps` passes, CUDA events on the
    library's stream; fraction of the measured HBM peak per cell."""
    import numpy as np
    from hq_inputs import haar_sweep_gate
    peak, _ = peaks()
    es = 8 if dtype == "c64" else 16
    nbytes = 2 * es * 2 ** n
    s = hq.hq_state_create_from_buffers(n, dtype, psi_t.data_ptr(), stream.cuda_stream)
    cells = {}
    for k in ks:
        for pl in placements:
            g = haar_sweep_gate(n, k, pl, 2000 + k)
            hq.hq_apply_matrix(s, g.U, g.qubits)
            ev = []
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                hq.hq_apply_matrix(s, g.U, g.qubits)
                b.record(stream)
                ev.append((a, b))
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(b) for a, b in ev)
            cells["k%d_%s" % (k, pl)] = {"phys_bits": sorted(n - 1 - q for q in g.qubits), "median_ms": ms,
                                         "frac": nbytes / (ms * 1e-3) / 1e9 / peak}
    nrm = hq.hq_norm(s)
    s.close()
    return {"workload": "BASELINE configs[2] cells on the %dq bench state (dense after the circuit), "
                        "median of %d passes" % (n, reps),
            "cells": cells, "min_frac_k_le_5": min(v["frac"] for key, v in cells.items() if int(key[1]) <= 5),
            "norm_after": nrm}


def run_other_configs(hq, torch, stream, reps=5, names=("12q", "30q")):
    """BASELINE configs[0] (12q d10, k <= 6) and configs[1] (30q d20, 2-qubit
    fused gates) on their own PyTorch buffers beside the bench state: the
    compiled circuit from |0> with the planned layout, 2 warm-up + `reps`
    timed runs (CUDA events on the library's stream), median."""
    from hq_inputs import sycamore_circuit
    peak, _ = peaks()
    out = {}
    for name in names:
        n, cycles, seed, kmax, cidx = CONFIGS[name]
        gates = sycamore_circuit(n, cycles, seed)
        fused = hq.hq_fuse(gates, kmax, blocks=True)
        psi = torch.empty(2 ** n, dtype=torch.complex64, device="cuda")
        s = hq.hq_state_create_from_buffers(n, "c64", psi.data_ptr(), stream.cuda_stream)
        hq.hq_state_set_layout(s, hq.hq_plan_layout(n, 0, fused, "c64")[0])
        circ = hq.hq_circuit_create(s, fused)
        P = hq.hq_circuit_info(circ)["passes"]
        ms = []
        for i in range(reps + 2):
            hq.hq_state_init_basis(s, 0)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            hq.hq_circuit_run(s, circ)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                ms.append(a.elapsed_time(b))
        nrm = hq.hq_norm(s)
        t = statistics.median(ms)
        gbs = P * 2 * 8 * 2 ** n / (t * 1e-3) / 1e9
        out[name] = {"workload": "%s Sycamore-style d%d, seed %d, fused k<=%d (BASELINE configs[%d]), c64"
                                 % (name, cycles, seed, kmax, cidx),
                     "gates": len(gates), "passes": P, "circuit_ms": t, "state_update_gbs": gbs,
                     "frac_of_hbm": gbs / peak, "norm_after": nrm}
        del circ                  # hq_circuit_destroy (Circuit.__del__) before the state
        s.close()
        del psi
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_hq(args)


if __name__ == "__main__":
    sys.exit(main())
