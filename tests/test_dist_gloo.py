"""Multi-process check of the distributed schedule's host logic (world_size 2,
gloo backend, CPU).  Each rank owns its shard of the physical index space and
executes the op stream hq_schedule emits: APPLY with the oracle on the local
shard, REMAP as the library's own transfer list (hq_remap_plan: the runs
exec_remap sends and receives with NCCL) over torch.distributed point-to-point,
PERMUTE as a local bit swap.  Rank 0 gathers the shards and
compares the logical state with the oracle (bit-exact for a reversible
circuit, 1e-12 for Haar gates).  This is the same exchange exec_remap issues
through NCCL on GPUs (one send/recv pair per contiguous run)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import oracle as O
        import paper_2111_06868_b200 as hq
        from hq_inputs import reversible_circuit, random_circuit, integer_state, random_state
        from sched_replay import apply_on_shard, permute_bits, to_logical

        m = world.bit_length() - 1
        nl = n - m
        if kind == "reversible":
            gates = reversible_circuit(n, 60, 13, kmax=3)
            psi0 = integer_state(n, 2)
        else:
            gates = random_circuit(n, 50, 17, kmax=4)
            psi0 = random_state(n, 4)
        ops, pi = hq.hq_schedule(n, m, gates)
        shard = psi0[rank << nl:(rank + 1) << nl].copy()
        for op in ops:
            if op["kind"] == "apply":
                g = gates[op["gate"]]
                apply_on_shard(shard, nl, g.U, op["bits"][:len(g.qubits)], rank)
            elif op["kind"] == "permute":
                pairs = [(op["bits"][2 * i], op["bits"][2 * i + 1]) for i in range(op["nbits"])]
                shard = permute_bits(shard, pairs)
            else:
                # the library's own transfer list (hq_remap_plan, the list
                # exec_remap issues as NCCL send/recv), moved over gloo
                new = np.empty_like(shard)
                reqs, recv_bufs = [], []
                for p, a, ln in hq.hq_remap_plan(n, m, op, rank):
                    src = shard[a:a + ln]
                    if p == rank:
                        new[a:a + ln] = src
                        continue
                    send = torch.from_numpy(np.ascontiguousarray(src).view(np.float64).copy())
                    recv = torch.empty_like(send)
                    reqs.append(dist.isend(send, p))
                    reqs.append(dist.irecv(recv, p))
                    recv_bufs.append((a, ln, recv))
                for r in reqs:
                    r.wait()
                for a, ln, recv in recv_bufs:
                    new[a:a + ln] = recv.numpy().view(np.complex128)
                shard = new
        parts = [torch.empty(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
        if rank == 0:
            shards = [p.numpy().view(np.complex128) for p in parts]
            got = to_logical(n, shards, pi)
            want = O.simulate(n, gates, psi0)
            nrem = sum(o["kind"] == "remap" for o in ops)
            if kind == "reversible":
                q.put(("ok" if np.array_equal(got, want) else "mismatch", nrem))
            else:
                q.put(("ok" if np.max(np.abs(got - want)) < 1e-12 else "mismatch", nrem))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["reversible", "haar"])
def test_schedule_over_gloo_world2(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 10, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    status, nrem = q.get(timeout=5)
    assert status == "ok"
    assert nrem > 0


def _traj_worker(rank, world, port, q):
    """Row f3 host logic over gloo: shots shard round robin (shard_shots),
    each with its private stream (shot_rng), per-rank sums added by the one
    all-reduce (reduce_sum).  The per-shot numerics here are the oracle's
    trajectory step (the GPU path does them with hq_kraus_sample)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle as O
        from paper_2111_06868_b200.trajectories import shard_shots, shot_rng, reduce_sum
        n, shots, seed = 3, 37, 11
        p = 0.2
        K = [np.sqrt(1 - p) * np.eye(2), np.sqrt(p) * np.diag([1.0, -1.0])]
        H = np.array([[1, 1], [1, -1]]) / np.sqrt(2)

        def run(shot):
            rng = shot_rng(seed, shot)
            psi = O.init_tokens(n, "0")
            for q_ in range(n):
                O.apply_gate(psi, H, [q_])
            for step in range(3):
                psi, _, _ = O.kraus_sample_step(psi, K, [step % n], rng.random())
            return O.reduced_dm(psi, [0, 2])

        acc = np.zeros((4, 4), dtype=complex)
        mine = shard_shots(shots, rank, world)
        for s in mine:
            acc += run(s)
        tot = reduce_sum(np.concatenate([acc.real.ravel(), acc.imag.ravel(), [len(mine)]]), dist.group.WORLD)
        if rank == 0:
            ref = sum(run(s) for s in range(shots)) / shots
            mean = (tot[:16] + 1j * tot[16:32]).reshape(4, 4) / tot[-1]
            ok = tot[-1] == shots and np.max(np.abs(mean - ref)) < 1e-14
            cover = sorted(shard_shots(shots, 0, world) + shard_shots(shots, 1, world)) == list(range(shots))
            q.put("ok" if ok and cover else "mismatch")
    finally:
        dist.destroy_process_group()


def test_trajectory_shots_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_traj_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == "ok"
