"""Noisy circuits by pure-state sampling of the Kraus operators (row f3).

PAPER P:1032-1041: "Noise can be simulated either at the density matrix
level, or by pure state sampling of the Kraus operators ... Pure state
sampling allows one to reach larger system sizes".  SPEC S:522-530, S:544:
per shot, evolve a pure state; at each channel compute p_i = ||K_i psi||^2,
sample i, set psi <- K_i psi / sqrt(p_i); averages converge at O(1/sqrt(shots));
shots are embarrassingly parallel, each with a private RNG stream
(seed = base_seed + shot index), results reduced by summation.

Everything numerical runs in the C ABI: the unitary stretches between
channels are fused (hq_fuse) and compiled once (hq_circuit_create), every
channel is one hq_kraus_sample (a reduced-density-matrix read pass plus one
apply pass), and the observable is hq_reduced_dm.  This module only orders the
calls, draws the uniforms and sums.  Shots shard round-robin over ranks with
no data-path collective; the per-rank sums are added with one all-reduce of a
few doubles at the end.

For small systems one shot per state is launch-bound, so `batch=B` advances B
shots in one state of n + log2(B) qubits (shot index on the top qubits): every
unitary pass serves all B shots, and a channel is one batched
reduced-density-matrix pass plus one apply pass with a per-shot matrix
(hq_reduced_dm_batched / hq_kraus_sample_batched).
"""
import numpy as np

from . import hq


class Channel:
    """A Kraus channel {K_i} on qubits (1 <= k <= 3)."""

    def __init__(self, qubits, kraus, name="K"):
        self.qubits = tuple(int(q) for q in qubits)
        self.kraus = [np.asarray(K, dtype=np.complex128) for K in kraus]
        self.name = name
        d = 2 ** len(self.qubits)
        if not 1 <= len(self.qubits) <= 3 or any(K.shape != (d, d) for K in self.kraus):
            raise ValueError("channel on %d qubits needs %dx%d Kraus matrices" % (len(self.qubits), d, d))


def shard_shots(n_shots, rank, world):
    """Shots of this rank: s = rank, rank + world, ... (round robin)."""
    return list(range(rank, n_shots, world))


def shot_rng(seed, shot):
    """The private uniform stream of one shot (seed = base + shot)."""
    return np.random.default_rng(seed + shot)


def split_segments(ops):
    """[gates..., Channel, gates..., ...] -> list of ('U', [gates]) / ('K', Channel)."""
    segs, cur = [], []
    for op in ops:
        if isinstance(op, Channel):
            if cur:
                segs.append(("U", cur))
                cur = []
            segs.append(("K", op))
        else:
            cur.append(op)
    if cur:
        segs.append(("U", cur))
    return segs


def reduce_sum(arr, group=None):
    """Sum a float64 array over the ranks of a torch.distributed group (no-op
    for a single process).  The only collective of the trajectory path."""
    if group is None:
        return np.asarray(arr, dtype=np.float64)
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.as_tensor(np.asarray(arr, dtype=np.float64), device=dev)
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def sample_trajectories(n, ops, n_shots, observe, seed=0, init="0", dtype="c64", kmax=6,
                        rank=0, world=1, group=None, per_step=None, batch=1):
    """Run this rank's share of `n_shots` trajectories of the noisy circuit
    `ops` (gates as (qubits, U) or objects with .qubits/.U, and Channel
    objects) from the token state `init`, and return the mean over ALL shots
    of the reduced density matrix of `observe` (k <= 3 qubits) at the end.

    per_step: optional list of op indices after which the reduced density
    matrix is also recorded (means returned as a list in that order).
    batch: shots advanced together in one state of n + log2(batch) qubits
    (a power of two; hq_kraus_sample_batched).  Each shot keeps its own
    uniform stream, so the branch choices are those of batch=1."""
    if batch > 1:
        return _sample_batched(n, ops, n_shots, observe, seed, init, dtype, kmax, rank, world, group,
                               per_step, batch)
    segs = split_segments(ops)
    marks = sorted(set(per_step or []))
    # op index -> segment boundary: record after segment j when its last op index is marked
    bounds, idx = [], -1
    for kind, body in segs:
        idx += len(body) if kind == "U" else 1
        bounds.append(idx)
    if any(m not in bounds for m in marks):
        raise ValueError("per_step indices must end a unitary stretch or be a channel")
    s = hq.hq_state_create(n, dtype, 1)
    compiled = []
    for kind, body in segs:
        compiled.append(hq.hq_circuit_create(s, hq.hq_fuse(body, kmax)) if kind == "U" else body)
    d = 2 ** len(observe)
    nrec = len(marks) + 1
    acc = np.zeros((nrec, d, d), dtype=np.complex128)
    chosen = []
    mine = shard_shots(n_shots, rank, world)
    for shot in mine:
        rng = shot_rng(seed, shot)
        hq.hq_state_init_tokens(s, init)
        picks, r = [], 0
        for j, ((kind, _), item) in enumerate(zip(segs, compiled)):
            if kind == "U":
                hq.hq_circuit_run(s, item)
            else:
                i, _ = hq.hq_kraus_sample(s, item.kraus, item.qubits, rng.random())
                picks.append(i)
            if r < len(marks) and bounds[j] == marks[r]:
                acc[r] += hq.hq_reduced_dm(s, observe)
                r += 1
        acc[-1] += hq.hq_reduced_dm(s, observe)
        chosen.append(picks)
    flat = np.concatenate([acc.real.ravel(), acc.imag.ravel(), [len(mine)]])
    tot = reduce_sum(flat, group)
    m = nrec * d * d
    mean = (tot[:m] + 1j * tot[m:2 * m]).reshape(nrec, d, d) / max(tot[-1], 1)
    return {"rho": mean[-1], "rho_steps": list(mean[:-1]), "shots": int(tot[-1]), "chosen": chosen}


def _sample_batched(n, ops, n_shots, observe, seed, init, dtype, kmax, rank, world, group, per_step, batch):
    nb = int(batch).bit_length() - 1
    if 1 << nb != batch:
        raise ValueError("batch must be a power of two")
    segs = split_segments(ops)
    marks = sorted(set(per_step or []))
    bounds, idx = [], -1
    for kind, body in segs:
        idx += len(body) if kind == "U" else 1
        bounds.append(idx)
    if any(m not in bounds for m in marks):
        raise ValueError("per_step indices must end a unitary stretch or be a channel")

    def shift(g):
        qs = g.qubits if hasattr(g, "qubits") else g[0]
        U = g.U if hasattr(g, "U") else g[1]
        return (tuple(int(q) + nb for q in qs), U)

    s = hq.hq_state_create(n + nb, dtype, 1)
    compiled = []
    for kind, body in segs:
        if kind == "U":
            compiled.append(hq.hq_circuit_create(s, hq.hq_fuse([shift(g) for g in body], kmax)))
        else:
            compiled.append(Channel([q + nb for q in body.qubits], body.kraus, body.name))
    tokens = "+" * nb + (init * n if len(init) == 1 else init)
    obs = [q + nb for q in observe]
    d = 2 ** len(observe)
    nrec = len(marks) + 1
    acc = np.zeros((nrec, d, d), dtype=np.complex128)
    chosen = []
    mine = shard_shots(n_shots, rank, world)
    for b0 in range(0, len(mine), batch):
        shots = mine[b0:b0 + batch]
        live = len(shots)
        rngs = [shot_rng(seed, sh) for sh in shots] + [np.random.default_rng(0)] * (batch - live)
        hq.hq_state_init_tokens(s, tokens)
        picks, r = [[] for _ in range(live)], 0

        def record(slot):
            acc[slot] += hq.hq_reduced_dm_batched_sum(s, nb, obs, live)

        for j, ((kind, _), item) in enumerate(zip(segs, compiled)):
            if kind == "U":
                hq.hq_circuit_run(s, item)
            else:
                u = np.array([g.random() for g in rngs[:live]] + [0.5] * (batch - live))
                ci, _ = hq.hq_kraus_sample_batched(s, nb, item.kraus, item.qubits, u)
                for t in range(live):
                    picks[t].append(int(ci[t]))
            if r < len(marks) and bounds[j] == marks[r]:
                record(r)
                r += 1
        record(-1)
        chosen.extend(picks)
    flat = np.concatenate([acc.real.ravel(), acc.imag.ravel(), [len(mine)]])
    tot = reduce_sum(flat, group)
    m = nrec * d * d
    mean = (tot[:m] + 1j * tot[m:2 * m]).reshape(nrec, d, d) / max(tot[-1], 1)
    return {"rho": mean[-1], "rho_steps": list(mean[:-1]), "shots": int(tot[-1]), "chosen": chosen}
