"""Test helper: replay an hq_schedule op stream on CPU shards.

APPLY ops run through the oracle (plain fp64 apply) on the local shard with the
op's physical target bits; REMAP ops exchange contiguous chunks exactly as
include/hq.h documents (chunk t of rank r -> peer with swapped rank bits = t,
landing in chunk bits(r)); PERMUTE ops swap local index bits.  Used by the
CPU tests of the distribution logic (single process and gloo world_size 2).
"""
import numpy as np

import oracle as O


def phys_apply(shard, nl, U, phys_bits):
    """Apply U with qubits[j] at physical bit phys_bits[j] of an nl-bit shard
    (oracle qubit label of physical bit p is nl-1-p)."""
    O.apply_gate(shard, U, [nl - 1 - p for p in phys_bits])


def cond_block(U, phys_bits, nl, rank):
    """Row f1: for an APPLY whose bits include global positions (>= nl), the
    block of U rank `rank` applies: rows/columns whose global-target bits equal
    the rank's bits, on the local targets.  Returns (V, local bits)."""
    k = len(phys_bits)
    fix, loc = 0, []
    for j, b in enumerate(phys_bits):
        if b >= nl:
            fix |= ((rank >> (b - nl)) & 1) << (k - 1 - j)
        else:
            loc.append(j)
    idx = []
    for a in range(2 ** len(loc)):
        x = fix
        for t, j in enumerate(loc):
            x |= ((a >> (len(loc) - 1 - t)) & 1) << (k - 1 - j)
        idx.append(x)
    return U[np.ix_(idx, idx)], [phys_bits[j] for j in loc]


def apply_on_shard(shard, nl, U, phys_bits, rank):
    """Apply a scheduled gate on one shard (conditioned when a bit is global)."""
    if all(b < nl for b in phys_bits):
        phys_apply(shard, nl, U, phys_bits)
        return
    V, lb = cond_block(np.asarray(U), phys_bits, nl, rank)
    if lb:
        phys_apply(shard, nl, V, lb)
    else:
        shard *= V[0, 0]


def permute_bits(shard, pairs):
    idx = np.arange(shard.size, dtype=np.int64)
    dst = idx.copy()
    for a, b in pairs:
        ba = (idx >> a) & 1
        bb = (idx >> b) & 1
        dst &= ~((1 << a) | (1 << b))
        dst |= (ba << b) | (bb << a)
    out = np.empty_like(shard)
    out[dst] = shard
    return out


def remap_runs(nl, pairs):
    """Run decomposition of a REMAP (see exec_remap): returns (mp, gsh, lmask,
    lmin, runlen, nruns, run_start(rho, t))."""
    mp = len(pairs)
    gsh = [a - nl for a, _ in pairs]
    lb = [b for _, b in pairs]
    lmask = sum(1 << b for b in lb)
    lmin = min(lb)

    def run_start(rho, t):
        x, src, b = 0, rho << lmin, 0
        for pos in range(nl):
            if (lmask >> pos) & 1:
                x |= ((t >> lb.index(pos)) & 1) << pos
            else:
                x |= ((src >> b) & 1) << pos
                b += 1
        return x
    return mp, gsh, lmask, lmin, 1 << lmin, 1 << (nl - mp - lmin), run_start


def peer_of(r, t, gsh):
    p = r
    for i, g in enumerate(gsh):
        p = (p & ~(1 << g)) | (((t >> i) & 1) << g)
    return p


def bits_of(r, gsh):
    return sum(((r >> g) & 1) << i for i, g in enumerate(gsh))


def replay_all_shards(n, m, gates, ops, psi_logical):
    """Single-process replay over all 2^m shards; returns the final shards."""
    nl = n - m
    G = 1 << m
    shards = [psi_logical[r << nl:(r + 1) << nl].copy() for r in range(G)]   # pi0 = identity
    for op in ops:
        if op["kind"] == "apply":
            g = gates[op["gate"]]
            k = len(g.qubits)
            for r, s in enumerate(shards):
                apply_on_shard(s, nl, g.U, op["bits"][:k], r)
        elif op["kind"] == "gather":
            # the gate across rank pairs: on the whole physical vector (rank
            # bits are the top m physical bits), then split back
            g = gates[op["gate"]]
            k = len(g.qubits)
            full = np.concatenate(shards)
            phys_apply(full, n, g.U, op["bits"][:k])
            shards = [full[r << nl:(r + 1) << nl].copy() for r in range(G)]
        elif op["kind"] == "permute":
            pairs = [(op["bits"][2 * i], op["bits"][2 * i + 1]) for i in range(op["nbits"])]
            shards = [permute_bits(s, pairs) for s in shards]
        else:
            pairs = [(op["bits"][2 * i], op["bits"][2 * i + 1]) for i in range(op["nbits"])]
            mp, gsh, lmask, lmin, runlen, nruns, run_start = remap_runs(nl, pairs)
            new = [np.empty_like(s) for s in shards]
            for r in range(G):
                u = bits_of(r, gsh)
                for t in range(1 << mp):
                    p = peer_of(r, t, gsh)
                    for rho in range(nruns):
                        a, b = run_start(rho, t), run_start(rho, u)
                        new[p][b:b + runlen] = shards[r][a:a + runlen]
            shards = new
    return shards


def to_logical(n, shards, pi):
    """Physical shards + final pi (logical q -> physical bit) -> logical psi."""
    phys = np.concatenate(shards)
    idx = np.arange(1 << n, dtype=np.int64)
    p = np.zeros_like(idx)
    for q in range(n):
        p |= ((idx >> (n - 1 - q)) & 1) << pi[q]
    return phys[p]
