"""Full-size parity at the BASELINE.json sizes and in the launch configuration
bench.py / bench_sweep.py time (n = 32 sweep, n = 34 circuit), where the full
oracle cannot run:

* sampled outputs: an index-addressable hash state (integers, exact in every
  dtype) is generated on the device; after one Haar k-qubit pass, randomly
  sampled gather sets are recomputed one by one by the oracle (its own apply on
  the gathered 2^k amplitudes) and compared with the device's outputs;
* mirror circuit (pin P9): the 34q d20 circuit fused to k <= 6 with the planned
  layout, followed by its inverse, returns |0> within the c64 bound;
* reversible circuit (pin P10): basis state through permutation gates of every
  k (SIMT and tensor-core paths) at 34 qubits, bit-exact against host bit ops.
"""
import numpy as np
import pytest
import torch

import oracle as O
from hq_inputs import (Gate, sycamore_circuit, haar_sweep_gate, permutation_matrix,
                       reversible_circuit)
from hq_inputs.states import hash_amplitudes_np, hash_state_torch
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu


def _gather_indices(n, qubits, outer):
    """Indices of the gather set of outer index `outer` (targets zeroed), in
    U-index order (qubits[0] = MSB of c)."""
    k = len(qubits)
    bits = sorted(n - 1 - q for q in qubits)
    base = int(outer)
    for b in bits:
        base = ((base >> b) << (b + 1)) | (base & ((1 << b) - 1))
    idx = []
    for c in range(2 ** k):
        x = base
        for j, q in enumerate(qubits):
            if (c >> (k - 1 - j)) & 1:
                x |= 1 << (n - 1 - q)
        idx.append(x)
    return np.array(idx, dtype=np.int64)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("placement", ["low", "high", "spread", "random0"])
def test_sampled_outputs_32q(k, placement):
    n = 32
    psi = hash_state_torch(n, "cuda")
    stream = torch.cuda.current_stream()
    s = hq.hq_state_create_from_buffers(n, "c64", psi.data_ptr(), stream.cuda_stream)
    g = haar_sweep_gate(n, k, placement, seed=2000 + k)
    hq.hq_apply_matrix(s, g.U, g.qubits)
    hq.hq_sync(s)
    rng = np.random.default_rng(k * 31 + len(placement))
    outers = rng.integers(0, 2 ** (n - k), size=128)
    all_idx = np.concatenate([_gather_indices(n, g.qubits, o) for o in outers])
    got = psi[torch.from_numpy(all_idx).cuda()].cpu().numpy().astype(np.complex128)
    worst = 0.0
    for t, o in enumerate(outers):
        idx = all_idx[t * 2 ** k:(t + 1) * 2 ** k]
        v = hash_amplitudes_np(idx)                       # inputs, regenerated on the host
        want = O.apply_gate(v.copy(), g.U, list(range(k)))  # oracle on the gathered set
        w = got[t * 2 ** k:(t + 1) * 2 ** k]
        worst = max(worst, np.linalg.norm(w - want) / np.linalg.norm(v))
    assert worst < 2e-6, worst
    s.close()
    del psi
    torch.cuda.empty_cache()


@pytest.mark.parametrize("blocks", [True, False])
def test_mirror_circuit_34q_k6_planned_layout(blocks):
    """P9 at the bench configuration (34q d20, k <= 6, hq_plan_layout; the
    bench planner (hq_fuse_blocks) and the plain C7 plan)."""
    n = 34
    gates = sycamore_circuit(n, 20, 3000)
    inv = [Gate(g.name + "^-1", g.qubits, g.U.conj().T) for g in reversed(gates)]
    fused = hq.hq_fuse(gates, 6, blocks=blocks) + hq.hq_fuse(inv, 6, blocks=blocks)
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_state_set_layout(s, hq.hq_plan_layout(n, 0, fused)[0])
    hq.hq_state_init_basis(s, 0)
    c = hq.hq_circuit_create(s, fused)
    hq.hq_circuit_run(s, c)
    a0 = hq.hq_get_amplitudes(s, 0, 1)[0]
    nrm = hq.hq_norm(s)
    # ||psi - |0>||^2 = (||psi||^2 - |psi_0|^2) + |psi_0 - 1|^2
    dist = np.sqrt(max(nrm ** 2 - abs(a0) ** 2, 0.0) + abs(a0 - 1) ** 2)
    print("34q mirror: passes=%d |psi - |0>| = %.3e, norm-1 = %.3e" % (len(fused), dist, nrm - 1))
    assert dist <= 1e-4


def _host_perm_apply(n, x, gates):
    y = x
    for g in gates:
        k = len(g.qubits)
        c = 0
        for j, q in enumerate(g.qubits):
            c |= ((y >> (n - 1 - q)) & 1) << (k - 1 - j)
        r = int(np.flatnonzero(np.abs(g.U[:, c]) > 0.5)[0])
        for j, q in enumerate(g.qubits):
            b = n - 1 - q
            y = (y & ~(1 << b)) | (((r >> (k - 1 - j)) & 1) << b)
    return y


def test_reversible_34q_all_k_bit_exact():
    """P10 at 34 qubits through every kernel family (k = 1..6)."""
    n = 34
    rng = np.random.default_rng(77)
    gates = reversible_circuit(n, 40, 5, kmax=4)
    for k in (5, 6, 5, 6):
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        gates.append(Gate("P", qs, permutation_matrix([int(p) for p in rng.permutation(2 ** k)])))
    x = int(rng.integers(0, 2 ** n))
    y = _host_perm_apply(n, x, gates)
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_state_init_basis(s, x)
    hq.hq_apply_circuit(s, gates)
    assert hq.hq_get_amplitudes(s, y, 1)[0] == 1.0
    assert hq.hq_norm(s) == 1.0


@pytest.mark.parametrize("G", [2, 8])
def test_block_plan_mirror_30q_virtual_shards_fused_remaps(G):
    """P9 through the distributed path at size: the 30q d20 circuit and its
    inverse, block plan k <= 6, planned layout with its first global set, on G
    virtual shards with fused remaps (the apply pass before each remap writes
    into the peer shards' buffers) -- |psi - |0>| <= 1e-4, and the remaps did
    fuse."""
    n = 30
    m = G.bit_length() - 1
    gates = sycamore_circuit(n, 20, 1000)
    inv = [Gate(g.name + "^-1", g.qubits, g.U.conj().T) for g in reversed(gates)]
    fused = hq.hq_fuse(gates, 6, blocks=True) + hq.hq_fuse(inv, 6, blocks=True)
    s = hq.hq_state_create_virtual(n, "c64", G)
    assert hq.hq_state_set_remap_mode(s, "fused+gather")
    hq.hq_state_set_layout(s, hq.hq_plan_layout(n, m, fused)[0])
    hq.hq_state_init_basis(s, 0)
    hq.hq_stats_reset(s)
    c = hq.hq_circuit_create(s, fused)
    hq.hq_circuit_run(s, c)
    st = hq.hq_stats_get(s)
    a0 = hq.hq_get_amplitudes(s, 0, 1)[0]
    nrm = hq.hq_norm(s)
    dist = np.sqrt(max(nrm ** 2 - abs(a0) ** 2, 0.0) + abs(a0 - 1) ** 2)
    print("30q mirror on %d virtual shards: passes=%d remaps=%d fused=%d |psi - |0>| = %.3e"
          % (G, len(fused), st["remaps"], st["remaps_fused"], dist))
    assert st["remaps"] > 0 and st["remaps_fused"] == st["remaps"]
    assert dist <= 1e-4
    del c
    s.close()
