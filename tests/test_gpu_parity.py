"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle.

Tolerances (BASELINE.json north_star): ||psi - psi_ref||_2 <= 1e-4 for complex64
and <= 1e-10 for complex128; permutation/index logic bit-exact (C11).
"""
import numpy as np
import pytest

import oracle as O
from hq_inputs import (Gate, sycamore_circuit, random_circuit, reversible_circuit,
                       haar_sweep_gate, haar_unitary, random_state, integer_state,
                       permutation_matrix, H, CX)
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu

TOL = {"c64": 1e-4, "c128": 1e-10}


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2111_06868_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _gpu_state(n, dtype, psi0=None, x=0):
    s = hq.hq_state_create(n, dtype, 1)
    if psi0 is None:
        hq.hq_state_init_basis(s, x)
    else:
        hq.hq_set_amplitudes(s, psi0)
    return s


def _err(a, b):
    return float(np.linalg.norm(a.astype(np.complex128) - b))


# ---------------------------------------------------------------- worked example / closed forms
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_P1_grover_on_gpu(dtype):
    s = _gpu_state(3, dtype, np.ones(8) / np.sqrt(8))
    hq.hq_apply_matrix(s, np.diag([-1, 1, 1, 1]).astype(complex), [1, 2])
    out = hq.hq_get_amplitudes(s)
    want = np.full(8, 1 / np.sqrt(8))
    want[[0, 4]] *= -1
    assert np.max(np.abs(out - want)) < 1e-6


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_ghz_and_norm(dtype):
    n = 20
    s = _gpu_state(n, dtype)
    hq.hq_apply_circuit(s, [Gate("H", (0,), H)] + [Gate("CX", (j, j + 1), CX) for j in range(n - 1)])
    out = hq.hq_get_amplitudes(s)
    nz = np.flatnonzero(np.abs(out) > 1e-6)
    assert list(nz) == [0, 2 ** n - 1]
    assert abs(hq.hq_norm(s) - 1.0) < (1e-6 if dtype == "c64" else 1e-13)


# ---------------------------------------------------------------- config [0]: 12q d10
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("kmax", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("blocks", [False, True])
def test_config0_12q_fused_vs_unfused_oracle(dtype, kmax, seed, blocks):
    n = 12
    gates = sycamore_circuit(n, 10, seed)
    want = O.simulate(n, gates)
    fused = hq.hq_fuse(gates, kmax, blocks=blocks)
    s = _gpu_state(n, dtype)
    hq.hq_apply_circuit(s, fused)
    got = hq.hq_get_amplitudes(s)
    assert _err(got, want) <= TOL[dtype]


# ---------------------------------------------------------------- single gates, every k, placements
PLACEMENTS = ["low", "high", "spread", "random0", "random1", "random2"]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("placement", PLACEMENTS)
@pytest.mark.parametrize("n", [11, 20])
def test_single_gate_all_placements(dtype, k, placement, n):
    g = haar_sweep_gate(n, k, placement, seed=2000 + k)
    psi0 = random_state(n, 17)
    want = O.apply_gate(psi0.copy(), g.U, g.qubits)
    s = _gpu_state(n, dtype, psi0)
    hq.hq_apply_matrix(s, g.U, g.qubits)
    got = hq.hq_get_amplitudes(s)
    assert _err(got, want) <= TOL[dtype] * 0.1


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_all_target_orders_k(dtype, k):
    """Every qubit order of targets spread over lane/register bit classes."""
    n = 18
    rng = np.random.default_rng(50 + k)
    psi0 = random_state(n, k)
    gates = []
    for t in range(6):
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        gates.append(Gate("U", qs, haar_unitary(k, rng)))
    want = O.simulate(n, gates, psi0)
    s = _gpu_state(n, dtype, psi0)
    hq.hq_apply_circuit(s, gates)
    assert _err(hq.hq_get_amplitudes(s), want) <= TOL[dtype]


# ---------------------------------------------------------------- bit-exact index logic (C11)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_permutation_bit_exact(dtype, k):
    n = 20
    rng = np.random.default_rng(900 + k)
    psi0 = integer_state(n, k)
    gates = []
    for t in range(5):
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        gates.append(Gate("P", qs, permutation_matrix([int(p) for p in rng.permutation(2 ** k)])))
    want = O.simulate(n, gates, psi0)
    s = _gpu_state(n, dtype, psi0)
    hq.hq_apply_circuit(s, gates)
    got = hq.hq_get_amplitudes(s).astype(np.complex128)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_reversible_circuit_bit_exact(dtype):
    n = 16
    gates = reversible_circuit(n, 120, 7, kmax=4)
    psi0 = integer_state(n, 3)
    want = O.simulate(n, gates, psi0)
    s = _gpu_state(n, dtype, psi0)
    hq.hq_apply_circuit(s, gates)
    assert np.array_equal(hq.hq_get_amplitudes(s).astype(np.complex128), want)


# ---------------------------------------------------------------- edge cases / errors
def test_errors_leave_state_unchanged():
    n = 8
    psi0 = random_state(n, 1)
    s = _gpu_state(n, "c128", psi0)
    for qs, U, status in [((0, 0), np.eye(4), "HQ_ERR_DUP_QUBIT"), ((8,), np.eye(2), "HQ_ERR_QUBIT"),
                          ((0, 1, 2, 3, 4, 5, 6), np.eye(128), "HQ_ERR_K")]:
        with pytest.raises(hq.HQError) as e:
            hq.hq_apply_matrix(s, U, qs)
        assert e.value.status == status
    with pytest.raises(hq.HQError) as e:
        hq.hq_apply_circuit(s, [Gate("H", (0,), H), Gate("bad", (9,), H)])
    assert e.value.status == "HQ_ERR_QUBIT"
    with pytest.raises(hq.HQError) as e:
        hq.hq_state_init_basis(s, 1 << n)
    assert e.value.status == "HQ_ERR_RANGE"
    assert np.array_equal(hq.hq_get_amplitudes(s), psi0)


@pytest.mark.parametrize("n", [1, 2, 5, 6])
def test_tiny_states(n):
    rng = np.random.default_rng(n)
    psi0 = random_state(n, n)
    gates = []
    for t in range(10):
        k = int(rng.integers(1, n + 1))
        k = min(k, 6)
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        gates.append(Gate("U", qs, haar_unitary(k, rng)))
    want = O.simulate(n, gates, psi0)
    s = _gpu_state(n, "c128", psi0)
    hq.hq_apply_circuit(s, gates)
    assert _err(hq.hq_get_amplitudes(s), want) <= 1e-12


def test_empty_circuit_and_identity():
    s = _gpu_state(10, "c64", random_state(10, 2))
    before = hq.hq_get_amplitudes(s)
    hq.hq_apply_circuit(s, [])
    hq.hq_apply_matrix(s, np.eye(16), [3, 1, 7, 9])
    assert np.array_equal(hq.hq_get_amplitudes(s), before)


def test_non_unitary_allowed():
    """C4: Projection-like U is applied as is, no renormalisation."""
    psi0 = random_state(6, 3)
    P0 = np.diag([1, 0]).astype(complex)
    s = _gpu_state(6, "c128", psi0)
    hq.hq_apply_matrix(s, P0, [2])
    want = O.apply_gate(psi0.copy(), P0, [2])
    assert _err(hq.hq_get_amplitudes(s), want) < 1e-15
    assert abs(hq.hq_norm(s) - np.linalg.norm(want)) < 1e-14


def test_partial_amplitude_ranges():
    n = 14
    psi0 = random_state(n, 9)
    s = _gpu_state(n, "c128", psi0)
    assert np.array_equal(hq.hq_get_amplitudes(s, 100, 37), psi0[100:137])
    hq.hq_set_amplitudes(s, np.arange(5) + 1j, first=2 ** n - 5)
    assert np.array_equal(hq.hq_get_amplitudes(s, 2 ** n - 5, 5), np.arange(5) + 1j)
    with pytest.raises(hq.HQError):
        hq.hq_get_amplitudes(s, 2 ** n - 2, 3)


# ---------------------------------------------------------------- compiled circuits
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_circuit_create_run_matches_apply(dtype):
    n = 18
    gates = hq.hq_fuse(sycamore_circuit(n, 12, 5), 4)
    s1 = _gpu_state(n, dtype)
    hq.hq_apply_circuit(s1, gates)
    s2 = _gpu_state(n, dtype)
    c = hq.hq_circuit_create(s2, gates)
    info = hq.hq_circuit_info(c)
    assert info["passes"] == len(gates) and info["remaps"] == 0
    hq.hq_circuit_run(s2, c)
    a, b = hq.hq_get_amplitudes(s1), hq.hq_get_amplitudes(s2)
    assert np.array_equal(a, b)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    assert _err(b, want) <= TOL[dtype]


# ---------------------------------------------------------------- virtual shards (distribution logic on 1 GPU)
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_virtual_shards_sycamore(G, dtype):
    n = 16
    gates = hq.hq_fuse(sycamore_circuit(n, 12, 6), 4)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    s = hq.hq_state_create_virtual(n, dtype, G)
    hq.hq_state_init_basis(s, 0)
    hq.hq_apply_circuit(s, gates)
    st = hq.hq_stats_get(s)
    assert st["remaps"] > 0
    assert _err(hq.hq_get_amplitudes(s), want) <= TOL[dtype]
    assert abs(hq.hq_norm(s) - 1) < 1e-5


@pytest.mark.parametrize("G", [2, 8])
def test_virtual_shards_reversible_bit_exact(G):
    n = 14
    gates = reversible_circuit(n, 100, 11, kmax=4)
    psi0 = integer_state(n, 5)
    want = O.simulate(n, gates, psi0)
    s = hq.hq_state_create_virtual(n, "c64", G)
    hq.hq_set_amplitudes(s, psi0)
    hq.hq_apply_circuit(s, gates)
    assert np.array_equal(hq.hq_get_amplitudes(s).astype(np.complex128), want)
    # readback of a sub-range through pi^-1
    assert np.array_equal(hq.hq_get_amplitudes(s, 77, 300).astype(np.complex128), want[77:377])


def test_virtual_circuit_rerun_requires_same_layout():
    n = 14
    gates = hq.hq_fuse(sycamore_circuit(n, 8, 1), 3)
    s = hq.hq_state_create_virtual(n, "c128", 4)
    hq.hq_state_init_basis(s, 0)
    c = hq.hq_circuit_create(s, gates)
    hq.hq_circuit_run(s, c)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    assert _err(hq.hq_get_amplitudes(s), want) <= 1e-10


# ---------------------------------------------------------------- full size: properties at any n
@pytest.mark.parametrize("n", [26, 30])
def test_mirror_circuit_full_size(n):
    """P9: C then C^dagger returns |0> (c64 tolerance 1e-4)."""
    gates = sycamore_circuit(n, 20 if n == 30 else 12, 1000)
    inv = [Gate(g.name + "^-1", g.qubits, g.U.conj().T) for g in reversed(gates)]
    fused = hq.hq_fuse(gates + inv, 2 if n == 30 else 4)
    s = _gpu_state(n, "c64")
    hq.hq_apply_circuit(s, fused)
    a0 = hq.hq_get_amplitudes(s, 0, 1)[0]
    nrm = hq.hq_norm(s)
    # ||psi - |0>||^2 = (||psi||^2 - |psi_0|^2) + |psi_0 - 1|^2
    dist = np.sqrt(max(nrm ** 2 - abs(a0) ** 2, 0.0) + abs(a0 - 1) ** 2)
    assert dist <= 1e-4


def test_reversible_full_size_bit_exact():
    """P10: basis state through reversible gates at 30q; f(x) by host bit ops."""
    n = 30
    gates = reversible_circuit(n, 60, 99, kmax=4)
    x = 0x2A5F3C1
    # host: push the basis index through the permutations
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
    s = _gpu_state(n, "c64", x=x)
    hq.hq_apply_circuit(s, gates)
    assert hq.hq_get_amplitudes(s, y, 1)[0] == 1.0
    assert hq.hq_norm(s) == 1.0


# ---------------------------------------------------------------- qubit layouts
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_layout_invariance(dtype):
    """Any logical->physical layout gives the same logical state (C14)."""
    n = 20
    gates = hq.hq_fuse(sycamore_circuit(n, 10, 8), 6)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    rng = np.random.default_rng(5)
    for trial in range(3):
        pi = [int(x) for x in rng.permutation(n)] if trial else hq.hq_plan_layout(n, 0, gates, dtype)[0]
        s = hq.hq_state_create(n, dtype, 1)
        hq.hq_state_set_layout(s, pi)
        assert hq.hq_state_get_layout(s) == pi
        hq.hq_state_init_basis(s, 0)
        c = hq.hq_circuit_create(s, gates)
        hq.hq_circuit_run(s, c)
        assert _err(hq.hq_get_amplitudes(s), want) <= TOL[dtype]
        assert np.allclose(hq.hq_get_amplitudes(s, 1000, 64), want[1000:1064], atol=1e-5)


def test_layout_bit_exact_permutations():
    n = 18
    gates = reversible_circuit(n, 80, 21, kmax=4)
    psi0 = integer_state(n, 9)
    want = O.simulate(n, gates, psi0)
    pi = [int(x) for x in np.random.default_rng(1).permutation(n)]
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_state_set_layout(s, pi)
    hq.hq_set_amplitudes(s, psi0)
    hq.hq_apply_circuit(s, gates)
    assert np.array_equal(hq.hq_get_amplitudes(s).astype(np.complex128), want)
    with pytest.raises(hq.HQError):
        hq.hq_state_set_layout(s, [0] * n)


# ---------------------------------------------------------------- CUDA graph replay
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_circuit_graph_replay(dtype):
    """hq_circuit_run captures the op stream into a CUDA graph (single shard,
    profiling off) and replays it; every replay must equal the oracle."""
    n = 17
    gates = hq.hq_fuse(sycamore_circuit(n, 12, 21), 6)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    s = hq.hq_state_create(n, dtype, 1)
    c = hq.hq_circuit_create(s, gates)
    hq.hq_stats_reset(s)
    for rep in range(3):
        hq.hq_state_init_basis(s, 0)
        hq.hq_circuit_run(s, c)
        assert _err(hq.hq_get_amplitudes(s), want) <= TOL[dtype]
    st = hq.hq_stats_get(s)
    assert st["passes"] == 3 * len(gates)
    # a run from a different starting state (no re-init) replays the same graph
    psi1 = hq.hq_get_amplitudes(s).astype(np.complex128)
    hq.hq_circuit_run(s, c)
    want2 = O.simulate(n, [Gate("F", q, U) for q, U in gates], psi1)
    assert _err(hq.hq_get_amplitudes(s), want2) <= 2 * TOL[dtype]
    # profiling disables the graph path; results stay identical
    hq.hq_state_init_basis(s, 0)
    hq.hq_profile_enable(s, True)
    hq.hq_circuit_run(s, c)
    hq.hq_profile_enable(s, False)
    t = hq.hq_kernel_times(s)
    assert t["count"] == len(gates)
    assert _err(hq.hq_get_amplitudes(s), want) <= TOL[dtype]


# ---------------------------------------------------------------- torch-owned memory

@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_rank_state_on_torch_buffers(dtype):
    """hq_state_create_rank_from_buffers (the bench's constructor): PyTorch owns
    the shard and the stream; results match the oracle and the amplitudes are
    visible through the torch tensor."""
    import torch
    n = 18
    gates = hq.hq_fuse(sycamore_circuit(n, 8, 21), 6)
    want = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    psi_t = torch.empty(2 ** n, dtype=cdt, device="cuda")
    stream = torch.cuda.Stream()
    s = hq.hq_state_create_rank_from_buffers(n, dtype, 1, 0, psi_t.data_ptr(), None, stream.cuda_stream)
    hq.hq_state_init_basis(s, 0)
    c = hq.hq_circuit_create(s, gates)
    hq.hq_circuit_run(s, c)
    hq.hq_sync(s)
    got = psi_t.cpu().numpy().astype(np.complex128)      # default layout: physical = logical
    assert np.linalg.norm(got - want) < (1e-4 if dtype == "c64" else 1e-10)
    with pytest.raises(hq.HQError) as e:
        hq.hq_state_create_rank_from_buffers(n, dtype, 1, 0, psi_t.data_ptr() + 8, None, None)
    assert e.value.status == "HQ_ERR_ARG"
    with pytest.raises(hq.HQError) as e:                # world 2 needs a receive buffer and an id
        hq.hq_state_create_rank_from_buffers(n, dtype, 2, 0, psi_t.data_ptr(), None, None)
    assert e.value.status == "HQ_ERR_ARG"


def test_borrowed_buffer_external_write_needs_invalidate():
    """the complex64 tensor-core passes scale amplitudes into FP16
    with the tracked norm bound.  After the caller scales a borrowed buffer
    by 2^20 outside the library, hq_state_invalidate_bound makes the next
    k = 6 pass correct (relative error within the single-pass bound)."""
    import torch
    n = 18
    psi0 = random_state(n, 41)
    psi_t = torch.from_numpy(psi0.astype(np.complex64)).cuda()
    stream = torch.cuda.Stream()
    s = hq.hq_state_create_from_buffers(n, "c64", psi_t.data_ptr(), stream.cuda_stream)
    hq.hq_set_amplitudes(s, psi0)
    assert abs(hq.hq_norm(s) - 1.0) < 1e-6          # bound is now ~1
    torch.cuda.synchronize()
    psi_t.mul_(2.0 ** 20)                           # external write: the bound is stale
    torch.cuda.synchronize()
    hq.hq_state_invalidate_bound(s)
    g = haar_sweep_gate(n, 6, "spread", 2206)
    hq.hq_apply_matrix(s, g.U, g.qubits)
    want = O.apply_gate(psi0.copy() * 2.0 ** 20, g.U, g.qubits)
    got = hq.hq_get_amplitudes(s).astype(np.complex128)
    assert np.all(np.isfinite(got))
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 2e-6


# ---------------------------------------------------------------- block plan at a tensor-core size

@pytest.mark.parametrize("kmax", [5, 6])
def test_block_plan_20q_tensor_cores_vs_oracle(kmax):
    """The bench's planner (hq_fuse_blocks) + hq_plan_layout at a size where
    the k = 5, 6 blocks run on the tensor cores, against the unfused oracle."""
    n = 20
    gates = sycamore_circuit(n, 14, 77)
    want = O.simulate(n, gates)
    fused = hq.hq_fuse(gates, kmax, blocks=True)
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_state_set_layout(s, hq.hq_plan_layout(n, 0, fused)[0])
    hq.hq_state_init_basis(s, 0)
    c = hq.hq_circuit_create(s, fused)
    hq.hq_circuit_run(s, c)
    got = hq.hq_get_amplitudes(s)
    assert _err(got, want) <= TOL["c64"]


# ---------------------------------------------------------------- small states: whole circuit in shared memory

@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [1, 2, 5, 8, 10, 11, 12])
def test_small_state_circuit_in_shared_memory(dtype, n):
    """hq_circuit_run for n_local <= 10 (and >= 2 passes) runs every pass in
    one CTA with the state in shared memory (11-12 qubits: per-pass kernels);
    results against the oracle, for
    fused gates of every k the state allows, twice in a row (re-run of the
    same compiled circuit) and with a random layout."""
    kmax = min(6, n)
    gates = [Gate("F", q, U) for q, U in hq.hq_fuse(random_circuit(n, 40, 7, kmax=min(kmax, 3)), kmax)]
    psi0 = random_state(n, 11)
    want1 = O.simulate(n, gates, psi0)
    want2 = O.simulate(n, gates, want1)
    for layout in (None, [int(x) for x in np.random.default_rng(n).permutation(n)]):
        s = _gpu_state(n, dtype)
        if layout is not None:
            hq.hq_state_set_layout(s, layout)
        hq.hq_set_amplitudes(s, psi0.astype(s.np_dtype))
        c = hq.hq_circuit_create(s, gates)
        hq.hq_stats_reset(s)
        hq.hq_circuit_run(s, c)
        assert _err(hq.hq_get_amplitudes(s), want1) <= TOL[dtype]
        hq.hq_circuit_run(s, c)
        assert _err(hq.hq_get_amplitudes(s), want2) <= TOL[dtype]
        st = hq.hq_stats_get(s)
        assert st["passes"] == 2 * len(gates)
