"""Row f2 on the GPU: density-matrix evolution by doubling (vec(rho) on 2N
qubits through the same apply kernels) vs the oracle's Kraus maps applied to
rho itself."""
import numpy as np
import pytest

import oracle as O
from hq_inputs import Gate, haar_unitary, random_state, X, Y
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu

TOL = {"c64": 1e-4, "c128": 1e-10}


def _depolarizing(p):
    s = np.sqrt(p / 4)
    return [np.sqrt(1 - 3 * p / 4) * np.eye(2), s * X, s * Y, s * np.diag([1, -1]).astype(complex)]


def _amp_damping(g):
    return [np.array([[1, 0], [0, np.sqrt(1 - g)]], dtype=complex),
            np.array([[0, np.sqrt(g)], [0, 0]], dtype=complex)]


def _random_channel(k, m, rng):
    """Random CPTP map with m Kraus operators (Stinespring: columns of a Haar
    isometry)."""
    d = 2 ** k
    Z = rng.standard_normal((d * m, d)) + 1j * rng.standard_normal((d * m, d))
    V, _ = np.linalg.qr(Z)                      # (d*m) x d isometry: sum_i K_i^H K_i = I
    return [V[i * d:(i + 1) * d, :] for i in range(m)]


def test_superop_matches_definition():
    rng = np.random.default_rng(1)
    K = _random_channel(2, 3, rng)
    S = hq.hq_dm_superop(K)
    want = sum(np.kron(k, k.conj()) for k in K)
    assert np.max(np.abs(S - want)) < 1e-15


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("shards", [1, 4])
def test_noisy_circuit_density_matrix(dtype, shards):
    N = 7
    rng = np.random.default_rng(11)
    psi = random_state(N, 5)
    rho = np.outer(psi, psi.conj())
    s = hq.hq_state_create(2 * N, dtype, 1) if shards == 1 else hq.hq_state_create_virtual(2 * N, dtype, shards)
    hq.hq_set_amplitudes(s, O.dm_vec(rho))
    for step in range(12):
        k = int(rng.integers(1, 5))
        qs = [int(q) for q in rng.choice(N, size=k, replace=False)]
        U = haar_unitary(k, rng)
        hq.hq_dm_apply_unitary(s, U, qs)
        rho = O.dm_apply_kraus(rho, [U], qs)
        q1 = [int(rng.integers(N))]
        ch = _depolarizing(0.05) if step % 3 == 0 else (_amp_damping(0.1) if step % 3 == 1
                                                         else _random_channel(2, 2, rng))
        if len(ch[0]) == 4:
            q1 = [int(q) for q in rng.choice(N, size=2, replace=False)]
        hq.hq_dm_apply_kraus(s, ch, q1)
        rho = O.dm_apply_kraus(rho, ch, q1)
    got = hq.hq_get_amplitudes(s).astype(np.complex128)
    assert np.linalg.norm(got - O.dm_vec(rho)) <= TOL[dtype]
    tr = hq.hq_dm_trace(s)
    assert abs(tr - np.trace(rho)) < (1e-5 if dtype == "c64" else 1e-12)
    assert abs(tr - 1) < (1e-5 if dtype == "c64" else 1e-12)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_super_circuit_block_plan_vs_oracle(dtype):
    """The bench_dm.py path: a noisy Sycamore-style circuit as a regular gate
    list on vec(rho) (every gate U (x) conj(U) on (q, q + N), a depolarising
    superoperator after each single-qubit gate), fused by the block planner
    and run with hq_apply_circuit, against the oracle's Kraus maps on rho."""
    from hq_inputs import sycamore_circuit
    N = 6
    pure = sycamore_circuit(N, 6, 5001)
    depol = _depolarizing(0.02)
    S1 = hq.hq_dm_superop(depol)
    gates = []
    rho = np.zeros((2 ** N, 2 ** N), dtype=complex)
    rho[0, 0] = 1.0
    for g in pure:
        gates.append(Gate("S", tuple(g.qubits) + tuple(q + N for q in g.qubits), np.kron(g.U, g.U.conj())))
        rho = O.dm_apply_kraus(rho, [g.U], list(g.qubits))
        if len(g.qubits) == 1:
            q = g.qubits[0]
            gates.append(Gate("D", (q, q + N), S1))
            rho = O.dm_apply_kraus(rho, depol, [q])
    fused = hq.hq_fuse(gates, 6, blocks=True)
    assert len(fused) <= len(hq.hq_fuse(gates, 6))
    s = hq.hq_state_create(2 * N, dtype, 1)
    hq.hq_state_init_basis(s, 0)
    hq.hq_apply_circuit(s, fused)
    got = hq.hq_get_amplitudes(s).astype(np.complex128)
    assert np.linalg.norm(got - O.dm_vec(rho)) <= TOL[dtype]
    assert abs(hq.hq_dm_trace(s) - 1) < (1e-5 if dtype == "c64" else 1e-12)


def test_dm_errors():
    s = hq.hq_state_create(7, "c64", 1)
    with pytest.raises(hq.HQError) as e:
        hq.hq_dm_trace(s)
    assert e.value.status == "HQ_ERR_STATE"
    s = hq.hq_state_create(8, "c64", 1)
    with pytest.raises(hq.HQError) as e:
        hq.hq_dm_apply_unitary(s, np.eye(2), [4])
    assert e.value.status == "HQ_ERR_QUBIT"
    with pytest.raises(hq.HQError) as e:
        hq.hq_dm_apply_kraus(s, [np.eye(16)], [0, 1, 2, 3])
    assert e.value.status == "HQ_ERR_K"
