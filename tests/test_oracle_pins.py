"""Pins of the CPU oracle against things other than itself (SURVEY §8(c) pins).

Each test names the pin and the passage it follows.  None of them imports the
product path.
"""
import os

import numpy as np
import pytest

import oracle as O
from hq_inputs import (SQRT_X, SQRT_Y, SQRT_W, H, X, Y, CX, SWAP, CCX, fsim,
                       cphase, cr_m, Gate, sycamore_circuit, random_circuit,
                       haar_unitary, random_state, integer_state,
                       permutation_matrix)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- P1 (C1)
def test_P1_grover_listing_pins_bit_order():
    """Grover gate on qubits [1,2] of the uniform 3-qubit
    state.  The oracle psi -= 2 P_0 psi on qubits (1,2) is U = diag(-1,1,1,1)."""
    psi = np.ones(8, dtype=np.complex128) / np.sqrt(8)
    O.apply_gate(psi, np.diag([-1, 1, 1, 1]).astype(np.complex128), [1, 2])
    for bits, val in _golden("grover_P403-422.txt"):
        i = int(bits, 2)
        assert abs(psi[i].imag) < 1e-15
        assert abs(psi[i].real - float(val)) < 1e-6, bits


# ---------------------------------------------------------------- P2 (C7/C8)
def test_P2_compress_worked_example():
    """CPHASE on all pairs of 5 qubits, max_n_qubits=3."""
    gates = [Gate("CPHASE", (q1, q2), cphase(1.0)) for q1 in range(5) for q2 in range(q1 + 1, 5)]
    fused = O.fused_gates(gates, 3)
    want = [tuple(int(x) for x in row) for row in _golden("compress_P510-529.txt")]
    assert [f[0] for f in fused] == want
    # and the fused circuit reproduces the original (C9)
    psi0 = random_state(5, 7)
    a = O.simulate(5, gates, psi0)
    b = O.simulate(5, [Gate("F", q, U) for q, U in fused], psi0)
    assert np.linalg.norm(a - b) < 1e-13


def test_C7_lenient_rule_counterexample_is_avoided():
    """[(0,1),(2,3),(0,1),(1,2)] with k_max=3.  The strict
    rule must keep the replay exact."""
    rng = np.random.default_rng(3)
    gates = [Gate("U", q, haar_unitary(2, rng)) for q in [(0, 1), (2, 3), (0, 1), (1, 2)]]
    psi0 = random_state(4, 1)
    a = O.simulate(4, gates, psi0)
    fused = O.fused_gates(gates, 3)
    b = O.simulate(4, [Gate("F", q, U) for q, U in fused], psi0)
    assert np.linalg.norm(a - b) < 1e-13
    for grp in O.compress(gates, 3):
        assert grp == sorted(grp)


@pytest.mark.parametrize("kmax", [2, 3, 4, 5, 6])
def test_fusion_preserves_state(kmax):
    """Fusion is associativity: fused == unfused to 1e-12."""
    n = 12
    gates = sycamore_circuit(n, 10, seed=0)
    psi0 = random_state(n, 11)
    a = O.simulate(n, gates, psi0)
    fused = O.fused_gates(gates, kmax)
    assert all(len(q) <= kmax for q, _ in fused)
    b = O.simulate(n, [Gate("F", q, U) for q, U in fused], psi0)
    assert np.linalg.norm(a - b) < 1e-12


def test_fusion_random_circuits():
    for seed in range(4):
        gates = random_circuit(7, 40, seed, kmax=3)
        psi0 = random_state(7, seed)
        a = O.simulate(7, gates, psi0)
        for kmax in (3, 4, 5):
            fused = O.fused_gates(gates, kmax)
            b = O.simulate(7, [Gate("F", q, U) for q, U in fused], psi0)
            assert np.linalg.norm(a - b) < 1e-12


# ---------------------------------------------------------------- P3-P5 closed forms
@pytest.mark.parametrize("n", list(range(1, 13)))
def test_P3_hadamard_uniform(n):
    psi = O.simulate(n, [Gate("H", (q,), H) for q in range(n)])
    assert np.allclose(psi, 2 ** (-n / 2), atol=1e-14, rtol=0)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_P4_ghz(n):
    gates = [Gate("H", (0,), H)] + [Gate("CX", (j, j + 1), CX) for j in range(n - 1)]
    psi = O.simulate(n, gates)
    nz = np.flatnonzero(np.abs(psi) > 1e-14)
    assert list(nz) == [0, 2 ** n - 1]
    assert np.allclose(psi[nz], 1 / np.sqrt(2), atol=1e-15)


def _qft_gates(n):
    gates = []
    for j in range(n):
        gates.append(Gate("H", (j,), H))
        for l in range(j + 1, n):
            gates.append(Gate("CR", (l, j), cr_m(l - j + 1)))
    for j in range(n // 2):
        gates.append(Gate("SWAP", (j, n - 1 - j), SWAP))
    return gates


@pytest.mark.parametrize("x", [0, 1, 6, 19, 31])
def test_P5_qft_phases(x):
    """QFT|x> = 2^(-n/2) sum_y e^{2 pi i x y / 2^n} |y> (closed form)."""
    n = 5
    psi = O.simulate(n, _qft_gates(n), x=x)
    y = np.arange(2 ** n)
    want = np.exp(2j * np.pi * x * y / 2 ** n) / 2 ** (n / 2)
    assert np.max(np.abs(psi - want)) < 1e-14


# ---------------------------------------------------------------- P6 invariants
def test_P6_norm_preserved():
    n = 12
    gates = random_circuit(n, 200, seed=5, kmax=3)
    psi = O.simulate(n, gates)
    assert abs(O.norm(psi) - 1.0) < 1e-10


def test_norm_closed_form():
    psi = np.zeros(4, dtype=np.complex128)
    psi[1] = 3.0
    psi[2] = 4.0j
    assert O.norm(psi) == 5.0
    v = random_state(10, 3, normalize=False)
    assert abs(O.norm(v) - np.linalg.norm(v)) < 1e-12 * np.linalg.norm(v)


def test_P12_identity_and_linearity():
    n = 6
    a = random_state(n, 1)
    b = O.simulate(n, [Gate("I", (1, 4, 2), np.eye(8, dtype=np.complex128))], a)
    assert np.array_equal(a, b)
    U = haar_unitary(3, np.random.default_rng(0))
    p1, p2 = random_state(n, 2), random_state(n, 3)
    al, be = 0.3 - 0.2j, -1.1 + 0.5j
    lhs = O.simulate(n, [Gate("U", (5, 0, 3), U)], al * p1 + be * p2)
    rhs = al * O.simulate(n, [Gate("U", (5, 0, 3), U)], p1) + be * O.simulate(n, [Gate("U", (5, 0, 3), U)], p2)
    assert np.max(np.abs(lhs - rhs)) < 1e-12


# ---------------------------------------------------------------- P7 brute force
def test_embed_dense_matches_textbook_kron():
    rng = np.random.default_rng(0)
    for n in (3, 5, 7):
        for k in (1, 2, 3):
            for q0 in range(0, n - k + 1):
                U = haar_unitary(k, rng)
                A = O.embed_dense(n, U, list(range(q0, q0 + k)))
                B = O.kron_embed_adjacent(n, U, q0)
                assert np.array_equal(A, B)


def test_circuit_matrix_cx_triple_is_swap():
    """[CX(0,1), CX(1,0), CX(0,1)] -> SWAP."""
    g = [Gate("CX", (0, 1), CX), Gate("CX", (1, 0), CX), Gate("CX", (0, 1), CX)]
    assert np.array_equal(O.circuit_matrix(2, g), SWAP)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_P7_oracle_vs_dense(k):
    rng = np.random.default_rng(100 + k)
    n = 8
    for trial in range(3):
        U = haar_unitary(k, rng)
        qs = [int(q) for q in rng.choice(n, size=k, replace=False)]
        psi = random_state(n, trial)
        want = O.embed_dense(n, U, qs) @ psi
        got = O.apply_gate(psi.copy(), U, qs)
        assert np.max(np.abs(got - want)) < 1e-14


def test_P7_circuit_vs_dense_matrix():
    """6-qubit 50-gate circuit vs circuit_matrix (1e-8; we use 1e-12)."""
    n = 6
    gates = random_circuit(n, 50, seed=9, kmax=3)
    psi0 = random_state(n, 4)
    assert np.max(np.abs(O.simulate(n, gates, psi0) - O.circuit_matrix(n, gates) @ psi0)) < 1e-12


# ---------------------------------------------------------------- P8 tensordot
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_P8_tensordot(k):
    rng = np.random.default_rng(7 + k)
    n = 14
    U = haar_unitary(k, rng)
    qs = [int(q) for q in rng.choice(n, size=k, replace=False)]
    psi = random_state(n, k)
    want = O.tensordot_apply(psi, U, qs)
    got = O.apply_gate(psi.copy(), U, qs)
    assert np.max(np.abs(got - want)) < 1e-14


# ---------------------------------------------------------------- C2 / C3
def test_C2_matrix_acts_on_column_vectors():
    """sqrt(Y)|0> = |+>; the transpose would give |->."""
    psi = O.simulate(1, [Gate("SY", (0,), SQRT_Y)])
    assert np.allclose(psi, [1 / np.sqrt(2), 1 / np.sqrt(2)], atol=1e-16)


def test_C2_kron_order_on_targets():
    """kron(A, B) on (a, b) == A on a then B on b (qubits[0] = MSB of U)."""
    rng = np.random.default_rng(1)
    A, B = haar_unitary(1, rng), haar_unitary(1, rng)
    n = 4
    psi = random_state(n, 5)
    lhs = O.simulate(n, [Gate("AB", (2, 0), np.kron(A, B))], psi)
    rhs = O.simulate(n, [Gate("A", (2,), A), Gate("B", (0,), B)], psi)
    assert np.max(np.abs(lhs - rhs)) < 1e-15


def test_C3_target_order_matters():
    rng = np.random.default_rng(2)
    U = haar_unitary(2, rng)
    psi = random_state(5, 6)
    a = O.simulate(5, [Gate("U", (1, 3), U)], psi)
    b = O.simulate(5, [Gate("U", (3, 1), SWAP @ U @ SWAP)], psi)
    c = O.simulate(5, [Gate("U", (3, 1), U)], psi)
    assert np.max(np.abs(a - b)) < 1e-15
    assert np.max(np.abs(a - c)) > 1e-3


def test_C11_permutation_on_integer_state_is_exact():
    """Reversible gates map |x> to |f(x)> computed by host bit operations."""
    n = 6
    psi = integer_state(n, 0)
    perm = [3, 0, 7, 1, 6, 2, 5, 4]
    qs = (4, 0, 2)
    got = O.apply_gate(psi.copy(), permutation_matrix(perm), qs)
    want = np.empty_like(psi)
    for i in range(2 ** n):
        c = 0
        for j, q in enumerate(qs):
            c |= ((i >> (n - 1 - q)) & 1) << (2 - j)
        r = perm[c]
        o = i
        for j, q in enumerate(qs):
            b = n - 1 - q
            o = (o & ~(1 << b)) | (((r >> (2 - j)) & 1) << b)
        want[o] = psi[i]
    assert np.array_equal(got, want)


def test_P15_determinism_across_threads():
    n = 16
    gates = random_circuit(n, 30, seed=1, kmax=4)
    psi0 = random_state(n, 0)
    O.set_threads(1)
    a = O.simulate(n, gates, psi0)
    na = O.norm(a)
    O.set_threads(4)
    b = O.simulate(n, gates, psi0)
    nb = O.norm(b)
    O.set_threads(os.cpu_count() or 1)
    assert np.array_equal(a, b) and na == nb


def test_oracle_rejects_bad_gates():
    psi = O.init_basis(3)
    with pytest.raises(O.OracleError):
        O.apply_gate(psi, np.eye(4), [0, 0])
    with pytest.raises(O.OracleError):
        O.apply_gate(psi, np.eye(2), [3])
    with pytest.raises(O.OracleError):
        O.apply_gate(psi, np.eye(4), [0])


# ---------------------------------------------------------------- inputs (C15, C16, C18)
def test_C15_gate_definitions():
    for U in (SQRT_X, SQRT_Y, SQRT_W, fsim()):
        assert np.allclose(U @ U.conj().T, np.eye(U.shape[0]), atol=1e-15)
    assert np.allclose(SQRT_X @ SQRT_X, -1j * X, atol=1e-15)
    W = (X + Y) / np.sqrt(2)
    ev, V = np.linalg.eigh(W)
    expw = V @ np.diag(np.exp(-1j * np.pi / 4 * ev)) @ V.conj().T
    assert np.allclose(SQRT_W, expw, atol=1e-15)
    assert np.allclose(CCX @ CCX, np.eye(8))


@pytest.mark.parametrize("n,cycles,count", [(12, 10, 163), (30, 20, 845), (34, 20, 960), (36, 24, 1224)])
def test_C16_generator_gate_counts(n, cycles, count):
    gates = sycamore_circuit(n, cycles, seed=0)
    assert len(gates) == count
    assert sum(len(g.qubits) == 1 for g in gates) == n * cycles


def test_C18_haar_unitary():
    rng = np.random.default_rng(0)
    for k in range(1, 7):
        U = haar_unitary(k, rng)
        assert np.max(np.abs(U @ U.conj().T - np.eye(2 ** k))) < 1e-14


# ---------------------------------------------------------------- f4: tokens, projection, probabilities
def test_tokens_spec_examples():
    """SPEC S:229-236 examples."""
    a = O.init_tokens(2, "00")
    assert a[0] == 1 and np.count_nonzero(a) == 1
    assert np.allclose(O.init_tokens(6, "++++++"), 2 ** -3, atol=1e-16)
    assert np.allclose(O.init_tokens(2, "+-"), [0.5, -0.5, 0.5, -0.5], atol=1e-16)
    assert np.array_equal(O.init_tokens(5, "+"), O.init_tokens(5, "+++++"))     # broadcast
    # qubit 0 is the MSB (C1): |1> on qubit 0 of 3 qubits is index 100
    assert np.flatnonzero(O.init_tokens(3, "100")).tolist() == [4]
    with pytest.raises(O.OracleError):
        O.init_tokens(3, "0.1")


def test_tokens_vs_gates():
    """'+'/'-' tokens equal H (and X then H) applied to |0> (closed form)."""
    n = 5
    tok = "+-01+"
    gates = []
    for q, t in enumerate(tok):
        if t in "1-":
            gates.append(Gate("X", (q,), X))
        if t in "+-":
            gates.append(Gate("H", (q,), H))
    assert np.max(np.abs(O.init_tokens(n, tok) - O.simulate(n, gates))) < 1e-15


def test_projection_spec_examples_and_grover():
    """SPEC S:252-255; the paper's own Grover oracle psi -= 2 * Projection(psi)
    on qubits [1, 2] reproduces the printed listing."""
    plus = O.init_tokens(1, "+")
    out, nrm = O.project(plus, [0], [0])
    assert np.allclose(out, [1 / np.sqrt(2), 0], atol=1e-16) and abs(nrm - 1 / np.sqrt(2)) < 1e-15
    psi = O.init_tokens(3, "+")
    psi0, _ = O.project(psi, [1, 2], [0, 0], renormalize=False)
    new = psi - 2 * psi0
    for bits, val in _golden("grover_P403-422.txt"):
        assert abs(new[int(bits, 2)].real - float(val)) < 1e-6
    basis = O.init_basis(4, 9)
    again, _ = O.project(basis, [0, 3], [1, 1], renormalize=True)
    assert np.array_equal(again, basis)
    with pytest.raises(O.OracleError):
        O.project(O.init_basis(2, 0), [0], [1], renormalize=True)


def test_probabilities_closed_forms():
    assert np.allclose(O.probabilities(O.init_basis(1, 1), [0]), [0, 1])
    assert np.allclose(O.probabilities(O.init_tokens(1, "+"), [0]), [0.5, 0.5])
    psi = random_state(6, 3)
    joint = O.probabilities(psi, [4, 1])
    # chain rule: marginal of qubit 4 = sum over qubit 1 of the joint
    assert np.allclose(joint.reshape(2, 2).sum(axis=1), O.probabilities(psi, [4]), atol=1e-15)
    assert abs(joint.sum() - 1) < 1e-14
    # brute force on tiny input
    brute = np.zeros(4)
    for i in range(64):
        brute[(((i >> 1) & 1) << 1) | ((i >> 4) & 1)] += abs(psi[i]) ** 2
    assert np.allclose(joint, brute, atol=1e-15)


# ---------------------------------------------------------------- f2: density matrices
def _depolarizing(p):
    s = np.sqrt(p / 4)
    return [np.sqrt(1 - 3 * p / 4) * np.eye(2), s * X, s * Y, s * np.diag([1, -1]).astype(complex)]


def _amp_damping(g):
    return [np.array([[1, 0], [0, np.sqrt(1 - g)]], dtype=complex),
            np.array([[0, np.sqrt(g)], [0, 0]], dtype=complex)]


def test_dm_closed_forms():
    """Depolarizing: rho -> (1-p) rho + p I/2 on one qubit; amplitude damping
    on |1><1|: gamma |0><0| + (1-gamma) |1><1| (textbook closed forms)."""
    psi = random_state(1, 4)
    rho = np.outer(psi, psi.conj())
    p = 0.3
    assert np.max(np.abs(O.dm_apply_kraus(rho, _depolarizing(p), [0]) - ((1 - p) * rho + p * np.eye(2) / 2))) < 1e-15
    one = np.diag([0, 1]).astype(complex)
    g = 0.25
    assert np.max(np.abs(O.dm_apply_kraus(one, _amp_damping(g), [0]) - np.diag([g, 1 - g]))) < 1e-15


def test_dm_pure_state_consistency_and_trace():
    """The paper's cross-check: evolving psi psi^dagger equals the
    density matrix of the evolved pure state; CPTP maps preserve the trace."""
    N = 4
    gates = random_circuit(N, 12, 3, kmax=2)
    psi = random_state(N, 2)
    rho = np.outer(psi, psi.conj())
    for gt in gates:
        rho = O.dm_apply_kraus(rho, [gt.U], list(gt.qubits))
    out = O.simulate(N, gates, psi)
    assert np.max(np.abs(rho - np.outer(out, out.conj()))) < 1e-14
    rho2 = O.dm_apply_kraus(rho, _amp_damping(0.4), [2])
    assert abs(np.trace(rho2) - 1) < 1e-14
    # vec(U rho U^dagger) = (U on rows) (conj U on columns) vec(rho): the doubling reading
    U = haar_unitary(2, np.random.default_rng(5))
    v = O.dm_vec(rho)
    v2 = O.apply_gate(O.apply_gate(v.copy(), U, [1, 3]), U.conj(), [1 + N, 3 + N])
    assert np.max(np.abs(v2 - O.dm_vec(O.dm_apply_kraus(rho, [U], [1, 3])))) < 1e-14


# ---------------------------------------------------------------- f3: reduced density matrix, trajectories

def _rdm_brute(psi, qubits):
    """rho[a][b] = sum over index pairs (i, j) that agree off the targets and
    read a, b on them (qubits[0] = MSB) of psi_i conj(psi_j): explicit loops."""
    n = int(np.log2(psi.size))
    k = len(qubits)
    rho = np.zeros((2 ** k, 2 ** k), dtype=complex)
    tmask = sum(1 << (n - 1 - q) for q in qubits)
    for i in range(2 ** n):
        a = sum(((i >> (n - 1 - q)) & 1) << (k - 1 - j) for j, q in enumerate(qubits))
        for j in range(2 ** n):
            if (i & ~tmask) != (j & ~tmask):
                continue
            b = sum(((j >> (n - 1 - q)) & 1) << (k - 1 - t) for t, q in enumerate(qubits))
            rho[a, b] += psi[i] * np.conj(psi[j])
    return rho


def test_reduced_dm_closed_forms():
    """Product state: the reduced state of a qubit is its own |v><v| (in the
    order asked for); GHZ: every 2-qubit marginal is diag(1/2, 0, 0, 1/2) and
    every 1-qubit marginal I/2 (textbook partial traces)."""
    psi = O.init_tokens(4, "0+1-")
    plus = np.array([1, 1]) / np.sqrt(2)
    minus = np.array([1, -1]) / np.sqrt(2)
    assert np.max(np.abs(O.reduced_dm(psi, [1]) - np.outer(plus, plus))) < 1e-15
    v = np.kron(minus, [1, 0])                      # qubits [3, 0]: qubit 3 is the MSB
    assert np.max(np.abs(O.reduced_dm(psi, [3, 0]) - np.outer(v, v))) < 1e-15
    ghz = np.zeros(8, dtype=complex)
    ghz[0] = ghz[7] = 1 / np.sqrt(2)
    for qs in ([0, 1], [2, 0], [1, 2]):
        assert np.max(np.abs(O.reduced_dm(ghz, qs) - np.diag([0.5, 0, 0, 0.5]))) < 1e-15
    assert np.max(np.abs(O.reduced_dm(ghz, [1]) - np.eye(2) / 2)) < 1e-15


@pytest.mark.parametrize("qubits", [[2], [4, 1], [0, 3, 2]])
def test_reduced_dm_brute_force_and_observables(qubits):
    """Against the explicit double loop, and Tr(O rho_T) = <psi| O (x) I |psi>
    with O embedded by embed_dense (an independent route, order-sensitive)."""
    n = 5
    psi = random_state(n, 31)
    rho = O.reduced_dm(psi, qubits)
    assert np.max(np.abs(rho - _rdm_brute(psi, qubits))) < 1e-14
    rng = np.random.default_rng(9)
    d = 2 ** len(qubits)
    A = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    Oh = A + A.conj().T
    want = np.vdot(psi, O.embed_dense(n, Oh, qubits) @ psi)
    assert abs(np.trace(Oh @ rho) - want) < 1e-12
    assert abs(np.trace(rho) - 1) < 1e-14 and np.max(np.abs(rho - rho.conj().T)) < 1e-15
    assert np.min(np.linalg.eigvalsh(rho)) > -1e-14


def _dephasing(p):
    return [np.sqrt(1 - p) * np.eye(2, dtype=complex), np.sqrt(p) * np.diag([1, -1]).astype(complex)]


def test_kraus_step_closed_forms():
    """Dephasing on |+>: p = (1 - p, p), branch 1 leaves |->; amplitude
    damping on |1>: p = (1 - g, g), branch 1 decays to |0>; a one-element
    channel {U} is the plain gate with p = (1,)."""
    plus = O.init_tokens(1, "+")
    out, i, p = O.kraus_sample_step(plus, _dephasing(0.3), [0], 0.2)
    assert i == 0 and np.allclose(p, [0.7, 0.3], atol=1e-15) and np.allclose(out, plus, atol=1e-15)
    out, i, p = O.kraus_sample_step(plus, _dephasing(0.3), [0], 0.8)
    assert i == 1 and np.allclose(out, O.init_tokens(1, "-"), atol=1e-15)
    one = O.init_tokens(1, "1")
    out, i, p = O.kraus_sample_step(one, _amp_damping(0.25), [0], 0.9)
    assert i == 1 and np.allclose(p, [0.75, 0.25], atol=1e-15) and np.allclose(out, [1, 0], atol=1e-15)
    psi = random_state(3, 4)
    U = haar_unitary(2, np.random.default_rng(3))
    out, i, p = O.kraus_sample_step(psi, [U], [2, 0], 0.5)
    assert i == 0 and abs(p[0] - 1) < 1e-14
    assert np.max(np.abs(out - O.simulate(3, [Gate("U", (2, 0), U)], psi))) < 1e-14
    with pytest.raises(O.OracleError):
        O.kraus_sample_step(O.init_tokens(1, "0"), [np.diag([0, 1]).astype(complex)], [0], 0.5)


def test_kraus_step_unravels_the_channel():
    """Averaging the post-step pure states over u (exactly: each branch with
    weight p_i / sum p) gives sum_i K_i rho K_i^dagger / sum p -- the
    trajectory unraveling of the density-matrix map."""
    n = 3
    psi = random_state(n, 8)
    rng = np.random.default_rng(4)
    Z = rng.standard_normal((12, 4)) + 1j * rng.standard_normal((12, 4))
    V, _ = np.linalg.qr(Z)
    K = [V[4 * i:4 * (i + 1)] for i in range(3)]            # CPTP 2-qubit channel
    _, _, p = O.kraus_sample_step(psi, K, [2, 0], 0.0)
    mean = np.zeros((2 ** n, 2 ** n), dtype=complex)
    cum = np.concatenate([[0], np.cumsum(p)])
    for i in range(3):
        u = (cum[i] + p[i] / 2) / p.sum()
        out, j, _ = O.kraus_sample_step(psi, K, [2, 0], u)
        assert j == i
        mean += p[i] / p.sum() * np.outer(out, out.conj())
    want = O.dm_apply_kraus(np.outer(psi, psi.conj()), K, [2, 0])
    assert abs(p.sum() - 1) < 1e-14
    assert np.max(np.abs(mean - want)) < 1e-14


# ---------------------------------------------------------------- P10 reversible image
def test_P10_reversible_image_textbook_sequence():
    """X, CX, SWAP, CCX on |0000> by hand (qubit 0 = MSB, C1; control first,
    C2): X(0) -> 1000, CX(0,3) -> 1001, SWAP(1,3) -> 1100, CCX(0,1,2) -> 1110."""
    n = 4
    seq = [Gate("X", (0,), X), Gate("CX", (0, 3), CX), Gate("SWAP", (1, 3), SWAP),
           Gate("CCX", (0, 1, 2), CCX)]
    want = [0b1000, 0b1001, 0b1100, 0b1110]
    for i in range(len(seq)):
        assert O.reversible_image(n, seq[:i + 1], 0) == want[i]
    with pytest.raises(O.OracleError):
        O.reversible_image(n, [Gate("H", (0,), H)], 0)


def test_P10_reversible_image_agrees_with_dense_simulation():
    from hq_inputs import reversible_circuit
    n = 8
    gates = reversible_circuit(n, 40, 5, kmax=3)
    for x in (0, 1, 77, 255):
        psi = O.simulate(n, gates, x=x)
        y = O.reversible_image(n, gates, x)
        assert psi[y] == 1.0 and np.count_nonzero(psi) == 1
