"""Row f3 on the GPU: reduced density matrices and Kraus trajectory steps
through the C ABI against the oracle (same states, same uniforms), on default
and permuted layouts and on virtual shards (targets on global qubits take the
remap path), plus the trajectory runner against closed forms."""
import numpy as np
import pytest

import oracle as O
from hq_inputs import Gate, random_state, haar_unitary
import paper_2111_06868_b200 as hq
from paper_2111_06868_b200.trajectories import Channel, sample_trajectories

pytestmark = pytest.mark.gpu

TOL = {"c64": 2e-6, "c128": 1e-13}


def _states(n, dtype, psi):
    out = []
    for name in ("default", "layout", "virtual4"):
        if name == "virtual4":
            s = hq.hq_state_create_virtual(n, dtype, 4)
        else:
            s = hq.hq_state_create(n, dtype, 1)
            if name == "layout":
                hq.hq_state_set_layout(s, [int(x) for x in np.random.default_rng(n).permutation(n)])
        hq.hq_set_amplitudes(s, psi.astype(s.np_dtype))
        out.append((name, s))
    return out


def _channel(k, m, seed):
    rng = np.random.default_rng(seed)
    d = 2 ** k
    Z = rng.standard_normal((d * m, d)) + 1j * rng.standard_normal((d * m, d))
    V, _ = np.linalg.qr(Z)
    return [V[i * d:(i + 1) * d, :] for i in range(m)]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("qubits", [[0], [13], [5, 2], [0, 13], [7, 1, 12]])
def test_reduced_dm_matches_oracle(dtype, qubits):
    n = 14
    psi = random_state(n, 3)
    want = O.reduced_dm(psi, qubits)
    for name, s in _states(n, dtype, psi):
        got = hq.hq_reduced_dm(s, qubits)
        assert np.max(np.abs(got - want)) < TOL[dtype], (name, qubits)
        # the layout may change (global targets), the state must not
        back = hq.hq_get_amplitudes(s).astype(np.complex128)
        assert np.max(np.abs(back - psi)) < (1e-7 if dtype == "c64" else 1e-15), name


def test_reduced_dm_large_state_trace():
    """Grid-stride path at a size where every block loops: trace = ||psi||^2."""
    n = 26
    s = hq.hq_state_create(n, "c64", 1)
    hq.hq_state_init_tokens(s, "+")
    rho = hq.hq_reduced_dm(s, [3, 20, 25])
    assert np.max(np.abs(rho - np.full((8, 8), 1 / 8))) < 1e-6


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k,m", [(1, 2), (1, 4), (2, 3), (3, 2)])
def test_kraus_sample_matches_oracle(dtype, k, m):
    n = 12
    psi = random_state(n, 10 + k)
    K = _channel(k, m, 100 * k + m)
    qubits = [11, 4, 0][:k] if k < 3 else [11, 4, 0]
    _, _, p = O.kraus_sample_step(psi, K, qubits, 0.0)
    cum = np.concatenate([[0], np.cumsum(p)]) / p.sum()
    for i in range(m):
        u = (cum[i] + cum[i + 1]) / 2           # the middle of branch i: no boundary ties
        want, wi, _ = O.kraus_sample_step(psi, K, qubits, u)
        assert wi == i
        for name, s in _states(n, dtype, psi):
            ci, probs = hq.hq_kraus_sample(s, K, qubits, u)
            assert ci == i, name
            assert np.max(np.abs(probs - p)) < (1e-6 if dtype == "c64" else 1e-13), name
            got = hq.hq_get_amplitudes(s).astype(np.complex128)
            assert np.linalg.norm(got - want) < (1e-5 if dtype == "c64" else 1e-12), (name, i)
            assert abs(hq.hq_norm(s) - 1) < (1e-6 if dtype == "c64" else 1e-13)


def test_kraus_sample_errors():
    s = hq.hq_state_create(4, "c64", 1)
    hq.hq_state_init_tokens(s, "0")
    with pytest.raises(hq.HQError) as e:              # ZeroNormBranch
        hq.hq_kraus_sample(s, [np.diag([0, 1]).astype(complex)], [2], 0.5)
    assert e.value.status == "HQ_ERR_RANGE"
    assert hq.hq_get_amplitudes(s)[0] == 1.0          # state unchanged
    with pytest.raises(hq.HQError):
        hq.hq_kraus_sample(s, [np.eye(2)], [2], 1.0)   # u not in [0, 1)
    with pytest.raises(hq.HQError):
        hq.hq_reduced_dm(s, [0, 1, 2, 3])              # k > 3


def test_trajectories_fig1_depolarizing_closed_form():
    """SPEC S:530 / paper Fig. 1 scenario: |+>, RZ(theta) steps each followed
    by single-qubit depolarizing p: <X>_t = (1 - p)^t cos(t theta) (Bloch
    vector shrinks by 1 - p per channel).  Trajectory means at 3000 shots
    within 4 sigma (sigma <= 1/sqrt(shots)) at every step."""
    theta, p, steps, shots = 0.3, 0.08, 6, 3000
    RZ = np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta)])
    s4 = np.sqrt(p / 4)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    Y = np.array([[0, -1j], [1j, 0]])
    Z = np.diag([1, -1]).astype(complex)
    depol = [np.sqrt(1 - 3 * p / 4) * np.eye(2), s4 * X, s4 * Y, s4 * Z]
    ops = []
    for t in range(steps):
        ops += [Gate("RZ", (0,), RZ), Channel([0], depol)]
    marks = [2 * t + 1 for t in range(steps - 1)]
    res = sample_trajectories(2, ops, shots, observe=[0], seed=7, init="+", per_step=marks)
    rhos = res["rho_steps"] + [res["rho"]]
    for t, rho in enumerate(rhos, start=1):
        ex = 2 * rho[0, 1].real                       # <X> = Tr(X rho)
        want = (1 - p) ** t * np.cos(t * theta)
        assert abs(ex - want) < 4 / np.sqrt(shots), (t, ex, want)
    assert res["shots"] == shots


def test_trajectories_noiseless_equal_statevector():
    """no channels -> every trajectory is the state-vector result."""
    n = 10
    gates = [Gate("U", (q, (q + 3) % n), haar_unitary(2, np.random.default_rng(q))) for q in range(n)]
    res = sample_trajectories(n, gates, 3, observe=[2, 7], seed=1)
    psi = O.simulate(n, gates)
    assert np.max(np.abs(res["rho"] - O.reduced_dm(psi, [2, 7]))) < 2e-6


def test_trajectories_mean_matches_density_matrix():
    """Trajectory average vs the exact density-matrix evolution (oracle) on a
    small noisy circuit with 2-qubit channels: within 5/sqrt(shots)."""
    n = 4
    rng = np.random.default_rng(3)
    ops = []
    rho = np.zeros((2 ** n, 2 ** n), dtype=complex)
    rho[0, 0] = 1
    for layer in range(3):
        for q in range(0, n, 2):
            U = haar_unitary(2, rng)
            ops.append(Gate("U", (q, q + 1), U))
            rho = O.dm_apply_kraus(rho, [U], [q, q + 1])
        K = _channel(2, 3, 50 + layer)
        ops.append(Channel([1, 2], K))
        rho = O.dm_apply_kraus(rho, K, [1, 2])
    shots = 2000
    res = sample_trajectories(n, ops, shots, observe=[0, 1], seed=5)
    # reduced density matrix of qubits (0, 1) from the full rho
    r = rho.reshape(4, 4, 4, 4)
    want = np.einsum("aibi->ab", r)
    assert np.max(np.abs(res["rho"] - want)) < 5 / np.sqrt(shots)


# ---------------------------------------------------------------- batched trajectories

def _batched_state(nb, n, dtype, seed):
    """2^nb shots, shot s holding random_state(n, seed + s) / sqrt(2^nb)."""
    S = 2 ** nb
    blocks = [random_state(n, seed + s) for s in range(S)]
    psi = np.concatenate(blocks) / np.sqrt(S)
    st = hq.hq_state_create(n + nb, dtype, 1)
    hq.hq_set_amplitudes(st, psi.astype(st.np_dtype))
    return st, blocks


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("qubits", [[0], [9, 2], [7, 0, 4]])
def test_reduced_dm_batched_matches_oracle(dtype, qubits):
    nb, n = 5, 10
    st, blocks = _batched_state(nb, n, dtype, 40)
    rho = hq.hq_reduced_dm_batched(st, nb, [q + nb for q in qubits])
    for s_, b in enumerate(blocks):
        want = O.reduced_dm(b, qubits) / 2 ** nb
        assert np.max(np.abs(rho[s_] - want)) < TOL[dtype] / 2 ** nb * 4, s_


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k,m", [(1, 4), (2, 3), (3, 2)])
def test_kraus_sample_batched_matches_oracle(dtype, k, m):
    nb, n = 4, 9
    S = 2 ** nb
    st, blocks = _batched_state(nb, n, dtype, 70)
    K = _channel(k, m, 7 * k + m)
    qubits = [8, 3, 0][:k]
    rng = np.random.default_rng(k)
    us, wants, idx = [], [], []
    for b in blocks:
        _, _, p = O.kraus_sample_step(b, K, qubits, 0.0)
        i = int(rng.integers(m))
        cum = np.concatenate([[0], np.cumsum(p)]) / p.sum()
        u = (cum[i] + cum[i + 1]) / 2
        w, wi, _ = O.kraus_sample_step(b, K, qubits, u)
        assert wi == i
        us.append(u)
        wants.append(w)
        idx.append(i)
    chosen, probs = hq.hq_kraus_sample_batched(st, nb, K, [q + nb for q in qubits], np.array(us))
    assert list(chosen) == idx
    got = hq.hq_get_amplitudes(st).astype(np.complex128).reshape(S, -1) * np.sqrt(S)
    for s_ in range(S):
        assert np.linalg.norm(got[s_] - wants[s_]) < (1e-5 if dtype == "c64" else 1e-12), s_
    assert abs(hq.hq_norm(st) - 1) < 1e-5


def test_batched_errors():
    st = hq.hq_state_create(8, "c64", 1)
    hq.hq_state_init_tokens(st, "+")
    with pytest.raises(hq.HQError) as e:
        hq.hq_reduced_dm_batched(st, 3, [1])          # target on a batch qubit
    assert e.value.status == "HQ_ERR_QUBIT"
    v = hq.hq_state_create_virtual(10, "c64", 2)
    hq.hq_state_init_tokens(v, "+")
    with pytest.raises(hq.HQError) as e:
        hq.hq_reduced_dm_batched(v, 2, [5])
    assert e.value.status == "HQ_ERR_STATE"
    lay = hq.hq_state_create(8, "c64", 1)
    hq.hq_state_set_layout(lay, list(range(8)))        # qubit 0 on physical bit 0
    hq.hq_state_init_tokens(lay, "+")
    with pytest.raises(hq.HQError) as e:
        hq.hq_reduced_dm_batched(lay, 2, [5])
    assert e.value.status == "HQ_ERR_STATE"


def test_batched_runner_equals_unbatched():
    """Same seeds -> same branch choices and the same mean as one shot per
    state (batch = 8 with a ragged last batch: 21 shots)."""
    n = 6
    rng = np.random.default_rng(12)
    ops = []
    for layer in range(3):
        for q in range(0, n - 1, 2):
            ops.append(Gate("U", (q, q + 1), haar_unitary(2, rng)))
        ops.append(Channel([layer % n, (layer + 2) % n], _channel(2, 3, 90 + layer)))
        ops.append(Channel([5], _channel(1, 2, 80 + layer)))
    a = sample_trajectories(n, ops, 21, observe=[1, 4], seed=3)
    b = sample_trajectories(n, ops, 21, observe=[1, 4], seed=3, batch=8)
    assert a["chosen"] == b["chosen"]
    assert np.max(np.abs(a["rho"] - b["rho"])) < 2e-6


def test_trajectories_fig1_batched():
    theta, p, steps, shots = 0.3, 0.08, 6, 4096
    RZ = np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta)])
    s4 = np.sqrt(p / 4)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    Y = np.array([[0, -1j], [1j, 0]])
    Z = np.diag([1, -1]).astype(complex)
    depol = [np.sqrt(1 - 3 * p / 4) * np.eye(2), s4 * X, s4 * Y, s4 * Z]
    ops = []
    for t in range(steps):
        ops += [Gate("RZ", (0,), RZ), Channel([0], depol)]
    marks = [2 * t + 1 for t in range(steps - 1)]
    res = sample_trajectories(1, ops, shots, observe=[0], seed=9, init="+", per_step=marks, batch=1024)
    for t, rho in enumerate(res["rho_steps"] + [res["rho"]], start=1):
        ex = 2 * rho[0, 1].real
        assert abs(ex - (1 - p) ** t * np.cos(t * theta)) < 4 / np.sqrt(shots), t
