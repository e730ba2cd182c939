"""f4 row on the GPU: token product states, projection, Born probabilities and
measurement through the C ABI vs the oracle, on default and permuted layouts
and on virtual shards (global qubits handled per rank)."""
import numpy as np
import pytest

import oracle as O
from hq_inputs import Gate, sycamore_circuit, random_state
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu

TOL = {"c64": 2e-6, "c128": 1e-13}


def _states(n, dtype):
    """(name, state) pairs: default layout, random layout, 4 virtual shards."""
    out = [("default", hq.hq_state_create(n, dtype, 1))]
    s = hq.hq_state_create(n, dtype, 1)
    hq.hq_state_set_layout(s, [int(x) for x in np.random.default_rng(n).permutation(n)])
    out.append(("layout", s))
    out.append(("virtual4", hq.hq_state_create_virtual(n, dtype, 4)))
    return out


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_init_tokens(dtype):
    n = 12
    rng = np.random.default_rng(3)
    for trial in range(4):
        tok = "".join(rng.choice(list("01+-"), size=n)) if trial else "+"
        want = O.init_tokens(n, tok)
        for name, s in _states(n, dtype):
            hq.hq_state_init_tokens(s, tok)
            got = hq.hq_get_amplitudes(s).astype(np.complex128)
            assert np.max(np.abs(got - want)) < TOL[dtype], (name, tok)


def test_init_tokens_errors():
    s = hq.hq_state_create(4, "c64", 1)
    for bad in ("0.1+", "abcd", "01", ""):
        with pytest.raises(hq.HQError) as e:
            hq.hq_state_init_tokens(s, bad)
        assert e.value.status == "HQ_ERR_ARG"


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_project_and_probabilities(dtype):
    n = 13
    gates = hq.hq_fuse(sycamore_circuit(n, 8, 4), 4)
    psi_ref = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    for name, s in _states(n, dtype):
        hq.hq_state_init_basis(s, 0)
        hq.hq_apply_circuit(s, gates)
        for qs in ([0], [12, 3], [5, 0, 9], list(range(10))):
            p = hq.hq_probabilities(s, qs)
            want = O.probabilities(psi_ref, qs)
            assert np.max(np.abs(p - want)) < (1e-6 if dtype == "c64" else 1e-13), (name, qs)
        qs, bits = [2, 11, 0], [1, 0, 1]
        nrm = hq.hq_project(s, qs, bits, renormalize=True)
        want, wn = O.project(psi_ref, qs, bits, renormalize=True)
        assert abs(nrm - wn) < 1e-6
        got = hq.hq_get_amplitudes(s).astype(np.complex128)
        assert np.linalg.norm(got - want) < (1e-4 if dtype == "c64" else 1e-10), name


def test_grover_via_projection_on_gpu():
    """The paper's Grover oracle psi - 2 P_0 psi assembled from
    hq_project on two GPU states; matches the printed listing."""
    a = hq.hq_state_create(3, "c128", 1)
    b = hq.hq_state_create(3, "c128", 1)
    hq.hq_state_init_tokens(a, "+")
    hq.hq_state_init_tokens(b, "+")
    hq.hq_project(b, [1, 2], [0, 0], renormalize=False)
    new = hq.hq_get_amplitudes(a) - 2 * hq.hq_get_amplitudes(b)
    want = np.full(8, 1 / np.sqrt(8))
    want[[0, 4]] *= -1
    assert np.max(np.abs(new - want)) < 1e-15


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_measure_collapses_consistently(dtype):
    n = 12
    gates = hq.hq_fuse(sycamore_circuit(n, 8, 9), 4)
    psi_ref = O.simulate(n, [Gate("F", q, U) for q, U in gates])
    qs = [7, 1]
    probs = O.probabilities(psi_ref, qs)
    cum = np.cumsum(probs)
    for u in (0.0, 0.3, 0.77, 0.999):
        s = hq.hq_state_create(n, dtype, 1)
        hq.hq_state_init_basis(s, 0)
        hq.hq_apply_circuit(s, gates)
        x = hq.hq_measure(s, qs, u)
        assert x == int(np.searchsorted(cum, u * cum[-1], side="right"))
        bits = [(x >> 1) & 1, x & 1]
        want, _ = O.project(psi_ref, qs, bits, renormalize=True)
        got = hq.hq_get_amplitudes(s).astype(np.complex128)
        assert np.linalg.norm(got - want) < (1e-4 if dtype == "c64" else 1e-10)
        assert abs(hq.hq_norm(s) - 1) < 1e-6


def test_measure_basis_and_plus():
    s = hq.hq_state_create(6, "c64", 1)
    hq.hq_state_init_tokens(s, "010101")
    assert hq.hq_measure(s, [1, 3], 0.5) == 3
    hq.hq_state_init_tokens(s, "+")
    p = hq.hq_probabilities(s, [0])
    assert np.allclose(p, [0.5, 0.5], atol=1e-7)
    assert hq.hq_measure(s, [0], 0.25) == 0
    assert np.allclose(hq.hq_probabilities(s, [0]), [1, 0], atol=1e-7)
    with pytest.raises(hq.HQError):
        hq.hq_project(s, [0], [1], renormalize=True)      # ZeroNormProjection
