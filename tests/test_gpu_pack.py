"""apply+pack (row f1): the scheduler packs the evictees of a
remap onto the top local bits with a PERMUTE that the executor folds into
the preceding apply pass (out-of-place, bit-permuted write into the exchange
buffer).  Checked on virtual shards (the real kernels, scheduler and chunk
arithmetic on one B200) against the fp64 oracle, for every kernel family that
can fold (tensor-core modes H and L, SIMT, generic) and through both the
direct (hq_apply_circuit) and the compiled (hq_circuit_run) executor; the
reversible circuits are bit-exact (pin P10)."""
import numpy as np
import pytest

import oracle as O
from hq_inputs import Gate, sycamore_circuit, reversible_circuit, integer_state, haar_sweep_gate, random_state
import paper_2111_06868_b200 as hq

pytestmark = pytest.mark.gpu
TOL = {"c64": 1e-4, "c128": 1e-10}


def _run(n, dtype, G, fused, planned, compiled, psi0=None, x=0, mode="fused+gather"):
    m = G.bit_length() - 1
    s = hq.hq_state_create_virtual(n, dtype, G)
    hq.hq_state_set_remap_mode(s, mode)
    if planned:
        pi0, _, _ = hq.hq_plan_layout(n, m, fused, dtype)
        hq.hq_state_set_layout(s, pi0)
    if psi0 is None:
        hq.hq_state_init_basis(s, x)
    else:
        hq.hq_set_amplitudes(s, psi0)
    hq.hq_stats_reset(s)
    if compiled:
        c = hq.hq_circuit_create(s, fused)
        hq.hq_circuit_run(s, c)
    else:
        hq.hq_apply_circuit(s, fused)
    return s, hq.hq_stats_get(s)


@pytest.mark.parametrize("compiled", [False, True])
@pytest.mark.parametrize("planned", [False, True])
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kmax", [4, 6])
def test_pack_sycamore_vs_oracle(kmax, G, planned, compiled):
    """20 qubits: k<=6 blocks run on the tensor cores (n_local >= 16), k<=4 on
    the SIMT kernel; every pack is folded (no standalone permute pass)."""
    n = 20
    gates = sycamore_circuit(n, 14, 77)
    fused = hq.hq_fuse(gates, kmax, blocks=True)
    s, st = _run(n, "c64", G, fused, planned, compiled)
    assert st["remaps"] > 0
    assert st["packs"] > 0 and st["permutes"] == 0, st
    err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.simulate(n, gates))
    assert err <= 1e-4, err


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,G,kmax", [(12, 4, 3), (12, 8, 6), (18, 4, 4), (20, 4, 6)])
def test_pack_every_kernel_family(dtype, n, G, kmax):
    """Small n (generic kernel), SIMT, complex128 (SIMT; its k = 5, 6 tile
    kernel cannot fold, so those packs run as standalone permute passes)."""
    gates = sycamore_circuit(n, 12, 5)
    fused = hq.hq_fuse(gates, kmax)
    s, st = _run(n, dtype, G, fused, True, False)
    assert st["remaps"] > 0
    err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.simulate(n, gates))
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("kmax", [3, 6])
@pytest.mark.parametrize("G", [4, 8])
def test_pack_reversible_bit_exact(kmax, G):
    """Permutation gates on an integer-valued state through packs and remaps:
    every amplitude equal (C11), and a basis state lands exactly on f(x) (P10)."""
    n = 20
    gates = reversible_circuit(n, 120, 31, kmax=3)
    fused = hq.hq_fuse(gates, kmax)
    psi0 = integer_state(n, 4)
    s, st = _run(n, "c64", G, fused, True, True, psi0=psi0)
    assert st["remaps"] > 0 and st["permutes"] == 0, st
    assert np.array_equal(hq.hq_get_amplitudes(s).astype(np.complex128), O.simulate(n, gates, psi0))
    x = 0xBEEF5
    s, st = _run(n, "c64", G, fused, True, False, x=x)
    y = O.reversible_image(n, gates, x)
    got = hq.hq_get_amplitudes(s)
    assert got[y] == 1.0 and np.count_nonzero(got) == 1


def test_pack_single_pass_every_tc_mode():
    """One k = 6 gate at mode-H and mode-L placements, then a segment that
    needs global qubit 0 and the top local bits 10..17: the remap's evictee
    lies below the run window, so the k = 6 pass carries the pack
    (2e-6 single-pass bound)."""
    from hq_inputs import haar_unitary
    n, G = 20, 4
    rng = np.random.default_rng(5)
    H = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    tail = [Gate("H0", (0,), H),
            Gate("U6", tuple(n - 1 - b for b in range(11, 17)), haar_unitary(6, rng)),
            Gate("U2", (n - 1 - 17, n - 1 - 10), haar_unitary(2, rng))]
    for placement in ("low", "b:0-3-7-9-14-15", "b:1-2-3-7-8-9", "b:0-2-5-9-12-15"):
        g = haar_sweep_gate(n, 6, placement, 2301)
        gates = [g] + tail
        psi0 = random_state(n, 12)
        s, st = _run(n, "c64", G, [(tuple(x.qubits), x.U) for x in gates], False, False, psi0=psi0,
                     mode="exchange")
        assert st["remaps"] == 1 and st["packs"] == 1 and st["permutes"] == 0, (placement, st)
        want = O.simulate(n, gates, psi0)
        err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - want)
        assert err < 4e-6, (placement, err)


# ---------------------------------------------------------------- fused remaps
@pytest.mark.parametrize("kmax", [4, 6])
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("compiled", [False, True])
def test_fused_remap_vs_exchange_and_oracle(kmax, G, compiled):
    """Fused remaps (the apply pass writes each element into its destination
    shard's exchange buffer) give bit-identical amplitudes to the separate
    exchange path (same kernels, only the output addresses differ) and match
    the oracle; on virtual shards every packed remap fuses."""
    n = 20
    gates = sycamore_circuit(n, 14, 78)
    fused = hq.hq_fuse(gates, kmax, blocks=True)
    m = G.bit_length() - 1
    out = {}
    for mode in ("exchange", "fused"):                         # fused without gathers: same kernels
        s = hq.hq_state_create_virtual(n, "c64", G)
        assert hq.hq_state_set_remap_mode(s, mode)            # virtual shards: always mappable
        pi0, _, _ = hq.hq_plan_layout(n, m, fused)
        hq.hq_state_set_layout(s, pi0)
        hq.hq_state_init_basis(s, 0)
        hq.hq_stats_reset(s)
        if compiled:
            hq.hq_circuit_run(s, hq.hq_circuit_create(s, fused))
        else:
            hq.hq_apply_circuit(s, fused)
        out[mode] = (hq.hq_get_amplitudes(s), hq.hq_stats_get(s))
    a_x, st_x = out["exchange"]
    a_f, st_f = out["fused"]
    assert st_x["remaps_fused"] == 0 and st_f["remaps"] == st_x["remaps"] > 0
    assert st_f["remaps_fused"] > 0, st_f
    assert np.array_equal(a_x, a_f)
    err = np.linalg.norm(a_f.astype(np.complex128) - O.simulate(n, gates))
    assert err <= 1e-4, err


@pytest.mark.parametrize("G", [4, 8])
def test_fused_remap_reversible_bit_exact(G):
    n = 20
    gates = reversible_circuit(n, 150, 37, kmax=3)
    fused = hq.hq_fuse(gates, 6)
    m = G.bit_length() - 1
    s = hq.hq_state_create_virtual(n, "c64", G)
    hq.hq_state_set_remap_mode(s, "fused")
    hq.hq_state_set_layout(s, hq.hq_plan_layout(n, m, fused)[0])
    x = 0x5C3A7
    hq.hq_state_init_basis(s, x)
    hq.hq_apply_circuit(s, fused)
    y = O.reversible_image(n, gates, x)
    got = hq.hq_get_amplitudes(s)
    assert got[y] == 1.0 and np.count_nonzero(got) == 1


# ---------------------------------------------------------------- pair gathers (row f1)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("compiled", [False, True])
def test_pair_gather_qft_no_remaps(dtype, G, compiled):
    """QFT on virtual shards: the Hadamards on global qubits run as pair
    gathers (each shard reads its partner's shard and writes its half), the
    controlled phases in place (block-diagonal), so the circuit needs no remap
    at all; matches the oracle."""
    from hq_inputs import qft_circuit
    n = 18
    gates = qft_circuit(n)
    s = hq.hq_state_create_virtual(n, dtype, G)
    psi0 = random_state(n, 21)
    hq.hq_set_amplitudes(s, psi0)
    hq.hq_stats_reset(s)
    if compiled:
        hq.hq_circuit_run(s, hq.hq_circuit_create(s, [(tuple(g.qubits), g.U) for g in gates]))
    else:
        hq.hq_apply_circuit(s, gates)
    st = hq.hq_stats_get(s)
    assert st["gathers"] > 0 and st["remaps"] == 0, st
    err = np.linalg.norm(hq.hq_get_amplitudes(s).astype(np.complex128) - O.simulate(n, gates, psi0))
    assert err <= TOL[dtype], err
    # the exchange mode (no peer gathers) gives the same result through remaps
    s2 = hq.hq_state_create_virtual(n, dtype, G)
    hq.hq_state_set_remap_mode(s2, "exchange")
    hq.hq_set_amplitudes(s2, psi0)
    hq.hq_stats_reset(s2)
    hq.hq_apply_circuit(s2, gates)
    assert hq.hq_stats_get(s2)["gathers"] == 0 and hq.hq_stats_get(s2)["remaps"] > 0
    err2 = np.linalg.norm(hq.hq_get_amplitudes(s2).astype(np.complex128) - O.simulate(n, gates, psi0))
    assert err2 <= TOL[dtype], err2


def test_pair_gather_reversible_bit_exact():
    """A permutation gate with one global target through a pair gather is exact."""
    from hq_inputs import CX, X, CCX
    n, G = 16, 4
    gates = [Gate("X", (0,), X), Gate("CX", (0, 9), CX), Gate("CCX", (3, 1, 12), CCX), Gate("X", (1,), X)]
    x = 0x1234
    s = hq.hq_state_create_virtual(n, "c64", G)
    hq.hq_state_init_basis(s, x)
    hq.hq_apply_circuit(s, gates)
    y = O.reversible_image(n, gates, x)
    got = hq.hq_get_amplitudes(s)
    assert got[y] == 1.0 and np.count_nonzero(got) == 1
    assert hq.hq_stats_get(s)["gathers"] > 0
