"""CPU-side tests of the C-ABI library: it loads, exports every symbol that
include/hq.h declares, fails loudly without a GPU, and its host logic (fusion
planner, distributed schedule) matches the oracle.  No compute calls here."""
import os
import re

import numpy as np
import pytest

import oracle as O
from hq_inputs import (Gate, sycamore_circuit, random_circuit, reversible_circuit, cphase,
                       random_state, haar_unitary)
import paper_2111_06868_b200 as hq
from paper_2111_06868_b200 import build as hqbuild

from sched_replay import replay_all_shards, to_logical

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    hqbuild.build()


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "hq.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    declared = set(re.findall(r"\b(hq_[a-z_0-9]+)\s*\(", header))
    assert len(declared) >= 30
    L = hq.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hq.HQError) as e:
        hq.hq_state_create(8, "c64", 1)
    assert e.value.status == "HQ_ERR_NO_DEVICE"


def _groups_from_oracle(gates, kmax):
    g = O.compress(gates, kmax)
    out = np.empty(len(gates), dtype=np.int32)
    for gi, members in enumerate(g):
        out[members] = gi
    return out, len(g)


def test_fuse_P2_worked_example():
    """PAPER P:510-529."""
    gates = [Gate("CPHASE", (q1, q2), cphase(1.0)) for q1 in range(5) for q2 in range(q1 + 1, 5)]
    fused = hq.hq_fuse(gates, 3)
    assert [f[0] for f in fused] == [(0, 1, 2), (0, 3, 4), (1, 3, 4), (2, 3, 4)]


@pytest.mark.parametrize("kmax", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("n,cycles,seed", [(12, 10, 0), (12, 10, 3), (30, 20, 1000), (34, 20, 3000)])
def test_fuse_groups_bit_exact_vs_oracle(n, cycles, seed, kmax):
    gates = sycamore_circuit(n, cycles, seed)
    got, ng = hq.hq_fuse_plan(gates, kmax)
    want, nw = _groups_from_oracle(gates, kmax)
    assert ng == nw
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", range(6))
def test_fuse_groups_random_circuits(seed):
    gates = random_circuit(9, 80, seed, kmax=3)
    for kmax in (3, 4, 5, 6):
        got, _ = hq.hq_fuse_plan(gates, kmax)
        want, _ = _groups_from_oracle(gates, kmax)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("kmax", [2, 4, 5, 6])
def test_fused_matrices_vs_oracle(kmax):
    gates = sycamore_circuit(12, 10, 2)
    got = hq.hq_fuse(gates, kmax)
    want = O.fused_gates(gates, kmax)
    assert len(got) == len(want)
    for (qg, Ug), (qw, Uw) in zip(got, want):
        assert qg == qw
        assert np.max(np.abs(Ug - Uw)) < 1e-13


def test_fuse_errors():
    gates = [Gate("U", (0, 1, 2), np.eye(8))]
    with pytest.raises(hq.HQError) as e:
        hq.hq_fuse(gates, 2)
    assert e.value.status == "HQ_ERR_K"
    with pytest.raises(hq.HQError) as e:
        hq.hq_fuse([Gate("U", (1, 1), np.eye(4))], 3)
    assert e.value.status == "HQ_ERR_DUP_QUBIT"
    with pytest.raises(hq.HQError) as e:
        hq.hq_fuse(gates, 7)
    assert e.value.status == "HQ_ERR_K"
    assert hq.hq_fuse([], 3) == []


# ---------------------------------------------------------------- distributed schedule

@pytest.mark.parametrize("m", [0, 1, 2, 3])
@pytest.mark.parametrize("kind", ["sycamore", "random"])
def test_schedule_replay_matches_oracle(m, kind):
    n = 12
    if kind == "sycamore":
        gates = [Gate("F", q, U) for q, U in O.fused_gates(sycamore_circuit(n, 10, 1), 4)]
    else:
        gates = random_circuit(n, 60, 5, kmax=4)
    ops, pi = hq.hq_schedule(n, m, gates)
    assert sum(o["kind"] == "apply" for o in ops) == len(gates)
    if m == 0:
        assert all(o["kind"] == "apply" for o in ops)
    # every APPLY target is local, or the gate is block-diagonal in its
    # global targets (row f1), checked here independently on U
    for o in ops:
        if o["kind"] == "apply":
            g = gates[o["gate"]]
            _assert_local_or_block_diag(g.U, o["bits"][:len(g.qubits)], n - m)
    psi0 = random_state(n, 3)
    shards = replay_all_shards(n, m, gates, ops, psi0)
    got = to_logical(n, shards, pi)
    want = O.simulate(n, gates, psi0)
    assert np.max(np.abs(got - want)) < 1e-12


def _assert_local_or_block_diag(U, bits, nl):
    k = len(bits)
    gmask = sum(1 << (k - 1 - j) for j, b in enumerate(bits) if b >= nl)
    if gmask == 0:
        return
    D = 2 ** k
    for r in range(D):
        for c in range(D):
            if (r ^ c) & gmask:
                assert U[r, c] == 0, "APPLY on a global target with a non-block-diagonal U"


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("kind", ["qft", "qaoa"])
def test_schedule_global_diagonal_gates_skip_remaps(m, kind):
    """Row f1: controlled-phase / ZZ gates on global qubits run in place with
    rank-selected blocks; the replay (cond_block per rank) matches the oracle
    and the op stream needs fewer remaps than the same circuit with every
    diagonal gate replaced by a dense one on the same qubits."""
    from hq_inputs import qft_circuit, qaoa_circuit
    n = 12
    gates = qft_circuit(n) if kind == "qft" else qaoa_circuit(n, 3, 7)
    ops, pi = hq.hq_schedule(n, m, gates)
    cond = [o for o in ops if o["kind"] == "apply"
            and any(b >= n - m for b in o["bits"][:len(gates[o["gate"]].qubits)])]
    assert cond, "expected in-place applies on global qubits"
    for o in cond:
        g = gates[o["gate"]]
        _assert_local_or_block_diag(g.U, o["bits"][:len(g.qubits)], n - m)
    psi0 = random_state(n, 5)
    got = to_logical(n, replay_all_shards(n, m, gates, ops, psi0), pi)
    assert np.max(np.abs(got - O.simulate(n, gates, psi0))) < 1e-12
    rng = np.random.default_rng(1)
    dense = [Gate(g.name, g.qubits, haar_unitary(len(g.qubits), rng))
             if np.count_nonzero(g.U - np.diag(np.diag(g.U))) == 0 else g for g in gates]
    ops_d, _ = hq.hq_schedule(n, m, dense)
    r_diag = sum(o["kind"] == "remap" for o in ops)
    r_dense = sum(o["kind"] == "remap" for o in ops_d)
    assert r_diag < r_dense, (r_diag, r_dense)


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("kind", ["qft", "random"])
def test_schedule_gather_ops_replay(m, kind):
    """Row f1, GATHER ops: with gathers allowed, isolated global accesses
    (a global qubit not needed local again within the lookahead) run across
    the rank pair instead of triggering a remap; the replay (the gate on the
    whole physical vector) matches the oracle and needs no more remaps."""
    from hq_inputs import qft_circuit
    n = 12
    gates = qft_circuit(n) if kind == "qft" else random_circuit(n, 40, 8, kmax=3)
    ops_g, pi = hq.hq_schedule(n, m, gates, gather=True)
    ops_r, _ = hq.hq_schedule(n, m, gates)
    assert sum(o["kind"] == "remap" for o in ops_g) <= sum(o["kind"] == "remap" for o in ops_r)
    if kind == "qft":
        assert sum(o["kind"] == "gather" for o in ops_g) > 0
        assert sum(o["kind"] == "remap" for o in ops_g) == 0      # H on globals gathered, phases in place
    for o in ops_g:
        if o["kind"] == "gather":
            k = len(gates[o["gate"]].qubits)
            assert sum(b >= n - m for b in o["bits"][:k]) == 1
    psi0 = random_state(n, 4)
    got = to_logical(n, replay_all_shards(n, m, gates, ops_g, psi0), pi)
    assert np.max(np.abs(got - O.simulate(n, gates, psi0))) < 1e-12


def test_schedule_phase_only_on_global_qubits():
    """A diagonal gate whose targets are all global is a per-rank phase."""
    n, m = 8, 2
    from hq_inputs import CZ, H
    gates = [Gate("H", (q,), H) for q in range(2, n)] + [Gate("CZ", (0, 1), CZ),
                                                         Gate("CP", (1, 0), np.diag([1, 1j, -1j, -1]).astype(complex))]
    ops, pi = hq.hq_schedule(n, m, gates)
    assert all(o["kind"] == "apply" for o in ops)              # no remap at all
    tail = [o for o in ops if o["gate"] >= n - 2]
    assert len(tail) == 2 and all(all(b >= n - m for b in o["bits"][:2]) for o in tail)
    psi0 = random_state(n, 2)
    got = to_logical(n, replay_all_shards(n, m, gates, ops, psi0), pi)
    assert np.max(np.abs(got - O.simulate(n, gates, psi0))) < 1e-13


def test_schedule_reversible_bit_exact():
    n, m = 10, 2
    gates = reversible_circuit(n, 80, 4, kmax=3)
    ops, pi = hq.hq_schedule(n, m, gates)
    from hq_inputs import integer_state
    psi0 = integer_state(n, 1)
    got = to_logical(n, replay_all_shards(n, m, gates, ops, psi0), pi)
    want = O.simulate(n, gates, psi0)
    assert np.array_equal(got, want)


def _segments_lower_bound(n, m, fused):
    """Fewest remaps any schedule can have when the first global set is free:
    greedy maximal runs of gates whose qubits fit on n - m local bits (the
    Sycamore blocks are dense, so every target must be local), minus one."""
    cnt, used = 0, set()
    for q, _ in fused:
        if len(used | set(q)) > n - m:
            cnt, used = cnt + 1, set()
        used |= set(q)
    return cnt


@pytest.mark.parametrize("n,cycles,seed", [(34, 20, 3000), (36, 24, 4000)])
@pytest.mark.parametrize("kmax,blocks", [(4, False), (5, False), (6, True)])
def test_schedule_remap_counts(n, cycles, seed, kmax, blocks):
    """the segment scheduler stays within two
    remaps of the lower bound (one remap per segment boundary; a segment
    ends early when a folded pack could not move enough evictees, which
    must not sit on bits 0, 1), from the planned first global set and from
    the default layout; at 34q m=3, k<=5: R <= 11 and R/P <= 0.106, the
    6x-at-8-GPUs threshold of the survey's cost model."""
    fused = hq.hq_fuse(sycamore_circuit(n, cycles, seed), kmax, blocks=blocks)
    gates = [Gate("F", q, U) for q, U in fused]
    for m in (1, 2, 3):
        lb = _segments_lower_bound(n, m, fused)
        ops, _ = hq.hq_schedule(n, m, gates)
        R0 = sum(o["kind"] == "remap" for o in ops)
        for i, o in enumerate(ops):
            if o["kind"] == "permute":
                assert i > 0 and ops[i - 1]["kind"] == "apply"
        pi0, _, _ = hq.hq_plan_layout(n, m, fused)
        assert sorted(pi0) == list(range(n))
        ops, _ = hq.hq_schedule(n, m, gates, pi0)
        R = sum(o["kind"] == "remap" for o in ops)
        assert sum(o["kind"] == "apply" for o in ops) == len(fused)
        assert lb <= R <= lb + 2, (m, R, lb)
        assert R0 <= lb + 3, (m, R0, lb)
        # every PERMUTE (pack) directly follows an apply, so the executor can fold it
        for i, o in enumerate(ops):
            if o["kind"] == "permute":
                assert i > 0 and ops[i - 1]["kind"] == "apply"
                assert all(b >= 2 for b in o["bits"][:2 * o["nbits"]])
                g = fused[ops[i - 1]["gate"]]
                assert all(b < n - m for b in ops[i - 1]["bits"][:len(g[0])])
        if n == 34 and kmax == 5 and m == 3:
            assert R <= 11 and R0 <= 12 and R / len(fused) <= 0.106


def test_schedule_errors():
    with pytest.raises(hq.HQError) as e:
        hq.hq_schedule(8, 3, [Gate("U", (0,), np.eye(2))])
    assert e.value.status == "HQ_ERR_NGPUS"
    with pytest.raises(hq.HQError) as e:
        hq.hq_schedule(8, 0, [Gate("U", (8,), np.eye(2))])
    assert e.value.status == "HQ_ERR_QUBIT"


@pytest.mark.parametrize("kmax", [4, 6])
def test_plan_layout_is_permutation_and_improves(kmax):
    fused = hq.hq_fuse(sycamore_circuit(34, 20, 3000), kmax)
    pi, before, after = hq.hq_plan_layout(34, 0, fused)
    assert sorted(pi) == list(range(34))
    assert after <= before
    if kmax == 6:
        # the cost model charges tensor-core passes with >= 2 targets in bits
        # 0..3 (1.19x) or in mode L (1.29x); on this circuit the planner finds
        # a layout with none of them, i.e. every pass at the base cost
        for q, _ in fused:
            if len(q) >= 5:
                b = [pi[x] for x in q]
                assert sum(x < 4 for x in b) <= 1 and not (0 in b and 1 in b), b
        assert abs(after - len(fused)) < 1e-9


def test_plan_layout_errors():
    with pytest.raises(hq.HQError):
        hq.hq_plan_layout(8, 0, [Gate("U", (9,), np.eye(2))])


# ---------------------------------------------------------------- block planner (hq_fuse_blocks)

@pytest.mark.parametrize("kind", ["sycamore", "random", "reversible"])
@pytest.mark.parametrize("kmax", [2, 3, 4, 5, 6])
def test_fuse_blocks_is_valid_and_no_worse(kind, kmax):
    """The block plan is the same circuit (oracle: fused vs unfused, fp64),
    every block has <= kmax qubits, and it never has more blocks than C7."""
    n = 12
    if kind == "sycamore":
        gates = sycamore_circuit(n, 10, 7)
    elif kind == "random":
        gates = random_circuit(n, 150, 9, kmax=min(kmax, 3))
    else:
        gates = reversible_circuit(n, 150, 9, kmax=min(kmax, 3))
    gates = [g for g in gates if len(g.qubits) <= kmax]
    c7 = hq.hq_fuse(gates, kmax)
    mg = hq.hq_fuse(gates, kmax, blocks=True)
    assert len(mg) <= len(c7)
    assert all(1 <= len(q) <= kmax and list(q) == sorted(q) for q, _ in mg)
    psi = random_state(n, 3)
    want = O.simulate(n, gates, psi)
    got = O.simulate(n, [Gate("F", q, U) for q, U in mg], psi)
    assert np.max(np.abs(got - want)) < 1e-12


_PASS_COST = {1: 1.0, 2: 1.0, 3: 1.06, 4: 1.15, 5: 1.13, 6: 1.24}   # DESIGN.md §6 pass-cost model


@pytest.mark.parametrize("seed", range(8))
def test_fuse_blocks_cost_not_above_c7_and_deterministic(seed):
    """On random circuits of random width the block plan never costs more
    than the C7 plan under the planner's own cost model (the C7 plan is the
    fallback), is the same circuit (oracle, fp64), and two calls return the
    identical plan (the rollouts run on host threads; the choice must not
    depend on their timing)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(6, 15))
    kmax = int(rng.integers(2, 7))
    gates = random_circuit(n, 250, 100 + seed, kmax=min(kmax, 3))
    c7 = hq.hq_fuse(gates, kmax)
    b1 = hq.hq_fuse(gates, kmax, blocks=True)
    b2 = hq.hq_fuse(gates, kmax, blocks=True)
    cost = lambda f: sum(_PASS_COST[len(q)] for q, _ in f)
    assert cost(b1) <= cost(c7) + 1e-9
    assert [q for q, _ in b1] == [q for q, _ in b2]
    assert all(np.array_equal(u1, u2) for (_, u1), (_, u2) in zip(b1, b2))
    psi = random_state(n, 5)
    got = O.simulate(n, [Gate("F", q, U) for q, U in b1], psi)
    assert np.max(np.abs(got - O.simulate(n, gates, psi))) < 1e-12


def test_fuse_blocks_bench_circuits():
    """The bench circuits (bench.py UNIT_PASSES): 34q d20 at
    kmax = 6, 80 C7 blocks -> 36; 36q d24, 96 -> 42; 30q d20, 67 -> 33."""
    for (n, c, s), c7, blk in [((34, 20, 3000), 80, 36), ((36, 24, 4000), 96, 42), ((30, 20, 1000), 67, 33)]:
        gates = sycamore_circuit(n, c, s)
        assert len(hq.hq_fuse(gates, 6)) == c7
        assert len(hq.hq_fuse(gates, 6, blocks=True)) == blk


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("kmax", [3, 4, 6])
def test_fuse_blocks_dense_matrix_equals_original(seed, kmax):
    """The block plan is a regrouping, so its circuit matrix (product of the
    embedded block matrices, brute force P7) equals the original
    circuit's; every gate is in one block of <= kmax ascending qubits.  The
    grouping itself is a planner choice the paper does not fix,
    so it is not compared with any reference grouping."""
    n = 8
    gates = [g for g in random_circuit(n, 70, 17 + seed, kmax=min(kmax, 3)) if len(g.qubits) <= kmax]
    mg = hq.hq_fuse(gates, kmax, blocks=True)
    assert len(mg) <= len(hq.hq_fuse(gates, kmax))
    assert all(1 <= len(q) <= kmax and list(q) == sorted(q) for q, _ in mg)
    got = O.circuit_matrix(n, [Gate("F", q, U) for q, U in mg])
    assert np.max(np.abs(got - O.circuit_matrix(n, gates))) < 1e-12
