"""Property-based checks of the block planner (hq_fuse_blocks)
on arbitrary small gate lists: whatever the grouping, the fused list is the
same circuit (its dense matrix, S:139-147 brute force pin P7, equals the
original's), every block acts on at most kmax ascending qubits, the plan is
never costlier than C7 under the planner's pass-cost model, and two calls
return the same plan.  CPU only: the planner is host code."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st, HealthCheck

import oracle as O
from hq_inputs import Gate, haar_unitary
import paper_2111_06868_b200 as hq

_PASS_COST = {1: 1.0, 2: 1.0, 3: 1.06, 4: 1.15, 5: 1.13, 6: 1.24}


@st.composite
def circuits(draw):
    n = draw(st.integers(2, 7))
    ng = draw(st.integers(0, 40))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(ng):
        k = int(rng.integers(1, min(3, n) + 1))
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        gates.append(Gate("U", qs, haar_unitary(k, rng)))
    kmin = max([len(g.qubits) for g in gates], default=1)
    kmax = draw(st.integers(kmin, 6))
    return n, gates, kmax


@settings(max_examples=200, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(circuits())
def test_block_plan_is_the_same_circuit(c):
    n, gates, kmax = c
    b1 = hq.hq_fuse(gates, kmax, blocks=True)
    c7 = hq.hq_fuse(gates, kmax)
    assert all(1 <= len(q) <= kmax and list(q) == sorted(q) for q, _ in b1)
    cost = lambda f: sum(_PASS_COST[len(q)] for q, _ in f)
    assert cost(b1) <= cost(c7) + 1e-9
    b2 = hq.hq_fuse(gates, kmax, blocks=True)
    assert [q for q, _ in b1] == [q for q, _ in b2]
    if not gates:
        assert b1 == []
        return
    want = O.circuit_matrix(n, gates)
    got = O.circuit_matrix(n, [Gate("F", q, U) for q, U in b1])
    assert np.max(np.abs(got - want)) < 1e-11
