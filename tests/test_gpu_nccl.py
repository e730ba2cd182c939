"""NCCL transport of the remap (row a5) with one process per GPU: two ranks
(hq_state_create_rank, ncclCommInitRank) run circuits whose gates force
global<->local qubit swaps through ncclSend/ncclRecv, and the combined
amplitudes are checked against the fp64 oracle (Sycamore circuit, 1e-4) and
bit-exactly (reversible circuit, pin P10).  Needs >= 2 visible GPUs; skipped
otherwise (NCCL refuses two ranks on one device)."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

import oracle as O
from hq_inputs import sycamore_circuit, reversible_circuit

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _rank_main(rank, world, nccl_id, q):
    try:
        sys.path.insert(0, ROOT)
        import paper_2111_06868_b200 as hq
        n = 16
        out = {}
        for name, gates, x, kmax in (("sycamore", sycamore_circuit(n, 8, 3), 0, 4),
                                     ("reversible", reversible_circuit(n, 80, 11, kmax=3), 0x5A3C, 3)):
            s = hq.hq_state_create_rank(n, "c64", world, rank, rank, nccl_id)
            hq.hq_state_init_basis(s, x)
            hq.hq_apply_circuit(s, hq.hq_fuse(gates, kmax))
            st = hq.hq_stats_get(s)
            amps = np.full(2 ** n, np.nan + 1j * np.nan, dtype=np.complex64)
            hq.hq_get_amplitudes(s, 0, 2 ** n, amps)
            out[name] = (amps, st["remaps"], hq.hq_norm(s))
            s.close()
        q.put((rank, out, None))
    except Exception as e:      # report instead of hanging the parent
        q.put((rank, None, repr(e)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (NCCL refuses two ranks on one device)")
def test_nccl_remap_two_ranks_vs_oracle():
    sys.path.insert(0, ROOT)
    import paper_2111_06868_b200 as hq
    hq.lib()
    nid = hq.hq_nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, nid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    n = 16
    for name in ("sycamore", "reversible"):
        a0, R0, nrm0 = res[0][name]
        a1, R1, nrm1 = res[1][name]
        assert R0 > 0 and R0 == R1                      # remaps really ran over NCCL
        own0, own1 = ~np.isnan(a0.real), ~np.isnan(a1.real)
        assert np.all(own0 ^ own1)                      # every amplitude owned by exactly one rank
        psi = np.where(own0, a0, a1).astype(np.complex128)
        if name == "sycamore":
            want = O.simulate(n, sycamore_circuit(n, 8, 3))
            assert np.linalg.norm(psi - want) <= 1e-4
            assert abs(nrm0 - 1) < 1e-5 and nrm0 == nrm1
        else:
            y = O.reversible_image(n, reversible_circuit(n, 80, 11, kmax=3), 0x5A3C)
            assert psi[y] == 1.0 and np.count_nonzero(psi) == 1
            assert nrm0 == 1.0 and nrm1 == 1.0
