"""ORACLE -- test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product path (``paper_2111_06868_b200``) never imports it and shares no code
with it; the only common dependency is the input generator package
``hq_inputs`` (which holds no method arithmetic).

Contents, each following the passage cited:

* ``apply_gate`` / ``simulate`` -- the plain fp64 gate-by-gate apply of
  ``sv_oracle.c``.
* ``norm`` -- ||psi||_2 (reading C13).
* ``embed_dense`` -- the 2^n x 2^n matrix of one gate written out from its
  definition M[i][i'] = U[r(i)][r(i')] if i, i' agree off the target bits,
  else 0 (brute-force pin P7, n <= 10).
* ``kron_embed_adjacent`` -- textbook kron(I, U, I) for ascending adjacent
  qubits (independent check of ``embed_dense``).
* ``circuit_matrix`` -- product of embedded gate matrices in application
  order.
* ``tensordot_apply`` -- the paper's own einsum engine idea (P:644-648,
  pin P8): numpy.tensordot on a (2,)*n array, axis j = qubit j.
* ``compress`` / ``fused_gates`` -- the greedy fusion rule, reading C7 of
  PAPER P:499-504 (worked example P:510-529), and the fused matrix
  U_group = U_last ... U_first embedded on the ascending support (P:493-494,
  readings C8, C9).  The product's block planner (``hq_fuse_blocks``) is a
  planner choice the paper does not fix (many groupings are valid,
  P:499-504); the oracle holds no transcript of it.  Block plans are checked
  only through the state they produce (fused vs unfused, and the dense
  circuit matrix), never grouping against grouping.

* ``reversible_image`` -- pin P10: a basis state |x> through permutation
  gates (0/1 matrices) is the basis state |f(x)>, with f computed by host bit
  operations on the index (qubit q <-> index bit n-1-q, reading C1; U acts on
  column vectors, reading C2).

* ``init_tokens`` / ``project`` / ``probabilities`` -- token product states
   as a Kronecker product of single-qubit
  vectors, projection and Born
  probabilities written out from their definitions.

* ``dm_apply_kraus`` -- a Kraus map rho -> sum_m K_m rho K_m^dagger on the
  density matrix itself, with embedded K_m, and
  ``dm_vec`` -- the row-major vectorisation vec(rho)[i 2^N + j] = rho[i][j]
  that the doubling reading (row f2) applies gates to.

* ``reduced_dm`` / ``kraus_sample_step`` -- the partial trace written out as
  M M^H of the reshaped state, and one trajectory step by explicit branches
  (row f3).

Parity pins for every function live in ``tests/test_oracle_pins.py``.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force=False):
    """Compile sv_oracle.c (plain C, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_apply.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_int]
        lib.oracle_apply.restype = ctypes.c_int
        lib.oracle_norm.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.oracle_norm.restype = ctypes.c_double
        lib.oracle_init_basis.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64]
        lib.oracle_init_basis.restype = None
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def set_threads(t):
    _get().oracle_set_threads(int(t))


def max_threads():
    return int(_get().oracle_max_threads())


class OracleError(RuntimeError):
    pass


def _nqubits(psi):
    N = psi.shape[0]
    n = N.bit_length() - 1
    if 1 << n != N:
        raise OracleError("length is not a power of two")
    return n


def apply_gate(psi, U, qubits):
    """In place: psi <- (U embedded on qubits) psi.  psi is complex128 1-D."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    n = _nqubits(psi)
    U = np.ascontiguousarray(U, dtype=np.complex128)
    k = len(qubits)
    if U.shape != (2 ** k, 2 ** k):
        raise OracleError("matrix shape does not match arity")
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    rc = _get().oracle_apply(psi.ctypes.data, n, U.ctypes.data, q.ctypes.data, k)
    if rc != 0:
        raise OracleError("oracle_apply failed with code %d" % rc)
    return psi


def init_basis(n, x=0):
    psi = np.empty(2 ** n, dtype=np.complex128)
    _get().oracle_init_basis(psi.ctypes.data, n, int(x))
    return psi


def simulate(n, gates, psi0=None, x=0):
    """Apply ``gates`` (leftmost first) to psi0 (copied) or |x>."""
    psi = init_basis(n, x) if psi0 is None else np.array(psi0, dtype=np.complex128, copy=True)
    for g in gates:
        apply_gate(psi, g.U if hasattr(g, "U") else g[1], g.qubits if hasattr(g, "qubits") else g[0])
    return psi


def norm(psi):
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    return float(_get().oracle_norm(psi.ctypes.data, _nqubits(psi)))


# ---------------------------------------------------------------- brute force

def embed_dense(n, U, qubits):
    """M[i][i'] = U[r(i)][r(i')] when i and i' agree off the target bits,
    else 0; r(i) = sum_j bit_(n-1-q_j)(i) 2^(k-1-j)."""
    k = len(qubits)
    idx = np.arange(2 ** n, dtype=np.int64)
    r = np.zeros_like(idx)
    mask = 0
    for j, q in enumerate(qubits):
        b = n - 1 - q
        r |= ((idx >> b) & 1) << (k - 1 - j)
        mask |= 1 << b
    rest = idx & ~mask
    same = rest[:, None] == rest[None, :]
    return np.where(same, np.asarray(U)[r[:, None], r[None, :]], 0).astype(np.complex128)


def kron_embed_adjacent(n, U, q0):
    """Textbook kron(I_{2^q0}, U, I_{2^(n-q0-k)}) for qubits q0..q0+k-1 in
    ascending order, qubit 0 being the leftmost Kronecker factor (C1)."""
    k = int(np.log2(np.asarray(U).shape[0]))
    return np.kron(np.kron(np.eye(2 ** q0), U), np.eye(2 ** (n - q0 - k)))


def circuit_matrix(n, gates):
    """Product of embedded gate matrices in application order."""
    M = np.eye(2 ** n, dtype=np.complex128)
    for g in gates:
        M = embed_dense(n, g.U, g.qubits) @ M
    return M


def tensordot_apply(psi, U, qubits):
    """numpy.tensordot engine (pin P8): psi as (2,)*n with axis j
    = qubit j; U as (2,)*2k with output axes first."""
    n = _nqubits(psi)
    k = len(qubits)
    T = np.asarray(psi).reshape((2,) * n)
    Ut = np.asarray(U).reshape((2,) * (2 * k))
    out = np.tensordot(Ut, T, axes=(list(range(k, 2 * k)), list(qubits)))
    out = np.moveaxis(out, list(range(k)), list(qubits))
    return np.ascontiguousarray(out).reshape(-1)


# ---------------------------------------------------------------- compress

def compress(gates, kmax):
    """Greedy fusion into groups of support <= kmax (rule C7):
    gate g joins the earliest-created group G with |supp(G) u supp(g)| <= kmax
    such that no non-member gate between G's first member and g touches a
    qubit of g; otherwise it opens a new group.  Groups are returned in
    first-member order as lists of gate indices."""
    for g in gates:
        if len(g.qubits) > kmax:
            raise OracleError("GateTooWide")
    groups = []           # each: dict(first, members(list), support(set), mset)
    touch = {}            # qubit -> indices of the gates (so far) that touch it
    for i, g in enumerate(gates):
        qs = set(g.qubits)
        placed = False
        for G in groups:
            if len(G["support"] | qs) > kmax:
                continue
            # non-member gates between G's first member and g touching g's qubits
            blocked = any(G["first"] < j < i and j not in G["mset"]
                          for q in qs for j in touch.get(q, ()))
            if blocked:
                continue
            G["members"].append(i)
            G["mset"].add(i)
            G["support"] |= qs
            placed = True
            break
        if not placed:
            groups.append({"first": i, "members": [i], "mset": {i}, "support": set(qs)})
        for q in qs:
            touch.setdefault(q, []).append(i)
    return [G["members"] for G in groups]


def fused_gates(gates, kmax):
    """Fused gate list: (ascending support, U_last ... U_first embedded on it)
    (P:493-494 to_matrix_gate; readings C8, C9)."""
    out = []
    groups = compress(gates, kmax)
    for members in groups:
        support = sorted(set().union(*[set(gates[i].qubits) for i in members]))
        pos = {q: j for j, q in enumerate(support)}
        m = len(support)
        M = np.eye(2 ** m, dtype=np.complex128)
        for i in members:
            M = embed_dense(m, gates[i].U, [pos[q] for q in gates[i].qubits]) @ M
        out.append((tuple(support), M))
    return out


def reversible_image(n, gates, x):
    """f(x) for a circuit of permutation gates (pin P10): for each gate read
    the target bits of the index as the column c (qubits[0] = MSB, C2), find
    the row r with U[r][c] = 1, write r back into the target bits."""
    y = int(x)
    for g in gates:
        k = len(g.qubits)
        c = 0
        for j, q in enumerate(g.qubits):
            c |= ((y >> (n - 1 - q)) & 1) << (k - 1 - j)
        col = np.asarray(g.U)[:, c]
        rows = np.flatnonzero(np.abs(col) > 0.5)
        if len(rows) != 1 or np.count_nonzero(col) != 1 or col[rows[0]] != 1:
            raise OracleError("not a permutation gate")
        r = int(rows[0])
        for j, q in enumerate(g.qubits):
            b = n - 1 - q
            y = (y & ~(1 << b)) | (((r >> (k - 1 - j)) & 1) << b)
    return y


# ---------------------------------------------------------------- f4: tokens, projection

_TOKENS = {"0": np.array([1.0, 0.0]), "1": np.array([0.0, 1.0]),
           "+": np.array([1.0, 1.0]) / np.sqrt(2.0), "-": np.array([1.0, -1.0]) / np.sqrt(2.0)}


def init_tokens(n, tokens):
    """Tensor product of single-qubit states, qubit 0 the leftmost (most
    significant) factor (C1); a single character is broadcast."""
    if len(tokens) == 1:
        tokens = tokens * n
    if len(tokens) != n or any(t not in _TOKENS for t in tokens):
        raise OracleError("BadToken")
    psi = np.array([1.0 + 0j])
    for t in tokens:
        psi = np.kron(psi, _TOKENS[t])
    return psi.astype(np.complex128)


def _qubit_bits(n, qubits):
    idx = np.arange(2 ** n, dtype=np.int64)
    return [((idx >> (n - 1 - q)) & 1) for q in qubits]


def project(psi, qubits, bits, renormalize=False):
    """Zero the amplitudes inconsistent with bits on qubits; optionally
    renormalise.  Returns (new psi, projected norm)."""
    n = _nqubits(psi)
    keep = np.ones(2 ** n, dtype=bool)
    for b, col in zip(bits, _qubit_bits(n, qubits)):
        keep &= col == b
    out = np.where(keep, psi, 0).astype(np.complex128)
    nrm = norm(out)
    if renormalize:
        if nrm < 1e-14:
            raise OracleError("ZeroNormProjection")
        out = out / nrm
    return out, nrm


def probabilities(psi, qubits):
    """P[x] = sum of |psi_i|^2 over indices whose qubits read x (qubits[0] MSB)."""
    n = _nqubits(psi)
    x = np.zeros(2 ** n, dtype=np.int64)
    k = len(qubits)
    for j, col in enumerate(_qubit_bits(n, qubits)):
        x |= col << (k - 1 - j)
    return np.bincount(x, weights=np.abs(psi) ** 2, minlength=2 ** k)


# ---------------------------------------------------------------- f2: density matrices

def dm_apply_kraus(rho, K, qubits):
    """rho -> sum_m E_m rho E_m^dagger, E_m = K_m embedded on qubits of N."""
    N = int(np.log2(rho.shape[0]))
    out = np.zeros_like(rho, dtype=np.complex128)
    for k in K:
        E = embed_dense(N, k, qubits)
        out += E @ rho @ E.conj().T
    return out


def dm_vec(rho):
    """vec(rho)[i 2^N + j] = rho[i][j] (logical qubits 0..N-1 = rows)."""
    return np.ascontiguousarray(rho, dtype=np.complex128).reshape(-1)


# ---------------------------------------------------------------- f3: trajectories

def reduced_dm(psi, qubits):
    """rho_T[a][b] = sum_r psi[a, r] conj(psi[b, r]) -- the partial trace of
    |psi><psi| over every qubit not in ``qubits`` (a, b read qubits[0] as the
    MSB, reading C1): psi reshaped to (2,)*n, target axes moved to the front
    in ``qubits`` order, flattened to a 2^k x 2^(n-k) matrix M, rho = M M^H."""
    n = _nqubits(psi)
    k = len(qubits)
    t = np.asarray(psi, dtype=np.complex128).reshape((2,) * n)
    t = np.moveaxis(t, list(qubits), list(range(k)))
    M = t.reshape(2 ** k, -1)
    return M @ M.conj().T


def kraus_sample_step(psi, K, qubits, u):
    """One trajectory step ("pure state sampling of the
    Kraus operators"): every branch K_i psi by the plain
    apply, p_i = ||K_i psi||^2, i = the first index with
    u * sum(p) < p_0 + ... + p_i (and p_i > 0), psi <- K_i psi / sqrt(p_i).
    Returns (new psi, i, p)."""
    branches = []
    for Ki in K:
        b = np.array(psi, dtype=np.complex128, copy=True)
        apply_gate(b, Ki, list(qubits))
        branches.append(b)
    p = np.array([float(np.vdot(b, b).real) for b in branches])
    if not np.any(p >= 1e-14):
        raise OracleError("ZeroNormBranch")
    target = u * p.sum()
    cum = 0.0
    i = len(p) - 1
    for j, pj in enumerate(p):
        cum += pj
        if target < cum and pj > 0:
            i = j
            break
    while i > 0 and p[i] == 0:
        i -= 1
    return branches[i] / np.sqrt(p[i]), i, p
