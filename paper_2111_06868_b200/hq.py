"""Thin ctypes binding of the C ABI in include/hq.h -- argument marshalling only.

Every function here has the name of the C entry point it calls and does no
arithmetic of the method: all of the hot path runs in libhq.so's CUDA
kernels.  If the library (or a CUDA device) is missing the calls raise; there
is no CPU fallback.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# HQ_LIB selects another build of the same library, e.g. the checked variant
# lib/libhq_check.so (device-side bounds checks and mbarrier watchdogs)
LIB_PATH = os.environ.get("HQ_LIB") or os.path.join(_PKG, "lib", "libhq.so")

HQ_C64, HQ_C128 = 0, 1
_DTYPES = {"c64": HQ_C64, "complex64": HQ_C64, HQ_C64: HQ_C64,
           "c128": HQ_C128, "complex128": HQ_C128, HQ_C128: HQ_C128}
_NP = {HQ_C64: np.complex64, HQ_C128: np.complex128}

STATUS = {0: "HQ_OK", 1: "HQ_ERR_ARG", 2: "HQ_ERR_NGPUS", 3: "HQ_ERR_OOM", 4: "HQ_ERR_CUDA",
          5: "HQ_ERR_NCCL", 6: "HQ_ERR_QUBIT", 7: "HQ_ERR_DUP_QUBIT", 8: "HQ_ERR_K",
          9: "HQ_ERR_RANGE", 10: "HQ_ERR_STATE", 11: "HQ_ERR_NO_DEVICE"}


class HQError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__("%s: %s" % (self.status, msg))


class hq_gate(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("qubits", ctypes.c_int32 * 6),
                ("U", ctypes.POINTER(ctypes.c_double))]


class hq_op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gate", ctypes.c_int32),
                ("nbits", ctypes.c_int32), ("bits", ctypes.c_int32 * 12)]


class hq_stats(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_uint64), ("remaps", ctypes.c_uint64),
                ("permutes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("hbm_bytes", ctypes.c_uint64), ("link_bytes", ctypes.c_uint64),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64), ("packs", ctypes.c_uint64),
                ("remaps_fused", ctypes.c_uint64), ("gathers", ctypes.c_uint64)]


_lib = None
P = ctypes.c_void_p


def lib():
    """Load libhq.so (build it first with paper_2111_06868_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HQError(-1, "libhq.so not built (%s); run python -m paper_2111_06868_b200.build"
                          % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "hq_state_create": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)],
            "hq_state_create_rank": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, P, ctypes.POINTER(P)],
            "hq_state_create_virtual": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)],
            "hq_state_create_from_buffers": [ctypes.c_int, ctypes.c_int, P, P, ctypes.POINTER(P)],
            "hq_state_create_rank_from_buffers": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P,
                                                  ctypes.POINTER(P)],
            "hq_nccl_unique_id": [P],
            "hq_state_destroy": [P],
            "hq_state_set_stream": [P, P],
            "hq_state_info": [P] + [ctypes.POINTER(ctypes.c_int)] * 5,
            "hq_state_init_basis": [P, ctypes.c_uint64],
            "hq_get_amplitudes": [P, ctypes.c_uint64, ctypes.c_uint64, P],
            "hq_set_amplitudes": [P, ctypes.c_uint64, ctypes.c_uint64, P],
            "hq_norm": [P, ctypes.POINTER(ctypes.c_double)],
            "hq_apply_matrix": [P, P, P, ctypes.c_int],
            "hq_apply_circuit": [P, P, ctypes.c_size_t],
            "hq_circuit_create": [P, P, ctypes.c_size_t, ctypes.POINTER(P)],
            "hq_circuit_run": [P, P],
            "hq_circuit_info": [P] + [ctypes.POINTER(ctypes.c_uint64)] * 3,
            "hq_circuit_destroy": [P],
            "hq_fuse": [P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.POINTER(hq_gate)),
                        ctypes.POINTER(ctypes.c_size_t)],
            "hq_free_gates": [P, ctypes.c_size_t],
            "hq_fuse_plan": [P, ctypes.c_size_t, ctypes.c_int, P, ctypes.POINTER(ctypes.c_size_t)],
            "hq_schedule": [ctypes.c_int, ctypes.c_int, P, ctypes.c_size_t,
                            ctypes.POINTER(ctypes.POINTER(hq_op)), ctypes.POINTER(ctypes.c_size_t), P],
            "hq_free_ops": [P],
            "hq_remap_plan": [ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, P, P, ctypes.c_size_t,
                              ctypes.POINTER(ctypes.c_size_t)],
            "hq_schedule_from": [ctypes.c_int, ctypes.c_int, P, ctypes.c_size_t, P, ctypes.c_int,
                                 ctypes.POINTER(ctypes.POINTER(hq_op)), ctypes.POINTER(ctypes.c_size_t), P],
            "hq_plan_layout": [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_size_t, P,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
            "hq_state_set_layout": [P, P],
            "hq_state_invalidate_bound": [P],
            "hq_state_set_remap_mode": [P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
            "hq_state_init_tokens": [P, ctypes.c_char_p],
            "hq_dm_superop": [P, ctypes.c_int, ctypes.c_int, P],
            "hq_dm_apply_unitary": [P, P, P, ctypes.c_int],
            "hq_dm_apply_kraus": [P, P, ctypes.c_int, P, ctypes.c_int],
            "hq_dm_trace": [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
            "hq_project": [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)],
            "hq_probabilities": [P, P, ctypes.c_int, P],
            "hq_measure": [P, P, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_uint64)],
            "hq_reduced_dm": [P, P, ctypes.c_int, P],
            "hq_fuse_blocks": [P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.POINTER(hq_gate)),
                               ctypes.POINTER(ctypes.c_size_t)],
            "hq_reduced_dm_batched": [P, ctypes.c_int, P, ctypes.c_int, P],
            "hq_reduced_dm_batched_sum": [P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P],
            "hq_kraus_sample_batched": [P, ctypes.c_int, P, ctypes.c_int, P, ctypes.c_int, P, P, P],
            "hq_kraus_sample": [P, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int), P],
            "hq_state_get_layout": [P, P],
            "hq_sync": [P],
            "hq_stats_get": [P, ctypes.POINTER(hq_stats)],
            "hq_stats_reset": [P],
            "hq_profile_enable": [P, ctypes.c_int],
            "hq_kernel_times": [P, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.hq_last_error.restype = ctypes.c_char_p
        L.hq_last_error.argtypes = []
        L.hq_version.restype = ctypes.c_char_p
        L.hq_version.argtypes = []
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise HQError(rc, lib().hq_last_error().decode(errors="replace"))


class State:
    """Owning handle of an ``hq_state*``."""

    def __init__(self, ptr, n, dtype):
        self.ptr = ptr
        self.n = n
        self.dtype = dtype
        self.np_dtype = _NP[dtype]

    def __del__(self):
        try:
            if self.ptr:
                lib().hq_state_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass

    def close(self):
        if self.ptr:
            _check(lib().hq_state_destroy(self.ptr))
            self.ptr = None


class Circuit:
    def __init__(self, ptr, state, keep):
        self.ptr = ptr
        self.state = state
        self._keep = keep

    def __del__(self):
        try:
            if self.ptr:
                lib().hq_circuit_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def _dt(dtype):
    if dtype not in _DTYPES:
        raise ValueError("dtype must be c64 or c128")
    return _DTYPES[dtype]


# ------------------------------------------------------------------ create

def hq_state_create(n, dtype="c64", ngpus=1):
    d = _dt(dtype)
    out = P()
    _check(lib().hq_state_create(int(n), d, int(ngpus), ctypes.byref(out)))
    return State(out, n, d)


def hq_nccl_unique_id():
    buf = (ctypes.c_char * 128)()
    _check(lib().hq_nccl_unique_id(buf))
    return bytes(buf)


def hq_state_create_rank(n, dtype, world_size, rank, device, nccl_id=None):
    d = _dt(dtype)
    out = P()
    idbuf = None
    if nccl_id is not None:
        idbuf = (ctypes.c_char * 128).from_buffer_copy(nccl_id)
    _check(lib().hq_state_create_rank(int(n), d, int(world_size), int(rank), int(device),
                                      idbuf, ctypes.byref(out)))
    return State(out, n, d)


def hq_state_create_virtual(n, dtype, nshards):
    d = _dt(dtype)
    out = P()
    _check(lib().hq_state_create_virtual(int(n), d, int(nshards), ctypes.byref(out)))
    return State(out, n, d)


def hq_state_create_from_buffers(n, dtype, psi_device_ptr, stream_ptr=None):
    d = _dt(dtype)
    out = P()
    _check(lib().hq_state_create_from_buffers(int(n), d, P(psi_device_ptr), P(stream_ptr or 0),
                                              ctypes.byref(out)))
    return State(out, n, d)


def hq_state_create_rank_from_buffers(n, dtype, world_size, rank, psi_device_ptr, buf_device_ptr=None,
                                      stream_ptr=None, nccl_id=None):
    """One rank's state on caller-owned device buffers (e.g. torch.empty):
    psi (and buf, the receive buffer, when world_size > 1) must outlive it."""
    d = _dt(dtype)
    out = P()
    idbuf = None
    if nccl_id is not None:
        idbuf = (ctypes.c_char * 128).from_buffer_copy(nccl_id)
    _check(lib().hq_state_create_rank_from_buffers(int(n), d, int(world_size), int(rank), idbuf,
                                                   P(psi_device_ptr), P(buf_device_ptr or 0),
                                                   P(stream_ptr or 0), ctypes.byref(out)))
    return State(out, n, d)


def hq_state_destroy(state):
    state.close()


def hq_state_set_stream(state, stream_ptr):
    _check(lib().hq_state_set_stream(state.ptr, P(stream_ptr)))


def hq_state_info(state):
    vals = [ctypes.c_int() for _ in range(5)]
    _check(lib().hq_state_info(state.ptr, *[ctypes.byref(v) for v in vals]))
    return dict(zip(["n", "dtype", "world", "local_shards", "first_rank"], [v.value for v in vals]))


# ------------------------------------------------------------------ state I/O

def hq_state_init_basis(state, x=0):
    _check(lib().hq_state_init_basis(state.ptr, int(x)))


def hq_state_init_tokens(state, tokens):
    _check(lib().hq_state_init_tokens(state.ptr, tokens.encode()))


def hq_project(state, qubits, bits, renormalize=False):
    """Returns the norm of the projected state (before renormalisation)."""
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    b = np.ascontiguousarray(bits, dtype=np.int32)
    out = ctypes.c_double()
    _check(lib().hq_project(state.ptr, q.ctypes.data, b.ctypes.data, int(q.size), int(bool(renormalize)),
                            ctypes.byref(out)))
    return out.value


def hq_probabilities(state, qubits):
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    out = np.zeros(2 ** q.size, dtype=np.float64)
    _check(lib().hq_probabilities(state.ptr, q.ctypes.data, int(q.size), out.ctypes.data))
    return out


def hq_measure(state, qubits, u):
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    out = ctypes.c_uint64()
    _check(lib().hq_measure(state.ptr, q.ctypes.data, int(q.size), float(u), ctypes.byref(out)))
    return out.value


def _kraus_array(K):
    mats = [np.ascontiguousarray(k, dtype=np.complex128) for k in K]
    ptrs = (ctypes.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
    return ptrs, mats


def hq_reduced_dm(state, qubits):
    """Reduced density matrix of k <= 3 qubits (complex128 2^k x 2^k;
    qubits[0] = MSB of the row index)."""
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    rho = np.zeros((2 ** q.size, 2 ** q.size), dtype=np.complex128)
    _check(lib().hq_reduced_dm(state.ptr, q.ctypes.data, int(q.size), rho.ctypes.data))
    return rho


def hq_kraus_sample(state, K, qubits, u):
    """One trajectory step of the Kraus channel K on qubits with uniform u in
    [0, 1): returns (chosen index, branch probabilities p_i = ||K_i psi||^2)."""
    ptrs, mats = _kraus_array(K)
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    probs = np.zeros(len(mats), dtype=np.float64)
    chosen = ctypes.c_int()
    _check(lib().hq_kraus_sample(state.ptr, ptrs, len(mats), q.ctypes.data, int(q.size), float(u),
                                 ctypes.byref(chosen), probs.ctypes.data))
    return chosen.value, probs


def hq_reduced_dm_batched(state, nb, qubits):
    """Per-shot reduced density matrices (2^nb, 2^k, 2^k), unnormalised."""
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    d = 2 ** q.size
    rho = np.zeros((2 ** nb, d, d), dtype=np.complex128)
    _check(lib().hq_reduced_dm_batched(state.ptr, int(nb), q.ctypes.data, int(q.size), rho.ctypes.data))
    return rho


def hq_reduced_dm_batched_sum(state, nb, qubits, nlive):
    """Sum over the first nlive shots of the trace-normalised reduced density
    matrices (the trajectory average's numerator), computed in the library."""
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    d = 2 ** q.size
    rho = np.zeros((d, d), dtype=np.complex128)
    _check(lib().hq_reduced_dm_batched_sum(state.ptr, int(nb), q.ctypes.data, int(q.size), int(nlive),
                                           rho.ctypes.data))
    return rho


def hq_kraus_sample_batched(state, nb, K, qubits, u):
    """One trajectory step for each of the 2^nb shots with uniforms u (2^nb):
    returns (chosen indices int32 array, probabilities (2^nb, nkraus))."""
    ptrs, mats = _kraus_array(K)
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    assert uu.size == 2 ** nb
    chosen = np.zeros(2 ** nb, dtype=np.int32)
    probs = np.zeros((2 ** nb, len(mats)), dtype=np.float64)
    _check(lib().hq_kraus_sample_batched(state.ptr, int(nb), ptrs, len(mats), q.ctypes.data, int(q.size),
                                         uu.ctypes.data, chosen.ctypes.data, probs.ctypes.data))
    return chosen, probs


def hq_dm_superop(K):
    """Superoperator sum_m K_m (x) conj(K_m) as a complex128 (4^k x 4^k) array."""
    ptrs, mats = _kraus_array(K)
    k = int(np.log2(mats[0].shape[0]))
    S = np.zeros((4 ** k, 4 ** k), dtype=np.complex128)
    _check(lib().hq_dm_superop(ptrs, len(mats), k, S.ctypes.data))
    return S


def hq_dm_apply_unitary(state, U, qubits):
    U, Uf = _u_buffer(U)
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    _check(lib().hq_dm_apply_unitary(state.ptr, Uf.ctypes.data, q.ctypes.data, int(q.size)))


def hq_dm_apply_kraus(state, K, qubits):
    ptrs, mats = _kraus_array(K)
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    _check(lib().hq_dm_apply_kraus(state.ptr, ptrs, len(mats), q.ctypes.data, int(q.size)))


def hq_dm_trace(state):
    re, im = ctypes.c_double(), ctypes.c_double()
    _check(lib().hq_dm_trace(state.ptr, ctypes.byref(re), ctypes.byref(im)))
    return complex(re.value, im.value)


def hq_get_amplitudes(state, first=0, count=None, out=None):
    if count is None:
        count = (1 << state.n) - first
    if out is None:
        out = np.zeros(count, dtype=state.np_dtype)
    assert out.dtype == state.np_dtype and out.flags.c_contiguous and out.size >= count
    _check(lib().hq_get_amplitudes(state.ptr, int(first), int(count), out.ctypes.data))
    return out


def hq_set_amplitudes(state, values, first=0):
    v = np.ascontiguousarray(values, dtype=state.np_dtype)
    _check(lib().hq_set_amplitudes(state.ptr, int(first), int(v.size), v.ctypes.data))


def hq_norm(state):
    out = ctypes.c_double()
    _check(lib().hq_norm(state.ptr, ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------ apply

def _u_buffer(U):
    U = np.ascontiguousarray(U, dtype=np.complex128)
    return U, U.view(np.float64)


def hq_apply_matrix(state, U, qubits):
    U, Uf = _u_buffer(U)
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    _check(lib().hq_apply_matrix(state.ptr, Uf.ctypes.data, q.ctypes.data, int(q.size)))


_GATE_DT = np.dtype({"names": ["k", "q", "U"], "formats": ["<i4", ("<i4", 6), "<u8"],
                     "offsets": [hq_gate.k.offset, hq_gate.qubits.offset, hq_gate.U.offset],
                     "itemsize": ctypes.sizeof(hq_gate)})


def _gate_array(gates):
    """gates: iterable of (qubits, U) or objects with .qubits/.U.  Builds the
    hq_gate array in one numpy structured buffer (all matrices in one
    complex128 buffer) instead of one ctypes object per gate."""
    gates = list(gates)
    ng = len(gates)
    recs = np.zeros(max(ng, 1), dtype=_GATE_DT)
    mats = []
    offs = np.zeros(ng + 1, dtype=np.int64)
    for i, g in enumerate(gates):
        qs = g.qubits if hasattr(g, "qubits") else g[0]
        U = g.U if hasattr(g, "U") else g[1]
        k = len(qs)
        recs["k"][i] = k
        recs["q"][i, :] = -1
        recs["q"][i, :k] = qs
        mats.append(np.asarray(U, dtype=np.complex128).reshape(-1))
        offs[i + 1] = offs[i] + mats[-1].size
    buf = np.concatenate(mats) if mats else np.zeros(1, dtype=np.complex128)
    base = buf.ctypes.data
    if ng:
        recs["U"][:ng] = base + 16 * offs[:ng]
    arr = ctypes.cast(recs.ctypes.data, ctypes.POINTER(hq_gate))
    return arr, ng, (recs, buf)


def hq_apply_circuit(state, gates):
    arr, ng, keep = _gate_array(gates)
    _check(lib().hq_apply_circuit(state.ptr, arr, ng))


def hq_circuit_create(state, gates):
    arr, ng, keep = _gate_array(gates)
    out = P()
    _check(lib().hq_circuit_create(state.ptr, arr, ng, ctypes.byref(out)))
    return Circuit(out, state, None)


def hq_circuit_run(state, circuit):
    _check(lib().hq_circuit_run(state.ptr, circuit.ptr))


def hq_circuit_info(circuit):
    v = [ctypes.c_uint64() for _ in range(3)]
    _check(lib().hq_circuit_info(circuit.ptr, *[ctypes.byref(x) for x in v]))
    return dict(passes=v[0].value, remaps=v[1].value, permutes=v[2].value)


# ------------------------------------------------------------------ planner

def hq_fuse(gates, kmax, blocks=False):
    """Returns list of (qubits tuple, U complex128 ndarray); blocks=True runs
    the block planner hq_fuse_blocks instead of the C7 greedy hq_fuse."""
    arr, ng, keep = _gate_array(gates)
    out = ctypes.POINTER(hq_gate)()
    nout = ctypes.c_size_t()
    fn = lib().hq_fuse_blocks if blocks else lib().hq_fuse
    _check(fn(arr, ng, int(kmax), ctypes.byref(out), ctypes.byref(nout)))
    res = []
    try:
        for i in range(nout.value):
            g = out[i]
            k = g.k
            d = 2 ** k
            U = np.ctypeslib.as_array(g.U, shape=(2 * d * d,)).copy().view(np.complex128).reshape(d, d)
            res.append((tuple(g.qubits[j] for j in range(k)), U))
    finally:
        lib().hq_free_gates(out, nout.value)
    return res


def hq_fuse_plan(gates, kmax):
    arr, ng, keep = _gate_array(gates)
    group_of = np.zeros(max(ng, 1), dtype=np.int32)
    ngroups = ctypes.c_size_t()
    _check(lib().hq_fuse_plan(arr, ng, int(kmax), group_of.ctypes.data, ctypes.byref(ngroups)))
    return group_of[:ng].copy(), ngroups.value


def hq_schedule(n, m, gates, pi0=None, gather=False):
    """Returns (ops list of dict, final pi list); pi0: initial layout (default
    q -> n-1-q); gather: allow GATHER ops (isolated global accesses)."""
    arr, ng, keep = _gate_array(gates)
    ops = ctypes.POINTER(hq_op)()
    nops = ctypes.c_size_t()
    pi = np.zeros(max(n, 1), dtype=np.int32)
    p0 = None if pi0 is None else np.ascontiguousarray(pi0, dtype=np.int32)
    _check(lib().hq_schedule_from(int(n), int(m), arr, ng, None if p0 is None else p0.ctypes.data,
                                  1 if gather else 0, ctypes.byref(ops), ctypes.byref(nops), pi.ctypes.data))
    res = []
    try:
        for i in range(nops.value):
            o = ops[i]
            res.append({"kind": ("apply", "remap", "permute", "gather")[o.kind], "gate": o.gate,
                        "nbits": o.nbits, "bits": [o.bits[t] for t in range(12)]})
    finally:
        lib().hq_free_ops(ops)
    return res, [int(x) for x in pi[:n]]


def hq_remap_plan(n, m, op, rank):
    """The library's transfer list of a REMAP op (dict from hq_schedule) for
    `rank`: list of (peer, offset, length) in amplitudes."""
    o = hq_op()
    o.kind, o.gate, o.nbits = 1, -1, int(op["nbits"])
    for t in range(12):
        o.bits[t] = int(op["bits"][t])
    cnt = ctypes.c_size_t()
    _check(lib().hq_remap_plan(int(n), int(m), ctypes.byref(o), int(rank), None, None, None, 0, ctypes.byref(cnt)))
    k = cnt.value
    peer = np.zeros(max(k, 1), dtype=np.int32)
    off = np.zeros(max(k, 1), dtype=np.uint64)
    ln = np.zeros(max(k, 1), dtype=np.uint64)
    _check(lib().hq_remap_plan(int(n), int(m), ctypes.byref(o), int(rank), peer.ctypes.data, off.ctypes.data,
                               ln.ctypes.data, k, ctypes.byref(cnt)))
    return [(int(peer[i]), int(off[i]), int(ln[i])) for i in range(k)]


def hq_plan_layout(n, m, gates, dtype="c64"):
    """Returns (pi list, model cost before, model cost after)."""
    arr, ng, keep = _gate_array(gates)
    pi = np.zeros(max(n, 1), dtype=np.int32)
    cb, ca = ctypes.c_double(), ctypes.c_double()
    _check(lib().hq_plan_layout(int(n), int(m), _dt(dtype), arr, ng, pi.ctypes.data,
                                ctypes.byref(cb), ctypes.byref(ca)))
    return [int(x) for x in pi[:n]], cb.value, ca.value


def hq_state_set_layout(state, pi):
    v = np.ascontiguousarray(pi, dtype=np.int32)
    _check(lib().hq_state_set_layout(state.ptr, v.ctypes.data))


REMAP_MODES = {"exchange": 0, "fused": 1, "gather": 2, "fused+gather": 3}


def hq_state_set_remap_mode(state, mode="fused+gather"):
    """'fused+gather' (default): remaps folded into the preceding apply pass
    and isolated global accesses as pair gathers, when peer buffers are
    mapped; 'fused' / 'gather' one of them; 'exchange': always a separate
    exchange.  Returns whether peer buffers are mapped."""
    avail = ctypes.c_int()
    _check(lib().hq_state_set_remap_mode(state.ptr, REMAP_MODES[mode], ctypes.byref(avail)))
    return bool(avail.value)


def hq_state_invalidate_bound(state):
    """Call after writing a borrowed state buffer outside the library (hq.h)."""
    _check(lib().hq_state_invalidate_bound(state.ptr))


def hq_state_get_layout(state):
    v = np.zeros(state.n, dtype=np.int32)
    _check(lib().hq_state_get_layout(state.ptr, v.ctypes.data))
    return [int(x) for x in v]


# ------------------------------------------------------------------ diagnostics

def hq_last_error():
    return lib().hq_last_error().decode(errors="replace")


def hq_version():
    return lib().hq_version().decode()


def hq_sync(state):
    _check(lib().hq_sync(state.ptr))


def hq_stats_get(state):
    s = hq_stats()
    _check(lib().hq_stats_get(state.ptr, ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in hq_stats._fields_}


def hq_stats_reset(state):
    _check(lib().hq_stats_reset(state.ptr))


def hq_profile_enable(state, on=True):
    _check(lib().hq_profile_enable(state.ptr, 1 if on else 0))


KERNEL_PATHS = {"all": -1, "simt": 0, "generic": 1, "tc": 2}


def hq_kernel_times(state, path="all"):
    """path: 'all', 'simt' (apply_reg), 'generic' (apply_gen), 'tc' (apply_tc)."""
    c, t, m, b = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    _check(lib().hq_kernel_times(state.ptr, KERNEL_PATHS[path], ctypes.byref(c), ctypes.byref(t),
                                 ctypes.byref(m), ctypes.byref(b)))
    return dict(count=c.value, total_ms=t.value, max_ms=m.value, bytes=b.value)
