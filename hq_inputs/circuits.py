"""Seeded circuit generators (inputs only).

A circuit is a list of :class:`Gate` = (name, qubits, U) applied leftmost first
(SPEC S:127).  U is a complex128 2^k x 2^k matrix in the C2 convention.

* ``sycamore_circuit``: the paper's ``get_rqc`` is undefined, so
  the benchmark circuits follow the Sycamore-style reading C16: per cycle one
  layer of single-qubit gates drawn from {sqrtX, sqrtY, sqrtW} (never repeating
  the qubit's previous gate), then one fSim(pi/2, pi/6) layer with pattern
  "ABCDCDAB"[c mod 8] on a cols = ceil(sqrt n) grid.
* ``haar_unitary``: Mezzadri's QR-with-phase-fix Haar sampler (C18).
* RNG: ``numpy.random.default_rng(seed)`` (PCG64), draws in loop order (C17).
"""
import hashlib
import json
import math
from collections import namedtuple

import numpy as np

from . import gates as G

Gate = namedtuple("Gate", ["name", "qubits", "U"])

#: seeds per BASELINE.json config index (C17)
CONFIG_SEEDS = {0: [0, 1, 2, 3, 4], 1: [1000], 2: 2000, 3: [3000], 4: [4000]}

_SINGLES = (("SQRT_X", G.SQRT_X), ("SQRT_Y", G.SQRT_Y), ("SQRT_W", G.SQRT_W))


def grid_shape(n):
    cols = math.ceil(math.sqrt(n))
    rows = math.ceil(n / cols)
    return rows, cols


def _coupler_pairs(n, layer):
    rows, cols = grid_shape(n)
    pairs = []
    for r in range(rows):
        for c in range(cols):
            q = r * cols + c
            if q >= n:
                continue
            if layer in "AB":
                if c % 2 == (0 if layer == "A" else 1) and c + 1 < cols:
                    q2 = q + 1
                    if q2 < n:
                        pairs.append((q, q2))
            else:
                if r % 2 == (0 if layer == "C" else 1) and r + 1 < rows:
                    q2 = q + cols
                    if q2 < n:
                        pairs.append((q, q2))
    return pairs


def sycamore_circuit(n, cycles, seed, theta=np.pi / 2, phi=np.pi / 6,
                     final_single_layer=False):
    """Sycamore-style random circuit with ``cycles`` cycles (C16)."""
    rng = np.random.default_rng(seed)
    fs = G.fsim(theta, phi)
    prev = [-1] * n
    out = []
    pattern = "ABCDCDAB"

    def single_layer():
        for q in range(n):
            if prev[q] < 0:
                choice = int(rng.integers(3))
            else:
                allowed = [i for i in range(3) if i != prev[q]]
                choice = allowed[int(rng.integers(2))]
            prev[q] = choice
            name, U = _SINGLES[choice]
            out.append(Gate(name, (q,), U))

    for c in range(cycles):
        single_layer()
        for (a, b) in _coupler_pairs(n, pattern[c % 8]):
            out.append(Gate("FSIM", (a, b), fs))
    if final_single_layer:
        single_layer()
    return out


def haar_unitary(k, rng):
    """Haar-random U(2^k): QR of a complex Ginibre matrix, phases fixed by
    diag(R)/|diag(R)| (Mezzadri 2007; C18)."""
    d = 2 ** k
    Z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2)
    Q, R = np.linalg.qr(Z)
    ph = np.diag(R) / np.abs(np.diag(R))
    return (Q * ph[None, :]).astype(np.complex128)


def haar_sweep_gate(n, k, placement, seed):
    """One Haar k-qubit gate for the fused-gate sweep (BASELINE config [2]).

    placement: 'low'  -> physical bits 0..k-1, i.e. qubits n-1..n-k
               'high' -> physical bits n-k..n-1, i.e. qubits 0..k-1
               'spread' -> evenly spread over the n bits
               'random<j>' -> k distinct random qubits (seeded by j)
               'b:<b0>-<b1>-...' -> these physical bits
    Qubit q sits at index bit n-1-q (C1).  Returns a Gate.
    """
    rng = np.random.default_rng(seed)
    U = haar_unitary(k, rng)
    if placement == "low":
        bits = list(range(k))
    elif placement == "high":
        bits = list(range(n - k, n))
    elif placement == "spread":
        bits = sorted({int(round(i * (n - 1) / max(k - 1, 1))) for i in range(k)})
        assert len(bits) == k
    elif placement.startswith("b:"):
        bits = [int(x) for x in placement[2:].split("-")]
        assert len(bits) == k
    elif placement.startswith("random"):
        j = int(placement[6:] or 0)
        r2 = np.random.default_rng(10_000 + 97 * j + seed)
        bits = [int(b) for b in r2.choice(n, size=k, replace=False)]
    else:
        raise ValueError(placement)
    qubits = tuple(n - 1 - b for b in bits)
    return Gate("HAAR%d" % k, qubits, U)


def random_circuit(n, n_gates, seed, kmax=2, kmin=1):
    """Random Haar gates of arity kmin..kmax on random distinct qubits."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_gates):
        k = int(rng.integers(kmin, kmax + 1))
        k = min(k, n)
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        out.append(Gate("HAAR%d" % k, qs, haar_unitary(k, rng)))
    return out


def reversible_circuit(n, n_gates, seed, kmax=3):
    """Random permutation gates (X, CX, SWAP, CCX, random 2^k permutations)
    on random qubits: maps basis states to basis states (pin P10, C11)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_gates):
        kind = int(rng.integers(5))
        if kind == 0:
            k, name, U = 1, "X", G.X
        elif kind == 1:
            k, name, U = 2, "CX", G.CX
        elif kind == 2:
            k, name, U = 2, "SWAP", G.SWAP
        elif kind == 3:
            k, name, U = 3, "CCX", G.CCX
        else:
            k = int(rng.integers(1, kmax + 1))
            perm = [int(p) for p in rng.permutation(2 ** k)]
            name, U = "PERM%d" % k, G.permutation_matrix(perm)
        k = min(k, n)
        if U.shape[0] != 2 ** k:
            continue
        qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
        out.append(Gate(name, qs, U))
    return out


def qft_circuit(n, with_swaps=False):
    """Quantum Fourier transform: for q = 0..n-1, H on q then controlled-R_m
    (m = 2, 3, ...) from each later qubit (textbook; pin P5's gates).  Most of
    its gates are diagonal controlled phases (row f1 workload)."""
    out = []
    for q in range(n):
        out.append(Gate("H", (q,), G.H))
        for j in range(q + 1, n):
            out.append(Gate("CR%d" % (j - q + 1), (j, q), G.cr_m(j - q + 1)))
    if with_swaps:
        for q in range(n // 2):
            out.append(Gate("SWAP", (q, n - 1 - q), G.SWAP))
    return out


def qaoa_circuit(n, layers, seed):
    """QAOA-style circuit on a ring plus random chords: per layer ZZ(gamma)
    phases (diagonal) on every edge, then RX(beta) on every qubit; starts
    from H on every qubit.  Diagonal-heavy (row f1 workload)."""
    rng = np.random.default_rng(seed)
    edges = [(q, (q + 1) % n) for q in range(n)]
    edges += [tuple(int(x) for x in rng.choice(n, size=2, replace=False)) for _ in range(n // 2)]
    out = [Gate("H", (q,), G.H) for q in range(n)]
    for _ in range(layers):
        gamma, beta = rng.uniform(0, np.pi, size=2)
        zz = np.diag(np.exp(-0.5j * gamma * np.array([1, -1, -1, 1]))).astype(np.complex128)
        for a, b in edges:
            out.append(Gate("ZZ", (a, b), zz))
        c, s = np.cos(beta / 2), np.sin(beta / 2)
        rx = np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
        for q in range(n):
            out.append(Gate("RX", (q,), rx))
    return out


def circuit_to_json(n, gates, meta=None):
    return json.dumps({
        "n": n, "meta": meta or {},
        "gates": [{"name": g.name, "qubits": list(g.qubits),
                   "matrix": [[float(repr_float(z.real)), float(repr_float(z.imag))]
                              for z in np.asarray(g.U).ravel()]}
                  for g in gates]})


def repr_float(x):
    return "%.17g" % x


def circuit_from_json(text):
    d = json.loads(text)
    gates = []
    for g in d["gates"]:
        k = len(g["qubits"])
        m = np.array([complex(a, b) for a, b in g["matrix"]],
                     dtype=np.complex128).reshape(2 ** k, 2 ** k)
        gates.append(Gate(g["name"], tuple(g["qubits"]), m))
    return d["n"], gates


def circuit_bytes(gates):
    h = bytearray()
    for g in gates:
        h += np.asarray(g.qubits, dtype=np.int32).tobytes()
        h += np.ascontiguousarray(g.U, dtype=np.complex128).tobytes()
    return bytes(h)


def circuit_sha256(gates):
    return hashlib.sha256(circuit_bytes(gates)).hexdigest()
