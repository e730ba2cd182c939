"""Seeded input states (no method arithmetic).

Index convention (C1, pinned by the paper's Grover listing P:403-422): qubit q
is index bit n-1-q, i.e. qubit 0 is the most significant bit.
"""
import numpy as np


def random_state(n, seed, normalize=True):
    """Complex normal state, complex128, optionally normalised."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    if normalize:
        v /= np.sqrt(np.sum(np.abs(v) ** 2))
    return v.astype(np.complex128)


def integer_state(n, seed, bound=2 ** 10):
    """Re/im parts are integers with |v| < 2^11: exact in FP32, TF32 and FP64,
    so permutation gates must reproduce them bit-exactly (C11)."""
    rng = np.random.default_rng(seed)
    re = rng.integers(-bound, bound, size=2 ** n)
    im = rng.integers(-bound, bound, size=2 ** n)
    return (re + 1j * im).astype(np.complex128)


def basis_index(bits):
    """Index of |b_0 b_1 ... b_{n-1}> with qubit 0 the MSB (C1)."""
    x = 0
    for b in bits:
        x = (x << 1) | int(b)
    return x
