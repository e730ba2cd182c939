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


# ---------------------------------------------------------------- hash states
# A deterministic, index-addressable integer-valued state: re/im are integers
# in [-2^10, 2^10) (exact in FP32/TF32/FP64), computed from the amplitude index
# alone so that any single amplitude can be regenerated on the host while the
# full state (up to 2^34 amplitudes) is generated on the device by torch.
_HM1, _HM2 = 0x9E3779B97F4A7C15 & ((1 << 63) - 1), 0xBF58476D1CE4E5B9 & ((1 << 63) - 1)


def hash_amplitudes_np(idx):
    """numpy: complex128 values of the hash state at int64 indices idx."""
    i = np.asarray(idx, dtype=np.int64)
    a = (i * np.int64(_HM1)) ^ (i >> np.int64(7))
    b = (i * np.int64(_HM2)) ^ (i >> np.int64(11))
    re = ((a >> np.int64(20)) & np.int64(2047)) - 1024
    im = ((b >> np.int64(24)) & np.int64(2047)) - 1024
    return re.astype(np.float64) + 1j * im.astype(np.float64)


def hash_state_torch(n, device, chunk=1 << 26):
    """torch: the same hash state as complex64 on `device` (2^n amplitudes)."""
    import torch
    out = torch.empty(1 << n, dtype=torch.complex64, device=device)
    view = torch.view_as_real(out)
    for s in range(0, 1 << n, chunk):
        i = torch.arange(s, min(s + chunk, 1 << n), dtype=torch.int64, device=device)
        a = (i * _HM1) ^ (i >> 7)
        b = (i * _HM2) ^ (i >> 11)
        view[s:s + i.numel(), 0] = (((a >> 20) & 2047) - 1024).to(torch.float32)
        view[s:s + i.numel(), 1] = (((b >> 24) & 2047) - 1024).to(torch.float32)
    return out


def random_state_torch(n, device, seed=0, dtype="c64"):
    """torch: a dense random-normal state of 2^n amplitudes on `device`,
    normalised (SURVEY §8(d) config [2]: "random-normal normalized state,
    device fill").  Every amplitude is non-zero, so timed passes see the
    operand activity of a generic state, not of a sparse |0>-derived one."""
    import torch
    dt = torch.complex64 if dtype == "c64" else torch.complex128
    out = torch.empty(1 << n, dtype=dt, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    flat = torch.view_as_real(out).reshape(-1)
    flat.normal_(generator=g)
    chunk = 1 << 27
    nrm2 = torch.zeros((), dtype=torch.float64, device=device)
    for i in range(0, flat.numel(), chunk):
        nrm2 += flat[i:i + chunk].double().square().sum()
    flat.div_(nrm2.sqrt().to(flat.dtype))
    return out
