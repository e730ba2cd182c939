"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no gate application, no
fusion, no norm).  It only *defines inputs*: gate matrices of the Sycamore-style
generator, Haar-random unitaries (C18), seeded random
states, and permutation matrices for the bit-exact tests (C11).  Both `oracle/`
and the product path consume these as plain numpy arrays.
"""
from .gates import (SQRT_X, SQRT_Y, SQRT_W, H, X, Y, Z, CX, CZ, SWAP, CCX,
                    fsim, cphase, cr_m, rz, permutation_matrix)
from .circuits import (Gate, sycamore_circuit, haar_unitary, haar_sweep_gate,
                       random_circuit, grid_shape, circuit_bytes, circuit_sha256,
                       circuit_to_json, circuit_from_json, reversible_circuit,
                       qft_circuit, qaoa_circuit, CONFIG_SEEDS)
from .states import random_state, integer_state, basis_index

__all__ = [
    "SQRT_X", "SQRT_Y", "SQRT_W", "H", "X", "Y", "Z", "CX", "CZ", "SWAP", "CCX",
    "fsim", "cphase", "cr_m", "rz", "permutation_matrix",
    "Gate", "sycamore_circuit", "haar_unitary", "haar_sweep_gate",
    "random_circuit", "grid_shape", "circuit_bytes", "circuit_sha256",
    "circuit_to_json", "circuit_from_json", "reversible_circuit", "qft_circuit",
    "qaoa_circuit", "CONFIG_SEEDS",
    "random_state", "integer_state", "basis_index",
]
