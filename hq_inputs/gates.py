"""Fixed fp64 gate matrices used as *inputs* (SURVEY.md §8(c) C15).

Convention (C2): row-major 2^k x 2^k, qubits[0] is the most
significant bit of the row/column index, and the gate acts on column vectors
(psi' = U psi).  These are definitions of inputs, not method arithmetic.
"""
import numpy as np

_s = 1.0 / np.sqrt(2.0)

#: sqrt(X) = RX(pi/2) = (1/sqrt2)[[1,-i],[-i,1]]                    (C15)
SQRT_X = _s * np.array([[1, -1j], [-1j, 1]], dtype=np.complex128)
#: sqrt(Y) = RY(pi/2) = (1/sqrt2)[[1,-1],[1,1]]                     (C15)
SQRT_Y = _s * np.array([[1, -1], [1, 1]], dtype=np.complex128)
#: sqrt(W) = RW(pi/2), W = (X+Y)/sqrt2:
#: (1/sqrt2)[[1, -e^{i pi/4}], [e^{-i pi/4}, 1]]                     (C15)
SQRT_W = _s * np.array([[1, -np.exp(1j * np.pi / 4)],
                        [np.exp(-1j * np.pi / 4), 1]], dtype=np.complex128)

H = _s * np.array([[1, 1], [1, -1]], dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
#: CX with qubits[0] = control (MSB), qubits[1] = target
CX = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]],
              dtype=np.complex128)
CZ = np.diag([1, 1, 1, -1]).astype(np.complex128)
SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]],
                dtype=np.complex128)
#: Toffoli, qubits[0], qubits[1] controls, qubits[2] target
CCX = np.eye(8, dtype=np.complex128)
CCX[[6, 7]] = CCX[[7, 6]]


def fsim(theta=np.pi / 2, phi=np.pi / 6):
    """fSim(theta, phi) in the Arute et al. 2019 convention (C15):
    [[1,0,0,0],[0,cos t,-i sin t,0],[0,-i sin t,cos t,0],[0,0,0,e^{-i phi}]]."""
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def cphase(phi):
    """CPHASE(phi) = diag(1,1,1,e^{i phi})."""
    return np.diag([1, 1, 1, np.exp(1j * phi)]).astype(np.complex128)


def cr_m(m):
    """Controlled R_m, R_m = diag(1, e^{2 pi i / 2^m}) (QFT pin P5)."""
    return cphase(2 * np.pi / 2 ** m)


def rz(theta):
    return np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta)]).astype(np.complex128)


def permutation_matrix(perm):
    """U with U[perm[c], c] = 1: maps basis |c> to |perm[c]> (C11)."""
    d = len(perm)
    U = np.zeros((d, d), dtype=np.complex128)
    for c, r in enumerate(perm):
        U[r, c] = 1.0
    return U
