"""Dense companion oracle (numpy/scipy, n <= 8) -- TEST INFRASTRUCTURE ONLY.

Builds Pauli strings as Kronecker products of the textbook 2x2 matrices and
rotations with the textbook matrix exponential ``scipy.linalg.expm(1j*phi*P)`` -- deliberately
*not* the closed form cos(phi) I + i sin(phi) P, so that the closed form used by
``oracle.apply`` is checked against an independent routine.

Bit convention: factor k acts on bit k-1 of the basis index.  With numpy's kron
the leftmost operand owns the most significant bit, so P_1 (x) ... (x) P_n as an index-space
matrix is ``kron(P_n, ..., P_1)``.  ``tests/test_oracle.py`` pins this reading on the paper's
worked example before it is used anywhere else.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

I2 = np.array([[1, 0], [0, 1]], dtype=np.complex128)
SX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
SY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
SZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
MATS = [I2, SX, SY, SZ]  # indexed by factor code, letters "IXYZ"

MAX_QUBITS = 8


def dense_pauli(factors_row) -> np.ndarray:
    f = list(np.asarray(factors_row, dtype=np.int64))
    if len(f) > MAX_QUBITS:
        raise ValueError("dense oracle is capped at 8 qubits")
    m = np.array([[1.0 + 0j]])
    for code in reversed(f):  # factor n leftmost ... factor 1 rightmost
        m = np.kron(m, MATS[code]) if m.size > 1 else MATS[code].copy()
    return m


def dense_rotation(factors_row, phi: float) -> np.ndarray:
    return scipy.linalg.expm(1j * float(phi) * dense_pauli(factors_row))


def dense_apply(psi: np.ndarray, factors: np.ndarray, angles) -> np.ndarray:
    out = np.asarray(psi, dtype=np.complex128).copy()
    for row, phi in zip(factors, angles):
        out = dense_rotation(row, phi) @ out
    return out


def dense_layer(factors: np.ndarray, angles) -> np.ndarray:
    n = factors.shape[1]
    u = np.eye(1 << n, dtype=np.complex128)
    for row, phi in zip(factors, angles):
        u = dense_rotation(row, phi) @ u
    return u
