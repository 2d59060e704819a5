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

import math

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


# ------------------------------------------------------------------ textbook gates (converter pins)
# Standard gate matrices as written in textbooks (H, S, T, Paulis, RX/RY/RZ(t) = exp(-i t P/2),
# CNOT, CZ, SWAP, CPHASE(l) = diag(1, 1, 1, e^{il}), RZZ(t) = exp(-i t ZZ/2)), embedded with qubit q
# = bit q of the index.  Used to check ps_gate_to_rotations and converted circuits.

_H = np.array([[1, 1], [1, -1]]) / math.sqrt(2)
_S = np.diag([1, 1j])
_T = np.diag([1, np.exp(1j * math.pi / 4)])
_X = np.array([[0, 1], [1, 0]])
_Y = np.array([[0, -1j], [1j, 0]])
_Z = np.diag([1, -1])


def _rx(t):
    return np.array([[math.cos(t / 2), -1j * math.sin(t / 2)], [-1j * math.sin(t / 2), math.cos(t / 2)]])


def _ry(t):
    return np.array([[math.cos(t / 2), -math.sin(t / 2)], [math.sin(t / 2), math.cos(t / 2)]])


def _rz(t):
    return np.diag([np.exp(-1j * t / 2), np.exp(1j * t / 2)])


def textbook_gate(name, qubits, params, n):
    """Gate matrix on n qubits, qubit q = bit q of the index, built from textbook definitions."""
    dim = 1 << n
    if len(qubits) == 1:
        m1 = {"H": _H, "S": _S, "T": _T, "X": _X, "Y": _Y, "Z": _Z}.get(name)
        if m1 is None:
            m1 = {"RX": _rx, "RY": _ry, "RZ": _rz}[name](params[0])
        q = qubits[0]
        u = np.zeros((dim, dim), complex)
        for i in range(dim):
            b = (i >> q) & 1
            for b2 in (0, 1):
                j = (i & ~(1 << q)) | (b2 << q)
                u[j, i] += m1[b2, b]
        return u
    c, t = qubits
    u = np.zeros((dim, dim), complex)
    for i in range(dim):
        bc, bt = (i >> c) & 1, (i >> t) & 1
        if name == "CNOT":
            j = i ^ (1 << t) if bc else i
            u[j, i] = 1
        elif name == "CZ":
            u[i, i] = -1 if (bc and bt) else 1
        elif name == "CPHASE":
            u[i, i] = np.exp(1j * params[0]) if (bc and bt) else 1
        elif name == "SWAP":
            j = i & ~((1 << c) | (1 << t)) | (bt << c) | (bc << t)
            u[j, i] = 1
        elif name == "RZZ":
            u[i, i] = np.exp(-1j * params[0] / 2 * (1 if bc == bt else -1))
    return u




def apply_gates(n: int, psi, gates) -> np.ndarray:
    """Applies a gate list [(name, qubits, params), ...] as dense textbook matrices (n <= 8)."""
    if n > MAX_QUBITS:
        raise ValueError("dense oracle is capped at 8 qubits")
    out = np.asarray(psi, dtype=np.complex128).copy()
    for name, qubits, params in gates:
        out = textbook_gate(name.upper(), tuple(qubits), tuple(params), n) @ out
    return out
