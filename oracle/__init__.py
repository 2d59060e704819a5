"""CPU oracle for the Pauli-rotation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2504_17881_b200``) never imports it and shares no code with it.

What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):

* ``apply``: psi <- exp(i phi_{L-1} P_{L-1}) ... exp(i phi_0 P_0) psi, each rotation by the
  closed form exp(i phi P) = cos(phi) I + i sin(phi) P (Introduction), with
  P = P_1 (x) ... (x) P_n decoded qubit by qubit and factor k on bit k-1
  (worked example P:483-484).  Implemented in plain C (``ps_oracle.c``), fp64.
* ``decode_masks``: the paper's two-integer representation (p1, p2) -> factors.
* ``expectation`` / ``norm`` / ``inner``: plain sums (P:667-671 signals are overlaps).
* ``apply_coset``: the same definition restricted to a coset i0 + span{p1_l}, exact because
  every rotation maps that coset to itself.
* ``random_state``: the seeded counter-based input generator of DESIGN.md "Input recipe"
  (input generation, not the method).

Pins (``tests/test_oracle.py``): dense matrix exponentials (``oracle.dense``, n <= 8), the
paper's worked example, SPEC/closed-form examples in ``tests/golden/``, unitarity, the
commuting-swap invariance, inverse layers, bit-exact basis permutations.  Every function here
is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libps_oracle.so")
_SRC = os.path.join(_HERE, "ps_oracle.c")

LETTERS = "IXYZ"  # factor code = index in this string


def build(force: bool = False) -> str:
    """Compile ps_oracle.c with plain gcc (no FMA contraction, OpenMP on the gather loop)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
            "-std=c11", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        dp = ctypes.POINTER(ctypes.c_double)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.oracle_decode_masks.argtypes = [ctypes.c_int, ctypes.c_size_t, u64p, u64p, u8p]
        L.oracle_decode_masks.restype = ctypes.c_int
        L.oracle_apply_factors.argtypes = [ctypes.c_int, dp, ctypes.c_size_t, u8p, dp]
        L.oracle_apply_factors.restype = ctypes.c_int
        L.oracle_pauli_apply.argtypes = [ctypes.c_int, u8p, dp, dp]
        L.oracle_pauli_apply.restype = ctypes.c_int
        L.oracle_norm.argtypes = [ctypes.c_int, dp]
        L.oracle_norm.restype = ctypes.c_double
        L.oracle_inner.argtypes = [ctypes.c_int, dp, dp, dp]
        L.oracle_inner.restype = None
        L.oracle_expectation.argtypes = [ctypes.c_int, dp, ctypes.c_size_t, u8p, dp, dp]
        L.oracle_expectation.restype = ctypes.c_int
        L.oracle_random_amplitudes.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, dp]
        L.oracle_random_amplitudes.restype = None
        L.oracle_generator_raw.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_generator_raw.restype = ctypes.c_uint64
        L.oracle_apply_coset.argtypes = [ctypes.c_int, ctypes.c_size_t, u64p, dp, ctypes.c_size_t, u8p, dp]
        L.oracle_apply_coset.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def word_to_factors(word: str) -> np.ndarray:
    """Pauli word P_1 P_2 ... P_n (leftmost letter = factor 1 = qubit 0) -> codes."""
    return np.array([LETTERS.index(ch) for ch in word.upper()], dtype=np.uint8)


def words_to_factors(words) -> np.ndarray:
    return np.stack([word_to_factors(w) for w in words]) if len(words) else np.zeros((0, 0), np.uint8)


def decode_masks(n: int, p1, p2) -> np.ndarray:
    """(p1, p2) masks -> factor codes, shape (count, n).  P:478-482."""
    p1 = np.ascontiguousarray(p1, dtype=np.uint64)
    p2 = np.ascontiguousarray(p2, dtype=np.uint64)
    out = np.zeros((len(p1), n), dtype=np.uint8)
    rc = lib().oracle_decode_masks(n, len(p1), _ptr(p1, ctypes.c_uint64), _ptr(p2, ctypes.c_uint64),
                                   _ptr(out, ctypes.c_uint8))
    if rc != 0:
        raise ValueError("mask bit at position >= n")
    return out


def _as_state(psi: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(psi, dtype=np.complex128).copy()


def apply(n: int, psi: np.ndarray, factors: np.ndarray, angles) -> np.ndarray:
    """Sequentially apply exp(i angles[l] P_l), l = 0 first.  Returns a new array."""
    out = _as_state(psi)
    assert out.shape == (1 << n,)
    f = np.ascontiguousarray(factors, dtype=np.uint8).reshape(-1, n) if n else np.zeros((len(angles), 0), np.uint8)
    ang = np.ascontiguousarray(angles, dtype=np.float64)
    assert f.shape[0] == ang.shape[0]
    if len(ang) == 0:
        return out
    rc = lib().oracle_apply_factors(n, _ptr(out.view(np.float64), ctypes.c_double), len(ang),
                                    _ptr(f, ctypes.c_uint8), _ptr(ang, ctypes.c_double))
    if rc != 0:
        raise MemoryError("oracle_apply_factors")
    return out


def apply_masks(n: int, psi: np.ndarray, p1, p2, angles) -> np.ndarray:
    return apply(n, psi, decode_masks(n, p1, p2), angles)


def pauli_apply(n: int, psi: np.ndarray, factors_row: np.ndarray) -> np.ndarray:
    a = _as_state(psi)
    out = np.zeros_like(a)
    f = np.ascontiguousarray(factors_row, dtype=np.uint8)
    lib().oracle_pauli_apply(n, _ptr(f, ctypes.c_uint8), _ptr(a.view(np.float64), ctypes.c_double),
                             _ptr(out.view(np.float64), ctypes.c_double))
    return out


def norm(n: int, psi: np.ndarray) -> float:
    a = _as_state(psi)
    return float(lib().oracle_norm(n, _ptr(a.view(np.float64), ctypes.c_double)))


def inner(n: int, a: np.ndarray, b: np.ndarray) -> complex:
    a = _as_state(a)
    b = _as_state(b)
    out = np.zeros(2)
    lib().oracle_inner(n, _ptr(a.view(np.float64), ctypes.c_double), _ptr(b.view(np.float64), ctypes.c_double),
                       _ptr(out, ctypes.c_double))
    return complex(out[0], out[1])


def expectation(n: int, psi: np.ndarray, factors: np.ndarray, coeffs) -> float:
    a = _as_state(psi)
    f = np.ascontiguousarray(factors, dtype=np.uint8).reshape(-1, n)
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros(1)
    rc = lib().oracle_expectation(n, _ptr(a.view(np.float64), ctypes.c_double), len(c), _ptr(f, ctypes.c_uint8),
                                  _ptr(c, ctypes.c_double), _ptr(out, ctypes.c_double))
    if rc != 0:
        raise MemoryError("oracle_expectation")
    return float(out[0])


def random_amplitudes(seed: int, first: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.complex128)
    lib().oracle_random_amplitudes(seed, first, count, _ptr(out.view(np.float64), ctypes.c_double))
    return out


def random_amplitudes_at(seed: int, indices) -> np.ndarray:
    """Generator values at arbitrary (e.g. coset) indices."""
    idx = np.asarray(indices, dtype=np.uint64)
    return np.array([random_amplitudes(seed, int(i), 1)[0] for i in idx], dtype=np.complex128)


def random_state(seed: int, n: int) -> np.ndarray:
    return random_amplitudes(seed, 0, 1 << n)


def generator_raw(seed: int, k: int) -> int:
    return int(lib().oracle_generator_raw(seed, k))


def apply_coset(n: int, members, amps: np.ndarray, factors: np.ndarray, angles) -> np.ndarray:
    mem = np.ascontiguousarray(members, dtype=np.uint64)
    a = _as_state(amps)
    f = np.ascontiguousarray(factors, dtype=np.uint8).reshape(-1, n)
    ang = np.ascontiguousarray(angles, dtype=np.float64)
    rc = lib().oracle_apply_coset(n, len(mem), _ptr(mem, ctypes.c_uint64), _ptr(a.view(np.float64), ctypes.c_double),
                                  len(ang), _ptr(f, ctypes.c_uint8), _ptr(ang, ctypes.c_double))
    if rc == -2:
        raise ValueError("coset not closed under the rotations' p1 masks")
    if rc != 0:
        raise MemoryError("oracle_apply_coset")
    return a


def coset_members(n: int, i0: int, p1_masks) -> np.ndarray:
    """Enumerate i0 + span_GF(2){p1_l} by closure (plain set construction, no elimination)."""
    members = {int(i0)}
    for x in p1_masks:
        x = int(x)
        if x == 0:
            continue
        new = {m ^ x for m in members}
        members |= new
    return np.array(sorted(members), dtype=np.uint64)
