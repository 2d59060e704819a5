"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against things other than
itself -- the paper's worked example, textbook matrix exponentials, closed forms, invariants and
brute force -- before any CUDA result is compared with it.

Citations: PAPER.md line numbers (P:n), SPEC.md line numbers (S:n).
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import oracle
from oracle import dense
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        for raw in fh:
            line = raw.split("#", 1)[0].strip()
            if line:
                yield line


def _phi(expr: str) -> float:
    allowed = set("0123456789.+-*/ ()pi")
    assert set(expr) <= allowed, expr
    return float(eval(expr, {"__builtins__": {}}, {"pi": math.pi}))


def _basis(n, i):
    v = np.zeros(1 << n, dtype=np.complex128)
    v[i] = 1.0
    return v


def _rand_state(rng, n):
    return rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)


# ---------------------------------------------------------------- encoding

def test_worked_example_decode():
    """sx (x) I (x) sy  <->  p1 = 5, p2 = 4."""
    f = oracle.decode_masks(3, [5], [4])
    assert f.tolist() == [[1, 0, 2]]  # X, I, Y on qubits 0, 1, 2
    assert oracle.word_to_factors("XIY").tolist() == [1, 0, 2]


@pytest.mark.parametrize("line", list(_lines("encode_examples.txt")))
def test_golden_encode(line):
    word, p1, p2 = line.split()
    f = oracle.decode_masks(len(word), [int(p1)], [int(p2)])
    assert f[0].tolist() == oracle.word_to_factors(word).tolist()


def test_decode_rejects_bits_above_n():
    with pytest.raises(ValueError):
        oracle.decode_masks(3, [8], [0])
    with pytest.raises(ValueError):
        oracle.decode_masks(3, [0], [1 << 3])


def test_dense_bit_convention_matches_worked_example():
    """The dense companion's kron order must put factor k on bit k-1: the XIY matrix
    maps |i> to a multiple of |i xor 5>, and its phase flips with bit 2 of i (the sy factor)."""
    m = dense.dense_pauli(oracle.word_to_factors("XIY"))
    for i in range(8):
        col = m[:, i]
        nz = np.flatnonzero(np.abs(col) > 0.5)
        assert nz.tolist() == [i ^ 5]
        expected = 1j if (i >> 2) & 1 == 0 else -1j
        assert col[i ^ 5] == expected


# ---------------------------------------------------------------- basis action

@pytest.mark.parametrize("line", list(_lines("basis_action.txt")))
def test_golden_basis_action(line):
    word, i, j, wr, wi = line.split()
    n = len(word)
    out = oracle.pauli_apply(n, _basis(n, int(i)), oracle.word_to_factors(word))
    expected = _basis(n, int(j)) * complex(float(wr), float(wi))
    assert np.array_equal(out, expected)


def test_basis_action_matches_dense_all_strings_n3():
    """Every one of the 64 three-qubit strings, every basis column, entry for entry."""
    n = 3
    for code in range(4 ** n):
        f = np.array([(code >> (2 * q)) & 3 for q in range(n)], dtype=np.uint8)
        m = dense.dense_pauli(f)
        for i in range(1 << n):
            out = oracle.pauli_apply(n, _basis(n, i), f)
            assert np.array_equal(out, m[:, i])


def test_involution_and_hermiticity():
    rng = np.random.default_rng(1)
    n = 5
    for _ in range(20):
        f = rng.integers(0, 4, size=n).astype(np.uint8)
        psi = _rand_state(rng, n)
        twice = oracle.pauli_apply(n, oracle.pauli_apply(n, psi, f), f)
        assert np.array_equal(twice, psi)  # P^2 = I exactly (phases are +-1, +-i)


# ---------------------------------------------------------------- rotations

@pytest.mark.parametrize("line", list(_lines("rotation_examples.txt")))
def test_golden_rotation_examples(line):
    lhs, rhs = line.split("=>")
    word, phi, i = lhs.split()
    n = len(word)
    out = oracle.apply(n, _basis(n, int(i)), oracle.word_to_factors(word)[None, :], [_phi(phi)])
    expected = np.zeros(1 << n, dtype=np.complex128)
    for tok in rhs.split():
        idx, re, im = tok.split(":")
        expected[int(idx)] = complex(float(re), float(im))
    assert np.max(np.abs(out - expected)) <= 1e-15


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8])
@pytest.mark.parametrize("kind", ["R4", "R10", "D", "S8"])
def test_oracle_matches_expm(n, kind):
    """Textbook routine: product of scipy expm(i phi P) (dense, kron of 2x2 matrices)."""
    codes, angles = workloads.random_layer(n, 12 if n == 8 else 25, seed=n, kind=kind)
    rng = np.random.default_rng(n)
    psi = _rand_state(rng, n)
    got = oracle.apply(n, psi, codes, angles)
    want = dense.dense_apply(psi, codes, angles)
    assert np.max(np.abs(got - want)) <= 1e-12


def test_closed_forms():
    rng = np.random.default_rng(2)
    n = 6
    for _ in range(10):
        f = rng.integers(0, 4, size=n).astype(np.uint8)
        psi = _rand_state(rng, n)
        # phi = 0 -> identity, bitwise
        assert np.array_equal(oracle.apply(n, psi, f[None], [0.0]), psi)
        # phi = pi/2 -> i P (cos(pi/2) = 6.1e-17 in fp64)
        ip = 1j * oracle.pauli_apply(n, psi, f)
        assert np.max(np.abs(oracle.apply(n, psi, f[None], [math.pi / 2]) - ip)) <= 1e-15 * np.max(np.abs(psi)) * 4
        # phi = pi -> -I
        assert np.max(np.abs(oracle.apply(n, psi, f[None], [math.pi]) + psi)) <= 1e-15 * np.max(np.abs(psi)) * 4
    # identity string -> global phase e^{i phi}
    psi = _rand_state(rng, n)
    phi = 0.3711
    got = oracle.apply(n, psi, np.zeros((1, n), np.uint8), [phi])
    assert np.max(np.abs(got - np.exp(1j * phi) * psi)) <= 1e-15 * 8


def test_config1_unitarity_and_norm():
    """Config 1 (BASELINE.json): 10 qubits, 200 random rotations of weight 1-10; the norm is
    preserved (relative 1e-12)."""
    n = 10
    codes, angles = workloads.random_layer(n, 200, seed=1, kind="R10")
    psi = oracle.random_state(250417881, n)
    out = oracle.apply(n, psi, codes, angles)
    n0, n1 = oracle.norm(n, psi), oracle.norm(n, out)
    assert abs(n1 - n0) <= 1e-12 * n0


def test_commuting_swap_invariance():
    """Rotations with commuting strings commute (S:64-69 symplectic rule, checked here by dense
    commutators, not by the rule); anticommuting ones do not -- so the oracle is order-sensitive."""
    rng = np.random.default_rng(3)
    n = 6
    seen_comm = seen_anti = 0
    for _ in range(60):
        f1 = rng.integers(0, 4, size=n).astype(np.uint8)
        f2 = rng.integers(0, 4, size=n).astype(np.uint8)
        m1, m2 = dense.dense_pauli(f1), dense.dense_pauli(f2)
        commute = np.allclose(m1 @ m2, m2 @ m1)
        a, b = rng.uniform(-np.pi, np.pi, 2)
        psi = _rand_state(rng, n)
        ab = oracle.apply(n, psi, np.stack([f1, f2]), [a, b])
        ba = oracle.apply(n, psi, np.stack([f2, f1]), [b, a])
        d = np.max(np.abs(ab - ba))
        if commute:
            seen_comm += 1
            assert d <= 1e-13
        else:
            seen_anti += 1
            assert d > 1e-3
    assert seen_comm > 5 and seen_anti > 5


def test_inverse_layer_returns_to_zero():
    """BASELINE north_star pin: a layer followed by its inverse (reversed order, negated angles)
    returns |0> (and any state)."""
    n = 10
    codes, angles = workloads.random_layer(n, 200, seed=4, kind="R10")
    psi = _basis(n, 0)
    fwd = oracle.apply(n, psi, codes, angles)
    back = oracle.apply(n, fwd, codes[::-1], -angles[::-1])
    assert np.max(np.abs(back - psi)) <= 1e-12
    assert np.max(np.abs(fwd - psi)) > 1e-3


def test_bit_exact_basis_permutation():
    """X-only rotations at phi = pi/2 are exactly i*X (up to cos(pi/2) residue): the basis index
    is b xor x_1 xor ... xor x_k, bit-exact, with phase i^k and a component exactly +-1
    (reading R8)."""
    rng = np.random.default_rng(5)
    n = 12
    for trial in range(20):
        k = int(rng.integers(1, 41))
        b = int(rng.integers(0, 1 << n))
        codes = (rng.integers(0, 2, size=(k, n)) * 1).astype(np.uint8)  # letters I / X
        codes[codes.sum(axis=1) == 0, 0] = 1
        out = oracle.apply(n, _basis(n, b), codes, [math.pi / 2] * k)
        target = b
        for row in codes:
            for q in range(n):
                if row[q] == 1:
                    target ^= 1 << q
        big = np.flatnonzero(np.abs(out) > 0.5)
        assert big.tolist() == [target]
        ph = 1j ** k
        v = out[target]
        if ph.real != 0:
            assert v.real == ph.real and abs(v.imag) <= 1e-30
        else:
            assert v.imag == ph.imag and abs(v.real) <= 1e-30
        rest = np.delete(out, target)
        assert np.max(np.abs(rest)) <= k * 1e-16


def test_eq1_suffix_identity():
    """Eq. (1): prod_l exp(i phi_l P_l (x) Q) =
    prod_l exp(i phi_l P_l) (x) (I+Q)/2 + prod_l exp(-i phi_l P_l) (x) (I-Q)/2,
    with P_l on the lower qubits and Q on the upper ones."""
    rng = np.random.default_rng(6)
    n_lo, n_hi = 4, 2
    n = n_lo + n_hi
    for _ in range(5):
        L = 6
        lo = rng.integers(0, 4, size=(L, n_lo)).astype(np.uint8)
        q = rng.integers(0, 4, size=n_hi).astype(np.uint8)
        full = np.concatenate([lo, np.repeat(q[None], L, 0)], axis=1)  # upper qubits = high bits
        phis = rng.uniform(-np.pi, np.pi, L)
        psi = _rand_state(rng, n)
        lhs = oracle.apply(n, psi, full, phis)
        up = dense.dense_layer(lo, phis)
        um = dense.dense_layer(lo, -phis)
        qm = dense.dense_pauli(q)
        eye = np.eye(1 << n_hi)
        # index = lower bits + 2^n_lo * upper bits  ->  kron(upper, lower)
        rhs_op = np.kron((eye + qm) / 2, up) + np.kron((eye - qm) / 2, um)
        assert np.max(np.abs(lhs - rhs_op @ psi)) <= 1e-12


def test_expectation_matches_dense():
    rng = np.random.default_rng(7)
    n = 6
    psi = _rand_state(rng, n)
    codes = rng.integers(0, 4, size=(15, n)).astype(np.uint8)
    coeffs = rng.standard_normal(15)
    got = oracle.expectation(n, psi, codes, coeffs)
    want = sum(c * np.vdot(psi, dense.dense_pauli(f) @ psi).real for f, c in zip(codes, coeffs))
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    assert abs(oracle.norm(n, psi) - np.vdot(psi, psi).real) <= 1e-12 * np.vdot(psi, psi).real
    phi = _rand_state(rng, n)
    ip = oracle.inner(n, psi, phi)
    assert abs(ip - np.vdot(psi, phi)) <= 1e-12 * np.sqrt(np.vdot(psi, psi).real * np.vdot(phi, phi).real)


# ---------------------------------------------------------------- coset oracle

def test_coset_oracle_equals_full_restriction():
    """Coset restriction (P|i> ~ |i xor p1>) reproduces the full oracle on the coset."""
    n = 11
    rng = np.random.default_rng(8)
    codes = np.zeros((30, n), np.uint8)
    nd_positions = [0, 3, 4, 7, 10]
    for l in range(30):
        row = rng.integers(0, 2, size=n).astype(np.uint8) * 3  # I/Z everywhere
        for p in nd_positions:
            if rng.integers(0, 3) == 0:
                row[p] = rng.integers(1, 3)  # X or Y
        codes[l] = row
    angles = rng.uniform(-np.pi, np.pi, 30)
    psi = oracle.random_state(99, n)
    full = oracle.apply(n, psi, codes, angles)
    xs = [sum(1 << q for q in range(n) if row[q] in (1, 2)) for row in codes]
    for i0 in (0, 2, 5 | 2 | 256):
        mem = oracle.coset_members(n, i0, xs)
        got = oracle.apply_coset(n, mem, psi[mem.astype(np.int64)], codes, angles)
        assert np.max(np.abs(got - full[mem.astype(np.int64)])) <= 1e-13


# ---------------------------------------------------------------- input generator (DESIGN.md Input recipe)

def test_generator_matches_published_splitmix64():
    """Output k of our counter generator is output k+1 of Vigna's splitmix64; published test
    vector for seed 1234567 (the xoshiro reference seeding), and seed 0 -> 0xe220a8397b1dcdaf."""
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
            16408922859458223821]
    assert [oracle.generator_raw(1234567, k) for k in range(5)] == want
    assert oracle.generator_raw(0, 0) == 0xE220A8397B1DCDAF


def test_random_amplitudes_exact_grid():
    a = oracle.random_amplitudes(250417881, 1000, 4096)
    v = np.concatenate([a.real, a.imag])
    assert np.all(v >= -1.0) and np.all(v < 1.0)
    assert np.all((v + 1.0) * 2.0 ** 52 == np.round((v + 1.0) * 2.0 ** 52))
    # counter-based: any window regenerates bitwise
    b = oracle.random_amplitudes(250417881, 1000 + 17, 100)
    assert np.array_equal(a[17:117], b)
    k = 2 * 1000
    assert a[0].real == (oracle.generator_raw(250417881, k) >> 11) * 2.0 ** -52 - 1.0
