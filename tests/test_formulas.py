"""NEXT-3 product formulas (host builders) pinned against textbook matrix exponentials (dense,
n <= 5) and the oracle; RPE estimation on synthetic signals.  CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.linalg

import oracle
from oracle import dense
import workloads
from paper_2504_17881_b200 import formulas, rpe
import paper_2504_17881_b200 as P


def _ham(n, terms, seed):
    """Random Hamiltonian: distinct R10-style strings, coefficients in [-1, 1]."""
    codes, _ = workloads.random_layer(n, terms, seed=seed, kind="R10")
    codes = np.unique(codes, axis=0)
    coeffs = np.random.default_rng(seed).uniform(-1, 1, len(codes))
    x, z = P.pauli_encode_codes(codes)
    return formulas.from_masks(n, x, z, coeffs), codes


def _dense_h(H):
    f = oracle.decode_masks(H.n, H.x, H.z)
    return sum(h * dense.dense_pauli(row) for h, row in zip(H.h, f))


def _dense_stream(n, x, z, a):
    return dense.dense_layer(oracle.decode_masks(n, x, z), a)


def test_trotter2_is_a_palindrome_with_exact_inverse():
    """trotter2(delta) followed by trotter2(-delta) is the identity."""
    H, _ = _ham(4, 40, 1)
    x, z, a = formulas.trotter2_step(H, 0.37)
    assert np.array_equal(x, x[::-1]) and np.array_equal(z, z[::-1])
    psi = oracle.random_state(3, 4)
    xi, zi, ai = formulas.trotter2_step(H, -0.37)
    out = oracle.apply_masks(4, oracle.apply_masks(4, psi, x, z, a), xi, zi, ai)
    assert np.max(np.abs(out - psi)) <= 1e-13


@pytest.mark.parametrize("order,ratio", [(1, 4.0), (2, 8.0)])
def test_trotter_error_exponents(order, ratio):
    """||U_k(delta) - e^{i delta H}|| = O(delta^{k+1}): halving delta divides the
    one-step error by ~2^{k+1} (textbook matrix exponential as the reference)."""
    H, _ = _ham(4, 40, 2)
    Hd = _dense_h(H)
    errs = []
    for d in (0.02, 0.01):
        x, z, a = (formulas.trotter1_step if order == 1 else formulas.trotter2_step)(H, d)
        U = _dense_stream(4, x, z, a)
        errs.append(np.linalg.norm(U - scipy.linalg.expm(1j * d * Hd), 2))
    assert abs(errs[0] / errs[1] - ratio) < 0.15 * ratio


def test_qdrift_single_term_is_exact():
    """a single-term H_R gives r equal rotations composing to e^{i t h P} exactly."""
    H = formulas.from_masks(3, [5], [4], [-0.7])
    x, z, a = formulas.qdrift_stage(H, 0.9, 7, seed=11, counter=0)
    assert len(a) == 7 and np.allclose(a, np.sign(-0.7) * 0.7 * 0.9 / 7)
    U = _dense_stream(3, x, z, a)
    f = oracle.decode_masks(3, [5], [4])
    assert np.max(np.abs(U - scipy.linalg.expm(1j * 0.9 * -0.7 * dense.dense_pauli(f[0])))) <= 1e-13


def test_qdrift_sampling_frequencies_and_replay():
    H, _ = _ham(6, 60, 3)
    r = 40000
    x, z, a = formulas.qdrift_stage(H, 1.0, r, seed=5, counter=0)
    keys = {(int(xx), int(zz)): k for k, (xx, zz) in enumerate(zip(H.x, H.z))}
    counts = np.zeros(len(H))
    for xx, zz in zip(x, z):
        counts[keys[(int(xx), int(zz))]] += 1
    p = np.abs(H.h) / H.lam
    chi2 = np.sum((counts - r * p) ** 2 / (r * p))
    assert chi2 < len(H) + 6 * math.sqrt(2 * len(H))  # ~6 sigma
    assert np.allclose(np.abs(a), H.lam / r)
    x2, z2, a2 = formulas.qdrift_stage(H, 1.0, r, seed=5, counter=0)
    assert np.array_equal(x, x2) and np.array_equal(a, a2)  # counter-based replay
    x3, _, _ = formulas.qdrift_stage(H, 1.0, r, seed=5, counter=r)
    assert not np.array_equal(x, x3)


def test_sample_count_examples():
    """S:461-465 examples for r = ceil(kappa lambda_R^2 delta^2 2^M), kappa = delta/(0.2 pi)."""
    assert formulas.sample_count(0.0, 0.3, 4) == 0
    assert formulas.sample_count(1.0, 0.2 * math.pi, 0) == 1
    a = 0.31 / (0.2 * math.pi) * 1.7 ** 2 * 0.31 ** 2
    assert formulas.sample_count(1.7, 0.31, 5) == math.ceil(a * 32)
    assert formulas.sample_count(1.7, 0.31, 6) == math.ceil(a * 64)


def test_partially_randomized_structure():
    H, _ = _ham(5, 60, 4)
    HD, HR = formulas.split_deterministic(H, 20)
    assert len(HD) + len(HR) == len(H)
    assert np.abs(HD.h).min() >= np.abs(HR.h).max()
    x, z, a = formulas.partially_randomized_step(HD, HR, 0.2, 9, seed=1, step=0)
    assert len(a) == 2 * len(HD) + 2 * 9
    # lambda_R = 0 -> second-order Trotter on H_D
    empty = H.take([])
    x0, z0, a0 = formulas.partially_randomized_step(HD, empty, 0.2, 0, seed=1, step=0)
    xt, zt, at = formulas.trotter2_step(HD, 0.2)
    assert np.array_equal(x0, xt) and np.array_equal(a0, at)
    with pytest.raises(ValueError):
        formulas.partially_randomized_step(HD, HR, 0.2, 0, seed=1, step=0)


def test_rpe_estimate_synthetic():
    """noiseless signals Z_m = e^{i phi 2^m}."""
    for phi in (0.3, 0.0, math.pi - 0.01, -2.0):
        zs = [complex(math.cos(phi * 2 ** m), math.sin(phi * 2 ** m)) for m in range(11)]
        est = rpe.estimate(zs, 1.0)
        d = (est - phi + math.pi) % (2 * math.pi) - math.pi
        assert abs(d) <= math.pi / 2 ** 11
