"""GPU parity tests (``-m gpu``): the CUDA path, called through the C ABI, against the CPU oracle.

Tolerances (BASELINE.json north_star): max |a_gpu - a_oracle| <= 1e-10 for fp64 and <= 1e-4 for
fp32 after up to 1000 rotations, on unnormalised O(1) amplitudes (reading R10); index
and mask handling bit-exact (basis permutations under X-only rotations at phi = pi/2, R8).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads
import paper_2504_17881_b200 as P
from paper_2504_17881_b200 import ps

pytestmark = pytest.mark.gpu

SEED = 250417881
TOL = {"c128": 1e-10, "c64": 1e-4}

_oracle_cache: dict = {}


def _want(n, kind, count, seed):
    key = (n, kind, count, seed)
    if key not in _oracle_cache:
        codes, ang = workloads.random_layer(n, count, seed=seed, kind=kind)
        _oracle_cache[key] = (codes, ang, oracle.apply(n, oracle.random_state(SEED, n), codes, ang))
    return _oracle_cache[key]


def _run(n, dtype, codes, ang, fusion=2, tile_bits=None, init="random", specialize=None):
    x, z = P.pauli_encode_codes(codes)
    with P.State(n, dtype) as st:
        st.set_option(ps.OPT_FUSION, fusion)
        if specialize is not None:
            st.set_option(ps.OPT_SPECIALIZE, specialize)
        if tile_bits:
            st.set_option(ps.OPT_TILE_BITS, tile_bits)
        if init == "random":
            st.init_random(SEED)
        else:
            st.init_basis(init)
        st.apply_rotations(x, z, ang)
        out = st.get_amplitudes()
        stats = st.stats()
    return out, stats


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("fusion", [0, 1, 2])
def test_config1(dtype, fusion):
    """BASELINE config 1: 10 qubits, 200 random rotations of weight 1-10."""
    codes, ang, want = _want(10, "R10", 200, 1)
    got, _ = _run(10, dtype, codes, ang, fusion=fusion, tile_bits=6)
    assert np.max(np.abs(got - want)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind,n,count,tb", [("R10", 12, 400, 8), ("S8", 13, 640, 9), ("LOW", 12, 300, 11),
                                             ("D", 11, 200, 7), ("R4", 14, 500, 10)])
def test_specialised_kernel_identical(dtype, kind, n, count, tb):
    """The specialised tile kernel (compile-time sign-pattern cases, PS_OPT_SPECIALIZE=2) performs
    the same operations as the generic one: bitwise-identical results, both at the oracle.  A
    quarter of the angles sit at +-pi/2 or +-pi/4 so SFORM and CFORM records mix in one pass."""
    codes, ang, _ = _want(n, kind, count, 7)
    ang = ang.copy()
    rng = np.random.default_rng(5)
    pick = rng.random(count) < 0.25
    ang[pick] = rng.choice([np.pi / 2, -np.pi / 2, np.pi / 4, -3 * np.pi / 4], size=int(pick.sum()))
    want = oracle.apply(n, oracle.random_state(SEED, n), codes, ang)
    outs = [_run(n, dtype, codes, ang, tile_bits=tb, specialize=sp)[0] for sp in (0, 1, 2)]
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[0], outs[1])
    assert np.max(np.abs(outs[2] - want)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind,n,count,tb", [("R10", 12, 400, 8), ("S8", 13, 640, 9), ("R4", 14, 500, 10),
                                             ("D", 11, 200, 7)])
def test_param_block_records_identical(dtype, kind, n, count, tb):
    """Records read from the launch's parameter block (PS_OPT_TILE_TUNE bit 10, the default) and
    from global memory (bit 10 clear), with or without the shared-memory prefetch of the next
    tile (bit 11), drive the same arithmetic: bitwise-identical results."""
    codes, ang, want = _want(n, kind, count, 11)
    x, z = P.pauli_encode_codes(codes)
    outs = []
    for tune in (512, 1536, 512 | 2048, 1536 | 2048):
        with P.State(n, dtype) as st:
            st.set_option(ps.OPT_TILE_BITS, tb)
            st.set_option(ps.OPT_TILE_TUNE, tune)
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            outs.append(st.get_amplitudes())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    assert np.max(np.abs(outs[1] - want)) <= TOL[dtype]


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 14, 17])
@pytest.mark.parametrize("kind", ["R4", "R10", "D", "S8", "LOW"])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("tile_bits", [None, 6])
def test_sizes_and_kinds(n, kind, dtype, tile_bits):
    count = 1000 if n <= 14 else 300
    codes, ang, want = _want(n, kind, count, 2)
    got, stats = _run(n, dtype, codes, ang, fusion=2, tile_bits=tile_bits)
    err = np.max(np.abs(got - want))
    assert err <= TOL[dtype], (err, stats["launches"])


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["R10", "LOW", "S8", "R4"])
def test_fusion_levels_agree(dtype, kind):
    """Fusion changes traffic and rounding order only: K1 one-rotation passes and same-x runs are
    bitwise identical (same per-pair arithmetic); tile passes (deferred-scale arithmetic) agree
    to a few ulps per rotation (R9)."""
    n = 16
    codes, ang = workloads.random_layer(n, 400, seed=3, kind=kind)
    outs = {}
    for fusion, tb, mode in ((0, None, 2), (1, None, 2), (2, None, 2), (2, 7, 2), (2, None, 0), (2, 9, 1), (2, None, 3)):
        x, z = P.pauli_encode_codes(codes)
        with P.State(n, dtype) as st:
            st.set_option(ps.OPT_FUSION, fusion)
            if tb:
                st.set_option(ps.OPT_TILE_BITS, tb)
            st.set_option(ps.OPT_TILE_TMA, mode)
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            outs[(fusion, tb, mode)] = st.get_amplitudes()
    ref = outs[(0, None, 2)]
    if kind in ("S8",):
        assert np.array_equal(outs[(1, None, 2)].view(np.uint8), ref.view(np.uint8))
    # every fusion level / tile variant within the north_star tolerance of the oracle (so any two
    # within twice that), and fp64 variants within 1e-12 of each other (R9: rounding order only)
    want = oracle.apply(n, oracle.random_state(SEED, n), codes, ang)
    for key, o in outs.items():
        assert np.max(np.abs(o - want)) <= TOL[dtype], key
        if dtype == "c128":
            assert np.max(np.abs(o - ref)) <= 1e-12, key


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("fusion", [0, 2])
def test_bit_exact_basis_permutation(dtype, fusion):
    """X-only rotations at phi = pi/2 from |b>: the index is b xor x_1 ... xor x_k bit-exactly,
    the surviving amplitude is i^k with a component exactly +-1 (R8)."""
    rng = np.random.default_rng(5)
    n = 14
    for trial in range(6):
        k = int(rng.integers(1, 41))
        b = int(rng.integers(0, 1 << n))
        codes = rng.integers(0, 2, size=(k, n)).astype(np.uint8)
        codes[codes.sum(axis=1) == 0, 0] = 1
        got, _ = _run(n, dtype, codes, [math.pi / 2] * k, fusion=fusion, init=b)
        target = b
        for row in codes:
            for q in range(n):
                if row[q]:
                    target ^= 1 << q
        big = np.flatnonzero(np.abs(got) > 0.5)
        assert big.tolist() == [target]
        ph = 1j ** k
        v = got[target]
        if ph.real != 0:
            assert v.real == ph.real
        else:
            assert v.imag == ph.imag
        rest_tol = k * (1e-16 if dtype == "c128" else 1e-7)
        assert np.max(np.abs(np.delete(got, target))) <= rest_tol


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_closed_forms(dtype):
    n = 12
    rng = np.random.default_rng(6)
    codes = rng.integers(0, 4, size=(20, n)).astype(np.uint8)
    with P.State(n, dtype) as st:
        st.init_random(SEED)
        a0 = st.get_amplitudes()
        x, z = P.pauli_encode_codes(codes)
        st.apply_rotations(x, z, np.zeros(20))
        assert np.array_equal(st.get_amplitudes(), a0)  # phi = 0 -> identity, bitwise
        st.apply_rotations([0], [0], [0.37])  # identity string -> e^{i phi}
        assert np.max(np.abs(st.get_amplitudes() - np.exp(0.37j) * a0)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_init_random_matches_generator(dtype):
    n = 15
    with P.State(n, dtype) as st:
        st.init_random(SEED)
        got = st.get_amplitudes()
    want = oracle.random_state(SEED, n)
    if dtype == "c128":
        assert np.array_equal(got, want)
    else:
        assert np.array_equal(got, want.astype(np.complex64))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_norm_expectation_inner(dtype):
    n = 13
    codes, ang, psi = _want(n, "R10", 300, 4)
    hcodes = np.random.default_rng(7).integers(0, 4, size=(40, n)).astype(np.uint8)
    hcodes[:10, :] = np.where(hcodes[:10, :] % 2 == 1, 3, 0)  # some diagonal terms
    hcodes[10:14] = hcodes[14]  # shared x groups
    coeffs = np.random.default_rng(8).standard_normal(40)
    x, z = P.pauli_encode_codes(codes)
    hx, hz = P.pauli_encode_codes(hcodes)
    tol = 1e-10 if dtype == "c128" else 2e-3
    with P.State(n, dtype) as st, P.State(n, dtype) as st2:
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        nrm = oracle.norm(n, psi)
        assert abs(st.norm() - nrm) <= tol * nrm
        e_want = oracle.expectation(n, psi, hcodes, coeffs)
        assert abs(st.expectation(hx, hz, coeffs) - e_want) <= tol * max(1.0, nrm)
        st2.init_random(SEED + 1)
        ip_want = oracle.inner(n, psi, oracle.random_state(SEED + 1, n))
        assert abs(st.inner(st2) - ip_want) <= tol * nrm
        st.normalize()
        assert abs(st.norm() - 1.0) <= (1e-12 if dtype == "c128" else 1e-5)


def test_set_get_and_errors():
    n = 9
    rng = np.random.default_rng(9)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    with P.State(n, "c128") as st:
        st.set_state(psi)
        assert np.array_equal(st.get_amplitudes(), psi)
        assert np.array_equal(st.get_amplitudes(100, 50), psi[100:150])
        st.set_state(psi[:7] * 2, first=500)
        psi2 = psi.copy()
        psi2[500:507] = psi[:7] * 2
        assert np.array_equal(st.get_amplitudes(), psi2)
        # validation failures leave the state unchanged
        with pytest.raises(P.PsError) as ei:
            st.apply_rotations([1, 1 << n], [0, 0], [0.1, 0.2])
        assert ei.value.code == -2
        with pytest.raises(P.PsError) as ei:
            st.apply_rotations([1], [0], [float("nan")])
        assert ei.value.code == -1
        with pytest.raises(P.PsError):
            st.get_amplitudes(510, 10)
        with pytest.raises(P.PsError):
            st.init_basis(1 << n)
        assert np.array_equal(st.get_amplitudes(), psi2)


def test_torch_memory_and_stream():
    import torch
    n = 12
    codes, ang, want = _want(n, "R10", 200, 10)
    x, z = P.pauli_encode_codes(codes)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with P.State(n, "c128", torch_memory=True) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            t = st._tensor.view(torch.complex128).cpu().numpy()
    assert np.max(np.abs(t - want)) <= 1e-10


def test_stats_and_profile():
    n = 14
    codes, ang = workloads.random_layer(n, 100, seed=11, kind="R10")
    x, z = P.pauli_encode_codes(codes)
    with P.State(n, "c128") as st:
        st.set_option(ps.OPT_PROFILE, 1)
        st.init_random(SEED)
        st.reset_stats()
        st.apply_rotations(x, z, ang)
        st.synchronize()
        s = st.stats()
    assert s["rotations"] == 100
    assert sum(s["rotations_by"].values()) == 100
    assert s["passes"] == sum(s["launches"][k] for k in ("stream", "tile", "coset"))
    assert sum(s["kernel_ms"][k] for k in ("stream", "tile", "coset")) > 0


# ------------------------------------------------------------------ full size (BASELINE config 2)

def test_30q_inverse_layer_and_norm():
    """30 qubits fp64 (16 GiB), the bench workload and launch configuration: a 1000-rotation R10
    layer followed by its inverse returns the seeded initial amplitudes, which the oracle
    regenerates one by one at sampled indices; the norm is preserved."""
    n = 30
    codes, ang = workloads.random_layer(n, 1000, seed=0, kind="R10")
    x, z = P.pauli_encode_codes(codes)
    rng = np.random.default_rng(12)
    sample = np.unique(np.concatenate([rng.integers(0, 1 << n, 2000), [0, (1 << n) - 1]]))
    with P.State(n, "c128", torch_memory=True) as st:
        st.init_random(SEED)
        n0 = st.norm()
        st.apply_rotations(x, z, ang)
        n1 = st.norm()
        st.apply_rotations(x[::-1], z[::-1], -ang[::-1])
        got = np.array([st.get_amplitudes(int(i), 1)[0] for i in sample[:300]])
    want = np.array([oracle.random_amplitudes(SEED, int(i), 1)[0] for i in sample[:300]])
    assert abs(n1 - n0) <= 1e-12 * n0
    assert np.max(np.abs(got - want)) <= 1e-10


def test_30q_coset_oracle():
    """30 qubits with X-support restricted to 16 qubits (Z anywhere): every coset of the X-span is
    invariant, so the coset oracle computes those amplitudes exactly (R13)."""
    n = 30
    rng = np.random.default_rng(13)
    xq = np.sort(rng.choice(n, 16, replace=False))
    L = 200
    codes = rng.integers(0, 2, size=(L, n)).astype(np.uint8) * 3
    for l in range(L):
        w = rng.integers(1, 6)
        pos = rng.choice(xq, w, replace=False)
        codes[l, pos] = rng.integers(1, 3, size=w)
    ang = rng.uniform(-np.pi, np.pi, L)
    x, z = P.pauli_encode_codes(codes)
    with P.State(n, "c128", torch_memory=True) as st:
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        for i0 in (0, int(rng.integers(0, 1 << n))):
            mem = oracle.coset_members(n, i0, x)
            init = np.array([oracle.random_amplitudes(SEED, int(m), 1)[0] for m in mem])
            want = oracle.apply_coset(n, mem, init, codes, ang)
            sel = rng.choice(len(mem), 200, replace=False)
            got = np.array([st.get_amplitudes(int(mem[s]), 1)[0] for s in sel])
            assert np.max(np.abs(got - want[sel])) <= 1e-10


# ------------------------------------------------------------------ NEXT-3: RPE signals

def test_rpe_signal_matches_oracle():
    """Z_m = <psi|e^{i delta H~ 2^m}|psi> for the second-order partially randomized
    method, through ps_apply_rotations + ps_inner, against the oracle applying the same stream."""
    from paper_2504_17881_b200 import formulas, rpe
    n = 10
    codes, _ = workloads.random_layer(n, 80, seed=21, kind="R10")
    codes = np.unique(codes, axis=0)
    coeffs = np.random.default_rng(21).uniform(-1, 1, len(codes))
    x, z = P.pauli_encode_codes(codes)
    H = formulas.from_masks(n, x, z, coeffs)
    HD, HR = formulas.split_deterministic(H, 30)
    delta = 0.3
    r = formulas.sample_count(HR.lam, delta, 3)
    psi0 = oracle.random_state(SEED, n)
    psi0 = psi0 / np.sqrt(oracle.norm(n, psi0))
    for m in (0, 2, 3):
        got = rpe.signal(n, HD, HR, delta, m, r, seed=7)
        sx, sz, sa = formulas.evolution_stream(HD, HR, delta, 2 ** m, r, 7)
        want = oracle.inner(n, psi0, oracle.apply_masks(n, psi0, sx, sz, sa))
        assert abs(got - want) <= 1e-10
        assert abs(got) <= 1 + 1e-9


def test_rpe_eigenstate_signal():
    """H = {h Z}, psi = |1> -> Z_m = e^{-i delta h 2^m} exactly (up to rounding)."""
    from paper_2504_17881_b200 import formulas, rpe
    H = formulas.from_masks(1, [0], [1], [0.7])
    empty = H.take([])
    for m in (0, 3, 6):
        got = rpe.signal(1, H, empty, 0.4, m, 0, seed=1, init=1)
        assert abs(got - np.exp(-1j * 0.4 * 0.7 * 2 ** m)) <= 1e-12


def test_option_validation_and_restore():
    with P.State(10, "c128") as st:
        for opt, bad in ((ps.OPT_FUSION, 5), (ps.OPT_TILE_BITS, 14), (ps.OPT_TILE_BITS, 3), (ps.OPT_CHUNK_BYTES, 1000),
                         (ps.OPT_MAX_PASS_ROTS, 0), (ps.OPT_TILE_TMA, 7), (ps.OPT_LAYOUT, 3), (ps.OPT_SPECIALIZE, 3), (ps.OPT_OVERLAP, 3),
                         (ps.OPT_OVERLAP, 5 << 16), (ps.OPT_SWAP_CTAS, 1 << 20), (99, 1)):
            with pytest.raises(P.PsError) as ei:
                st.set_option(opt, bad)
            assert ei.value.code == -1
        st.init_random(SEED)
        a0 = st.get_amplitudes()
        st.set_option(ps.OPT_TILE_BITS, 5)  # valid options leave the state alone
        assert np.array_equal(st.get_amplitudes(), a0)


def test_create_entry_points_directly():
    """ps_create and ps_create_dist called through the C ABI (not via the State class): |0> after
    creation, a layer against the oracle, and every argument check of include/ps.h."""
    import ctypes
    L = P.lib()
    h = ctypes.c_void_p()
    assert L.ps_create(10, ps.C128, ctypes.byref(h)) == 0
    nq, nl, rk, wd, dt = (ctypes.c_int() for _ in range(5))
    assert L.ps_info(h, ctypes.byref(nq), ctypes.byref(nl), ctypes.byref(rk), ctypes.byref(wd), ctypes.byref(dt), None) == 0
    assert (nq.value, nl.value, rk.value, wd.value, dt.value) == (10, 10, 0, 1, ps.C128)
    out = np.zeros(1 << 10, np.complex128)
    assert L.ps_get_amplitudes(h, 0, 1 << 10, out.ctypes.data_as(ctypes.c_void_p)) == 0
    assert out[0] == 1 and np.count_nonzero(out) == 1
    codes, ang, want = _want(10, "R10", 200, 1)
    x, z = P.pauli_encode_codes(codes)
    assert L.ps_init_random(h, SEED) == 0
    assert L.ps_apply_rotations(h, x.ctypes.data_as(ctypes.c_void_p), z.ctypes.data_as(ctypes.c_void_p),
                                np.ascontiguousarray(ang).ctypes.data_as(ctypes.c_void_p), len(ang)) == 0
    assert L.ps_get_amplitudes(h, 0, 1 << 10, out.ctypes.data_as(ctypes.c_void_p)) == 0
    assert np.max(np.abs(out - want)) <= 1e-10
    assert L.ps_destroy(h) == 0
    h2 = ctypes.c_void_p()
    assert L.ps_create_dist(9, ps.C64, 0, 1, None, ctypes.byref(h2)) == 0  # world 1: no NCCL id needed
    assert L.ps_info(h2, ctypes.byref(nq), ctypes.byref(nl), None, ctypes.byref(wd), ctypes.byref(dt), None) == 0
    assert (nq.value, nl.value, wd.value, dt.value) == (9, 9, 1, ps.C64)
    assert L.ps_destroy(h2) == 0
    bad = ctypes.c_void_p()
    assert L.ps_create(0, ps.C128, ctypes.byref(bad)) == -1
    assert L.ps_create(63, ps.C128, ctypes.byref(bad)) == -1
    assert L.ps_create(10, 7, ctypes.byref(bad)) == -1
    assert L.ps_create_dist(10, ps.C128, 0, 3, None, ctypes.byref(bad)) == -1   # world not a power of two
    assert L.ps_create_dist(10, ps.C128, 2, 2, None, ctypes.byref(bad)) == -1   # rank >= world
    assert L.ps_create_dist(10, ps.C128, 0, 2, None, ctypes.byref(bad)) == -1   # world > 1 without an id
    assert L.ps_create_dist(1, ps.C128, 0, 2, None, ctypes.byref(bad)) == -1    # no local qubit left
    assert L.ps_create(10, ps.C128, None) == -1
    assert not bad.value
