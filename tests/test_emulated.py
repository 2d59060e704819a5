"""Multi-rank path on ONE GPU (``-m gpu``): ps_create_emulated runs G virtual ranks -- G slices of
one device buffer, each with its own SPMD plan (per-rank signs, exchange sides), the same kernels
as real ranks (P2P swap, full exchange, local transpositions, mirror butterfly, the fused
exchange + tile kernel), peer pointers into the other slices -- so the driver's single-GPU run
checks the partitioned path (e; NEXT-2; NEXT-4) against the CPU oracle.

P:357-430 (partitioned layout, pairwise exchange k <-> k xor gx), P:403-404 (diagonal upper part),
P:126-148 Eq. (1) (one exchange per run), P:458-474 (mirror + butterfly), P:122-125 / P:676-680
(exchange overlap).  Tolerances as in test_gpu_parity.py (BASELINE.json north_star).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads
import paper_2504_17881_b200 as P
from paper_2504_17881_b200 import ps

pytestmark = pytest.mark.gpu

SEED = 250417881
TOL = {"c128": 1e-10, "c64": 1e-4}
_cache: dict = {}


def layer_with_global(n, count, seed, world):
    """R10 layer plus rotations with X on the top (global) qubits, runs sharing an upper X-part
    and Z-only global terms (the same recipe as tests/mp_worker.py)."""
    codes, ang = workloads.random_layer(n, count, seed=seed, kind="R10")
    rng = np.random.default_rng(seed)
    m = world.bit_length() - 1
    for l in range(0, count, 7):
        q = n - 1 - int(rng.integers(0, max(1, m)))
        codes[l, q] = rng.integers(1, 4)
    for l in range(3, count, 11):
        codes[l:l + 4, n - 1] = 1
    return codes, ang


def _want(n, count, seed, world):
    key = (n, count, seed, world)
    if key not in _cache:
        codes, ang = layer_with_global(n, count, seed, world)
        _cache[key] = (codes, ang, oracle.apply(n, oracle.random_state(SEED, n), codes, ang))
    return _cache[key]


def _emu(n, world, dtype="c128", **opts):
    st = P.State(n, dtype, emulate=world)
    for k, v in opts.items():
        st.set_option(getattr(ps, "OPT_" + k.upper()), v)
    return st


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("layout", [0, 1, 2])
@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("fusion,tile_bits", [(0, 6), (1, 6), (2, 6), (2, 0)])
def test_emulated_ranks_against_oracle(world, layout, fused, fusion, tile_bits):
    n = 11
    codes, ang, want = _want(n, 300, 41, world)
    x, z = P.pauli_encode_codes(codes)
    opts = dict(layout=layout, fused_exchange=fused, fusion=fusion, chunk_bytes=4096)
    if tile_bits:
        opts["tile_bits"] = tile_bits
    with _emu(n, world, **opts) as st:
        st.init_random(SEED)
        h = len(ang) // 2
        st.apply_rotations(x[:h], z[:h], ang[:h])  # the lazy layout persists across the two calls
        nrm_mid = st.norm()
        st.apply_rotations(x[h:], z[h:], ang[h:])
        got = st.get_amplitudes()
        stats = st.stats()
    n0 = oracle.norm(n, oracle.random_state(SEED, n))
    assert abs(nrm_mid - n0) <= 1e-12 * n0
    assert np.max(np.abs(got - want)) <= 1e-10, stats
    if world > 1:
        assert stats["exchanges"] > 0


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("cap", [0, 1, 3])
def test_fused_exchange_identical_to_swap(world, dtype, cap):
    """The fused exchange + tile kernel performs the same per-element arithmetic as swap-then-pass:
    bitwise-identical amplitudes, with many tiles per CTA (grid cap) so the per-tile flag protocol
    runs several rounds, and tiles where 2^ell is a free bit (partner tile tau ^ dtau) or inside the
    tile space (dtau = 0)."""
    n = 14
    codes, ang, want = _want(n, 400, 42, world)
    x, z = P.pauli_encode_codes(codes)
    outs = []
    for fused in (0, 1):
        with _emu(n, world, dtype, fused_exchange=fused, tile_bits=8, grid_cap=cap) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            outs.append(st.get_amplitudes())
    assert np.array_equal(outs[0], outs[1])
    assert np.max(np.abs(outs[1] - want)) <= TOL[dtype]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_full_exchange_fallback(world):
    """Rotations whose local X-part covers every local bit (no free pivot): chunked full exchange
    (two phases over the virtual ranks)."""
    m = world.bit_length() - 1
    n = m + 3
    words = ["X" * n, "Y" + "X" * (n - 2) + "Z", "Z" * n, ("XY" * n)[:n], "I" + "X" * (n - 1)]
    codes = oracle.words_to_factors(words)
    x, z = P.pauli_encode_codes(codes)
    ang = np.array([0.3, -1.2, 0.7, 2.0, -0.5])
    for layout in (0, 1):
        with _emu(n, world, layout=layout, chunk_bytes=4096) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
        assert np.max(np.abs(got - oracle.apply(n, oracle.random_state(SEED, n), codes, ang))) <= 1e-12


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_jw_trotter_expectation_norm_inner(world, dtype):
    """A JW-shaped first-order Trotter step (x-major order for this world), then
    the Hamiltonian's expectation (global-X terms need exchanges), the norm and an overlap."""
    n = 14
    m = world.bit_length() - 1
    hc, hco = workloads.jw_hamiltonian(n, 2000, 27.0, seed=1, n_local=n - m)
    ang = workloads.trotter1_angles(hco, 0.5)
    x, z = P.pauli_encode_codes(hc)
    want = oracle.apply(n, oracle.random_state(SEED, n), hc, ang)
    tol = TOL[dtype]
    with _emu(n, world, dtype) as st, _emu(n, world, dtype) as st2:
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        got = st.get_amplitudes()
        e = st.expectation(x, z, hco)
        nrm = st.norm()
        st2.init_random(SEED + 1)
        ip = st.inner(st2)
    scale = oracle.norm(n, want)
    assert np.max(np.abs(got - want)) <= tol
    etol = 1e-9 if dtype == "c128" else 2e-3
    assert abs(e - oracle.expectation(n, want, hc, hco)) <= etol * scale
    assert abs(nrm - scale) <= etol * scale
    assert abs(ip - oracle.inner(n, want, oracle.random_state(SEED + 1, n))) <= etol * scale


@pytest.mark.parametrize("world", [2, 4])
def test_expectation_without_free_pivot(world):
    """Terms whose local X-part covers every local bit and that have X on a global qubit: the
    read-only full exchange (k_expect_cross), against the oracle."""
    m = world.bit_length() - 1
    n = m + 4
    rng = np.random.default_rng(43)
    words = ["X" * n, "Y" * n, "Z" + "X" * (n - 1), "XZ" * (n // 2) + "X" * (n % 2)]
    words = [w[:n - 1] + ("Y" if i % 2 else "X") for i, w in enumerate(words)] + ["X" * (n - 1) + "Z"]
    words = [("X" * (n - m)) + "".join(rng.choice(list("XYZ"), m)) for _ in range(3)] + words
    codes = oracle.words_to_factors(words)
    coeffs = rng.standard_normal(len(words))
    x, z = P.pauli_encode_codes(codes)
    psi = oracle.random_state(SEED, n)
    with _emu(n, world, chunk_bytes=4096) as st:
        st.init_random(SEED)
        e = st.expectation(x, z, coeffs)
    assert abs(e - oracle.expectation(n, psi, codes, coeffs)) <= 1e-12 * oracle.norm(n, psi)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["R10", "R4", "S8"])
def test_emulated_large_default_options(world, dtype, kind):
    """22 qubits, default options (2^12 tiles, fused exchange, lazy layout): the bench's
    launch configuration on the multi-rank path, full-state oracle comparison."""
    n = 22
    codes, ang = workloads.random_layer(n, 150, seed=44, kind=kind)
    key = ("L", n, kind)
    if key not in _cache:
        _cache[key] = oracle.apply(n, oracle.random_state(SEED, n), codes, ang)
    want = _cache[key]
    x, z = P.pauli_encode_codes(codes)
    with _emu(n, world, dtype) as st:
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        got = st.get_amplitudes()
        stats = st.stats()
    assert stats["exchanges"] > 0
    assert np.max(np.abs(got - want)) <= TOL[dtype], stats


def test_g_invariance_and_single_rank():
    """world = 1 emulation is a plain state; the same layer on 1, 2, 4, 8 virtual ranks agrees with
    the single-GPU run to a few ulps."""
    n = 16
    codes, ang, _ = _want(n, 300, 45, 8)
    x, z = P.pauli_encode_codes(codes)
    with P.State(n, "c128") as one:
        one.init_random(SEED)
        one.apply_rotations(x, z, ang)
        ref = one.get_amplitudes()
    for world in (1, 2, 4, 8):
        with _emu(n, world) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
        if world == 1:
            assert np.array_equal(got, ref)
        else:
            assert np.max(np.abs(got - ref)) <= 1e-12


def test_rpe_signal_emulated():
    """NEXT-3: Z_m of the partially randomized second-order method on 2 virtual ranks, vs oracle."""
    from paper_2504_17881_b200 import formulas, rpe
    n = 12
    codes, _ = workloads.random_layer(n, 120, seed=31, kind="R10")
    codes = np.unique(codes, axis=0)
    coeffs = np.random.default_rng(31).uniform(-1, 1, len(codes))
    hx, hz = P.pauli_encode_codes(codes)
    H = formulas.from_masks(n, hx, hz, coeffs)
    HD, HR = formulas.split_deterministic(H, 40, n_local=n - 1)
    r = formulas.sample_count(HR.lam, 0.3, 2)
    psi0 = oracle.random_state(SEED, n)
    psi0 = psi0 / np.sqrt(oracle.norm(n, psi0))
    for m in (0, 2):
        zm = rpe.signal(n, HD, HR, 0.3, m, r, seed=3, emulate=2)
        sx, sz, sa = formulas.evolution_stream(HD, HR, 0.3, 2 ** m, r, 3)
        want = oracle.inner(n, psi0, oracle.apply_masks(n, psi0, sx, sz, sa))
        assert abs(zm - want) <= 1e-10


def test_z0_basis_coset_oracle():
    """NEXT-3 (Fig. 4 analog): Z_0 = <b|e^{i delta H~}|b> of one partially randomized
    second-order step of a JW-shaped Hamiltonian whose X support lies on 14 qubits of a 24-qubit
    register (Z letters everywhere), on 1 GPU and on 4 virtual ranks, against the coset oracle."""
    from paper_2504_17881_b200 import formulas, rpe
    n = 24
    pos = list(range(n - 14, n))
    codes, coeffs = workloads.jw_embedded(n, pos, 3000, 20.0, seed=3)
    x, z = P.pauli_encode_codes(codes)
    H = formulas.from_masks(n, x, z, coeffs)
    HD, HR = formulas.split_deterministic(H, 400)
    b = sum(1 << q for q in range(0, n, 2))
    for d in (0.05, 0.3):
        r = formulas.sample_count(HR.lam, d, 0)
        sx, sz, sa = formulas.evolution_stream(HD, HR, d, 1, r, 11)
        mem = oracle.coset_members(n, b, np.unique(sx))
        out = oracle.apply_coset(n, mem, (mem == b).astype(np.complex128), oracle.decode_masks(n, sx, sz), sa)
        want = complex(out[np.searchsorted(mem, b)])
        assert abs(rpe.z0_basis(n, HD, HR, d, r, 11, b) - want) <= 1e-10
        assert abs(rpe.z0_basis(n, HD, HR, d, r, 11, b, emulate=4) - want) <= 1e-10
        assert 0.0 < abs(want) <= 1.0 + 1e-12
