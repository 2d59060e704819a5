"""GPU parity at the sizes and launch configurations the bench uses (``-m gpu``), through the C ABI.

* large-n sweeps (22 and 24 qubits, default options): full-state comparison with the CPU oracle
  for every random-layer kind, fp64 and fp32.  At 24 qubits both dtypes run several tiles per CTA
  of the persistent grid (2^12 fp64 tiles on a 1184-CTA grid, 2^12 fp32 tiles on a 2368-CTA grid),
  so the incremental tile bases and the next-tile prefetch run exactly as in the 30-qubit bench;
* a grid cap (PS_OPT_GRID_CAP) forces many tiles per CTA at 14-18 qubits;
* 2^13 / 2^14-amplitude tiles (one CTA of 512 / 1024 threads per SM);
* minimum chunk sizes of 2^3 amplitudes (one more gathered dimension per tile).

Tolerances: BASELINE.json north_star (1e-10 fp64, 1e-4 fp32 max abs amplitude error) on the
unnormalised O(1) amplitudes of the seeded generator (R10).
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


def _want(n, kind, count, seed):
    key = (n, kind, count, seed)
    if key not in _cache:
        codes, ang = workloads.random_layer(n, count, seed=seed, kind=kind)
        _cache[key] = (codes, ang, oracle.apply(n, oracle.random_state(SEED, n), codes, ang))
    return _cache[key]


def _run(n, dtype, codes, ang, **opts):
    x, z = P.pauli_encode_codes(codes)
    with P.State(n, dtype) as st:
        for k, v in opts.items():
            st.set_option(getattr(ps, "OPT_" + k.upper()), v)
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        return st.get_amplitudes(), st.stats()


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["R10", "R4", "S8", "LOW", "D"])
@pytest.mark.parametrize("n,count", [(22, 200), (24, 100)])
def test_large_n_default_options(n, count, kind, dtype):
    codes, ang, want = _want(n, kind, count, 31)
    got, stats = _run(n, dtype, codes, ang)
    err = float(np.max(np.abs(got - want)))
    assert err <= TOL[dtype], (err, stats["launches"])


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["R10", "R4", "S8"])
@pytest.mark.parametrize("n,cap", [(14, 1), (16, 3), (18, 7)])
@pytest.mark.parametrize("tune", [0, 1536])
def test_grid_cap_many_tiles_per_cta(n, cap, kind, dtype, tune):
    """Many tiles per CTA, with (default fp64) and without (tune 1536) the next-tile prefetch."""
    codes, ang, want = _want(n, kind, 300, 32)
    opts = dict(grid_cap=cap)
    if tune:
        opts["tile_tune"] = tune
    got, _ = _run(n, dtype, codes, ang, **opts)
    assert np.max(np.abs(got - want)) <= TOL[dtype]
    ref, _ = _run(n, dtype, codes, ang)
    assert np.array_equal(got, ref)  # the tile schedule and the prefetch do not change any arithmetic


@pytest.mark.parametrize("dtype,tile_bits", [("c128", 13), ("c64", 12), ("c64", 13), ("c64", 14)])
@pytest.mark.parametrize("kind", ["R10", "R4", "S8", "LOW"])
@pytest.mark.parametrize("chunk_bits", [0, 3])
def test_big_tiles_and_small_chunks(dtype, tile_bits, kind, chunk_bits):
    n = 18
    codes, ang, want = _want(n, kind, 400, 33)
    opts = dict(tile_bits=tile_bits, grid_cap=5)
    if chunk_bits:
        opts["chunk_bits"] = chunk_bits
    got, stats = _run(n, dtype, codes, ang, **opts)
    assert np.max(np.abs(got - want)) <= TOL[dtype], stats["launches"]
