"""Multi-GPU parity worker: run under torchrun, one rank per GPU (tests/test_multigpu.py).

Every check compares the sharded CUDA path (NCCL half-vector exchanges, per-rank signs) with the
CPU oracle or with a single-GPU run; rank 0 writes a JSON report and exits non-zero on failure.
"""
from __future__ import annotations

import json
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402
import paper_2504_17881_b200 as P  # noqa: E402
from paper_2504_17881_b200 import ps  # noqa: E402

SEED = 250417881


class _SkipSmall(Exception):
    pass


def layer_with_global(n, count, seed, world):
    """R10 layer plus runs of rotations with X on the top (global) qubits and Z-only global terms."""
    codes, ang = workloads.random_layer(n, count, seed=seed, kind="R10")
    rng = np.random.default_rng(seed)
    m = world.bit_length() - 1
    for l in range(0, count, 7):
        q = n - 1 - int(rng.integers(0, m))
        codes[l, q] = rng.integers(1, 4)
    for l in range(3, count, 11):  # a run sharing an upper X-part
        codes[l:l + 4, n - 1] = 1
    return codes, ang


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    report = {"world": world, "checks": []}
    ok = True

    def check(name, err, tol):
        nonlocal ok
        good = bool(err <= tol)
        ok &= good
        report["checks"].append({"name": name, "err": float(err), "tol": tol, "ok": good})

    only_large = os.environ.get("PS_MP_ONLY_LARGE") == "1"
    try:
        # (a) small n against the oracle, all fusion levels, small exchange chunks
        for n in (() if only_large else (6, 10, 13)):
            codes, ang = layer_with_global(n, 300, n, world)
            x, z = P.pauli_encode_codes(codes)
            want = oracle.apply(n, oracle.random_state(SEED, n), codes, ang) if rank == 0 else None
            for fusion, chunk, layout, transport, ovl, fused in (
                    (0, 4096, 0, 0, 1, 0), (1, 1 << 28, 0, 1, 1, 0), (2, 4096, 0, 0, 1, 0), (2, 1 << 28, 1, 1, 1, 0),
                    (0, 1 << 28, 1, 0, 1, 0), (2, 4096, 1, 1, 0, 0), (2, 1 << 28, 2, 1, 1, 0), (1, 4096, 2, 0, 1, 0),
                    (2, 1 << 28, 1, 1, 1, 1), (2, 4096, 0, 1, 0, 1), (2, 1 << 28, 1, 1, 2, 0), (2, 1 << 28, 0, 1, 2, 0),
                    (2, 1 << 28, 1, 1, 11, 0), (2, 1 << 28, 1, 1, 12, 0), (2, 1 << 28, 2, 1, 2, 0),
                    (1, 4096, 2, 1, 2, 0)):
                # ovl >= 10: overlap mode ovl - 10 with 32 full-size swap CTAs (else the slim kernel)
                with P.State(n, "c128", world=world, rank=rank) as st:
                    st.set_option(ps.OPT_FUSED_EXCHANGE, fused)
                    st.set_option(ps.OPT_OVERLAP, ovl % 10)
                    st.set_option(ps.OPT_SWAP_CTAS, 32 if ovl >= 10 else 0)
                    st.set_option(ps.OPT_FUSION, fusion)
                    st.set_option(ps.OPT_TILE_BITS, 6)
                    st.set_option(ps.OPT_CHUNK_BYTES, chunk)
                    st.set_option(ps.OPT_LAYOUT, layout)
                    st.set_option(ps.OPT_TRANSPORT, transport)
                    st.init_random(SEED)
                    # two calls: the lazy layout persists across them; the norm needs no restore
                    h = len(ang) // 2
                    st.apply_rotations(x[:h], z[:h], ang[:h])
                    nrm_mid = st.norm()
                    st.apply_rotations(x[h:], z[h:], ang[h:])
                    got = st.get_amplitudes()
                    stats = st.stats()
                if rank == 0:
                    tag = (f"n={n} fusion={fusion} chunk={chunk} layout={layout} transport={transport} overlap={ovl} "
                           f"fused={fused}")
                    check(f"oracle {tag} exch={stats['exchanges']} perm={stats['launches']['permute']}",
                          np.max(np.abs(got - want)), 1e-10)
                    check(f"mid-call norm {tag}", abs(nrm_mid - oracle.norm(n, oracle.random_state(SEED, n))) /
                          oracle.norm(n, oracle.random_state(SEED, n)), 1e-12)
        # (a2) 18 qubits with default tiles: overlapped swap pieces whose runs reach 1 KB go through the
        # TMA swap kernel; the register kernels must give bitwise the same state
        for n in (() if only_large else (18,)):
            codes, ang = layer_with_global(n, 200, n, world)
            x, z = P.pauli_encode_codes(codes)
            want = oracle.apply(n, oracle.random_state(SEED, n), codes, ang) if rank == 0 else None
            ref = None
            for ovl, swap_tma, swap_ctas in ((2, 1, 0), (1, 1, 0), (2, 0, 0), (2, 1, -1), (1, 0, 32), (0, 1, 0)):
                with P.State(n, "c128", world=world, rank=rank) as st:
                    st.set_option(ps.OPT_OVERLAP, ovl)
                    st.set_option(ps.OPT_SWAP_TMA, swap_tma)
                    st.set_option(ps.OPT_SWAP_CTAS, swap_ctas)
                    st.init_random(SEED)
                    st.apply_rotations(x, z, ang)
                    got = st.get_amplitudes()
                    stats = st.stats()
                if rank == 0:
                    tag = f"n={n} overlap={ovl} swap_tma={swap_tma} swap_ctas={swap_ctas} exch={stats['exchanges']}"
                    check(f"oracle {tag}", np.max(np.abs(got - want)), 1e-10)
                    if ref is None:
                        ref = got
                    check(f"swap kernels bitwise {tag}", 0.0 if np.array_equal(got, ref) else 1.0, 0.0)
        if only_large:
            raise _SkipSmall()
        # (b) full-exchange fallback: local X-part covering every local bit
        n = world.bit_length() - 1 + 3
        words = ["X" * n, "Y" + "X" * (n - 2) + "Z", "Z" * n, "XY" * (n // 2) + "X" * (n % 2), "I" + "X" * (n - 1)]
        codes = oracle.words_to_factors(words)
        x, z = P.pauli_encode_codes(codes)
        ang = np.array([0.3, -1.2, 0.7, 2.0, -0.5])
        with P.State(n, "c128", world=world, rank=rank) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
        if rank == 0:
            check(f"full-exchange fallback n={n}", np.max(np.abs(got - oracle.apply(n, oracle.random_state(SEED, n), codes, ang))), 1e-12)
        # (c) JW-shaped first-order Trotter step, x-major order for this world size
        n = 16
        m = world.bit_length() - 1
        hc, hco = workloads.jw_hamiltonian(n, 3000, 27.0, seed=1, n_local=n - m)
        ang = workloads.trotter1_angles(hco, 0.5)
        x, z = P.pauli_encode_codes(hc)
        want = oracle.apply(n, oracle.random_state(SEED, n), hc, ang) if rank == 0 else None
        with P.State(n, "c128", world=world, rank=rank) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
            stats = st.stats()
            # (d) expectation of the same Hamiltonian (global-X terms need exchanges), norm, inner
            e = st.expectation(x, z, hco)
            nrm = st.norm()
            with P.State(n, "c128", world=world, rank=rank) as st2:
                st2.init_random(SEED + 1)
                ip = st.inner(st2)
        if rank == 0:
            check(f"JW Trotter n=16 ({len(ang)} terms, {stats['exchanges']} exchanges)", np.max(np.abs(got - want)), 1e-10)
            check("expectation", abs(e - oracle.expectation(n, want, hc, hco)), 1e-9)
            check("norm", abs(nrm - oracle.norm(n, want)) / oracle.norm(n, want), 1e-12)
            check("inner", abs(ip - oracle.inner(n, want, oracle.random_state(SEED + 1, n))), 1e-9)
        # (e) fp32 against the oracle
        n = 12
        codes, ang = layer_with_global(n, 400, 5, world)
        x, z = P.pauli_encode_codes(codes)
        with P.State(n, "c64", world=world, rank=rank) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
        if rank == 0:
            check("fp32 n=12", np.max(np.abs(got - oracle.apply(n, oracle.random_state(SEED, n), codes, ang))), 1e-4)
        # (f) G-invariance at 24 qubits against a single-GPU run of the same layer
        n = 24
        codes, ang = layer_with_global(n, 500, 24, world)
        x, z = P.pauli_encode_codes(codes)
        with P.State(n, "c128", world=world, rank=rank) as st:
            st.init_random(SEED)
            st.apply_rotations(x, z, ang)
            got = st.get_amplitudes()
        if rank == 0:
            with P.State(n, "c128") as one:
                one.init_random(SEED)
                one.apply_rotations(x, z, ang)
                ref = one.get_amplitudes()
            check("G-invariance n=24 vs 1 GPU", np.max(np.abs(got - ref)), 1e-12)
        # (h) NEXT-3: RPE signal of the partially randomized second-order method, sharded
        from paper_2504_17881_b200 import formulas, rpe
        n = 12
        codes, _ = workloads.random_layer(n, 120, seed=31, kind="R10")
        codes = np.unique(codes, axis=0)
        coeffs = np.random.default_rng(31).uniform(-1, 1, len(codes))
        hx, hz = P.pauli_encode_codes(codes)
        H = formulas.from_masks(n, hx, hz, coeffs)
        HD, HR = formulas.split_deterministic(H, 40, n_local=n - (world.bit_length() - 1))
        r = formulas.sample_count(HR.lam, 0.3, 2)
        for m in (0, 2):
            zm = rpe.signal(n, HD, HR, 0.3, m, r, seed=3, world=world, rank=rank)
            if rank == 0:
                psi0 = oracle.random_state(SEED, n)
                psi0 = psi0 / np.sqrt(oracle.norm(n, psi0))
                sx, sz, sa = formulas.evolution_stream(HD, HR, 0.3, 2 ** m, r, 3)
                want = oracle.inner(n, psi0, oracle.apply_masks(n, psi0, sx, sz, sa))
                check(f"RPE Z_{m} (r={r})", abs(zm - want), 1e-10)
    except _SkipSmall:
        pass
    except Exception:  # noqa: BLE001
        ok = False
        report["error"] = traceback.format_exc()
    try:
        # (g) large n (PS_MP_LARGE=n): JW-shaped Trotter step with X-support on 16 qubits (incl. the
        # global ones) and Z letters everywhere, checked on whole cosets by the coset oracle
        big = int(os.environ.get("PS_MP_LARGE", "0"))
        if big:
            rng = np.random.default_rng(big)
            m = world.bit_length() - 1
            pos = sorted(set([big - 1 - j for j in range(m)]) | set(int(v) for v in rng.choice(big - m, 16 - m, replace=False)))
            hc, hco = workloads.jw_embedded(big, pos, 2000, 20.0, seed=2, n_local=big - m)
            ang = workloads.trotter1_angles(hco, 0.5)
            x, z = P.pauli_encode_codes(hc)
            import time
            with P.State(big, "c128", world=world, rank=rank) as st:
                st.init_random(SEED)
                st.synchronize()
                t0 = time.perf_counter()
                st.apply_rotations(x, z, ang)
                st.synchronize()
                el = time.perf_counter() - t0
                stats = st.stats()
                nrm = st.norm()
                for trial in range(2):
                    i0 = int(rng.integers(0, 1 << big)) if trial else 0
                    mem = oracle.coset_members(big, i0, x)
                    sel = np.sort(rng.choice(len(mem), 200, replace=False))
                    got = np.array([st.get_amplitudes(int(mem[k]), 1)[0] for k in sel])
                    if rank == 0:
                        init = oracle.random_amplitudes_at(SEED, mem)
                        want = oracle.apply_coset(big, mem, init, hc, ang)
                        check(f"coset oracle n={big} ({len(mem)} members, {len(ang)} terms, {stats['exchanges']} exchanges, "
                              f"{el:.1f} s)", np.max(np.abs(got - want[sel])), 1e-10)
                if rank == 0:
                    n0 = float(np.sum(np.abs(oracle.random_amplitudes(SEED, 0, 1 << 20)) ** 2)) * 2 ** (big - 20)
                    report["large_norm_ratio"] = nrm / n0
    except Exception:  # noqa: BLE001
        ok = False
        report["error"] = traceback.format_exc()
    report["ok"] = ok
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        path = os.environ.get("PS_MP_REPORT", "mp_report.json")
        with open(path, "w") as fh:
            json.dump(report, fh, indent=1)
        print(json.dumps(report))
    dist.destroy_process_group()
    sys.exit(0 if all(flags) else 1)


if __name__ == "__main__":
    main()
