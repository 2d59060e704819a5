"""Benchmark: Pauli rotations/s (and HBM GB/s) on a 30-qubit fp64 state (BASELINE.json configs[1]).

One step = one ps_apply_rotations call applying a layer of 1000 random Pauli rotations of weight
1-10 (the R10 generator of DESIGN.md "Input recipe") to the full 2^30-amplitude state, inputs
resident in HBM; value = rotations / second (whole job).  N > 1 GPUs (torchrun): the same
30-qubit state sharded over N ranks by its top qubits (strong scaling), exchanges over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--qubits 30] [--layer 1000] [--kind R10] [--dtype c128] [--fusion 2]

--impl reference times the CPU oracle (the slow from-definition program) on the host cores,
on a bounded sample of the same workload (scaled to the 30-qubit metric), and prints the same
line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "Pauli rotations/sec and HBM GB/s at 30-36 qubits, 1/2/4/8 B200"
UNIT = "rotations/s"
FALLBACK_HBM_GBS = 6650.0
SPEC_HBM_GBS = 8000.0  # BASELINE.json north_star "roughly 8 TB/s" (B200 DGX figure)
PASS_FAMS = ("stream", "tile", "coset", "xtile")  # kernel families that make one HBM pass


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", dest="n", type=int, default=30)
    ap.add_argument("--layer", type=int, default=1000)
    ap.add_argument("--kind", default="R10", help="R10 R4 D S8 LOW (random layers), JW (Trotter step), QAOA, GATES, UCC, HEA (VQE), SUFFIX (L-groups)")
    ap.add_argument("--terms", type=int, default=92968, help="JW: Hamiltonian terms (Table 3: 92,968 at 32q)")
    ap.add_argument("--lam", type=float, default=27.0, help="JW: lambda = sum |h| (Table 3)")
    ap.add_argument("--delta", type=float, default=0.5, help="JW: Trotter step size")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--fusion", type=int, default=2)
    ap.add_argument("--tile-bits", type=int, default=0)
    ap.add_argument("--tile-mode", type=int, default=2,
                    help="0 cp.async prefetch, 1 TMA ring, 2 register-direct, 3 TMA-bulk prefetch")
    ap.add_argument("--chunk-bits", type=int, default=0)
    ap.add_argument("--tile-tune", type=int, default=-1)
    ap.add_argument("--layout", type=int, default=1, help="world > 1: 1 lazy qubit swaps, 0 runs + swap-back")
    ap.add_argument("--transport", type=int, default=1, help="world > 1: 1 NVLink P2P, 0 NCCL send/recv")
    ap.add_argument("--overlap", type=int, default=2, help="world > 1: overlap swaps with the next pass (2: and the previous one)")
    ap.add_argument("--swap-tma", type=int, default=1, help="overlapped swap pieces through the TMA swap kernel (1) or the register kernel (0)")
    ap.add_argument("--swap-ctas", type=int, default=0, help="overlapped swap pieces: 0 default (slim kernel, 2 per SM); -k slim (per SM if k <= 8); k full-size")
    ap.add_argument("--specialize", type=int, default=-1,
                    help="tile-kernel variant: -1 library default (fp64 2, fp32 0), 0 generic, 2 unit-dx specialised, "
                         "1 planner's per-pass choice")
    ap.add_argument("--group", type=int, default=10, help="SUFFIX: rotations per group sharing an upper string")
    ap.add_argument("--fused", type=int, default=0, help="world > 1: fused exchange + tile kernel (1) or swaps (0, default)")
    ap.add_argument("--emulate", type=int, default=0,
                    help="run the multi-rank path as G virtual ranks on this one GPU (ps_create_emulated)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_name(args):
    prec = "fp64" if args.dtype == "c128" else "fp32"
    if args.kind == "JW":
        return (f"{args.n}q {prec} first-order Trotter step of a JW-shaped molecular Hamiltonian "
                f"({args.terms} terms, lambda {args.lam}, delta {args.delta}, x-major order)")
    if args.kind == "QAOA":
        return f"{args.n}q {prec} QAOA MaxCut, random 3-regular graph, p = {args.layer} layers"
    if args.kind == "GATES":
        return f"{args.n}q {prec} random gate brickwork of depth {args.layer}, converted to rotations"
    if args.kind == "SUFFIX":
        return (f"{args.n}q {prec} groups of L={args.group} rotations sharing an upper string on the "
                f"partitioned qubits (P:502-508), {args.layer} rotations/step")
    if args.kind == "UCC":
        return (f"{args.n}q {prec} UCCSD-shaped VQE layer (JW; {args.n // 3} occupied spin orbitals, "
                f"singles + {args.layer} sampled doubles x 8 strings)")
    if args.kind == "HEA":
        return f"{args.n}q {prec} hardware-efficient VQE ansatz, {args.layer} RY/RZ + CNOT-ladder layers"
    return (f"{args.n}q {prec} random Pauli-rotation layer "
            f"({args.kind}: weight 1-10, phi~U[-pi,pi)), {args.layer} rotations/step")


def layers(args, count, world=1):
    """(codes or None, x, z, angles) per step; structured workloads repeat one step."""
    import paper_2504_17881_b200 as P
    out = []
    if args.kind == "JW":
        m = world.bit_length() - 1
        codes, coeffs = workloads.jw_hamiltonian(args.n, args.terms, args.lam, seed=0, n_local=args.n - m)
        x, z = P.pauli_encode_codes(codes)
        ang = workloads.trotter1_angles(coeffs, args.delta)
        return [(x, z, ang)] * count
    if args.kind == "QAOA":
        codes, ang = workloads.qaoa_layers(args.n, args.layer, seed=0)
        x, z = P.pauli_encode_codes(codes)
        return [(x, z, ang)] * count
    if args.kind == "GATES":
        x, z, ang = P.circuit_to_rotations(workloads.gate_circuit(args.n, args.layer, seed=0))
        return [(x, z, ang)] * count
    if args.kind == "SUFFIX":
        m = max(1, world.bit_length() - 1)
        out = []
        for s in range(count):
            codes, ang = workloads.suffix_groups(args.n, args.layer, args.group, m, seed=1000 + s)
            x, z = P.pauli_encode_codes(codes)
            out.append((x, z, ang))
        return out
    if args.kind == "UCC":
        codes, ang = workloads.ucc_layers(args.n, args.n // 3, seed=0, max_doubles=args.layer)
        x, z = P.pauli_encode_codes(codes)
        return [(x, z, ang)] * count
    if args.kind == "HEA":
        x, z, ang = P.circuit_to_rotations(workloads.hardware_efficient_vqe(args.n, args.layer, seed=0))
        return [(x, z, ang)] * count
    for s in range(count):
        codes, ang = workloads.random_layer(args.n, args.layer, seed=1000 + s, kind=args.kind)
        x, z = P.pauli_encode_codes(codes)
        out.append((x, z, ang))
    return out


# ------------------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            sm.append(s)
            mx = max(mx, m)
            for b, name in self.REASONS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def fma_roofline(stats, fam, args, world, clk):
    kms = stats["kernel_ms"][fam]
    rot = stats["rotations_by"][fam]
    if kms <= 0 or rot <= 0:
        return None
    nl = args.n - (world.bit_length() - 1)
    fma = 2.0 * rot * float(1 << nl)  # per rank (rank 0's stats)
    achieved = fma / (kms / 1e3)
    lanes = 64 if args.dtype == "c128" else 128
    mhz = (clk or {}).get("sm_max_mhz") or 1965.0
    peak = 148 * lanes * mhz * 1e6
    return {"bound": "alu", "unit": "FMA/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "algorithmic_fma_per_rotation": 2.0 * float(1 << nl)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(kernel: str, bytes_per_launch: float, dtype: str):
    """dram bytes per launch from the committed ncu --set full summary, when that capture was of a
    launch of the same size and dtype as this run's (else null: per-launch traffic of another
    configuration says nothing about this one)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        alg = float(d[kernel + "_algorithmic"])
        if d.get(kernel + "_dtype") != dtype or abs(bytes_per_launch - alg) > 0.01 * alg:
            return None
        return d.get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------------------------ CPU oracle

def _set_omp_threads(k):
    """The oracle's OpenMP runtime is the system libgomp; its thread count is set process-wide
    (torchrun exports OMP_NUM_THREADS=1, which would otherwise pin it to one core)."""
    import ctypes
    import oracle
    oracle.lib()
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(k))
        return int(k)
    except OSError:
        return int(os.environ.get("OMP_NUM_THREADS", "1"))


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _host_copy_gbs(cores, gib=1.0):
    """STREAM-like host copy: numpy copy of a 1 GiB buffer split over `cores` threads (numpy
    releases the GIL), best of 3, read + write bytes counted."""
    from concurrent.futures import ThreadPoolExecutor
    n = int(gib * 2 ** 30) // 8
    a = np.ones(n)
    b = np.empty_like(a)
    parts = np.array_split(np.arange(n), cores)
    bounds = [(int(p[0]), int(p[-1]) + 1) for p in parts if len(p)]

    def cp(r):
        b[r[0]:r[1]] = a[r[0]:r[1]]

    best = 0.0
    with ThreadPoolExecutor(max_workers=cores) as ex:
        for _ in range(3):
            t0 = time.perf_counter()
            list(ex.map(cp, bounds))
            el = time.perf_counter() - t0
            best = max(best, 2 * n * 8 / el / 1e9)
    return best


def _oracle_rate(n_s, kind, layer, budget_s, seed=1000):
    """rotations/s of the oracle applying a `kind` layer at n_s qubits until budget_s is spent
    (at least one rotation), rotation by rotation; also the sample description"""
    import oracle
    codes, ang = workloads.random_layer(n_s, layer, seed=seed, kind=kind)
    psi = oracle.random_state(workloads.BASE_SEED, n_s)
    done, t0 = 0, time.perf_counter()
    while done < len(ang):
        psi = oracle.apply(n_s, psi, codes[done:done + 1], ang[done:done + 1])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return done / el, done, el


def cpu_oracle_sample(args, n_sample=26):
    """the oracle as it stands on the host cores -- OpenMP over all cores and
    single-threaded, R10 and R4 layers at 24/26 qubits, the config-1 set, a STREAM-like host copy and
    the CPU model.  value = the all-core R10 rate at n_sample qubits scaled by 2^(n_sample - n) to the
    benchmark's n (the oracle's cost is linear in 2^n); ~20 s of host work in total."""
    cores = os.cpu_count() or 1
    used = _set_omp_threads(cores)
    n_s = min(n_sample, args.n)
    kind = args.kind if args.kind in ("R10", "R4", "D", "S8", "LOW") else "R10"
    rate, done, el = _oracle_rate(n_s, kind, args.layer, 8.0)
    scale = 2.0 ** (n_s - args.n)
    runs = [{"threads": used, "qubits": n_s, "kind": kind, "rotations": done, "seconds": round(el, 2),
             "rot_per_s": rate, "gb_per_s": rate * 2 * 16 * 2 ** n_s / 1e9}]
    n24 = min(24, args.n)
    r4, d4, e4 = _oracle_rate(n24, "R4", 20, 3.0)
    runs.append({"threads": used, "qubits": n24, "kind": "R4", "rotations": d4, "seconds": round(e4, 2),
                 "rot_per_s": r4, "gb_per_s": r4 * 2 * 16 * 2 ** n24 / 1e9})
    _set_omp_threads(1)
    r1, d1, e1 = _oracle_rate(n24, kind, args.layer, 4.0)
    runs.append({"threads": 1, "qubits": n24, "kind": kind, "rotations": d1, "seconds": round(e1, 2),
                 "rot_per_s": r1, "gb_per_s": r1 * 2 * 16 * 2 ** n24 / 1e9})
    rc, dc, ec = _oracle_rate(10, "R10", 200, 2.0, seed=1)
    runs.append({"threads": 1, "qubits": 10, "kind": "R10 (config 1)", "rotations": dc, "seconds": round(ec, 4),
                 "rot_per_s": rc})
    _set_omp_threads(cores)
    copy = _host_copy_gbs(cores)
    return {"value": rate * scale, "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"{done} rotations of a {kind} layer on a {n_s}-qubit fp64 state in {el:.1f} s on {used} "
                      f"threads, scaled by 2^({n_s}-{args.n}) to the {args.n}-qubit state",
            "extrapolated": {"from_qubits": n_s, "to_qubits": args.n, "factor": scale},
            "cpu_model": _cpu_model(), "host_copy_gbs": copy,
            "oracle_frac_of_host_copy": runs[0]["gb_per_s"] / copy if copy > 0 else None,
            "runs": runs}


def run_reference(args):
    """The base contract's reference arm for this tier: the oracle, as it stands, on the host cores.
    Each step is a bounded sample (~5 s) of the workload: the layer's rotations applied one by one
    at 26 qubits; ms_per_step is that sample's measured time and value its rate scaled to the
    benchmark's qubit count (the scaling is stated in "extrapolated")."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = _set_omp_threads(os.cpu_count() or 1)
    n_s = min(26, args.n)
    kind = args.kind if args.kind in ("R10", "R4", "D", "S8", "LOW") else "R10"
    scale = 2.0 ** (n_s - args.n)
    rates, times, dones = [], [], []
    for s in range(args.warmup + args.steps):
        rate, done, el = _oracle_rate(n_s, kind, args.layer, 5.0, seed=1000 + s)
        if s >= args.warmup:
            rates.append(rate)
            times.append(el)
            dones.append(done)
    value = statistics.mean(rates) * scale
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(args), "n_qubits": args.n,
                                        "rotations_per_step": args.layer},
        "extrapolated": {"from_qubits": n_s, "to_qubits": args.n, "factor": scale,
                         "sample_rotations_per_step": dones,
                         "note": "each step applies the first rotations of the layer at the sample size "
                                 "for ~5 s; value = sample rate x factor (cost linear in 2^n)"},
        "cpu_baseline": {"kind": "oracle", "cores": cores, "value": value, "unit": UNIT,
                         "sample": f"{sum(dones)} rotations of {kind} layers at {n_s} qubits over "
                                   f"{args.steps} timed steps", "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ ours

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_17881_b200 as P
    from paper_2504_17881_b200 import ps

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    if args.emulate and world > 1:
        raise SystemExit("--emulate runs on one GPU (no torchrun)")
    if args.emulate:
        st = P.State(args.n, args.dtype, emulate=args.emulate, torch_memory=True)
    else:
        st = P.State(args.n, args.dtype, world=world, rank=rank, torch_memory=True)
    st.set_option(ps.OPT_FUSION, args.fusion)
    if args.tile_bits:
        st.set_option(ps.OPT_TILE_BITS, args.tile_bits)
    st.set_option(ps.OPT_TILE_TMA, args.tile_mode)
    if args.chunk_bits:
        st.set_option(ps.OPT_CHUNK_BITS, args.chunk_bits)
    if args.tile_tune >= 0:
        st.set_option(ps.OPT_TILE_TUNE, args.tile_tune)
    st.set_option(ps.OPT_LAYOUT, args.layout)
    st.set_option(ps.OPT_TRANSPORT, args.transport)
    st.set_option(ps.OPT_OVERLAP, args.overlap)
    st.set_option(ps.OPT_SWAP_CTAS, args.swap_ctas)
    st.set_option(ps.OPT_SWAP_TMA, args.swap_tma)
    if args.specialize >= 0:
        st.set_option(ps.OPT_SPECIALIZE, args.specialize)
    st.set_option(ps.OPT_FUSED_EXCHANGE, args.fused)
    st.set_option(ps.OPT_PROFILE, 1)
    enc = layers(args, args.warmup + args.steps, args.emulate or world)
    rot_per_step = len(enc[0][2])
    st.init_random(workloads.BASE_SEED)

    stream = st.torch_stream  # the stream libps enqueues on
    for w in range(args.warmup):
        x, z, a = enc[w]
        st.apply_rotations(x, z, a)
    st.synchronize()
    st.reset_stats()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for s in range(args.steps):
        x, z, a = enc[args.warmup + s]
        st.apply_rotations(x, z, a)
        evs[s + 1].record(stream)
    st.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[s].elapsed_time(evs[s + 1]) for s in range(args.steps)]
    clk = clocks.stop()
    stats = st.stats()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = rot_per_step / (ms_per_step / 1e3)
    amp_bytes = 16 if args.dtype == "c128" else 8
    # emulation: every virtual rank's slice lives on this GPU; stats are rank 0's
    ranks = args.emulate or world
    local_state = amp_bytes << (args.n - (world.bit_length() - 1))
    hbm_alg = sum(stats["algo_bytes"][k] for k in PASS_FAMS) / (ms / 1e3) / 1e9 * ranks

    # dominant kernel roofline (CUDA events around each launch on the launching stream)
    fam = max(PASS_FAMS, key=lambda k: stats["kernel_ms"][k])
    launches = max(1, stats["launches"][fam])
    kms = stats["kernel_ms"][fam]
    bytes_per_launch = stats["algo_bytes"][fam] / launches
    achieved = stats["algo_bytes"][fam] / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    peak, peak_src = peaks()
    rotations = stats["rotations"]
    passes = max(1, stats["passes"])
    gpu_launches = sum(stats["launches"].values())  # every libps kernel family (exchanges: swap kernels / NCCL)

    # e2e through the public API with host buffers (pinned): H2D of the initial state + rotation
    # arrays, the layer, D2H of the norm (the step's scalar result)
    e2e = None
    if not args.no_e2e:
        tdt = torch.float64 if args.dtype == "c128" else torch.float32
        host = torch.empty((amp_bytes << args.n if args.emulate else local_state) // (amp_bytes // 2), dtype=tdt,
                           pin_memory=True)
        st.init_random(workloads.BASE_SEED)
        host.copy_(st._tensor)  # the seeded initial state, staged in pinned host memory (untimed)
        h2d = (amp_bytes << args.n if args.emulate else local_state) + 24 * rot_per_step
        e_steps = min(args.steps, 2)
        x, z, a = enc[0]
        cnt, first = (1 << args.n, 0) if args.emulate else (1 << st.n_local, rank << st.n_local)
        st.set_state_ptr(host.data_ptr(), cnt, first=first)
        st.apply_rotations(x, z, a)
        st.norm()
        barrier()
        t0 = time.perf_counter()
        for s in range(e_steps):
            x, z, a = enc[(args.warmup + s) % len(enc)]
            st.set_state_ptr(host.data_ptr(), cnt, first=first)
            st.apply_rotations(x, z, a)
            st.norm()
        barrier()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": rot_per_step * e_steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": 8, "steps": e_steps,
               "path": "ps_set_state(pinned host) + ps_apply_rotations(host arrays) + ps_norm -> host"}
        del host

    if rank == 0:
        cpu = None if args.no_cpu else cpu_oracle_sample(args)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.dtype == "c128" else "f32",
            "data": "synthetic",
            "config": {"workload": workload_name(args), "n_qubits": args.n, "rotations_per_step": rot_per_step,
                       "fusion": args.fusion, "tile_mode": args.tile_mode, "tile_bits": args.tile_bits or 12,
                       "layout": args.layout, "transport": args.transport, "overlap": args.overlap, "swap_ctas": args.swap_ctas, "swap_tma": args.swap_tma, "specialize": args.specialize if args.specialize >= 0 else (2 if args.dtype == "c128" else 0),
                       "parallelism": (f"state sharded over {args.emulate} virtual ranks on 1 GPU (emulation)"
                                       if args.emulate else f"state sharded over {world} GPU(s) by top qubits"),
                       "fused_exchange": args.fused, "group": args.group if args.kind == "SUFFIX" else None,
                       "l2": "inputs larger than L2 (state %.1f GiB per GPU)" % (local_state / 2 ** 30)},
            "hbm_gbs": hbm_alg,
            "bytes_per_rotation": stats["algo_bytes"]["stream"] / max(1, stats["rotations_by"]["stream"])
            if fam == "stream" else sum(stats["algo_bytes"][k] for k in PASS_FAMS) / max(1, rotations),
            "rotations_per_pass": rotations / passes,
            "passes": {k: stats["launches"][k] for k in PASS_FAMS},
            "exchanges": stats["exchanges"],
            "exchange_ms": stats["kernel_ms"]["exchange"],
            # per direction per GPU: swap exchanges over their own (CUDA-event) time; fused exchange +
            # tile passes over theirs (NVLink 5: 900 GB/s per direction nominal, 770 measured peer copy).
            # With overlap (modes 1, 2) a swap's time runs on its stream from the first piece to the last
            # and includes the waits for pass pieces, so this is a lower bound on the link rate; the
            # serialised rate is the --overlap 0 line (profiles/r02/multi_gpu.md)
            "nvlink_gbs": (stats["nvlink_bytes"] / (stats["kernel_ms"]["exchange"] / 1e3) / 1e9
                           if stats["kernel_ms"]["exchange"] > 0 and stats["nvlink_bytes"] > 0 else None),
            "nvlink_gbs_includes_overlap_waits": bool(world > 1 and args.overlap > 0),
            "nvlink_fused_gbs": (stats["nvlink_fused_bytes"] / (stats["kernel_ms"]["xtile"] / 1e3) / 1e9
                                 if stats["kernel_ms"]["xtile"] > 0 else None),
            "best_step_ms": min(step_ms) if step_ms else None,
            "roofline": {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "frac_of_spec": achieved / SPEC_HBM_GBS, "spec_gbs": SPEC_HBM_GBS,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": kms / launches,
                         "traffic": traffic_for(fam, bytes_per_launch, args.dtype)},
            # the fp64/fp32 FMA pipe roofline of the same kernel family: the deferred-scale pair update
            # costs 2 FMA per amplitude and rotation (4 per pair); peak = 148 SMs x 64 fp64 (128 fp32)
            # FMA lanes x the max SM clock (B200_PROFILING.md: 148 SMs, 1965 MHz)
            "roofline_fma": fma_roofline(stats, fam, args, world, clk),
            # exchange rotations (world > 1): swap NVLink rate per direction per GPU against NVLink 5's
            # nominal 900 GB/s per direction (770 GB/s = our measured peer copy, DESIGN.md section 5
            # K3); with overlap the swap time includes waits (a lower bound)
            "roofline_nvlink": ({"bound": "nvlink", "unit": "GB/s",
                                 "achieved": stats["nvlink_bytes"] / (stats["kernel_ms"]["exchange"] / 1e3) / 1e9,
                                 "peak": 900.0, "peak_source": "NVLink 5 nominal per direction",
                                 "frac": stats["nvlink_bytes"] / (stats["kernel_ms"]["exchange"] / 1e3) / 1e9 / 900.0,
                                 "measured_peer_copy_gbs": 770.0,
                                 "includes_overlap_waits": bool(args.overlap > 0)}
                                if world > 1 and stats["kernel_ms"]["exchange"] > 0 and stats["nvlink_bytes"] > 0
                                else None),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
