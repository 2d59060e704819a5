"""Thin Python binding of libps (include/ps.h): argument marshalling only.

Every step of the hot path runs in libps's CUDA kernels (or NCCL for exchanges).  There is no
CPU fallback: if libps.so is missing or a call fails, this module raises.  PyTorch is used only
for device memory, streams and process groups (torch.distributed bootstrap of the NCCL id).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PS_LIB_PATH") or os.path.join(_HERE, "libps.so")  # override for A/B builds

C128, C64 = 0, 1
K_STREAM, K_TILE, K_COSET, K_REDUCE, K_INIT, K_EXCHANGE, K_PERMUTE, K_MIRROR, K_XTILE = range(9)
KERNEL_NAMES = ["stream", "tile", "coset", "reduce", "init", "exchange", "permute", "mirror", "xtile"]
NK = len(KERNEL_NAMES)
OP_MIRROR_BEGIN, OP_MIRROR_SWITCH, OP_MIRROR_END = 16, 17, 18
OPT_PROFILE, OPT_FUSION, OPT_TILE_BITS, OPT_CHUNK_BYTES, OPT_MAX_PASS_ROTS, OPT_VEC256, OPT_TILE_TMA, OPT_CHUNK_BITS, OPT_TILE_TUNE, OPT_LAYOUT, OPT_TRANSPORT, OPT_OVERLAP, OPT_SPECIALIZE, OPT_GRID_CAP, OPT_FUSED_EXCHANGE, OPT_SWAP_CTAS, OPT_SWAP_TMA = range(17)


class PsError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [
        ("rotations", ctypes.c_uint64),
        ("passes", ctypes.c_uint64),
        ("exchanges", ctypes.c_uint64),
        ("launches", ctypes.c_uint64 * NK),
        ("rotations_by", ctypes.c_uint64 * NK),
        ("algo_bytes", ctypes.c_double * NK),
        ("nvlink_bytes", ctypes.c_double),
        ("kernel_ms", ctypes.c_double * NK),
        ("nvlink_fused_bytes", ctypes.c_double),
    ]

    def as_dict(self):
        return {
            "rotations": int(self.rotations),
            "passes": int(self.passes),
            "exchanges": int(self.exchanges),
            "launches": {k: int(self.launches[i]) for i, k in enumerate(KERNEL_NAMES)},
            "rotations_by": {k: int(self.rotations_by[i]) for i, k in enumerate(KERNEL_NAMES)},
            "algo_bytes": {k: float(self.algo_bytes[i]) for i, k in enumerate(KERNEL_NAMES)},
            "nvlink_bytes": float(self.nvlink_bytes),
            "kernel_ms": {k: float(self.kernel_ms[i]) for i, k in enumerate(KERNEL_NAMES)},
            "nvlink_fused_bytes": float(self.nvlink_fused_bytes),
        }


class PlanOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("first_rot", ctypes.c_int32), ("n_rot", ctypes.c_int32),
                ("exch_bit", ctypes.c_int32), ("exch_gx", ctypes.c_uint64), ("tile_bits", ctypes.c_uint32),
                ("n_sub", ctypes.c_uint32)]


class PlanRot(ctypes.Structure):
    _fields_ = [("x", ctypes.c_uint64), ("z", ctypes.c_uint64), ("y", ctypes.c_int32), ("sign", ctypes.c_int32),
                ("angle", ctypes.c_double)]


EXPORTS = [
    "ps_create", "ps_create_ex", "ps_create_dist", "ps_create_emulated", "ps_get_unique_id", "ps_destroy", "ps_info", "ps_set_option",
    "ps_init_basis", "ps_init_random", "ps_normalize", "ps_set_state", "ps_get_amplitudes", "ps_apply_rotations",
    "ps_norm", "ps_expectation", "ps_inner", "ps_synchronize", "ps_get_stats", "ps_reset_stats",
    "ps_status_string", "ps_last_error", "ps_pauli_encode", "ps_pauli_encode_codes", "ps_gate_to_rotations",
    "ps_plan_describe",
]

_lib = None


def lib():
    """Loads libps.so (built in-tree by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, i32, sz, dp = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
    H = ctypes.c_void_p
    sig = {
        "ps_create": [i32, i32, ctypes.POINTER(H)],
        "ps_create_ex": [i32, i32, vp, sz, vp, i32, i32, vp, ctypes.POINTER(H)],
        "ps_create_dist": [i32, i32, i32, i32, vp, ctypes.POINTER(H)],
        "ps_create_emulated": [i32, i32, i32, vp, sz, vp, ctypes.POINTER(H)],
        "ps_get_unique_id": [vp],
        "ps_destroy": [H],
        "ps_info": [H, vp, vp, vp, vp, vp, vp],
        "ps_set_option": [H, i32, ctypes.c_int64],
        "ps_init_basis": [H, u64],
        "ps_init_random": [H, u64],
        "ps_normalize": [H],
        "ps_set_state": [H, u64, u64, vp],
        "ps_get_amplitudes": [H, u64, u64, vp],
        "ps_apply_rotations": [H, vp, vp, vp, sz],
        "ps_norm": [H, vp],
        "ps_expectation": [H, vp, vp, vp, sz, vp],
        "ps_inner": [H, H, vp],
        "ps_synchronize": [H],
        "ps_get_stats": [H, vp],
        "ps_reset_stats": [H],
        "ps_pauli_encode": [ctypes.c_char_p, vp, vp],
        "ps_pauli_encode_codes": [vp, i32, sz, vp, vp],
        "ps_gate_to_rotations": [ctypes.c_char_p, vp, i32, vp, i32, vp, vp, vp, sz, vp],
        "ps_plan_describe": [i32, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp, sz, vp, vp, sz, vp],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.ps_status_string.argtypes = [ctypes.c_int]
    L.ps_status_string.restype = ctypes.c_char_p
    L.ps_last_error.argtypes = []
    L.ps_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(fn: str, rc: int):
    if rc != 0:
        msg = lib().ps_last_error().decode(errors="replace")
        raise PsError(fn, rc, msg)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------------- host helpers

def pauli_encode(word: str):
    x, z = ctypes.c_uint64(), ctypes.c_uint64()
    _check("ps_pauli_encode", lib().ps_pauli_encode(word.encode(), ctypes.byref(x), ctypes.byref(z)))
    return int(x.value), int(z.value)


def pauli_encode_codes(codes: np.ndarray):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    if codes.ndim != 2:
        raise ValueError("codes must be (count, n)")
    count, n = codes.shape
    x = np.zeros(count, np.uint64)
    z = np.zeros(count, np.uint64)
    _check("ps_pauli_encode_codes", lib().ps_pauli_encode_codes(_p(codes), n, count, _p(x), _p(z)))
    return x, z


def gate_to_rotations(gate: str, qubits, params=()):
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    p = _f64(params if len(params) else [0.0])
    cap = 8
    x = np.zeros(cap, np.uint64)
    z = np.zeros(cap, np.uint64)
    a = np.zeros(cap, np.float64)
    nout = ctypes.c_size_t()
    _check("ps_gate_to_rotations", lib().ps_gate_to_rotations(gate.encode(), _p(q), len(q), _p(p), len(params),
                                                             _p(x), _p(z), _p(a), cap, ctypes.byref(nout)))
    k = nout.value
    return x[:k].copy(), z[:k].copy(), a[:k].copy()


def circuit_to_rotations(gates):
    """[(name, qubits, params), ...] -> (x, z, angles) in application order."""
    xs, zs, angs = [], [], []
    for name, qubits, params in gates:
        x, z, a = gate_to_rotations(name, qubits, params)
        xs.append(x); zs.append(z); angs.append(a)
    if not xs:
        return np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0)
    return np.concatenate(xs), np.concatenate(zs), np.concatenate(angs)


def plan_describe(n: int, x, z, angles, world: int = 1, rank: int = 0, fusion: int = 2, tile_bits: int = 12,
                  layout: int = 1):
    x, z, a = _u64(x), _u64(z), _f64(angles)
    nops, nrots = ctypes.c_size_t(), ctypes.c_size_t()
    _check("ps_plan_describe", lib().ps_plan_describe(n, world, rank, fusion, tile_bits, layout, _p(x), _p(z), _p(a),
                                                      len(a), None, 0, ctypes.byref(nops), None, 0,
                                                      ctypes.byref(nrots)))
    ops = (PlanOp * max(1, nops.value))()
    rots = (PlanRot * max(1, nrots.value))()
    _check("ps_plan_describe", lib().ps_plan_describe(n, world, rank, fusion, tile_bits, layout, _p(x), _p(z), _p(a),
                                                      len(a), ops, nops.value, ctypes.byref(nops), rots, nrots.value,
                                                      ctypes.byref(nrots)))
    op_list = [dict(kind=o.kind, first_rot=o.first_rot, n_rot=o.n_rot, exch_bit=o.exch_bit, exch_gx=int(o.exch_gx),
                    tile_bits=o.tile_bits, n_sub=o.n_sub) for o in ops[: nops.value]]
    rot_list = [dict(x=int(r.x), z=int(r.z), y=r.y, sign=r.sign, angle=r.angle) for r in rots[: nrots.value]]
    return op_list, rot_list


def bootstrap_nccl_id(rank: int, group=None) -> bytes:
    """Rank 0 creates an ncclUniqueId (ps_get_unique_id); torch.distributed (any backend, e.g.
    gloo or nccl) broadcasts the 128 bytes to every rank of `group`."""
    import torch.distributed as dist
    obj = [None]
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        _check("ps_get_unique_id", lib().ps_get_unique_id(buf))
        obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=0, group=group)
    assert isinstance(obj[0], bytes) and len(obj[0]) == 128
    return obj[0]


# ---------------------------------------------------------------------------------- the state

class State:
    """A 2^n-amplitude state on this process's GPU (one rank of `world`).

    dtype: "c128" (complex double, the paper's precision P:354) or "c64".
    world > 1: call inside an initialised torch.distributed group (any backend); rank 0's NCCL
    unique id is broadcast with it, then libps runs its own NCCL communicator.
    torch_memory=True: the local slice is a torch tensor and work runs on torch's current stream.
    """

    def __init__(self, n: int, dtype: str = "c128", world: int = 1, rank: int = 0, torch_memory: bool = False,
                 group=None, emulate: int = 0):
        self.n = int(n)
        self.dtype = C128 if dtype in ("c128", "complex128", C128) else C64
        self.world, self.rank = int(world), int(rank)
        self._h = ctypes.c_void_p()
        self._tensor = None
        self.torch_stream = None
        L = lib()
        nid = None
        if emulate:
            # G virtual ranks on this device (ps_create_emulated): one handle, global indices
            self.world, self.rank, self.emulated = int(emulate), 0, True
            dev_ptr, nbytes, stream = None, 0, None
            if torch_memory:
                import torch
                tdt = torch.float64 if self.dtype == C128 else torch.float32
                self._tensor = torch.empty(2 << self.n, dtype=tdt, device="cuda")
                dev_ptr, nbytes = self._tensor.data_ptr(), self._tensor.numel() * self._tensor.element_size()
                cur = torch.cuda.current_stream()
                self.torch_stream = cur if cur.cuda_stream != 0 else torch.cuda.Stream()
                stream = self.torch_stream.cuda_stream
            _check("ps_create_emulated", L.ps_create_emulated(self.n, self.dtype, self.world, dev_ptr, nbytes, stream,
                                                              ctypes.byref(self._h)))
            nq, nl = ctypes.c_int(), ctypes.c_int()
            L.ps_info(self._h, ctypes.byref(nq), ctypes.byref(nl), None, None, None, None)
            self.n_local = nl.value
            return
        self.emulated = False
        if self.world > 1:
            nid = ctypes.create_string_buffer(bootstrap_nccl_id(self.rank, group), 128)
        dev_ptr, nbytes, stream = None, 0, None
        if torch_memory:
            import torch
            m = (self.world - 1).bit_length()
            nl = self.n - m
            tdt = torch.float64 if self.dtype == C128 else torch.float32
            self._tensor = torch.empty(2 << nl, dtype=tdt, device="cuda")
            dev_ptr = self._tensor.data_ptr()
            nbytes = self._tensor.numel() * self._tensor.element_size()
            cur = torch.cuda.current_stream()
            # the legacy default stream has handle 0, which libps reads as "make your own":
            # give libps a real torch stream so torch events on it see the work
            self.torch_stream = cur if cur.cuda_stream != 0 else torch.cuda.Stream()
            stream = self.torch_stream.cuda_stream
        _check("ps_create_ex", L.ps_create_ex(self.n, self.dtype, dev_ptr, nbytes, stream, self.rank, self.world,
                                              nid, ctypes.byref(self._h)))
        nq, nl = ctypes.c_int(), ctypes.c_int()
        L.ps_info(self._h, ctypes.byref(nq), ctypes.byref(nl), None, None, None, None)
        self.n_local = nl.value

    # lifetime
    def close(self):
        if self._h:
            lib().ps_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def np_dtype(self):
        return np.complex128 if self.dtype == C128 else np.complex64

    def set_option(self, opt: int, value: int):
        _check("ps_set_option", lib().ps_set_option(self._h, opt, int(value)))

    # init / access
    def init_basis(self, index: int = 0):
        _check("ps_init_basis", lib().ps_init_basis(self._h, int(index)))

    def init_random(self, seed: int):
        _check("ps_init_random", lib().ps_init_random(self._h, int(seed)))

    def normalize(self):
        _check("ps_normalize", lib().ps_normalize(self._h))

    def set_state(self, amps, first: int = 0):
        a = np.ascontiguousarray(amps, dtype=self.np_dtype)
        _check("ps_set_state", lib().ps_set_state(self._h, int(first), a.size, _p(a)))

    def set_state_ptr(self, host_ptr: int, count: int, first: int = 0):
        _check("ps_set_state", lib().ps_set_state(self._h, int(first), int(count), ctypes.c_void_p(host_ptr)))

    def get_amplitudes(self, first: int = 0, count: int | None = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - first
        out = np.zeros(int(count), dtype=self.np_dtype)
        _check("ps_get_amplitudes", lib().ps_get_amplitudes(self._h, int(first), int(count), _p(out)))
        return out

    # hot path
    def apply_rotations(self, x, z, angles):
        x, z, a = _u64(x), _u64(z), _f64(angles)
        if not (len(x) == len(z) == len(a)):
            raise ValueError("x, z, angles must have equal length")
        _check("ps_apply_rotations", lib().ps_apply_rotations(self._h, _p(x), _p(z), _p(a), len(a)))

    def apply_codes(self, codes, angles):
        x, z = pauli_encode_codes(codes)
        self.apply_rotations(x, z, angles)

    def norm(self) -> float:
        out = ctypes.c_double()
        _check("ps_norm", lib().ps_norm(self._h, ctypes.byref(out)))
        return out.value

    def expectation(self, x, z, coeffs) -> float:
        x, z, c = _u64(x), _u64(z), _f64(coeffs)
        out = ctypes.c_double()
        _check("ps_expectation", lib().ps_expectation(self._h, _p(x), _p(z), _p(c), len(c), ctypes.byref(out)))
        return out.value

    def inner(self, other: "State") -> complex:
        out = np.zeros(2)
        _check("ps_inner", lib().ps_inner(self._h, other._h, _p(out)))
        return complex(out[0], out[1])

    def synchronize(self):
        _check("ps_synchronize", lib().ps_synchronize(self._h))

    def stats(self) -> dict:
        s = Stats()
        _check("ps_get_stats", lib().ps_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check("ps_reset_stats", lib().ps_reset_stats(self._h))
