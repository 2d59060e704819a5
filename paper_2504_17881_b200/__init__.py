"""B200-native full-state-vector simulation of Pauli-rotation layers (arXiv 2504.17881, "phase2").

The hot path lives in libps.so (C ABI in include/ps.h, CUDA kernels for sm_100a in csrc/);
``paper_2504_17881_b200.ps`` is its thin ctypes binding.
"""
from .ps import (State, PsError, pauli_encode, pauli_encode_codes, gate_to_rotations, circuit_to_rotations,
                 plan_describe, lib)

__all__ = ["State", "PsError", "pauli_encode", "pauli_encode_codes", "gate_to_rotations", "circuit_to_rotations",
           "plan_describe", "lib"]
