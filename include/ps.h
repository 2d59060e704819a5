/*
 * ps.h -- C ABI of libps: full-state-vector simulation of Pauli-rotation layers on B200.
 *
 * The hot path of arXiv 2504.17881 ("phase2"): starting from a state |psi>, apply the sequence
 * of Pauli rotations exp(i phi P) (Introduction), each by the closed form
 * exp(i phi P) = cos(phi) I + i sin(phi) P, with P encoded as two 64-bit masks
 * (P:116-121).  One process per GPU; the state is partitioned over G = 2^m GPUs by its
 * top m qubits (Mathematical model).
 *
 * Citations "P:n" are PAPER.md line numbers; "S:n" SPEC.md line numbers; readings of ambiguous
 * passages are numbered R1.. in DESIGN.md.
 *
 * Conventions (all entry points)
 *   - Qubit q (0-based) is factor P_{q+1} of the string and bit q of the basis index.
 *   - Pauli string masks: xmask bit q set iff P_{q+1} in {X, Y}  (the paper's p1);
 *                         zmask bit q set iff P_{q+1} in {Y, Z}  (the paper's p2).
 *   - Amplitude storage: interleaved (re, im) of the handle's element type:
 *       PS_C128 -> two doubles per amplitude (the paper's C99 _Complex double),
 *       PS_C64  -> two floats per amplitude.
 *   - Rotation order: angle[0] is applied first: U = R_{count-1} ... R_1 R_0 (R7).
 *   - Multi-GPU (world > 1): every call is SPMD-collective -- all ranks call it with identical
 *     arguments (like MPI).  Index ranges are GLOBAL logical indices; rank r owns
 *     [r*2^(n-m), (r+1)*2^(n-m)) at every call boundary.
 *   - Errors: every entry point returns a ps_status (0 = PS_OK).  Arguments are validated before
 *     any device work, so a call that fails validation leaves the state unchanged.  An
 *     asynchronous CUDA or NCCL fault poisons the handle: later calls return PS_ESTATE.
 *     ps_last_error() gives a thread-local message for the last failure.
 *   - Ownership: the library owns handles and (unless ps_create_ex is given a buffer) the state
 *     memory.  Input arrays are borrowed for the duration of the call only.  Output buffers are
 *     caller-allocated.  One handle per host thread; no internal locking.
 *   - Stream semantics: device work is enqueued on the handle's stream.  ps_apply_rotations and
 *     ps_init_* return once the work is enqueued; ps_synchronize, ps_norm, ps_expectation,
 *     ps_inner, ps_get_amplitudes block until their result is available.
 */
#ifndef PS_H
#define PS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ps_state *ps_handle; /* opaque; owned by the library */

typedef enum { PS_C128 = 0, PS_C64 = 1 } ps_dtype;

typedef enum {
    PS_OK = 0,
    PS_EINVAL = -1,      /* bad argument: NULL with count > 0, n out of range, non-finite angle, bad letter */
    PS_ERANGE = -2,      /* mask bit >= n, or index range beyond 2^n */
    PS_ENOMEM = -3,      /* device or host allocation failed */
    PS_ECUDA = -4,       /* CUDA runtime error */
    PS_ENCCL = -5,       /* NCCL error */
    PS_ESTATE = -6,      /* handle poisoned by an earlier asynchronous fault */
    PS_EUNSUPPORTED = -7 /* valid request this build cannot serve (e.g. world > 1 without NCCL) */
} ps_status;

/* kernel families counted in ps_stats */
enum {
    PS_K_STREAM = 0,   /* K1: streaming pair-rotation pass (single rotation or same-x run)   */
    PS_K_TILE = 1,     /* K2: low-qubit fused tile pass (contiguous 2^k tile: gathered into registers,
                          shared memory between sub-groups; TMA only in the A/B modes)       */
    PS_K_COSET = 2,    /* K7: coset-tile fused pass (gathered 2^k tile)                       */
    PS_K_REDUCE = 3,   /* K5: norm / expectation / inner-product reductions                   */
    PS_K_INIT = 4,     /* K6: state initialisation                                            */
    PS_K_EXCHANGE = 5, /* K3: half-vector exchange (NVLink P2P swap or NCCL send/recv)       */
    PS_K_PERMUTE = 6,  /* local qubit transposition pass (restoring the canonical layout)     */
    PS_K_MIRROR = 7,   /* PS_OPT_LAYOUT=2: butterfly / recombine passes of Eq. (core_state)    */
    PS_K_XTILE = 8,    /* K8: fused half-vector exchange + tile pass (PS_OPT_FUSED_EXCHANGE)    */
    PS_K_COUNT = 9
};

/* extra plan-op kinds (ps_plan_describe only): the paper's three-step grouped execution */
enum {
    PS_OP_MIRROR_BEGIN = 16,  /* B <- conj(w_k) A_(k xor gx) (full exchange), butterfly A,B     */
    PS_OP_MIRROR_SWITCH = 17, /* following passes act on B (with negated angles)              */
    PS_OP_MIRROR_END = 18     /* A <- (A + B)/sqrt(2); passes act on A again                  */
};

typedef struct ps_stats {
    uint64_t rotations;                  /* rotations applied since the last reset */
    uint64_t passes;                     /* HBM passes over the local state (all kernel families) */
    uint64_t exchanges;                  /* half-vector exchanges, counting the swap-back */
    uint64_t launches[PS_K_COUNT];       /* kernel launches per family */
    uint64_t rotations_by[PS_K_COUNT];   /* rotations applied per family */
    double algo_bytes[PS_K_COUNT];       /* algorithmic HBM bytes per family (2*2^n_l*s per pass) */
    double nvlink_bytes;                 /* bytes sent to each peer by swap exchanges and mirror
                                            fetches, per direction (PS_K_EXCHANGE time) */
    double kernel_ms[PS_K_COUNT];        /* device time per family (CUDA events; PS_OPT_PROFILE=1 only) */
    double nvlink_fused_bytes;           /* bytes read from the partner by fused exchange + tile
                                            passes (PS_K_XTILE time) */
} ps_stats;

/* options for ps_set_option */
enum {
    PS_OPT_PROFILE = 0,       /* 1: time every launch with CUDA events on the handle's stream (default 0) */
    PS_OPT_FUSION = 1,        /* 0: one rotation per pass (K1 only); 1: same-x runs; 2: + tiles (default 2) */
    PS_OPT_TILE_BITS = 2,     /* log2 amplitudes per fused tile, 4..13 for C128 (default 12),
                                 4..14 for C64 (default 12); 2^13 / 2^14 tiles run one CTA of
                                 512 / 1024 threads per SM */
    PS_OPT_CHUNK_BYTES = 3,   /* exchange chunk size in bytes (default 256 MiB) */
    PS_OPT_MAX_PASS_ROTS = 4, /* cap on rotations fused into one tile pass (default: no cap) */
    PS_OPT_VEC256 = 5,        /* 1: 256-bit LDG/STG in K1 (default 1); 0: 128-bit */
    PS_OPT_TILE_TMA = 6,      /* tile-pass kernel: 2 = register-direct (default): first sub-group
                                 loads from HBM, last stores to HBM, smem between sub-groups;
                                 0 = cp.async-prefetched double buffer; 1 = 3-stage TMA ring;
                                 3 = TMA-bulk-prefetched double buffer (A/B) */
    PS_OPT_CHUNK_BITS = 7,    /* min log2 contiguous amplitudes per gathered chunk (0 = default 4:
                                 256 B for C128, 128 B for C64) */
    PS_OPT_TILE_TUNE = 8,     /* register-direct tile kernel tuning bits: 1-3 = CTAs per SM (0 per-dtype
                                 default: fp64 uncapped = 2, fp32 8; 1/2/3 register cap for 5/6/8
                                 CTAs of 128 threads), 4-7 = persistent-grid multiplier (default 4),
                                 9 = L2::256B sector promotion on the gathered loads, 10 = the pass's
                                 records in the launch's parameter block (uniform constant loads;
                                 passes of <= 256 rotations), 11 = LDGSTS prefetch of the next tile's
                                 first sub-group into shared memory while the current tile's last
                                 sub-group is computed and stored (default C128 3584 = bits
                                 9 + 10 + 11, C64 1536 = bits 9 + 10) */
    PS_OPT_LAYOUT = 9,        /* world > 1: 1 = lazy qubit-swap layout kept across calls, swaps chosen
                                 by furthest next use (default); 0 = one half-vector exchange per run
                                 sharing the upper X-part, swapped back at once (Eq. (1) economy);
                                 2 = the paper's three-step execution: a mirror buffer
                                 per GPU (doubles memory), one full-partition exchange per group
                                 sharing the upper string, butterfly, U+ on A and U- on B,
                                 recombine -- kept for A/B */
    PS_OPT_TRANSPORT = 10,    /* world > 1: 1 = NVLink P2P swap kernel on CUDA-IPC peer pointers when
                                 available (default); 0 = NCCL send/recv with staging */
    PS_OPT_OVERLAP = 11,      /* world > 1, P2P: 2 = each swap overlaps the tile passes before and
                                 after it (default): a chain pass, E, pass, ..., pass runs in 2^B
                                 pieces split by free bits outside every tile, a piece is swapped as
                                 soon as both ranks finished it (pairwise P2P flag barrier) and the
                                 next pass's piece runs as soon as it landed; 1 = only with the pass
                                 after it; 0 = serialise; bits 16-18 = B + 1 (default B = 2).  Like
                                 every option, it must be set identically on all ranks */
    PS_OPT_SPECIALIZE = 12    /* tile-kernel variant: 2 = specialised (default for C128): CFORM
                                 rotations whose sub-group xor mask dx is a unit vector or 0 run
                                 through one of 80 compile-time cases (per-pair signs and pairing
                                 fixed, no sign flips), the rest generically; 0 = generic (default
                                 for C64: per-pair signs at run time); 1 = planner's per-pass choice
                                 (specialised for passes of >= 16 rotations, half of them unit).
                                 Bitwise-identical results (same operations in the same order) */,
    PS_OPT_GRID_CAP = 13,     /* test knob: cap on the persistent tile grid (CTAs), so small states
                                 run several tiles per CTA (incremental tile bases, next-tile
                                 prefetch); 0 = no cap (default) */
    PS_OPT_FUSED_EXCHANGE = 14 /* world > 1 with peer access (P2P transport or emulation): 1 = a
                                 half-vector exchange followed by a tile pass runs as ONE kernel that
                                 reads the partner's half through the peer pointer and stores in the
                                 new layout, with per-tile release/acquire flags instead of a swap;
                                 0 = swap, then the pass, overlapped on two streams (default: the
                                 fused kernel measured slower, profiles/r02/multi_gpu.md)
                                  */,
    PS_OPT_SWAP_CTAS = 15     /* overlapped swap pieces: the slim swap kernel (128 threads, <= 64
                                 registers, fits next to the tile kernel's resident CTAs) with
                                 -k CTAs per SM for -8 <= -k < 0 or k CTAs for -k < -8; 0 = default
                                 (2 per SM); k > 0 = k full-size CTAs (512 threads: wait for whole
                                 SMs) */,
    PS_OPT_SWAP_TMA = 16      /* overlapped swap pieces: 1 = the TMA swap kernel (one thread per CTA
                                 moves 4 KB chunks through a 4-stage shared-memory ring with
                                 cp.async.bulk loads of the partner's and its own chunk and crosswise
                                 bulk stores; default) where the piece's contiguous runs are >= 1 KB,
                                 else the slim register kernel; 0 = always the register kernel */
};

/* ------------------------------------------------------------------------------------------ */
/* Lifetime                                                                                    */

/* Single GPU on the current CUDA device.  n_qubits in [1, 62] (memory permitting: 2^n amplitudes).
 * The state is allocated (2^n * 16 B for PS_C128) and set to |0>. */
int ps_create(int n_qubits, int dtype, ps_handle *out);

/* General constructor.
 *   dev_buf/bytes: optional caller-owned device buffer holding the LOCAL slice
 *                  (2^(n-m) amplitudes); NULL -> the library allocates.  The caller keeps it
 *                  alive until ps_destroy.
 *   stream:        optional cudaStream_t to enqueue on (e.g. torch's current stream); NULL ->
 *                  the library creates a non-blocking stream.
 *   rank, world:   this process's rank and the number of GPUs G = 2^m, 1 <= G, G | 2^(n-1)
 *                  (M = 2^m tasks, one per GPU).
 *   nccl_id:       128-byte ncclUniqueId from ps_get_unique_id on rank 0, broadcast by the
 *                  caller (torch.distributed); ignored when world == 1.
 * The state is set to |0>. */
int ps_create_ex(int n_qubits, int dtype, void *dev_buf, size_t bytes, void *stream, int rank,
                 int world, const void *nccl_id, ps_handle *out);

/* Rank emulation on ONE device (tests and single-GPU evidence of the multi-GPU path): the state is
 * split into `world` = G = 2^m slices of one device buffer (dev_buf, or library-owned when NULL;
 * 2^n amplitudes, slice r = global indices [r 2^(n-m), (r+1) 2^(n-m)) as on G GPUs), each driven by
 * a virtual rank with its own plan (per-rank signs and exchange sides), its own records
 * and the same kernels as a real rank; peer pointers are the other slices, NCCL barriers become
 * stream order on `stream` (NULL: the library creates one), all-reduces become host sums.  The
 * virtual ranks run their plans pass by pass in lockstep (two phases where ranks read each other's
 * data; one launch over all ranks for the fused exchange).  The handle is used like a single
 * state: calls are NOT collective, index ranges are global, ps_get_stats reports rank 0's
 * counters.  Transport is always peer access (PS_OPT_TRANSPORT is ignored) and the two-stream
 * overlap is off.  world in [1, 8] for the fused exchange kernel (larger groups fall back to
 * swaps).  The state is set to |0>. */
int ps_create_emulated(int n_qubits, int dtype, int world, void *dev_buf, size_t bytes, void *stream,
                       ps_handle *out);

/* Convenience: ps_create_ex with library-owned memory and stream. */
int ps_create_dist(int n_qubits, int dtype, int rank, int world, const void *nccl_id,
                   ps_handle *out);

/* Writes a fresh 128-byte ncclUniqueId into out (host only; call on rank 0). */
int ps_get_unique_id(void *out);

int ps_destroy(ps_handle h);

/* Introspection: qubits, local qubits n-m, rank, world, dtype, device pointer of the local slice. */
int ps_info(ps_handle h, int *n_qubits, int *n_local, int *rank, int *world, int *dtype,
            void **dev_ptr);

int ps_set_option(ps_handle h, int option, int64_t value);

/* ------------------------------------------------------------------------------------------ */
/* State initialisation and access (a7 row; P:519 random init for benchmarks, P:625 basis
 * states for guiding states)                                                                  */

/* |index>: all amplitudes zero except a_index = 1.  PS_ERANGE if index >= 2^n. */
int ps_init_basis(ps_handle h, uint64_t index);

/* Unnormalised seeded amplitudes a_i = u(seed, 2i) + i u(seed, 2i+1) with the counter-based
 * generator of DESIGN.md "Input recipe" (values in [-1, 1), exact in fp64; rounded once to fp32
 * for PS_C64).  Identical for any world size. */
int ps_init_random(ps_handle h, uint64_t seed);

/* Scales the state to unit norm (one reduction + one scaling pass). */
int ps_normalize(ps_handle h);

/* Copies count amplitudes from host memory amps (interleaved, handle dtype) into global indices
 * [first, first+count).  Every rank passes the same data; each keeps the part it owns.
 * PS_ERANGE if first+count > 2^n.  Pinned host memory gives full PCIe bandwidth. */
int ps_set_state(ps_handle h, uint64_t first, uint64_t count, const void *amps);

/* Copies global indices [first, first+count) to host memory amps_out (interleaved, handle
 * dtype).  With world > 1 the result appears on every rank.  Blocks. */
int ps_get_amplitudes(ps_handle h, uint64_t first, uint64_t count, void *amps_out);

/* ------------------------------------------------------------------------------------------ */
/* The hot path                                                                                */

/* Applies exp(i angle[l] P_l) for l = 0 .. count-1 in that order, P_l given by
 * (xmask[l], zmask[l]).  Pairs (i, i xor xmask) are updated by
 *   a'_i = cos(phi) a_i + i sin(phi) w(i xor x) a_(i xor x),
 *   w(i) = i^(popc(x & z) mod 4) (-1)^(popc(z & i))            (R3),
 * a direct sum of 2x2 blocks.  xmask = zmask = 0 is the global phase e^{i phi} (R5).
 * Rotations are grouped into HBM passes (same-x runs, fused tiles) and, for
 * world > 1, rotations whose xmask touches the top m qubits run after a pairwise half-vector
 * exchange with rank r xor gx (Eq. (1)); z-only support on the top qubits
 * becomes a per-rank sign.  The result equals the sequential product up to fp
 * rounding.  PS_EINVAL on NULL arrays with count > 0 or a non-finite angle; PS_ERANGE on a mask
 * bit >= n. */
int ps_apply_rotations(ps_handle h, const uint64_t *xmask, const uint64_t *zmask,
                       const double *angle, size_t count);

/* out = sum_i |a_i|^2 over all ranks, fp64 accumulation.  Blocks. */
int ps_norm(ps_handle h, double *out);

/* out = sum_l coeff[l] * Re <psi|P_l|psi> over all ranks (P:560-566 H = sum h_l P_l),
 * fp64 accumulation; terms sharing an xmask share one read pass.  Blocks. */
int ps_expectation(ps_handle h, const uint64_t *xmask, const uint64_t *zmask,
                   const double *coeff, size_t count, double *out);

/* out[0] + i out[1] = <a|b> = sum_i conj(a_i) b_i (the overlap behind Z_m).
 * a and b must have equal n, dtype and world.  Blocks. */
int ps_inner(ps_handle a, ps_handle b, double *out_re_im);

int ps_synchronize(ps_handle h);

int ps_get_stats(ps_handle h, ps_stats *out);
int ps_reset_stats(ps_handle h);

const char *ps_status_string(int code);
const char *ps_last_error(void);

/* ------------------------------------------------------------------------------------------ */
/* Host-only helpers (no GPU needed)                                                           */

/* Pauli word (letters I, X, Y, Z; leftmost = P_1 = qubit 0; length 1..64) -> masks.
 * "XIY" -> (5, 4).  PS_EINVAL on an empty word, a bad letter or length > 64. */
int ps_pauli_encode(const char *word, uint64_t *xmask, uint64_t *zmask);

/* Batch form: codes[l*n + q] in {0=I, 1=X, 2=Y, 3=Z} for qubit q of string l. */
int ps_pauli_encode_codes(const uint8_t *codes, int n, size_t count, uint64_t *xmask,
                          uint64_t *zmask);

/* Standard gate -> Pauli rotations under the paper's exp(+i phi P) convention (R1), universality
 * P:12.  gate: "H","S","T","X","Y","Z","RX","RY","RZ","CNOT"/"CX","CZ","SWAP",
 * "CPHASE","RZZ" (case-insensitive); qubits[0] = control / first qubit; params: angle for
 * RX/RY/RZ/CPHASE/RZZ.  The global phase is emitted as an identity-string rotation (x = z = 0), so
 * the product of the emitted rotations equals the gate matrix exactly (up to rounding).
 * Writes *n_out rotations (<= cap; 7 suffices) in application order.  PS_EINVAL on an unknown
 * gate or bad qubits, PS_ERANGE if cap is too small. */
int ps_gate_to_rotations(const char *gate, const int *qubits, int n_qubits_gate,
                         const double *params, int n_params, uint64_t *xmask, uint64_t *zmask,
                         double *angle, size_t cap, size_t *n_out);

/* Planner dump (host only; for tests and plan inspection).  Plans `count` rotations for an
 * n-qubit state on `world` GPUs as seen by `rank`, with the given fusion level, tile bits and
 * layout policy (PS_OPT_LAYOUT), starting from and returning to the canonical layout, and writes
 * up to cap ops.  Each op is one HBM pass, one exchange or one local transposition; for a pass,
 * the rotations it applies are given in PHYSICAL local coordinates. */
typedef struct ps_plan_op {
    int32_t kind;        /* PS_K_STREAM, PS_K_TILE, PS_K_COSET, PS_K_EXCHANGE, PS_K_PERMUTE or
                            PS_OP_MIRROR_*; MIRROR_BEGIN carries gx in exch_gx and the upper
                            Z-part in tile_bits (low 32 bits) */
    int32_t first_rot;   /* index of the first input rotation covered */
    int32_t n_rot;       /* rotations applied by this op (EXCHANGE: 0, or 1 for a full exchange) */
    int32_t exch_bit;    /* EXCHANGE: local pivot bit l swapped with the partner (-1: full exchange);
                            PERMUTE: first local bit of the transposition */
    uint64_t exch_gx;    /* EXCHANGE: partner = rank xor exch_gx; PERMUTE: second local bit */
    uint32_t tile_bits;  /* TILE/COSET: log2 tile size */
    uint32_t n_sub;      /* TILE/COSET: register sub-groups the pass is split into */
} ps_plan_op;

/* Physical rotation record as executed (one per rotation per pass, in order). */
typedef struct ps_plan_rot {
    uint64_t x;   /* physical local xor mask */
    uint64_t z;   /* physical local phase mask */
    int32_t y;    /* i^y factor of the ORIGINAL string, popc(x & z) mod 4 of the logical masks */
    int32_t sign; /* +1/-1: per-rank sign folded into sin(phi) */
    double angle; /* phi */
} ps_plan_rot;

int ps_plan_describe(int n_qubits, int world, int rank, int fusion, int tile_bits, int layout,
                     const uint64_t *xmask, const uint64_t *zmask, const double *angle,
                     size_t count, ps_plan_op *ops, size_t ops_cap, size_t *n_ops,
                     ps_plan_rot *rots, size_t rots_cap, size_t *n_rots);

#ifdef __cplusplus
}
#endif

#endif /* PS_H */
