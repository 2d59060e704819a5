// api.cpp -- the C ABI of libps (include/ps.h): handles, device memory, streams, NCCL, and the
// execution of plans produced by planner.cpp.  Argument marshalling and orchestration only;
// every step of the path runs in the kernels of kernels.cu (or NCCL for exchanges).
//
// Rank sets.  Every operation runs on a RANK SET: one handle for a real rank (one process per
// GPU, collectives over NCCL), or the G virtual ranks of an emulation group (ps_create_emulated:
// G slices of one device buffer, the same planner, plans and kernels, peer pointers into the
// other slices, stream order instead of NCCL barriers and host sums instead of all-reduces).
// The virtual ranks of a group execute their plans pass by pass in lockstep; a pass whose
// ranks read each other's data (full exchange, mirror fetch) runs as two phases over all ranks,
// and the fused exchange + tile pass runs as one kernel over all ranks' slices.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ps_internal.h"

namespace ps {

// kernels.cu
int kernel_max_red_blocks();
cudaError_t launch_stream(int dtype, void* a, int nl, const Pass& p, const DevRot* d_rots, int vec256,
                          cudaStream_t s);
cudaError_t launch_tile(int dtype, void* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                        const uint64_t* d_offs, int use_tma, int tune, cudaStream_t s, const DevSub* h_subs,
                        const DevTRot* h_trots, int grid_cap);
cudaError_t launch_full_update(int dtype, void* a, const void* stage, uint64_t base, uint64_t count, uint64_t pbase,
                               const DevRot* rec, cudaStream_t s);
cudaError_t launch_norm(int dtype, const void* a, uint64_t n, double* d_partial, double* d_out, cudaStream_t s);
cudaError_t launch_inner(int dtype, const void* a, const void* b, uint64_t n, double* d_partial, double* d_out,
                         cudaStream_t s);
cudaError_t launch_expect(int dtype, const void* a, uint64_t n, uint64_t x0, const DevTerm* terms, int nt,
                          double* d_partial, double* d_out_slot, cudaStream_t s);
cudaError_t launch_expect_cross(int dtype, const void* a, const void* stage, uint64_t base, uint64_t count,
                                uint64_t pbase, uint64_t xl, uint64_t zl, int y, int sgn, double* d_partial,
                                double* d_out_slot, cudaStream_t s);
cudaError_t launch_init_random(int dtype, void* a, uint64_t n, uint64_t seed, uint64_t goff, cudaStream_t s);
cudaError_t launch_set_one(int dtype, void* a, uint64_t idx, cudaStream_t s);
cudaError_t launch_scale(int dtype, void* a, uint64_t n, double f, cudaStream_t s);
cudaError_t launch_permute(int dtype, void* a, int nl, int b1, int b2, cudaStream_t s);
cudaError_t launch_butterfly(int dtype, void* A, void* B, uint64_t n, int wr, int wi, cudaStream_t s);
cudaError_t launch_recombine(int dtype, void* A, const void* B, uint64_t n, cudaStream_t s);
cudaError_t launch_p2p_copy(int dtype, void* dst, const void* src, uint64_t n, cudaStream_t s);
cudaError_t launch_pair_barrier(const uint32_t* mine, uint32_t* theirs, uint32_t epoch, cudaStream_t s);
cudaError_t launch_p2p_swap(int dtype, void* local, void* peer, uint64_t rows, uint64_t row_amps, uint64_t my_off,
                            uint64_t peer_off, uint64_t t0, uint64_t t1, uint64_t fmask, uint64_t fval,
                            cudaStream_t s, int ctas, int tma_chunk = 0);
cudaError_t launch_xtile(int dtype, const XTileRank* ranks, int nranks, const Pass& p, const uint64_t* d_offs,
                         const uint64_t* h_offs, int ell, uint32_t epoch, cudaStream_t s, int grid_cap);

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace ps

using namespace ps;

struct PendingTiming {
    int kind;
    cudaEvent_t e0, e1;
};

struct ps_state {
    int n = 0, nl = 0, rank = 0, world = 1, dtype = PS_C128;
    size_t amp_bytes = 16;
    int device = 0;
    void* d_state = nullptr;
    bool own_state = false;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool poisoned = false;
    // emulation: a virtual rank of a group (no NCCL; peers = the group's other slices), or the
    // group handle itself (vranks = its virtual ranks in rank order)
    bool emulated = false;
    std::vector<ps_state*> vranks;
    bool is_group() const { return !vranks.empty(); }
    // per-call plan buffers
    DevRot* d_rots = nullptr;
    size_t d_rots_cap = 0;
    uint64_t* d_offs = nullptr;
    size_t d_offs_cap = 0;
    DevSub* d_subs = nullptr;
    size_t d_subs_cap = 0;
    DevTRot* d_trots = nullptr;
    size_t d_trots_cap = 0;
    void* h_stage[2] = {nullptr, nullptr};
    size_t h_stage_cap[2] = {0, 0};
    cudaEvent_t h_stage_ev[2] = {nullptr, nullptr};
    int stage_flip = 0;
    // reductions
    double* d_partial = nullptr;
    double* d_result = nullptr;  // 64 doubles
    double* h_result = nullptr;  // pinned, 64 doubles
    DevTerm* d_terms = nullptr;
    size_t d_terms_cap = 0;
    // multi-GPU
    ncclComm_t comm = nullptr;
    void* d_xstage[2] = {nullptr, nullptr};
    size_t xstage_bytes = 0;
    size_t chunk_bytes = 256ull << 20;
    // layout (world > 1): physical bit -> logical qubit; identity = canonical
    std::vector<int> perm;
    int* d_barrier = nullptr;
    std::vector<void*> peers;  // peer pointers to every rank's local slice (CUDA IPC, or the group's slices)
    std::vector<void*> peer_bases;
    bool p2p = false;
    // fused exchange + tile pass (PS_OPT_FUSED_EXCHANGE): per-tile handshake flags of every rank
    uint32_t* d_flags = nullptr;
    size_t flags_cap = 0;
    std::vector<uint32_t*> peer_flags;
    uint32_t epoch = 0;
    // pairwise P2P barriers (overlapped swaps): words [flag_words + src * kBarSlots + slot] of a
    // rank's d_flags are raised by rank src; bar_epoch[partner * kBarSlots + slot] counts the uses
    static constexpr int kBarSlots = 4;
    std::vector<uint32_t> bar_epoch;
    int fused = 0;  // off by default: measured slower than swap + overlap (profiles/r02/multi_gpu.md)
    void* d_mirror = nullptr;  // PS_OPT_LAYOUT=2 mirror buffer B_k
    cudaStream_t xstream = nullptr;  // second stream: swaps overlapped with the next pass
    static constexpr int kMaxPieceBits = 3;
    static constexpr int kXev = 2 + 2 * (1 << kMaxPieceBits);  // overlap mode 2 uses 1 + 2P events
    cudaEvent_t xev[kXev] = {};
    int overlap = 2;      // PS_OPT_OVERLAP (2: the swap overlaps the passes before and after it)
    int swap_tma = 1;     // PS_OPT_SWAP_TMA: overlapped swap pieces through the TMA swap kernel
    int swap_ctas = -2;   // overlapped swap pieces: < 0 the slim kernel that co-resides with the
                          // tile kernel (-k: k per SM if k <= 8, else k CTAs), > 0 full-size CTAs
    int piece_bits = 2;   // an overlapped swap/pass pair runs in up to 2^piece_bits pieces
    const Plan* cur_plan = nullptr;  // the plan being executed (host copies of its records)
    int layout = 1, transport = 1;
    int specialize = 0;
    int grid_cap = 0;
    // options
    int profile = 0, fusion = 2, tile_bits = 11, vec256 = 1, max_pass_rots = 1 << 30, tile_tma = 2, chunk_bits = 0, tile_tune = 1536;
    ps_stats stats{};
    std::vector<PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    Plan plan;  // reused
};

using RankSet = std::vector<ps_state*>;

// ------------------------------------------------------------------------------------------
// error helpers

static int fail(int code, const std::string& msg) {
    set_last_error(msg);
    return code;
}

#define CUDA_TRY(h, expr)                                                                          \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            if ((h) && _e != cudaErrorMemoryAllocation && _e != cudaErrorInvalidValue)             \
                (h)->poisoned = true;                                                              \
            return fail(_e == cudaErrorMemoryAllocation ? PS_ENOMEM : PS_ECUDA,                    \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                       \
        }                                                                                          \
    } while (0)

#define NCCL_TRY(h, expr)                                                                          \
    do {                                                                                           \
        ncclResult_t _r = (expr);                                                                  \
        if (_r != ncclSuccess) {                                                                   \
            if (h) (h)->poisoned = true;                                                           \
            return fail(PS_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));             \
        }                                                                                          \
    } while (0)

static bool any_poisoned(ps_state* h) {
    if (h->poisoned) return true;
    for (ps_state* v : h->vranks)
        if (v->poisoned) return h->poisoned = true;
    return false;
}

#define CHECK_HANDLE(h)                                                                            \
    do {                                                                                           \
        if (!(h)) return fail(PS_EINVAL, "NULL handle");                                           \
        if (any_poisoned(h)) return fail(PS_ESTATE, "handle poisoned by an earlier fault");        \
        cudaSetDevice((h)->device);                                                                \
    } while (0)

static RankSet ranks_of(ps_state* h) { return h->is_group() ? h->vranks : RankSet{h}; }

static void poison_all(const RankSet& rs) {
    for (ps_state* r : rs) r->poisoned = true;
}

static cudaEvent_t get_event(ps_state* h) {
    if (!h->event_pool.empty()) {
        cudaEvent_t e = h->event_pool.back();
        h->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// CUDA events around a launch on the stream it runs on (PS_OPT_PROFILE)
struct Timed {
    ps_state* h;
    int kind;
    cudaStream_t st;
    cudaEvent_t e0 = nullptr;
    Timed(ps_state* hh, int k, cudaStream_t s = nullptr) : h(hh), kind(k), st(s ? s : hh->stream) {
        if (h->profile) {
            e0 = get_event(h);
            cudaEventRecord(e0, st);
        }
    }
    ~Timed() {
        if (h->profile && e0) {
            cudaEvent_t e1 = get_event(h);
            cudaEventRecord(e1, st);
            h->pending.push_back({kind, e0, e1});
        }
    }
};

static void drain_timings(ps_state* h) {
    for (auto& p : h->pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.e1) == cudaSuccess && cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess)
            h->stats.kernel_ms[p.kind] += ms;
        h->event_pool.push_back(p.e0);
        h->event_pool.push_back(p.e1);
    }
    h->pending.clear();
}

template <typename T>
static int ensure_dev(ps_state* h, T** buf, size_t* cap, size_t need) {
    if (need <= *cap) return PS_OK;
    size_t ncap = std::max(need, *cap * 2);
    if (*buf) CUDA_TRY(h, cudaFreeAsync(*buf, h->stream));
    *buf = nullptr;
    CUDA_TRY(h, cudaMallocAsync((void**)buf, ncap * sizeof(T), h->stream));
    *cap = ncap;
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// lifetime

extern "C" int ps_get_unique_id(void* out) {
    if (!out) return fail(PS_EINVAL, "NULL out");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(PS_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return PS_OK;
}

static void free_state(ps_state* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (ps_state* v : h->vranks) free_state(v);
    h->vranks.clear();
    drain_timings(h);
    for (auto e : h->event_pool) cudaEventDestroy(e);
    for (void* b : h->peer_bases)
        if (b) cudaIpcCloseMemHandle(b);
    if (h->d_barrier) cudaFree(h->d_barrier);
    if (h->d_flags) cudaFree(h->d_flags);
    if (h->d_mirror) cudaFree(h->d_mirror);
    if (h->xstream) cudaStreamDestroy(h->xstream);
    for (int t = 0; t < ps_state::kXev; ++t)
        if (h->xev[t]) cudaEventDestroy(h->xev[t]);
    if (h->comm) ncclCommDestroy(h->comm);
    for (int t = 0; t < 2; ++t) {
        if (h->d_xstage[t]) cudaFree(h->d_xstage[t]);
        if (h->h_stage[t]) cudaFreeHost(h->h_stage[t]);
        if (h->h_stage_ev[t]) cudaEventDestroy(h->h_stage_ev[t]);
    }
    if (h->d_rots) cudaFree(h->d_rots);
    if (h->d_offs) cudaFree(h->d_offs);
    if (h->d_subs) cudaFree(h->d_subs);
    if (h->d_trots) cudaFree(h->d_trots);
    if (h->d_terms) cudaFree(h->d_terms);
    if (h->d_partial) cudaFree(h->d_partial);
    if (h->d_result) cudaFree(h->d_result);
    if (h->h_result) cudaFreeHost(h->h_result);
    if (h->own_state && h->d_state) cudaFree(h->d_state);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

static int init_basis_rank(ps_state* h, uint64_t index);
static void reset_layout(ps_state* h);
static int restore_layout(const RankSet& rs);

// CUDA-IPC peer pointers to every rank's local slice and handshake flags: the allocation base is
// exported with its offset (cuMemGetAddressRange through the runtime's driver entry point),
// all-gathered with NCCL
struct IpcRec {
    cudaIpcMemHandle_t handle;
    uint64_t offset;
    cudaIpcMemHandle_t flag_handle;
    int32_t ok;
    int32_t pad;
};

static bool ipc_export(void* ptr, cudaIpcMemHandle_t* handle, uint64_t* offset) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
    typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
    CUdeviceptr base = 0;
    size_t size = 0;
    if (((GetRange)fn)(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return false;
    if (cudaIpcGetMemHandle(handle, (void*)base) != cudaSuccess) return false;
    *offset = (uint64_t)((CUdeviceptr)ptr - base);
    return true;
}

// handshake flags of the fused exchange + tile pass: one 32-bit word per tile of the smallest
// tiles a pass can have (2^4 amplitudes), so every pass's tile index has a word
static size_t flag_words(const ps_state* h) { return (size_t)1 << std::max(0, h->nl - 4); }
static size_t bar_words(const ps_state* h) { return (size_t)h->world * ps_state::kBarSlots; }

static void setup_p2p(ps_state* h) {
    h->p2p = false;
    IpcRec mine{};
    mine.ok = ipc_export(h->d_state, &mine.handle, &mine.offset) ? 1 : 0;
    uint64_t foff = 0;
    if (mine.ok && h->d_flags) mine.ok = ipc_export(h->d_flags, &mine.flag_handle, &foff) && foff == 0;
    cudaGetLastError();
    IpcRec* d_all = nullptr;
    if (cudaMalloc(&d_all, sizeof(IpcRec) * (h->world + 1)) != cudaSuccess) return;
    std::vector<IpcRec> all(h->world);
    bool ok = cudaMemcpyAsync(d_all + h->world, &mine, sizeof(IpcRec), cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
              ncclAllGather(d_all + h->world, d_all, sizeof(IpcRec), ncclChar, h->comm, h->stream) == ncclSuccess &&
              cudaMemcpyAsync(all.data(), d_all, sizeof(IpcRec) * h->world, cudaMemcpyDeviceToHost, h->stream) ==
                  cudaSuccess &&
              cudaStreamSynchronize(h->stream) == cudaSuccess;
    cudaFree(d_all);
    int my_ok = ok ? 1 : 0;
    h->peers.assign(h->world, nullptr);
    h->peer_bases.assign(2 * h->world, nullptr);
    h->peer_flags.assign(h->world, nullptr);
    for (int r = 0; r < h->world && my_ok; ++r) {
        if (!all[r].ok) {
            my_ok = 0;
            break;
        }
        if (r == h->rank) {
            h->peers[r] = h->d_state;
            h->peer_flags[r] = h->d_flags;
            continue;
        }
        void* b = nullptr;
        if (cudaIpcOpenMemHandle(&b, all[r].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            my_ok = 0;
            break;
        }
        h->peer_bases[r] = b;
        h->peers[r] = (char*)b + all[r].offset;
        void* f = nullptr;
        if (cudaIpcOpenMemHandle(&f, all[r].flag_handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            my_ok = 0;
            break;
        }
        h->peer_bases[h->world + r] = f;
        h->peer_flags[r] = (uint32_t*)f;
    }
    // every rank must agree (the transport is collective)
    int* d_flag = h->d_barrier;
    int agree = my_ok;
    if (cudaMemcpyAsync(d_flag, &agree, sizeof(int), cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
        ncclAllReduce(d_flag, d_flag, 1, ncclInt32, ncclMin, h->comm, h->stream) == ncclSuccess &&
        cudaMemcpyAsync(&agree, d_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream) == cudaSuccess &&
        cudaStreamSynchronize(h->stream) == cudaSuccess)
        h->p2p = agree == 1;
    cudaMemsetAsync(d_flag, 0, sizeof(int), h->stream);
    if (!h->p2p) h->fused = 0;
    if (h->p2p) {
        // high priority: swap (and barrier) CTAs are dispatched ahead of the pending CTAs of the
        // persistent tile grid they overlap with
        int lo_prio = 0, hi_prio = 0;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        bool sok = cudaStreamCreateWithPriority(&h->xstream, cudaStreamNonBlocking, hi_prio) == cudaSuccess;
        for (int t = 0; sok && t < ps_state::kXev; ++t)
            sok = cudaEventCreateWithFlags(&h->xev[t], cudaEventDisableTiming) == cudaSuccess;
        if (!sok) {
            cudaGetLastError();
            h->overlap = 0;
        }
    }
}

// one rank's state: device memory (or the caller's), scratch, layout; NCCL and P2P when world > 1
// and the rank is real
static int make_state(int n_qubits, int dtype, void* dev_buf, size_t bytes, void* stream, int rank, int world,
                      const void* nccl_id, bool emulated, ps_state** out) {
    *out = nullptr;
    const int m = __builtin_ctz((unsigned)world);
    ps_state* h = new ps_state();
    h->n = n_qubits;
    h->nl = n_qubits - m;
    h->rank = rank;
    h->world = world;
    h->dtype = dtype;
    h->emulated = emulated;
    h->amp_bytes = dtype == PS_C128 ? 16 : 8;
    // per-dtype defaults (profiles/r01/kernel_ab.md): fp64 2^12 tiles with the next tile's first
    // sub-group prefetched into shared memory (tune bit 11); fp32 2^11 tiles at 8 CTAs per SM,
    // where the prefetch costs more occupancy than it hides
    // 2^12-amplitude tiles for both dtypes (fp32 on 256 threads x 4 CTAs per SM: R10 +5.7 % over
    // 2^11 tiles, JW -1.6 %; profiles/r02/kernel_ab.md section 10)
    h->tile_bits = 12;
    h->tile_tune = dtype == PS_C128 ? (1536 | 2048) : 1536;
    // fp64: unit-dx CFORM rotations with compile-time signs (+6 % R10, +9 % JW, +15 % gates;
    // profiles/r02/kernel_ab.md); fp32 keeps the generic kernel (its 64-register 8-CTA build spills)
    h->specialize = dtype == PS_C128 ? 2 : 0;
    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess) {
        delete h;
        return fail(PS_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    }
    const size_t need = h->amp_bytes << h->nl;
    auto bail = [&](int code, const std::string& msg) {
        free_state(h);
        return fail(code, msg);
    };
    if (stream) {
        h->stream = (cudaStream_t)stream;
    } else {
        e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return bail(PS_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
        h->own_stream = true;
    }
    if (dev_buf) {
        if (bytes < need) return bail(PS_EINVAL, "dev_buf smaller than the local slice");
        // 256-byte aligned (slices smaller than 256 B, e.g. of an emulation group: aligned to their size)
        if (((uintptr_t)dev_buf) & (std::min<size_t>(256, need) - 1))
            return bail(PS_EINVAL, "dev_buf must be 256-byte aligned");
        h->d_state = dev_buf;
    } else {
        e = cudaMalloc(&h->d_state, need);
        if (e != cudaSuccess) return bail(PS_ENOMEM, std::string("cudaMalloc state: ") + cudaGetErrorString(e));
        h->own_state = true;
    }
    const int nred = kernel_max_red_blocks();
    if ((e = cudaMalloc(&h->d_partial, sizeof(double) * 2 * (size_t)nred)) != cudaSuccess ||
        (e = cudaMalloc(&h->d_result, sizeof(double) * 64)) != cudaSuccess ||
        (e = cudaMallocHost(&h->h_result, sizeof(double) * 64)) != cudaSuccess)
        return bail(PS_ENOMEM, std::string("scratch: ") + cudaGetErrorString(e));
    for (int t = 0; t < 2; ++t) {
        if ((e = cudaEventCreateWithFlags(&h->h_stage_ev[t], cudaEventDisableTiming)) != cudaSuccess)
            return bail(PS_ECUDA, std::string("event: ") + cudaGetErrorString(e));
    }
    h->perm.resize(n_qubits);
    for (int q = 0; q < n_qubits; ++q) h->perm[q] = q;
    if (world > 1) {
        // handshake flags of the fused exchange + tile pass (0 = no epoch raised yet)
        if ((e = cudaMalloc(&h->d_flags, sizeof(uint32_t) * (flag_words(h) + bar_words(h)))) != cudaSuccess)
            return bail(PS_ENOMEM, std::string("flags: ") + cudaGetErrorString(e));
        h->flags_cap = flag_words(h);
        h->bar_epoch.assign(bar_words(h), 0);
        if ((e = cudaMemsetAsync(h->d_flags, 0, sizeof(uint32_t) * (h->flags_cap + bar_words(h)), h->stream)) !=
            cudaSuccess)
            return bail(PS_ECUDA, std::string("flags: ") + cudaGetErrorString(e));
    }
    if (world > 1 && !emulated) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, 128);
        ncclResult_t r = ncclCommInitRank(&h->comm, world, id, rank);
        if (r != ncclSuccess) return bail(PS_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        if ((e = cudaMalloc(&h->d_barrier, sizeof(int) * 4)) != cudaSuccess)
            return bail(PS_ENOMEM, std::string("barrier: ") + cudaGetErrorString(e));
        // stream-ordered before setup_p2p's copies and all-reduces on the same words
        if ((e = cudaMemsetAsync(h->d_barrier, 0, sizeof(int) * 4, h->stream)) != cudaSuccess)
            return bail(PS_ECUDA, std::string("barrier: ") + cudaGetErrorString(e));
        setup_p2p(h);  // best effort; NCCL send/recv otherwise
    }
    if (emulated) h->overlap = 0;  // one stream per group; the fused kernel replaces the overlap
    int rc = init_basis_rank(h, 0);
    if (rc) {
        std::string msg = ps_last_error();
        free_state(h);
        return fail(rc, msg);
    }
    *out = h;
    return PS_OK;
}

static int check_create_args(int n_qubits, int dtype, int rank, int world) {
    if (dtype != PS_C128 && dtype != PS_C64) return fail(PS_EINVAL, "dtype must be PS_C128 or PS_C64");
    if (world < 1 || (world & (world - 1)) || world > (1 << 20)) return fail(PS_EINVAL, "world must be a power of two");
    if (rank < 0 || rank >= world) return fail(PS_EINVAL, "rank out of range");
    const int m = __builtin_ctz((unsigned)world);
    if (n_qubits < 1 || n_qubits > 62) return fail(PS_EINVAL, "n_qubits must be in [1, 62]");
    if (n_qubits - m < 1) return fail(PS_EINVAL, "need at least one local qubit (n - log2(world) >= 1)");
    return PS_OK;
}

extern "C" int ps_create_ex(int n_qubits, int dtype, void* dev_buf, size_t bytes, void* stream, int rank,
                            int world, const void* nccl_id, ps_handle* out) {
    if (!out) return fail(PS_EINVAL, "NULL out");
    *out = nullptr;
    int rc = check_create_args(n_qubits, dtype, rank, world);
    if (rc) return rc;
    if (world > 1 && !nccl_id) return fail(PS_EINVAL, "world > 1 needs an NCCL unique id");
    return make_state(n_qubits, dtype, dev_buf, bytes, stream, rank, world, nccl_id, false, out);
}

extern "C" int ps_create_dist(int n_qubits, int dtype, int rank, int world, const void* nccl_id, ps_handle* out) {
    return ps_create_ex(n_qubits, dtype, nullptr, 0, nullptr, rank, world, nccl_id, out);
}

extern "C" int ps_create(int n_qubits, int dtype, ps_handle* out) {
    return ps_create_ex(n_qubits, dtype, nullptr, 0, nullptr, 0, 1, nullptr, out);
}

extern "C" int ps_create_emulated(int n_qubits, int dtype, int world, void* dev_buf, size_t bytes, void* stream,
                                  ps_handle* out) {
    if (!out) return fail(PS_EINVAL, "NULL out");
    *out = nullptr;
    int rc = check_create_args(n_qubits, dtype, 0, world);
    if (rc) return rc;
    ps_state* g = new ps_state();
    g->n = n_qubits;
    g->nl = n_qubits - __builtin_ctz((unsigned)world);
    g->world = world;
    g->dtype = dtype;
    g->amp_bytes = dtype == PS_C128 ? 16 : 8;
    cudaError_t e = cudaGetDevice(&g->device);
    auto bail = [&](int code, const std::string& msg) {
        free_state(g);
        return fail(code, msg);
    };
    if (e != cudaSuccess) return bail(PS_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    const size_t slice = g->amp_bytes << g->nl, need = slice * (size_t)world;
    if (stream) {
        g->stream = (cudaStream_t)stream;
    } else {
        e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return bail(PS_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
        g->own_stream = true;
    }
    if (dev_buf) {
        if (bytes < need) return bail(PS_EINVAL, "dev_buf smaller than the state");
        if (((uintptr_t)dev_buf) & 255) return bail(PS_EINVAL, "dev_buf must be 256-byte aligned");
        g->d_state = dev_buf;
    } else {
        e = cudaMalloc(&g->d_state, need);
        if (e != cudaSuccess) return bail(PS_ENOMEM, std::string("cudaMalloc state: ") + cudaGetErrorString(e));
        g->own_state = true;
    }
    for (int r = 0; r < world; ++r) {
        ps_state* v = nullptr;
        rc = make_state(n_qubits, dtype, (char*)g->d_state + slice * r, slice, g->stream, r, world, nullptr,
                        world > 1, &v);
        if (rc) {
            std::string msg = ps_last_error();
            return bail(rc, msg);
        }
        g->vranks.push_back(v);
    }
    for (ps_state* v : g->vranks) {
        v->peers.resize(world);
        v->peer_flags.resize(world);
        for (int r = 0; r < world; ++r) {
            v->peers[r] = g->vranks[r]->d_state;
            v->peer_flags[r] = g->vranks[r]->d_flags;
        }
        v->p2p = world > 1;
    }
    g->tile_bits = g->vranks[0]->tile_bits;
    g->tile_tune = g->vranks[0]->tile_tune;
    *out = g;
    return PS_OK;
}

extern "C" int ps_destroy(ps_handle h) {
    if (!h) return fail(PS_EINVAL, "NULL handle");
    free_state(h);
    return PS_OK;
}

extern "C" int ps_info(ps_handle h, int* n_qubits, int* n_local, int* rank, int* world, int* dtype, void** dev_ptr) {
    if (!h) return fail(PS_EINVAL, "NULL handle");
    if (n_qubits) *n_qubits = h->n;
    if (n_local) *n_local = h->nl;
    if (rank) *rank = h->rank;
    if (world) *world = h->world;
    if (dtype) *dtype = h->dtype;
    if (dev_ptr) *dev_ptr = h->d_state;
    return PS_OK;
}

static int check_option(const ps_state* h, int option, int64_t value) {
    switch (option) {
    case PS_OPT_PROFILE:
    case PS_OPT_VEC256:
    case PS_OPT_TILE_TUNE:
    case PS_OPT_TRANSPORT:
    case PS_OPT_FUSED_EXCHANGE: return PS_OK;
    case PS_OPT_FUSION: return (value < 0 || value > 2) ? fail(PS_EINVAL, "fusion must be 0, 1 or 2") : PS_OK;
    case PS_OPT_TILE_BITS: {
        // <= 512 (fp64) / 1024 (fp32) threads x 16 amplitudes per tile: 128 KiB of shared memory
        const int kmax = h->dtype == PS_C128 ? 13 : 14;
        return (value < 4 || value > kmax) ? fail(PS_EINVAL, "tile bits out of range [4, 13] (C128) / [4, 14] (C64)")
                                           : PS_OK;
    }
    case PS_OPT_CHUNK_BYTES:
        return (value < 4096 || (value & (value - 1))) ? fail(PS_EINVAL, "chunk bytes must be a power of two >= 4096")
                                                        : PS_OK;
    case PS_OPT_MAX_PASS_ROTS: return value < 1 ? fail(PS_EINVAL, "max pass rotations must be >= 1") : PS_OK;
    case PS_OPT_LAYOUT: return (value < 0 || value > 2) ? fail(PS_EINVAL, "layout must be 0, 1 or 2") : PS_OK;
    case PS_OPT_OVERLAP:
        if ((value & 0xffff) > 2) return fail(PS_EINVAL, "overlap mode must be 0, 1 or 2");
        return (((value >> 16) & 7) > ps_state::kMaxPieceBits + 1) ? fail(PS_EINVAL, "overlap piece bits must be <= 3")
                                                                    : PS_OK;
    case PS_OPT_SWAP_TMA: return PS_OK;
    case PS_OPT_SWAP_CTAS:
        return (value < -(1 << 16) || value > (1 << 16)) ? fail(PS_EINVAL, "swap CTAs must be in [-65536, 65536]")
                                                         : PS_OK;
    case PS_OPT_CHUNK_BITS:
        return (value < 0 || value > 12) ? fail(PS_EINVAL, "chunk bits must be 0..12 (0 = default)") : PS_OK;
    case PS_OPT_SPECIALIZE: return (value < 0 || value > 2) ? fail(PS_EINVAL, "specialize must be 0, 1 or 2") : PS_OK;
    case PS_OPT_GRID_CAP: return (value < 0 || value > (1 << 20)) ? fail(PS_EINVAL, "grid cap must be 0..2^20") : PS_OK;
    case PS_OPT_TILE_TMA: return (value < 0 || value > 3) ? fail(PS_EINVAL, "tile mode must be 0..3") : PS_OK;
    default: return fail(PS_EINVAL, "unknown option");
    }
}

// applies a validated option to one rank
static int set_option_rank(ps_state* h, int option, int64_t value) {
    switch (option) {
    case PS_OPT_PROFILE: h->profile = value ? 1 : 0; break;
    case PS_OPT_FUSION: h->fusion = (int)value; break;
    case PS_OPT_TILE_BITS: h->tile_bits = (int)value; break;
    case PS_OPT_CHUNK_BYTES: h->chunk_bytes = (size_t)value; break;
    case PS_OPT_MAX_PASS_ROTS: h->max_pass_rots = (int)std::min<int64_t>(value, 1 << 30); break;
    case PS_OPT_VEC256: h->vec256 = value ? 1 : 0; break;
    case PS_OPT_TILE_TUNE: h->tile_tune = (int)value; break;
    case PS_OPT_LAYOUT:
        if (value == 2 && h->world > 1 && !h->d_mirror) {
            cudaSetDevice(h->device);
            cudaError_t e = cudaMalloc(&h->d_mirror, h->amp_bytes << h->nl);
            if (e != cudaSuccess) {
                h->d_mirror = nullptr;
                return fail(PS_ENOMEM, std::string("mirror buffer: ") + cudaGetErrorString(e));
            }
        }
        h->layout = (int)value;
        break;
    case PS_OPT_TRANSPORT: h->transport = (value || h->emulated) ? 1 : 0; break;
    case PS_OPT_OVERLAP: {
        // 0: off; 1: with the next pass; 2: with the passes before and after; bits 16-18 = piece bits + 1
        const int pb = (int)((value >> 16) & 7);
        h->overlap = (value && h->xstream) ? ((value & 0xffff) == 2 ? 2 : 1) : 0;
        if (pb) h->piece_bits = pb - 1;
        break;
    }
    case PS_OPT_SWAP_CTAS: h->swap_ctas = value == 0 ? -2 : (int)value; break;
    case PS_OPT_SWAP_TMA: h->swap_tma = value ? 1 : 0; break;
    case PS_OPT_CHUNK_BITS: h->chunk_bits = (int)value; break;
    case PS_OPT_SPECIALIZE: h->specialize = (int)value; break;
    case PS_OPT_GRID_CAP: h->grid_cap = (int)value; break;
    case PS_OPT_FUSED_EXCHANGE: h->fused = (value && h->p2p) ? 1 : 0; break;
    case PS_OPT_TILE_TMA: h->tile_tma = (int)value; break;
    default: return fail(PS_EINVAL, "unknown option");
    }
    return PS_OK;
}

extern "C" int ps_set_option(ps_handle h, int option, int64_t value) {
    if (!h) return fail(PS_EINVAL, "NULL handle");
    int rc = check_option(h, option, value);
    if (rc) return rc;
    RankSet rs = ranks_of(h);
    if (option == PS_OPT_LAYOUT && value == 2 && h->world > 1) {
        // the mirror mode starts from the canonical layout
        if (any_poisoned(h)) return fail(PS_ESTATE, "handle poisoned by an earlier fault");
        cudaSetDevice(h->device);
        if ((rc = restore_layout(rs))) return rc;
    }
    for (ps_state* r : rs)
        if ((rc = set_option_rank(r, option, value))) return rc;
    if (h->is_group()) {  // the group handle mirrors its ranks' options
        h->tile_bits = rs[0]->tile_bits;
        h->tile_tune = rs[0]->tile_tune;
        h->layout = rs[0]->layout;
        h->profile = rs[0]->profile;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// collectives over a rank set: NCCL for a real rank, stream order and host sums for a group

static int barrier(ps_state* h) {
    if (h->emulated || h->world == 1) return PS_OK;  // emulation: one stream orders everything
    NCCL_TRY(h, ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt32, ncclSum, h->comm, h->stream));
    return PS_OK;
}

static int barrier_on(ps_state* h, cudaStream_t st, int slot) {
    if (h->emulated || h->world == 1) return PS_OK;
    NCCL_TRY(h, ncclAllReduce(h->d_barrier + slot, h->d_barrier + slot, 1, ncclInt32, ncclSum, h->comm, st));
    return PS_OK;
}

// pairwise barrier with `partner` on stream st (P2P flags; NCCL barrier without peer access)
static int pair_barrier(ps_state* h, cudaStream_t st, int partner, int slot) {
    if (h->emulated || h->world == 1) return PS_OK;
    if (!h->p2p || !h->peer_flags[partner]) return barrier_on(h, st, slot);
    uint32_t& ep = h->bar_epoch[(size_t)partner * ps_state::kBarSlots + slot];
    ep += 1;
    const size_t fw = flag_words(h);
    CUDA_TRY(h, launch_pair_barrier(h->d_flags + fw + (size_t)partner * ps_state::kBarSlots + slot,
                                    h->peer_flags[partner] + fw + (size_t)h->rank * ps_state::kBarSlots + slot, ep,
                                    st));
    return PS_OK;
}

// vals[k] = sum over all ranks of d_result[k], k < nvals (blocks)
static int sum_results(const RankSet& rs, int nvals, double* vals) {
    ps_state* h0 = rs[0];
    if (!h0->emulated && h0->world > 1)
        NCCL_TRY(h0, ncclAllReduce(h0->d_result, h0->d_result, (size_t)nvals, ncclDouble, ncclSum, h0->comm, h0->stream));
    for (ps_state* r : rs)
        CUDA_TRY(r, cudaMemcpyAsync(r->h_result, r->d_result, sizeof(double) * nvals, cudaMemcpyDeviceToHost, r->stream));
    for (ps_state* r : rs) CUDA_TRY(r, cudaStreamSynchronize(r->stream));
    for (int k = 0; k < nvals; ++k) {
        double s = 0.0;
        for (ps_state* r : rs) s += r->h_result[k];
        vals[k] = s;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// init / access

static uint64_t local_amps(const ps_state* h) { return 1ull << h->nl; }

static int init_basis_rank(ps_state* h, uint64_t index) {
    reset_layout(h);  // the whole state is overwritten
    Timed t(h, PS_K_INIT);
    CUDA_TRY(h, cudaMemsetAsync(h->d_state, 0, h->amp_bytes * local_amps(h), h->stream));
    if ((index >> h->nl) == (uint64_t)h->rank)
        CUDA_TRY(h, launch_set_one(h->dtype, h->d_state, index & (local_amps(h) - 1), h->stream));
    h->stats.launches[PS_K_INIT] += 1;
    return PS_OK;
}

extern "C" int ps_init_basis(ps_handle h, uint64_t index) {
    CHECK_HANDLE(h);
    if (h->n < 64 && index >> h->n) return fail(PS_ERANGE, "basis index >= 2^n");
    for (ps_state* r : ranks_of(h)) {
        int rc = init_basis_rank(r, index);
        if (rc) return rc;
    }
    return PS_OK;
}

extern "C" int ps_init_random(ps_handle h, uint64_t seed) {
    CHECK_HANDLE(h);
    for (ps_state* r : ranks_of(h)) {
        reset_layout(r);  // the whole state is overwritten
        Timed t(r, PS_K_INIT);
        CUDA_TRY(r, launch_init_random(r->dtype, r->d_state, local_amps(r), seed, (uint64_t)r->rank << r->nl, r->stream));
        r->stats.launches[PS_K_INIT] += 1;
    }
    return PS_OK;
}

static int reduce_norm(const RankSet& rs, double* out);

extern "C" int ps_normalize(ps_handle h) {
    CHECK_HANDLE(h);
    RankSet rs = ranks_of(h);
    double nrm = 0.0;
    int rc = reduce_norm(rs, &nrm);
    if (rc) return rc;
    if (!(nrm > 0.0)) return fail(PS_EINVAL, "cannot normalise a zero state");
    for (ps_state* r : rs) {
        Timed t(r, PS_K_INIT);
        CUDA_TRY(r, launch_scale(r->dtype, r->d_state, local_amps(r), 1.0 / std::sqrt(nrm), r->stream));
    }
    return PS_OK;
}

static int check_range(const ps_state* h, uint64_t first, uint64_t count) {
    if (h->n < 64) {
        const uint64_t dim = 1ull << h->n;
        if (first > dim || count > dim - first) return fail(PS_ERANGE, "index range beyond 2^n");
    }
    return PS_OK;
}

extern "C" int ps_set_state(ps_handle h, uint64_t first, uint64_t count, const void* amps) {
    CHECK_HANDLE(h);
    if (count && !amps) return fail(PS_EINVAL, "NULL amps with count > 0");
    int rc = check_range(h, first, count);
    if (rc) return rc;
    RankSet rs = ranks_of(h);
    if (first == 0 && h->n < 64 && count == (1ull << h->n)) {
        for (ps_state* r : rs) reset_layout(r);  // the whole state is overwritten
    } else if ((rc = restore_layout(rs))) {
        return rc;
    }
    for (ps_state* r : rs) {
        const uint64_t lo = (uint64_t)r->rank << r->nl, hi = lo + local_amps(r);
        const uint64_t a = std::max(lo, first), b = std::min(hi, first + count);
        if (a < b)
            CUDA_TRY(r, cudaMemcpyAsync((char*)r->d_state + (a - lo) * r->amp_bytes,
                                        (const char*)amps + (a - first) * r->amp_bytes, (b - a) * r->amp_bytes,
                                        cudaMemcpyHostToDevice, r->stream));
    }
    for (ps_state* r : rs) CUDA_TRY(r, cudaStreamSynchronize(r->stream));
    return PS_OK;
}

static int ensure_xstage(ps_state* h, size_t bytes) {
    if (h->xstage_bytes >= bytes) return PS_OK;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int t = 0; t < 2; ++t) {
        if (h->d_xstage[t]) cudaFree(h->d_xstage[t]);
        h->d_xstage[t] = nullptr;
    }
    h->xstage_bytes = 0;
    for (int t = 0; t < 2; ++t) CUDA_TRY(h, cudaMalloc(&h->d_xstage[t], bytes));
    h->xstage_bytes = bytes;
    return PS_OK;
}

extern "C" int ps_get_amplitudes(ps_handle h, uint64_t first, uint64_t count, void* amps_out) {
    CHECK_HANDLE(h);
    if (count && !amps_out) return fail(PS_EINVAL, "NULL amps_out with count > 0");
    int rc = check_range(h, first, count);
    if (rc) return rc;
    RankSet rs = ranks_of(h);
    if ((rc = restore_layout(rs))) return rc;
    if (h->world == 1 || h->is_group()) {
        // every slice is on this device: copy each rank's part directly
        for (ps_state* r : rs) {
            const uint64_t lo = (uint64_t)r->rank << r->nl, hi = lo + local_amps(r);
            const uint64_t a = std::max(lo, first), b = std::min(hi, first + count);
            if (a < b)
                CUDA_TRY(r, cudaMemcpyAsync((char*)amps_out + (a - first) * r->amp_bytes,
                                            (const char*)r->d_state + (a - lo) * r->amp_bytes, (b - a) * r->amp_bytes,
                                            cudaMemcpyDeviceToHost, r->stream));
        }
        for (ps_state* r : rs) CUDA_TRY(r, cudaStreamSynchronize(r->stream));
        return PS_OK;
    }
    // world > 1: pieces broadcast from their owners (collective; all ranks pass the same range)
    const size_t piece_amps = std::max<size_t>(1, h->chunk_bytes / h->amp_bytes);
    rc = ensure_xstage(h, piece_amps * h->amp_bytes);
    if (rc) return rc;
    uint64_t done = 0;
    while (done < count) {
        const uint64_t g = first + done;
        const int owner = (int)(g >> h->nl);
        const uint64_t owner_end = ((uint64_t)owner + 1) << h->nl;
        const uint64_t len = std::min<uint64_t>({count - done, piece_amps, owner_end - g});
        if (owner == h->rank)
            CUDA_TRY(h, cudaMemcpyAsync(h->d_xstage[0], (const char*)h->d_state + (g & (local_amps(h) - 1)) * h->amp_bytes,
                                        len * h->amp_bytes, cudaMemcpyDeviceToDevice, h->stream));
        NCCL_TRY(h, ncclBroadcast(h->d_xstage[0], h->d_xstage[0], len * h->amp_bytes, ncclChar, owner, h->comm, h->stream));
        CUDA_TRY(h, cudaMemcpyAsync((char*)amps_out + done * h->amp_bytes, h->d_xstage[0], len * h->amp_bytes,
                                    cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        done += len;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// exchanges (K3): half-vector swap of slots with bit ell == 1-keep with partner rank^gx

static int exchange_half(ps_state* h, const Pass& p) {
    const int partner = h->rank ^ (int)p.gx;
    const size_t s = h->amp_bytes;
    const uint64_t rows = 1ull << (h->nl - 1 - p.ell);
    const size_t row_bytes = s << p.ell;
    const size_t start = (size_t)(1 - p.keep) * row_bytes;
    const size_t chunk = h->chunk_bytes;
    if (h->p2p && h->transport) {
        // both ranks of the pair swap their regions in place through NVLink peer pointers, each
        // doing half of the elements; barriers order it against all earlier and later work
        // (emulation: both halves run one after the other on the group's stream)
        const uint64_t row_amps = 1ull << p.ell, total = rows * row_amps;
        const uint64_t e0 = p.keep ? total / 2 : 0, e1 = p.keep ? total : total / 2;
        int rc = barrier(h);
        if (rc) return rc;
        CUDA_TRY(h, launch_p2p_swap(h->dtype, h->d_state, h->peers[partner], rows, row_amps,
                                    (uint64_t)(1 - p.keep) * row_amps, (uint64_t)p.keep * row_amps, e0, e1, 0, 0,
                                    h->stream, 0));
        rc = barrier(h);
        if (rc) return rc;
        h->stats.nvlink_bytes += (double)(rows * row_bytes);
        h->stats.exchanges += 1;
        h->stats.algo_bytes[PS_K_EXCHANGE] += (double)(rows * row_bytes) * 2.0;
        return PS_OK;
    }
    int rc = ensure_xstage(h, std::min(chunk, row_bytes * rows));
    if (rc) return rc;
    char* base = (char*)h->d_state;
    if (row_bytes >= chunk) {
        for (uint64_t r = 0; r < rows; ++r) {
            for (size_t off = 0; off < row_bytes; off += chunk) {
                char* reg = base + start + r * 2 * row_bytes + off;
                const size_t len = std::min(chunk, row_bytes - off);
                CUDA_TRY(h, cudaMemcpyAsync(h->d_xstage[0], reg, len, cudaMemcpyDeviceToDevice, h->stream));
                NCCL_TRY(h, ncclGroupStart());
                NCCL_TRY(h, ncclSend(h->d_xstage[0], len, ncclChar, partner, h->comm, h->stream));
                NCCL_TRY(h, ncclRecv(reg, len, ncclChar, partner, h->comm, h->stream));
                NCCL_TRY(h, ncclGroupEnd());
                h->stats.nvlink_bytes += (double)len;
            }
        }
    } else {
        const uint64_t rows_per = std::max<uint64_t>(1, chunk / row_bytes);
        for (uint64_t r0 = 0; r0 < rows; r0 += rows_per) {
            const uint64_t nr = std::min(rows_per, rows - r0);
            char* reg = base + start + r0 * 2 * row_bytes;
            CUDA_TRY(h, cudaMemcpy2DAsync(h->d_xstage[0], row_bytes, reg, 2 * row_bytes, row_bytes, nr,
                                          cudaMemcpyDeviceToDevice, h->stream));
            NCCL_TRY(h, ncclGroupStart());
            NCCL_TRY(h, ncclSend(h->d_xstage[0], nr * row_bytes, ncclChar, partner, h->comm, h->stream));
            NCCL_TRY(h, ncclRecv(h->d_xstage[1], nr * row_bytes, ncclChar, partner, h->comm, h->stream));
            NCCL_TRY(h, ncclGroupEnd());
            CUDA_TRY(h, cudaMemcpy2DAsync(reg, 2 * row_bytes, h->d_xstage[1], row_bytes, row_bytes, nr,
                                          cudaMemcpyDeviceToDevice, h->stream));
            h->stats.nvlink_bytes += (double)(nr * row_bytes);
        }
    }
    h->stats.exchanges += 1;
    h->stats.algo_bytes[PS_K_EXCHANGE] += (double)(rows * row_bytes) * 2.0;
    return PS_OK;
}

// contiguous elements per chunk of the TMA swap kernel for a piece of E(gx, ell) enumerated with
// element filter mask emask (runs end at a region row or at the lowest filter bit); 0 = use the
// register kernel (runs shorter than 1 KB, or the TMA form switched off)
static int swap_tma_chunk(const ps_state* h, uint64_t row_amps, uint64_t emask, uint64_t t0, uint64_t t1) {
    if (!h->swap_tma || t1 <= t0) return 0;
    uint64_t run = row_amps;
    if (emask) run = std::min<uint64_t>(run, 1ull << __builtin_ctzll(emask));
    uint64_t c = std::min<uint64_t>(4096 / h->amp_bytes, run);
    c = std::min<uint64_t>(c, t1 - t0);
    while (c > 1 && ((t1 - t0) % c || t0 % c)) c >>= 1;
    return c * h->amp_bytes >= 1024 ? (int)c : 0;
}

// a bit that splits the next pass's tiles into two halves whose elements all have that bit
// fixed: a free (tile-enumeration) bit in which no two elements of one tile differ
static uint64_t split_bits(const Pass& np) { return np.free_mask & ~np.touch_mask; }

static bool can_overlap(const ps_state* h, const Pass& ex, const Pass* np) {
    return h->overlap && h->xstream && h->p2p && h->transport && !ex.full && ex.kind == PASS_EXCHANGE && np &&
           (np->kind == PASS_TILE || np->kind == PASS_COSET) && h->tile_tma == 2 && split_bits(*np) != 0;
}

// swap E(gx, ell) overlapped with the following tile pass.  The pass is
// split into P = 2^B pieces by B of its free bits outside its tile space (so every tile lies in one
// piece); the region of the swap splits by the same bits.  The second stream swaps piece after
// piece (each closed by a barrier: both ranks' halves have landed) while the main stream runs
// each pass piece as soon as its data is in place.  If ell itself is such a bit, the tiles on the
// kept side need no swapped data and run during the whole swap.
static int exchange_overlap(ps_state* h, const Pass& ex, const Pass& np) {
    const int partner = h->rank ^ (int)ex.gx;
    const uint64_t rows = 1ull << (h->nl - 1 - ex.ell);
    const uint64_t row_amps = 1ull << ex.ell, total = rows * row_amps;
    const uint64_t my_off = (uint64_t)(1 - ex.keep) * row_amps, peer_off = (uint64_t)ex.keep * row_amps;
    const uint64_t sb = split_bits(np);
    const bool f_is_ell = (sb >> ex.ell) & 1;
    uint64_t pbits = 0;  // piece bits (local positions): the highest split bits other than ell
    int B = 0;
    for (int b = 63; b >= 0 && B < std::min(h->piece_bits, (int)ps_state::kMaxPieceBits); --b)
        if (((sb >> b) & 1) && b != ex.ell) {
            pbits |= 1ull << b;
            ++B;
        }
    if (!f_is_ell && B == 0) return fail(PS_EUNSUPPORTED, "overlap without a split bit");  // can_overlap excludes it
    const int P = 1 << B;
    // local bit f -> bit of the region element index (bit ell removed)
    auto elem_bits = [&](uint64_t m) {
        uint64_t r = 0;
        for (; m; m &= m - 1) {
            const int f = __builtin_ctzll(m);
            r |= 1ull << (f < ex.ell ? f : f - 1);
        }
        return r;
    };
    auto deposit = [](uint64_t v, uint64_t mask) {
        uint64_t r = 0;
        for (; mask; mask &= mask - 1, v >>= 1)
            if (v & 1) r |= mask & (~mask + 1);
        return r;
    };
    const uint64_t emask = elem_bits(pbits);
    const uint64_t piece = total >> B;  // elements per piece; each rank swaps half of them
    const uint64_t t0 = ex.keep ? piece / 2 : 0, t1 = ex.keep ? piece : piece / 2;
    auto swap_piece = [&](int j, cudaStream_t st, int ctas) {
        return launch_p2p_swap(h->dtype, h->d_state, h->peers[partner], rows, row_amps, my_off, peer_off, t0, t1,
                               emask, deposit((uint64_t)j, emask), st, ctas,
                               ctas < 0 ? swap_tma_chunk(h, row_amps, emask, t0, t1) : 0);
    };
    auto run_pass = [&](uint64_t fixed_mask, uint64_t fixed_val) -> int {
        Pass q = np;
        q.free_mask = np.free_mask & ~fixed_mask;
        q.or_mask = np.or_mask | fixed_val;
        Timed t(h, np.kind);
        CUDA_TRY(h, launch_tile(h->dtype, h->d_state, h->nl, q, h->d_subs, h->d_trots, h->d_offs, h->tile_tma,
                                h->tile_tune, h->stream, h->cur_plan->subs.data(), h->cur_plan->trots.data(),
                                h->grid_cap));
        return PS_OK;
    };
    int rc = barrier(h);  // every rank's earlier passes are done
    if (rc) return rc;
    const int first = f_is_ell ? 0 : 1;
    if (!f_is_ell) {
        // piece 0 is swapped with the whole GPU before anything can run
        Timed t(h, PS_K_EXCHANGE);
        CUDA_TRY(h, swap_piece(0, h->stream, 0));
        rc = barrier(h);
        if (rc) return rc;
    }
    CUDA_TRY(h, cudaEventRecord(h->xev[0], h->stream));
    CUDA_TRY(h, cudaStreamWaitEvent(h->xstream, h->xev[0], 0));
    {
        // the overlapped swap pieces, timed on the stream they run on: kernel_ms[EXCHANGE] then
        // covers every swapped byte (and overlaps the pass's own time)
        Timed t(h, PS_K_EXCHANGE, h->xstream);
        for (int j = first; j < P; ++j) {
            CUDA_TRY(h, swap_piece(j, h->xstream, h->swap_ctas));
            rc = pair_barrier(h, h->xstream, partner, 1);
            if (rc) return rc;
            CUDA_TRY(h, cudaEventRecord(h->xev[1 + j], h->xstream));
        }
    }
    const uint64_t lbit = 1ull << ex.ell;
    if (f_is_ell) {
        rc = run_pass(lbit, (uint64_t)ex.keep << ex.ell);  // kept side: no swapped slot
        if (rc) return rc;
    }
    for (int j = 0; j < P; ++j) {
        if (j >= first) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->xev[1 + j], 0));
        const uint64_t fm = pbits | (f_is_ell ? lbit : 0);
        const uint64_t fv = deposit((uint64_t)j, pbits) | (f_is_ell ? (uint64_t)(1 - ex.keep) << ex.ell : 0);
        rc = run_pass(fm, fv);
        if (rc) return rc;
    }
    const double region = (double)(rows * row_amps * h->amp_bytes);
    h->stats.nvlink_bytes += region;
    h->stats.exchanges += 1;
    h->stats.launches[PS_K_EXCHANGE] += 1;
    h->stats.algo_bytes[PS_K_EXCHANGE] += region * 2.0;
    // the pass pieces are one logical pass over the local state
    h->stats.launches[np.kind] += 1;
    h->stats.rotations_by[np.kind] += (uint64_t)np.rot_count;
    h->stats.algo_bytes[np.kind] += 2.0 * (double)h->amp_bytes * (double)local_amps(h);
    h->stats.passes += 1;
    return PS_OK;
}

// overlap mode 2: a chain  pass, E, pass, E, ..., pass  (tile passes and P2P half exchanges,
// consecutive exchanges allowed) as one pipeline.  Every pass and every swap region splits into
// P = 2^B pieces by B local bits that are free bits outside every pass's tile space and are no
// exchange's ell, so piece j of each step touches only elements whose piece bits equal j.  The
// main stream runs the passes piece by piece, a pass's piece j waiting for the preceding swap's
// piece j; the second stream swaps piece j of an exchange as soon as this rank finished the
// preceding step's piece j and the partner arrived at the same point (pairwise barrier).  A swap
// then overlaps the passes on both sides of it, and an exchange right after another one (4 and more
// ranks) still overlaps.
static bool chain_pass(const Pass& q) { return q.kind == PASS_TILE || q.kind == PASS_COSET; }
static bool chain_exchange(const ps_state* h, const Pass& q) {
    return q.kind == PASS_EXCHANGE && !q.full && h->overlap >= 2 && h->xstream && h->p2p && h->transport &&
           h->tile_tma == 2;
}

// end (exclusive) of the longest chain starting at tile pass passes[b], or 0 if there is none;
// *pbits_out = the piece bits (the highest common split bits, at most piece_bits of them)
static size_t overlap_chain_end(const ps_state* h, const std::vector<Pass>& passes, size_t b, uint64_t* pbits_out) {
    // with the fused exchange + tile kernel on, every fusable exchange runs fused instead
    if (h->overlap < 2 || h->fused || !chain_pass(passes[b])) return 0;
    uint64_t sb = split_bits(passes[b]);
    int want = 0;  // split bits the first segment keeps; later segments must keep as many
    size_t end = 0, k = b + 1;
    while (k < passes.size()) {
        uint64_t ells = 0;
        size_t m = k;
        while (m < passes.size() && chain_exchange(h, passes[m])) ells |= 1ull << passes[m++].ell;
        if (m == k || m >= passes.size() || !chain_pass(passes[m])) break;
        const uint64_t nsb = sb & ~ells & split_bits(passes[m]);
        const int have = __builtin_popcountll(nsb);
        if (have == 0 || (end && have < want)) break;
        if (!end) want = std::min(have, std::min(h->piece_bits, (int)ps_state::kMaxPieceBits));
        sb = nsb;
        end = m + 1;
        k = m + 1;
    }
    if (!end) return 0;
    uint64_t pbits = 0;
    int B = 0;
    for (int q = 63; q >= 0 && B < want; --q)
        if ((sb >> q) & 1) {
            pbits |= 1ull << q;
            ++B;
        }
    *pbits_out = pbits;
    return end;
}

static int overlap_chain(ps_state* h, const std::vector<Pass>& passes, size_t b, size_t e, uint64_t pbits) {
    const int P = 1 << __builtin_popcountll(pbits);  // <= 8: events xev[1..P] (passes), xev[1+P..2P] (swaps)
    auto deposit = [](uint64_t v, uint64_t mask) {
        uint64_t r = 0;
        for (; mask; mask &= mask - 1, v >>= 1)
            if (v & 1) r |= mask & (~mask + 1);
        return r;
    };
    const double pass_bytes = 2.0 * (double)h->amp_bytes * (double)local_amps(h);
    int rc = PS_OK;
    bool after_swap = false;
    for (size_t k = b; k < e; ++k) {
        const Pass& st = passes[k];
        if (chain_pass(st)) {
            for (int j = 0; j < P; ++j) {
                if (after_swap) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->xev[1 + P + j], 0));
                Pass q = st;
                q.free_mask = st.free_mask & ~pbits;
                q.or_mask = st.or_mask | deposit((uint64_t)j, pbits);
                {
                    Timed t(h, st.kind);
                    CUDA_TRY(h, launch_tile(h->dtype, h->d_state, h->nl, q, h->d_subs, h->d_trots, h->d_offs,
                                            h->tile_tma, h->tile_tune, h->stream, h->cur_plan->subs.data(),
                                            h->cur_plan->trots.data(), h->grid_cap));
                }
                CUDA_TRY(h, cudaEventRecord(h->xev[1 + j], h->stream));
            }
            after_swap = false;
            h->stats.launches[st.kind] += 1;  // the pieces are one logical pass over the local state
            h->stats.rotations_by[st.kind] += (uint64_t)st.rot_count;
            h->stats.algo_bytes[st.kind] += pass_bytes;
            h->stats.passes += 1;
            continue;
        }
        // a half exchange E(gx, ell), swapped piece by piece on the second stream
        const int partner = h->rank ^ (int)st.gx;
        const uint64_t rows = 1ull << (h->nl - 1 - st.ell);
        const uint64_t row_amps = 1ull << st.ell, total = rows * row_amps;
        const uint64_t my_off = (uint64_t)(1 - st.keep) * row_amps, peer_off = (uint64_t)st.keep * row_amps;
        uint64_t emask = 0;  // piece bits in region-element positions (bit ell removed)
        for (uint64_t m = pbits; m; m &= m - 1) {
            const int f = __builtin_ctzll(m);
            emask |= 1ull << (f < st.ell ? f : f - 1);
        }
        const uint64_t piece = total / (uint64_t)P;
        const uint64_t t0 = st.keep ? piece / 2 : 0, t1 = st.keep ? piece : piece / 2;
        {
            Timed t(h, PS_K_EXCHANGE, h->xstream);
            for (int j = 0; j < P; ++j) {
                // after a pass: this rank finished its piece j (event); after a swap the stream order
                // already holds.  Then the partner reached the same point (pair barrier).
                if (!after_swap) CUDA_TRY(h, cudaStreamWaitEvent(h->xstream, h->xev[1 + j], 0));
                if ((rc = pair_barrier(h, h->xstream, partner, 1))) return rc;
                CUDA_TRY(h, launch_p2p_swap(h->dtype, h->d_state, h->peers[partner], rows, row_amps, my_off, peer_off,
                                            t0, t1, emask, deposit((uint64_t)j, emask), h->xstream, h->swap_ctas,
                                            h->swap_ctas < 0 ? swap_tma_chunk(h, row_amps, emask, t0, t1) : 0));
                if ((rc = pair_barrier(h, h->xstream, partner, 2))) return rc;  // both halves of piece j landed
                CUDA_TRY(h, cudaEventRecord(h->xev[1 + P + j], h->xstream));
            }
        }
        after_swap = true;
        const double region = (double)(total * h->amp_bytes);
        h->stats.nvlink_bytes += region;
        h->stats.exchanges += 1;
        h->stats.launches[PS_K_EXCHANGE] += 1;
        h->stats.algo_bytes[PS_K_EXCHANGE] += region * 2.0;
    }
    return PS_OK;
}

// single-rotation full exchange (no free pivot): chunk pairs {t, t^delta}
static int exchange_full(ps_state* h, const Pass& p, const DevRot* d_rec, const DevRot& rec) {
    const int partner = h->rank ^ (int)p.gx;
    const size_t s = h->amp_bytes;
    const uint64_t N = local_amps(h);
    uint64_t C = std::max<uint64_t>(1, h->chunk_bytes / s);
    if (C > N) C = N;
    // C must be a power of two
    C = 1ull << highest_bit(C);
    const uint64_t xl = rec.x;
    const uint64_t delta = xl / C;
    int rc = ensure_xstage(h, 2 * C * s);
    if (rc) return rc;
    char* st = (char*)h->d_xstage[0];
    char* base = (char*)h->d_state;
    const uint64_t nchunks = N / C;
    for (uint64_t t = 0; t < nchunks; ++t) {
        const uint64_t u = t ^ delta;
        if (u < t) continue;
        NCCL_TRY(h, ncclGroupStart());
        NCCL_TRY(h, ncclSend(base + t * C * s, C * s, ncclChar, partner, h->comm, h->stream));
        if (u != t) NCCL_TRY(h, ncclSend(base + u * C * s, C * s, ncclChar, partner, h->comm, h->stream));
        NCCL_TRY(h, ncclRecv(st, C * s, ncclChar, partner, h->comm, h->stream));
        if (u != t) NCCL_TRY(h, ncclRecv(st + C * s, C * s, ncclChar, partner, h->comm, h->stream));
        NCCL_TRY(h, ncclGroupEnd());
        // st holds partner chunk t, st + C*s partner chunk u
        // own chunk t needs partner elements i^xl in chunk u; own chunk u needs partner chunk t
        const char* pu = (u != t) ? st + C * s : st;
        CUDA_TRY(h, launch_full_update(h->dtype, h->d_state, pu, t * C, C, u * C, d_rec, h->stream));
        if (u != t) CUDA_TRY(h, launch_full_update(h->dtype, h->d_state, st, u * C, C, t * C, d_rec, h->stream));
        h->stats.nvlink_bytes += (double)(C * s * (u != t ? 2 : 1));
    }
    h->stats.exchanges += 1;
    h->stats.rotations_by[PS_K_EXCHANGE] += 1;
    h->stats.algo_bytes[PS_K_EXCHANGE] += (double)(N * s) * 3.0;
    return PS_OK;
}

// the same full exchange for the virtual ranks of a group: per chunk step, every rank first stages
// its partner's chunks t and u (the "receive"), then every rank updates its own chunks
static int exchange_full_group(const RankSet& rs, const std::vector<Plan*>& plans, size_t pi) {
    ps_state* h0 = rs[0];
    const Pass& p0 = plans[0]->passes[pi];
    const size_t s = h0->amp_bytes;
    const uint64_t N = local_amps(h0);
    uint64_t C = std::max<uint64_t>(1, h0->chunk_bytes / s);
    if (C > N) C = N;
    C = 1ull << highest_bit(C);
    const uint64_t delta = plans[0]->rots[p0.rot_begin].x / C;
    for (ps_state* r : rs) {
        int rc = ensure_xstage(r, 2 * C * s);
        if (rc) return rc;
    }
    const uint64_t nchunks = N / C;
    for (uint64_t t = 0; t < nchunks; ++t) {
        const uint64_t u = t ^ delta;
        if (u < t) continue;
        for (ps_state* r : rs) {
            const ps_state* q = rs[r->rank ^ (int)p0.gx];
            char* st = (char*)r->d_xstage[0];
            CUDA_TRY(r, cudaMemcpyAsync(st, (const char*)q->d_state + t * C * s, C * s, cudaMemcpyDeviceToDevice, r->stream));
            if (u != t)
                CUDA_TRY(r, cudaMemcpyAsync(st + C * s, (const char*)q->d_state + u * C * s, C * s,
                                            cudaMemcpyDeviceToDevice, r->stream));
        }
        for (size_t k = 0; k < rs.size(); ++k) {
            ps_state* r = rs[k];
            const Pass& p = plans[k]->passes[pi];
            const char* st = (const char*)r->d_xstage[0];
            const char* pu = (u != t) ? st + C * s : st;
            CUDA_TRY(r, launch_full_update(r->dtype, r->d_state, pu, t * C, C, u * C, r->d_rots + p.rot_begin, r->stream));
            if (u != t)
                CUDA_TRY(r, launch_full_update(r->dtype, r->d_state, st, u * C, C, t * C, r->d_rots + p.rot_begin,
                                               r->stream));
            r->stats.nvlink_bytes += (double)(C * s * (u != t ? 2 : 1));
        }
    }
    for (ps_state* r : rs) {
        r->stats.exchanges += 1;
        r->stats.launches[PS_K_EXCHANGE] += 1;
        r->stats.rotations_by[PS_K_EXCHANGE] += 1;
        r->stats.algo_bytes[PS_K_EXCHANGE] += (double)(N * s) * 3.0;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// fused exchange + tile pass (NEXT-2): the half-vector exchange E(gx, ell)
// and the tile pass after it run as ONE kernel.  Each rank's tiles read their kept half from local
// memory and the other half straight from the partner's slots through the peer pointer, compute,
// and store every element locally in the new layout.  A store into a slot the partner still has to
// read waits on a per-tile flag the partner raises (release, system scope) once its reads of that
// tile are done; both ranks walk their tiles in the same order, so no swap, no staging and no
// barrier after the pass.  Emulated ranks run as one kernel over all ranks' slices.

static bool can_fuse(const ps_state* h, const Pass& ex, const Pass* np) {
    return h->fused && h->p2p && h->transport && h->world > 1 && ex.kind == PASS_EXCHANGE && !ex.full && np &&
           (np->kind == PASS_TILE || np->kind == PASS_COSET) && h->tile_tma == 2;
}

static int exchange_fused(const RankSet& rs, const std::vector<Plan*>& plans, size_t pi) {
    ps_state* h0 = rs[0];
    const Pass& ex0 = plans[0]->passes[pi];
    const Pass& np0 = plans[0]->passes[pi + 1];
    const size_t ntiles = (size_t)1 << __builtin_popcountll(np0.free_mask);
    if (ntiles > h0->flags_cap) return fail(PS_EUNSUPPORTED, "fused exchange: more tiles than flag words");
    int rc = barrier(h0);  // every rank's earlier passes are done before anyone reads a peer slot
    if (rc) return rc;
    std::vector<XTileRank> xr(rs.size());
    for (size_t k = 0; k < rs.size(); ++k) {
        ps_state* r = rs[k];
        const Pass& ex = plans[k]->passes[pi];
        const Pass& np = plans[k]->passes[pi + 1];
        const int partner = r->rank ^ (int)ex.gx;
        r->epoch += 1;
        xr[k].a = r->d_state;
        xr[k].peer = r->peers[partner];
        xr[k].flags = r->d_flags;
        xr[k].peer_flags = r->peer_flags[partner];
        xr[k].subs = r->d_subs + np.sub_begin;
        xr[k].trots = r->d_trots;
        xr[k].rank = r->rank;
        xr[k].keep = ex.keep;
    }
    {
        Timed t(h0, PS_K_XTILE);
        CUDA_TRY(h0, launch_xtile(h0->dtype, xr.data(), (int)xr.size(), np0, h0->d_offs + np0.off_begin,
                                  plans[0]->offsets.data() + np0.off_begin, ex0.ell, h0->epoch, h0->stream,
                                  h0->grid_cap));
    }
    for (size_t k = 0; k < rs.size(); ++k) {
        ps_state* r = rs[k];
        const Pass& np = plans[k]->passes[pi + 1];
        // one pass over the local state (half of it read through the peer pointer), no swap
        r->stats.nvlink_fused_bytes += (double)(local_amps(r) / 2 * r->amp_bytes);
        r->stats.exchanges += 1;
        r->stats.launches[PS_K_XTILE] += 1;
        r->stats.rotations_by[PS_K_XTILE] += (uint64_t)np.rot_count;
        r->stats.algo_bytes[PS_K_XTILE] += 2.0 * (double)r->amp_bytes * (double)local_amps(r);
        r->stats.passes += 1;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// the hot path

static int upload_plan(ps_state* h, const Plan& plan) {
    const size_t rb = plan.rots.size() * sizeof(DevRot);
    const size_t ob = plan.offsets.size() * sizeof(uint64_t);
    const size_t sb = plan.subs.size() * sizeof(DevSub);
    const size_t tb = plan.trots.size() * sizeof(DevTRot);
    const size_t total = rb + ob + sb + tb;
    if (total == 0) return PS_OK;
    int rc = ensure_dev(h, &h->d_rots, &h->d_rots_cap, std::max<size_t>(plan.rots.size(), 1));
    if (!rc) rc = ensure_dev(h, &h->d_offs, &h->d_offs_cap, std::max<size_t>(plan.offsets.size(), 1));
    if (!rc) rc = ensure_dev(h, &h->d_subs, &h->d_subs_cap, std::max<size_t>(plan.subs.size(), 1));
    if (!rc) rc = ensure_dev(h, &h->d_trots, &h->d_trots_cap, std::max<size_t>(plan.trots.size(), 1));
    if (rc) return rc;
    const int b = h->stage_flip;
    h->stage_flip ^= 1;
    CUDA_TRY(h, cudaEventSynchronize(h->h_stage_ev[b]));
    if (h->h_stage_cap[b] < total) {
        if (h->h_stage[b]) CUDA_TRY(h, cudaFreeHost(h->h_stage[b]));
        h->h_stage[b] = nullptr;
        const size_t cap = std::max(total, 2 * h->h_stage_cap[b]);
        CUDA_TRY(h, cudaMallocHost(&h->h_stage[b], cap));
        h->h_stage_cap[b] = cap;
    }
    char* hs = (char*)h->h_stage[b];
    size_t off = 0;
    auto put = [&](void* dst, const void* src, size_t bytes) -> int {
        if (!bytes) return PS_OK;
        std::memcpy(hs + off, src, bytes);
        CUDA_TRY(h, cudaMemcpyAsync(dst, hs + off, bytes, cudaMemcpyHostToDevice, h->stream));
        off += bytes;
        return PS_OK;
    };
    rc = put(h->d_rots, plan.rots.data(), rb);
    if (!rc) rc = put(h->d_offs, plan.offsets.data(), ob);
    if (!rc) rc = put(h->d_subs, plan.subs.data(), sb);
    if (!rc) rc = put(h->d_trots, plan.trots.data(), tb);
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->h_stage_ev[b], h->stream));
    return PS_OK;
}

static PlanConfig plan_config(const ps_state* h) {
    PlanConfig cfg;
    cfg.n = h->n;
    cfg.n_local = h->nl;
    cfg.world = h->world;
    cfg.rank = h->rank;
    cfg.fusion = h->fusion;
    cfg.tile_bits = h->tile_bits;
    cfg.min_chunk_bits = h->chunk_bits ? h->chunk_bits : 4;  // >= 16 amplitudes (256 B fp64, 128 B fp32)
    cfg.phase_bits = h->dtype == PS_C128 ? 3 : 4;      // 16-B vs 8-B shared-memory accesses
    cfg.max_pass_rots = h->max_pass_rots;
    cfg.layout = h->layout;
    cfg.specialize = h->specialize;
    cfg.perm = h->perm;
    return cfg;
}

// the paper's step (i): B <- A_(k xor gx) via a full-partition exchange
static int mirror_fetch(ps_state* h, const Pass& p) {
    if (!h->d_mirror) return fail(PS_ESTATE, "mirror buffer missing (PS_OPT_LAYOUT=2)");
    const int partner = h->rank ^ (int)p.gx;
    const uint64_t N = local_amps(h);
    const size_t bytes = h->amp_bytes * N;
    Timed t(h, PS_K_EXCHANGE);
    if (h->p2p && h->transport) {
        int rc = barrier(h);
        if (rc) return rc;
        CUDA_TRY(h, launch_p2p_copy(h->dtype, h->d_mirror, h->peers[partner], N, h->stream));
        rc = barrier(h);  // the partner may overwrite its A (butterfly) only after my read
        if (rc) return rc;
    } else {
        for (size_t off = 0; off < bytes; off += h->chunk_bytes) {
            const size_t len = std::min(h->chunk_bytes, bytes - off);
            NCCL_TRY(h, ncclGroupStart());
            NCCL_TRY(h, ncclSend((const char*)h->d_state + off, len, ncclChar, partner, h->comm, h->stream));
            NCCL_TRY(h, ncclRecv((char*)h->d_mirror + off, len, ncclChar, partner, h->comm, h->stream));
            NCCL_TRY(h, ncclGroupEnd());
        }
    }
    h->stats.exchanges += 1;
    h->stats.launches[PS_K_EXCHANGE] += 1;
    h->stats.nvlink_bytes += (double)bytes;
    h->stats.algo_bytes[PS_K_EXCHANGE] += (double)bytes * 2.0;
    return PS_OK;
}

// step (ii): B <- conj(w_k) B, butterfly A, B
static int mirror_butterfly(ps_state* h, const Pass& p) {
    const uint64_t N = local_amps(h);
    Timed t(h, PS_K_MIRROR);
    CUDA_TRY(h, launch_butterfly(h->dtype, h->d_state, h->d_mirror, N, (int)p.wr, (int)p.wi, h->stream));
    h->stats.launches[PS_K_MIRROR] += 1;
    h->stats.algo_bytes[PS_K_MIRROR] += 4.0 * (double)(h->amp_bytes * N);
    return PS_OK;
}

// one pass of one rank that needs no other rank's data in the same phase
static int execute_pass(ps_state* h, const Plan& plan, size_t pi, void** target) {
    const Pass& p = plan.passes[pi];
    const double pass_bytes = 2.0 * (double)h->amp_bytes * (double)local_amps(h);
    switch (p.kind) {
    case PASS_STREAM: {
        Timed t(h, PS_K_STREAM);
        CUDA_TRY(h, launch_stream(h->dtype, *target, h->nl, p, h->d_rots, h->vec256, h->stream));
        break;
    }
    case PASS_TILE:
    case PASS_COSET: {
        Timed t(h, p.kind);
        CUDA_TRY(h, launch_tile(h->dtype, *target, h->nl, p, h->d_subs, h->d_trots, h->d_offs, h->tile_tma,
                                h->tile_tune, h->stream, plan.subs.data(), plan.trots.data(), h->grid_cap));
        break;
    }
    case PASS_MIRROR_SWITCH:
        *target = h->d_mirror;
        return PS_OK;
    case PASS_MIRROR_END: {
        Timed t(h, PS_K_MIRROR);
        CUDA_TRY(h, launch_recombine(h->dtype, h->d_state, h->d_mirror, local_amps(h), h->stream));
        h->stats.launches[PS_K_MIRROR] += 1;
        h->stats.algo_bytes[PS_K_MIRROR] += 1.5 * pass_bytes;
        *target = h->d_state;
        return PS_OK;
    }
    case PASS_PERMUTE: {
        Timed t(h, PS_K_PERMUTE);
        CUDA_TRY(h, launch_permute(h->dtype, h->d_state, h->nl, p.ell, p.ell2, h->stream));
        h->stats.launches[PS_K_PERMUTE] += 1;
        h->stats.algo_bytes[PS_K_PERMUTE] += pass_bytes / 2;  // half the amplitudes move
        return PS_OK;
    }
    case PASS_EXCHANGE: {
        Timed t(h, PS_K_EXCHANGE);
        int rc = p.full ? exchange_full(h, p, h->d_rots + p.rot_begin, plan.rots[p.rot_begin]) : exchange_half(h, p);
        if (rc) return rc;
        h->stats.launches[PS_K_EXCHANGE] += 1;
        return PS_OK;
    }
    default:
        return fail(PS_EINVAL, "internal: unknown pass kind");
    }
    h->stats.launches[p.kind] += 1;
    h->stats.rotations_by[p.kind] += (uint64_t)p.rot_count;
    h->stats.algo_bytes[p.kind] += pass_bytes;
    h->stats.passes += 1;
    return PS_OK;
}

// executes one plan per rank of the set, pass by pass in lockstep (SPMD plans: the same passes on
// every rank, rank-specific signs and exchange sides)
static int execute_plans(const RankSet& rs, const std::vector<Plan*>& plans) {
    const size_t G = rs.size();
    const size_t np = plans[0]->passes.size();
    for (size_t k = 0; k < G; ++k) {
        if (plans[k]->passes.size() != np) return fail(PS_EINVAL, "internal: rank plans differ");
        int rc = upload_plan(rs[k], *plans[k]);
        if (rc) return rc;
        rs[k]->cur_plan = plans[k];
    }
    std::vector<void*> target(G);
    for (size_t k = 0; k < G; ++k) target[k] = rs[k]->d_state;
    int rc = PS_OK;
    for (size_t pi = 0; pi < np && !rc; ++pi) {
        const Pass& p0 = plans[0]->passes[pi];
        const Pass* next = pi + 1 < np ? &plans[0]->passes[pi + 1] : nullptr;
        if (p0.kind == PASS_EXCHANGE && G <= 8 && can_fuse(rs[0], p0, next)) {
            rc = exchange_fused(rs, plans, pi);
            ++pi;  // the next pass ran inside the fused kernel
            continue;
        }
        // the overlap pipelines run their passes on the state itself: not inside a mirror section
        const bool on_state = target[0] == rs[0]->d_state;
        if (G == 1 && on_state && rs[0]->overlap >= 2) {
            uint64_t pbits = 0;
            const size_t ce = overlap_chain_end(rs[0], plans[0]->passes, pi, &pbits);
            if (ce) {
                rc = overlap_chain(rs[0], plans[0]->passes, pi, ce, pbits);
                pi = ce - 1;  // the whole chain ran inside the pipeline
                continue;
            }
        }
        if (G == 1 && on_state && p0.kind == PASS_EXCHANGE && can_overlap(rs[0], p0, next)) {
            rc = exchange_overlap(rs[0], p0, *next);
            ++pi;  // the next pass ran inside the overlap
            continue;
        }
        if (p0.kind == PASS_EXCHANGE && p0.full && rs[0]->emulated) {
            rc = exchange_full_group(rs, plans, pi);
            continue;
        }
        if (p0.kind == PASS_MIRROR_BEGIN) {
            // every rank fetches its partner's A before any rank's butterfly overwrites its own
            for (size_t k = 0; k < G && !rc; ++k) rc = mirror_fetch(rs[k], plans[k]->passes[pi]);
            for (size_t k = 0; k < G && !rc; ++k) {
                rc = mirror_butterfly(rs[k], plans[k]->passes[pi]);
                target[k] = rs[k]->d_state;
            }
            continue;
        }
        for (size_t k = 0; k < G && !rc; ++k) rc = execute_pass(rs[k], *plans[k], pi, &target[k]);
    }
    if (rc && np > 0) {
        // passes already enqueued have transformed (part of) the state and its layout: the handle
        // no longer describes its amplitudes
        const std::string msg = ps_last_error();
        poison_all(rs);
        set_last_error(msg + " (handle poisoned: the plan failed after its first pass was enqueued)");
    }
    return rc;
}

static bool layout_canonical(const ps_state* h) {
    for (int q = 0; q < (int)h->perm.size(); ++q)
        if (h->perm[q] != q) return false;
    return true;
}

static void reset_layout(ps_state* h) {
    for (int q = 0; q < (int)h->perm.size(); ++q) h->perm[q] = q;
}

// brings the state back to the canonical layout (rank = top qubits, identity within ranks)
static int restore_layout(const RankSet& rs) {
    if (rs[0]->world == 1 || layout_canonical(rs[0])) return PS_OK;
    std::vector<Plan> rp(rs.size());
    std::vector<Plan*> pp(rs.size());
    for (size_t k = 0; k < rs.size(); ++k) {
        make_restore_plan(plan_config(rs[k]), rs[k]->perm, &rp[k]);
        pp[k] = &rp[k];
    }
    int rc = execute_plans(rs, pp);
    if (rc) return rc;
    for (ps_state* r : rs) reset_layout(r);
    return PS_OK;
}

extern "C" int ps_apply_rotations(ps_handle h, const uint64_t* xmask, const uint64_t* zmask, const double* angle,
                                  size_t count) {
    CHECK_HANDLE(h);
    std::string err;
    int rc = validate_rotations(h->n, xmask, zmask, angle, count, &err);
    if (rc) return fail(rc, "ps_apply_rotations: " + err);
    if (count == 0) return PS_OK;
    RankSet rs = ranks_of(h);
    std::vector<Plan*> plans;
    for (ps_state* r : rs) {
        make_plan(plan_config(r), xmask, zmask, angle, count, &r->plan);
        plans.push_back(&r->plan);
    }
    rc = execute_plans(rs, plans);
    if (rc) return rc;
    for (ps_state* r : rs) {
        if (r->plan.perm_out.size() == r->perm.size())
            r->perm = r->plan.perm_out;
        else
            reset_layout(r);
        r->stats.rotations += count;
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// reductions

static int reduce_norm(const RankSet& rs, double* out) {
    for (ps_state* h : rs) {
        Timed t(h, PS_K_REDUCE);
        CUDA_TRY(h, launch_norm(h->dtype, h->d_state, local_amps(h), h->d_partial, h->d_result, h->stream));
        h->stats.launches[PS_K_REDUCE] += 1;
        h->stats.algo_bytes[PS_K_REDUCE] += (double)h->amp_bytes * (double)local_amps(h);
    }
    return sum_results(rs, 1, out);
}

extern "C" int ps_norm(ps_handle h, double* out) {
    CHECK_HANDLE(h);
    if (!out) return fail(PS_EINVAL, "NULL out");
    return reduce_norm(ranks_of(h), out);
}

extern "C" int ps_inner(ps_handle a, ps_handle b, double* out) {
    CHECK_HANDLE(a);
    CHECK_HANDLE(b);
    if (!out) return fail(PS_EINVAL, "NULL out");
    if (a->n != b->n || a->dtype != b->dtype || a->world != b->world || a->rank != b->rank || a->device != b->device ||
        a->is_group() != b->is_group())
        return fail(PS_EINVAL, "ps_inner: handles differ in n, dtype, world, rank, device or emulation");
    RankSet ra = ranks_of(a), rb = ranks_of(b);
    int rc0 = restore_layout(ra);
    if (!rc0) rc0 = restore_layout(rb);
    if (rc0) return rc0;
    if (b->stream != a->stream) {
        CUDA_TRY(b, cudaStreamSynchronize(b->stream));
    }
    for (size_t k = 0; k < ra.size(); ++k) {
        ps_state* x = ra[k];
        Timed t(x, PS_K_REDUCE);
        CUDA_TRY(x, launch_inner(x->dtype, x->d_state, rb[k]->d_state, local_amps(x), x->d_partial, x->d_result, x->stream));
        x->stats.launches[PS_K_REDUCE] += 1;
        x->stats.algo_bytes[PS_K_REDUCE] += 2.0 * (double)x->amp_bytes * (double)local_amps(x);
    }
    return sum_results(ra, 2, out);
}

// expectation (R17): terms are grouped by their upper X-part gx; a gx != 0 group runs after a half
// exchange E(gx, ell) with a free local pivot ell (so every pair is local), grouped again by
// physical x (one read pass per x); a term whose local X-part covers every local bit
// (no free pivot) is summed against its partner's chunks (read-only full exchange)
struct ExpSeg {
    uint64_t gx = 0;
    int ell = 0, keep = 0;
    bool full = false;                // single term, no free pivot
    uint64_t fx = 0, fz = 0;          // full: local x / z parts
    int fy = 0, fsgn = 0;
    double fcoeff = 0.0;
    std::vector<uint64_t> xorder;
    std::vector<DevTerm> flat;
    std::vector<std::pair<size_t, size_t>> ranges;
};

static void expectation_plan(const ps_state* h, const uint64_t* xmask, const uint64_t* zmask, const double* coeff,
                             size_t count, std::vector<ExpSeg>* segs) {
    const int nl = h->nl;
    const uint64_t lmask = (1ull << nl) - 1;
    const uint64_t rank = (uint64_t)h->rank;
    std::vector<uint64_t> gorder;
    std::map<uint64_t, std::vector<size_t>> bygx;
    for (size_t l = 0; l < count; ++l) {
        const uint64_t gx = xmask[l] >> nl;
        if (!bygx.count(gx)) gorder.push_back(gx);
        bygx[gx].push_back(l);
    }
    std::stable_sort(gorder.begin(), gorder.end(), [](uint64_t a, uint64_t b) { return (a == 0) > (b == 0); });
    for (uint64_t gx : gorder) {
        const std::vector<size_t>& idx = bygx[gx];
        size_t pos = 0;
        while (pos < idx.size()) {
            ExpSeg sg;
            sg.gx = gx;
            size_t end = pos;
            uint64_t U = 0;
            if (gx == 0) {
                end = idx.size();
            } else {
                while (end < idx.size() && (U | (xmask[idx[end]] & lmask)) != lmask) U |= xmask[idx[end++]] & lmask;
                if (end == pos) {
                    const size_t l = idx[pos];
                    sg.full = true;
                    sg.fx = xmask[l] & lmask;
                    sg.fz = zmask[l] & lmask;
                    sg.fy = __builtin_popcountll(xmask[l] & zmask[l]) & 3;
                    sg.fsgn = __builtin_parityll((zmask[l] >> nl) & rank);
                    sg.fcoeff = coeff[l];
                    segs->push_back(std::move(sg));
                    ++pos;
                    continue;
                }
            }
            if (gx) {
                sg.ell = highest_bit(lmask & ~U);
                sg.keep = (int)((rank >> __builtin_ctzll(gx)) & 1);
            }
            std::map<uint64_t, std::vector<DevTerm>> byx;
            for (size_t q = pos; q < end; ++q) {
                const size_t l = idx[q];
                const uint64_t xh = xmask[l] >> nl, xl = xmask[l] & lmask, zh = zmask[l] >> nl, zl = zmask[l] & lmask;
                uint64_t xp = xl, zp = zl;
                int sgn = __builtin_parityll(zh & rank);
                if (gx) {
                    const int kappa = __builtin_parityll(zh & gx) ^ (int)((zl >> sg.ell) & 1);
                    xp = xl ^ (xh ? (1ull << sg.ell) : 0);
                    zp = zl ^ (kappa ? (1ull << sg.ell) : 0);
                    sgn ^= sg.keep & kappa;
                }
                const int y = __builtin_popcountll(xmask[l] & zmask[l]) & 3;
                // Re(i^y sigma t): y=0 -> tr, 1 -> -ti, 2 -> -tr, 3 -> ti ; pairs counted twice (i and j)
                const double w = (xp ? 2.0 : 1.0) * coeff[l] * (sgn ? -1.0 : 1.0);
                DevTerm t;
                t.z = zp;
                t.kr = (y == 0) ? w : (y == 2 ? -w : 0.0);
                t.ki = (y == 1) ? -w : (y == 3 ? w : 0.0);
                if (!byx.count(xp)) sg.xorder.push_back(xp);
                byx[xp].push_back(t);
            }
            for (uint64_t xp : sg.xorder) {
                sg.ranges.push_back({sg.flat.size(), byx[xp].size()});
                sg.flat.insert(sg.flat.end(), byx[xp].begin(), byx[xp].end());
            }
            segs->push_back(std::move(sg));
            pos = end;
        }
    }
}

// Re sum_i conj(psi_(i xor x)) w(i) psi_i over the local i of every rank, for one term without a
// free pivot: the partner's chunk u = t xor delta is staged (NCCL send/recv, or copied from the
// group's slices) against every own chunk t; nothing is modified
static int expectation_full(const RankSet& rs, const std::vector<const ExpSeg*>& sg, double* out) {
    ps_state* h0 = rs[0];
    const size_t s = h0->amp_bytes;
    const uint64_t N = local_amps(h0);
    uint64_t C = std::max<uint64_t>(1, h0->chunk_bytes / s);
    if (C > N) C = N;
    C = 1ull << highest_bit(C);
    const uint64_t delta = sg[0]->fx / C;
    for (ps_state* r : rs) {
        int rc = ensure_xstage(r, C * s);
        if (rc) return rc;
    }
    double total = 0.0;
    const uint64_t nchunks = N / C;
    for (uint64_t t0 = 0; t0 < nchunks; t0 += 64) {
        const uint64_t nb = std::min<uint64_t>(64, nchunks - t0);
        for (uint64_t q = 0; q < nb; ++q) {
            const uint64_t t = t0 + q, u = t ^ delta;
            for (size_t k = 0; k < rs.size(); ++k) {
                ps_state* r = rs[k];
                const int partner = r->rank ^ (int)sg[k]->gx;
                if (r->emulated) {
                    CUDA_TRY(r, cudaMemcpyAsync(r->d_xstage[0], (const char*)rs[partner]->d_state + u * C * s, C * s,
                                                cudaMemcpyDeviceToDevice, r->stream));
                } else {
                    // the partner's own chunk t' = u pairs with my chunk u ^ delta = t: it sends u
                    NCCL_TRY(r, ncclGroupStart());
                    NCCL_TRY(r, ncclSend((const char*)r->d_state + u * C * s, C * s, ncclChar, partner, r->comm, r->stream));
                    NCCL_TRY(r, ncclRecv(r->d_xstage[0], C * s, ncclChar, partner, r->comm, r->stream));
                    NCCL_TRY(r, ncclGroupEnd());
                }
            }
            for (size_t k = 0; k < rs.size(); ++k) {
                ps_state* r = rs[k];
                Timed tm(r, PS_K_REDUCE);
                CUDA_TRY(r, launch_expect_cross(r->dtype, r->d_state, r->d_xstage[0], t * C, C, u * C, sg[k]->fx,
                                                sg[k]->fz, sg[k]->fy, sg[k]->fsgn, r->d_partial, r->d_result + q,
                                                r->stream));
                r->stats.launches[PS_K_REDUCE] += 1;
                r->stats.algo_bytes[PS_K_REDUCE] += 2.0 * (double)(C * s);
                r->stats.nvlink_bytes += (double)(C * s);
            }
        }
        double vals[64];
        int rc = sum_results(rs, (int)nb, vals);
        if (rc) return rc;
        for (uint64_t q = 0; q < nb; ++q) total += vals[q];
    }
    *out = sg[0]->fcoeff * total;
    return PS_OK;
}

extern "C" int ps_expectation(ps_handle h, const uint64_t* xmask, const uint64_t* zmask, const double* coeff,
                              size_t count, double* out) {
    CHECK_HANDLE(h);
    if (!out) return fail(PS_EINVAL, "NULL out");
    std::string err;
    int rc = validate_rotations(h->n, xmask, zmask, coeff, count, &err);
    if (rc) return fail(rc, "ps_expectation: " + err);
    *out = 0.0;
    if (count == 0) return PS_OK;
    RankSet rs = ranks_of(h);
    if ((rc = restore_layout(rs))) return rc;
    std::vector<std::vector<ExpSeg>> segs(rs.size());
    for (size_t k = 0; k < rs.size(); ++k) expectation_plan(rs[k], xmask, zmask, coeff, count, &segs[k]);
    const uint64_t N = local_amps(rs[0]);
    double total = 0.0;
    for (size_t si = 0; si < segs[0].size(); ++si) {
        const ExpSeg& s0 = segs[0][si];
        if (s0.full) {
            std::vector<const ExpSeg*> sg;
            for (auto& v : segs) sg.push_back(&v[si]);
            double part = 0.0;
            if ((rc = expectation_full(rs, sg, &part))) return rc;
            total += part;
            continue;
        }
        auto exchange = [&]() -> int {
            for (size_t k = 0; k < rs.size(); ++k) {
                Pass ex;
                ex.kind = PASS_EXCHANGE;
                ex.gx = segs[k][si].gx;
                ex.ell = segs[k][si].ell;
                ex.keep = segs[k][si].keep;
                Timed t(rs[k], PS_K_EXCHANGE);
                int r2 = exchange_half(rs[k], ex);
                if (r2) {
                    poison_all(rs);  // the layout is half-way through an exchange
                    return r2;
                }
            }
            return PS_OK;
        };
        if (s0.gx && (rc = exchange())) return rc;
        for (size_t k = 0; k < rs.size(); ++k) {
            ps_state* r = rs[k];
            const ExpSeg& sg = segs[k][si];
            if ((rc = ensure_dev(r, &r->d_terms, &r->d_terms_cap, sg.flat.size()))) return rc;
            CUDA_TRY(r, cudaMemcpyAsync(r->d_terms, sg.flat.data(), sg.flat.size() * sizeof(DevTerm),
                                        cudaMemcpyHostToDevice, r->stream));
        }
        const size_t ng = s0.xorder.size();
        for (size_t gi = 0; gi < ng; gi += 64) {
            const size_t nb = std::min<size_t>(64, ng - gi);
            for (size_t k = 0; k < rs.size(); ++k) {
                ps_state* r = rs[k];
                const ExpSeg& sg = segs[k][si];
                for (size_t q = 0; q < nb; ++q) {
                    Timed t(r, PS_K_REDUCE);
                    CUDA_TRY(r, launch_expect(r->dtype, r->d_state, N, sg.xorder[gi + q], r->d_terms + sg.ranges[gi + q].first,
                                              (int)sg.ranges[gi + q].second, r->d_partial, r->d_result + q, r->stream));
                    r->stats.launches[PS_K_REDUCE] += 1;
                    r->stats.algo_bytes[PS_K_REDUCE] += (double)r->amp_bytes * (double)N;
                }
            }
            double vals[64];
            if ((rc = sum_results(rs, (int)nb, vals))) return rc;
            for (size_t q = 0; q < nb; ++q) total += vals[q];
        }
        if (s0.gx && (rc = exchange())) return rc;
    }
    *out = total;
    return PS_OK;
}

// ------------------------------------------------------------------------------------------

extern "C" int ps_synchronize(ps_handle h) {
    CHECK_HANDLE(h);
    for (ps_state* r : ranks_of(h)) {
        CUDA_TRY(r, cudaStreamSynchronize(r->stream));
        if (r->comm) {
            ncclResult_t async_err = ncclSuccess;
            ncclCommGetAsyncError(r->comm, &async_err);
            if (async_err != ncclSuccess) {
                r->poisoned = true;
                return fail(PS_ENCCL, std::string("NCCL async error: ") + ncclGetErrorString(async_err));
            }
        }
        drain_timings(r);
    }
    return PS_OK;
}

// a group reports its rank 0's counters (what rank 0 of a real run reports)
extern "C" int ps_get_stats(ps_handle h, ps_stats* out) {
    if (!h || !out) return fail(PS_EINVAL, "NULL argument");
    ps_state* r = h->is_group() ? h->vranks[0] : h;
    if (!any_poisoned(h)) {
        cudaSetDevice(r->device);
        if (!r->pending.empty()) {
            cudaStreamSynchronize(r->stream);
            drain_timings(r);
        }
    }
    *out = r->stats;
    return PS_OK;
}

extern "C" int ps_reset_stats(ps_handle h) {
    if (!h) return fail(PS_EINVAL, "NULL handle");
    for (ps_state* r : ranks_of(h)) {
        if (!r->poisoned) {
            cudaSetDevice(r->device);
            cudaStreamSynchronize(r->stream);
            drain_timings(r);
        }
        std::memset(&r->stats, 0, sizeof(r->stats));
    }
    return PS_OK;
}

extern "C" const char* ps_status_string(int code) {
    switch (code) {
    case PS_OK: return "PS_OK";
    case PS_EINVAL: return "PS_EINVAL: invalid argument";
    case PS_ERANGE: return "PS_ERANGE: mask bit or index out of range";
    case PS_ENOMEM: return "PS_ENOMEM: allocation failed";
    case PS_ECUDA: return "PS_ECUDA: CUDA error";
    case PS_ENCCL: return "PS_ENCCL: NCCL error";
    case PS_ESTATE: return "PS_ESTATE: handle poisoned by an earlier fault";
    case PS_EUNSUPPORTED: return "PS_EUNSUPPORTED: unsupported request";
    default: return "unknown status";
    }
}

extern "C" const char* ps_last_error(void) { return g_last_error.c_str(); }
