// gather_bw.cu -- microbenchmark: HBM read+write bandwidth of the coset-tile access pattern with
// no arithmetic, to separate the access-pattern ceiling from kernel latency hiding.
//
// A 2^n-amplitude fp64 state; tiles of 2^k amplitudes = 2^h chunks of 2^c contiguous amplitudes
// (k = c + h) at i0 xor off[u], off = span of h random vectors above bit c (like a coset tile);
// each thread loads 16 amplitudes (l = d*T + tid), adds 1 to the real part, stores them back.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bw tools/gather_bw.cu
//   ./gather_bw [n=30]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__device__ __forceinline__ uint64_t pdep(uint64_t v, uint64_t mask) {
    uint64_t out = 0;
    for (uint64_t m = mask; m; m &= m - 1) {
        if (v & 1) out |= m & (~m + 1);
        v >>= 1;
    }
    return out;
}

template <int LOADS>
__global__ void __launch_bounds__(512) gather(double2* a, int kbits, int cbits, uint64_t free_mask,
                                              const uint64_t* offs, uint64_t ntiles) {
    extern __shared__ uint64_t soff[];
    const int h = kbits - cbits;
    for (int u = threadIdx.x; u < (1 << h); u += blockDim.x) soff[u] = offs[u];
    __syncthreads();
    const uint32_t T = blockDim.x;
    const uint32_t cmask = (1u << cbits) - 1;
    for (uint64_t tau = blockIdx.x; tau < ntiles; tau += gridDim.x) {
        const uint64_t i0 = pdep(tau, free_mask);
        double2 v[LOADS];
        uint64_t g[LOADS];
#pragma unroll
        for (int d = 0; d < LOADS; ++d) {
            const uint32_t l = d * T + threadIdx.x;
            g[d] = (i0 ^ soff[l >> cbits]) | (l & cmask);
            v[d] = __ldcs(&a[g[d]]);
        }
#pragma unroll
        for (int d = 0; d < LOADS; ++d) {
            v[d].x += 1.0;
            __stcs(&a[g[d]], v[d]);
        }
    }
}

// 256-bit variant: each lane moves two consecutive amplitudes per access
template <int LOADS>
__global__ void __launch_bounds__(512) gather256(double2* a, int kbits, int cbits, uint64_t free_mask,
                                                 const uint64_t* offs, uint64_t ntiles) {
    extern __shared__ uint64_t soff[];
    const int h = kbits - cbits;
    for (int u = threadIdx.x; u < (1 << h); u += blockDim.x) soff[u] = offs[u];
    __syncthreads();
    const uint32_t T = blockDim.x;
    const uint32_t cmask = (1u << cbits) - 1;
    for (uint64_t tau = blockIdx.x; tau < ntiles; tau += gridDim.x) {
        const uint64_t i0 = pdep(tau, free_mask);
        double v[LOADS][4];
        uint64_t g[LOADS];
#pragma unroll
        for (int d = 0; d < LOADS; ++d) {
            const uint32_t l = 2 * (d * T + threadIdx.x);
            g[d] = (i0 ^ soff[l >> cbits]) | (l & cmask);
            asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(v[d][0]), "=d"(v[d][1]), "=d"(v[d][2]), "=d"(v[d][3])
                         : "l"(a + g[d]));
        }
#pragma unroll
        for (int d = 0; d < LOADS; ++d) {
            v[d][0] += 1.0;
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(a + g[d]), "d"(v[d][0]), "d"(v[d][1]),
                         "d"(v[d][2]), "d"(v[d][3])
                         : "memory");
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    double2* a;
    const size_t bytes = (sizeof(double2)) << n;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return 1;
    cudaMemset(a, 0, bytes);
    uint64_t* d_offs;
    cudaMalloc(&d_offs, 8 << 12);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::mt19937_64 rng(7);
    printf("n=%d state %.1f GiB\n", n, bytes / 1073741824.0);
    struct Cfg { int k, c, threads, vec; };
    const Cfg cfgs[] = {{11, 4, 128, 1}, {11, 4, 256, 1}, {11, 4, 64, 2}, {11, 4, 128, 2}, {11, 4, 256, 2},
                        {12, 4, 256, 1}, {12, 4, 512, 1}, {12, 4, 256, 2}, {10, 4, 64, 1}, {10, 4, 128, 1}};
    for (const Cfg cf : cfgs) {
        const int h = cf.k - cf.c;
        std::vector<uint64_t> basis;
        uint64_t pivmask = 0;
        while ((int)basis.size() < h) {
            const int p = cf.c + 3 + (int)(rng() % (uint64_t)(n - cf.c - 3));
            if ((pivmask >> p) & 1) continue;
            uint64_t v = (1ull << p) | (rng() & ((1ull << p) - 1) & ~((1ull << cf.c) - 1));
            basis.push_back(v);
            pivmask |= 1ull << p;
        }
        for (size_t i = 0; i < basis.size(); ++i)
            for (size_t j = 0; j < basis.size(); ++j)
                if (i != j && ((basis[j] >> (63 - __builtin_clzll(basis[i]))) & 1)) basis[j] ^= basis[i];
        std::vector<uint64_t> offs(1ull << h);
        for (uint64_t u = 0; u < offs.size(); ++u) {
            uint64_t o = 0;
            for (int t = 0; t < h; ++t)
                if ((u >> t) & 1) o ^= basis[t];
            offs[u] = o;
        }
        cudaMemcpy(d_offs, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice);
        const uint64_t free_mask = ((1ull << n) - 1) & ~((1ull << cf.c) - 1) & ~pivmask;
        const uint64_t ntiles = 1ull << (n - cf.k);
        const int loads = (1 << cf.k) / cf.threads / cf.vec;
        for (int occ : {2, 4, 8, 16}) {
            if (occ * cf.threads > 2048) continue;
            const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)nsm * occ);
            const size_t smem = std::max<size_t>(8ull << h, 200000 / occ);
            cudaFuncSetAttribute(gather<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaFuncSetAttribute(gather<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaFuncSetAttribute(gather<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaFuncSetAttribute(gather256<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaFuncSetAttribute(gather256<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaFuncSetAttribute(gather256<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            auto launch = [&]() {
                if (cf.vec == 1) {
                    if (loads == 8) gather<8><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                    if (loads == 16) gather<16><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                    if (loads == 32) gather<32><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                } else {
                    if (loads == 4) gather256<4><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                    if (loads == 8) gather256<8><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                    if (loads == 16) gather256<16><<<grid, cf.threads, smem>>>(a, cf.k, cf.c, free_mask, d_offs, ntiles);
                }
            };
            launch();
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int reps = 3;
            for (int r = 0; r < reps; ++r) launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const cudaError_t err = cudaGetLastError();
            int real_occ = 0;
            if (cf.vec == 1 && loads == 16) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&real_occ, gather<16>, cf.threads, smem);
            printf("k=%2d c=%d thr=%3d vec=%d loads/thr=%2d ctas/SM=%2d (occ %d) inflight/SM=%6d B : %7.1f GB/s %s\n", cf.k, cf.c,
                   cf.threads, cf.vec, loads, occ, real_occ, occ * (1 << cf.k) * 16, 2.0 * bytes * reps / (ms / 1e3) / 1e9,
                   err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
    }
    return 0;
}
