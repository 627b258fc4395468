// Building blocks of the reduce-then-scan kernels (scan.cu and the fused
// count + scan passes of connectivity.cu / refine.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace phg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

inline int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

__device__ __forceinline__ long long warp_incl_scan_ll(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// exclusive block scan of one value per thread (NT threads, NT <= 1024);
// *total (optional) receives the block total
template <int NT>
__device__ __forceinline__ long long block_excl_scan_ll(long long v, long long* total = nullptr) {
    __shared__ long long warp_sums[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long inc = warp_incl_scan_ll(v);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        long long s = lane < NT / 32 ? warp_sums[lane] : 0;
        s = warp_incl_scan_ll(s);
        if (lane < NT / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const long long base = warp ? warp_sums[warp - 1] : 0;
    if (total) *total = warp_sums[NT / 32 - 1];
    __syncthreads();
    return base + inc - v;
}

template <int NT>
__device__ __forceinline__ long long block_sum_ll(long long v) {
    __shared__ long long warp_sums[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
    __syncthreads();
    long long s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) s += warp_sums[i];
    return s;  // valid in thread 0
}

// In-place exclusive scan of n tile sums by one 1024-thread block (launched
// on s); *total (device) = grand total.  Defined in scan.cu.
void scan_sums(long long* sums, int64_t n, int64_t* total, cudaStream_t s);

// shared-memory staging index: one pad word per 16 (blocked writes of 16
// consecutive int64 per thread stay within 2-way bank conflicts)
__device__ __forceinline__ int scan_pad(int i) { return i + (i >> 4); }

// write a staged tile of kScanTile int64 to out[base ..) coalesced (16 B
// stores where the tile is complete and aligned)
__device__ __forceinline__ void store_tile_i64(const long long* stage, int64_t* __restrict__ out, int64_t base,
                                               int64_t n) {
    if (base + kScanTile <= n && (base & 1) == 0) {
        longlong2* o = reinterpret_cast<longlong2*>(out + base);
#pragma unroll
        for (int k = 0; k < kScanTile / 2 / kScanThreads; ++k) {
            const int j = (int)threadIdx.x + k * kScanThreads;  // pair index
            o[j] = make_longlong2(stage[scan_pad(2 * j)], stage[scan_pad(2 * j + 1)]);
        }
    } else {
        for (int i = threadIdx.x; i < kScanTile; i += kScanThreads)
            if (base + i < n) out[base + i] = stage[scan_pad(i)];
    }
}

}  // namespace phg
