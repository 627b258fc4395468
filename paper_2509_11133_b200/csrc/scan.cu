// Deterministic device-wide exclusive scan (int32 counts -> int64 offsets),
// the "unique/scan" half of the numbering pipeline.
// Three passes: tile reduce -> scan of tile sums (one block) -> tile scan.
#include <atomic>

#include <cuda_runtime.h>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

__device__ __forceinline__ long long warp_incl_scan(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// exclusive block scan of one value per thread; returns the block total
__device__ __forceinline__ long long block_excl_scan(long long v, long long* total) {
    __shared__ long long warp_sums[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        long long s = lane < kThreads / 32 ? warp_sums[lane] : 0;
        s = warp_incl_scan(s);
        if (lane < kThreads / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const long long base = warp ? warp_sums[warp - 1] : 0;
    *total = warp_sums[kThreads / 32 - 1];
    __syncthreads();
    return base + inc - v;
}

__global__ void __launch_bounds__(kThreads) tile_reduce(const int32_t* __restrict__ in, int64_t n,
                                                        long long* __restrict__ tile_sum) {
    const int64_t base = (int64_t)blockIdx.x * kTile;
    long long s = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int64_t idx = base + (int64_t)i * kThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    long long total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kThreads) scan_tile_sums(long long* __restrict__ tile_sum, int64_t ntiles,
                                                           int64_t* __restrict__ grand_total) {
    long long carry = 0;
    for (int64_t b = 0; b < ntiles; b += kThreads) {
        const int64_t idx = b + threadIdx.x;
        const long long v = idx < ntiles ? tile_sum[idx] : 0;
        long long total;
        const long long ex = block_excl_scan(v, &total);
        if (idx < ntiles) tile_sum[idx] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *grand_total = carry;
}

__global__ void __launch_bounds__(kThreads) tile_scan(const int32_t* __restrict__ in, int64_t n,
                                                      const long long* __restrict__ tile_off,
                                                      int64_t* __restrict__ out) {
    // blocked arrangement: thread i owns items [i*kItems, (i+1)*kItems) of the tile
    __shared__ int32_t sh[kTile];
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int64_t idx = base + (int64_t)i * kThreads + threadIdx.x;
        sh[i * kThreads + threadIdx.x] = idx < n ? in[idx] : 0;
    }
    __syncthreads();
    int32_t v[kItems];
    long long s = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        v[i] = sh[threadIdx.x * kItems + i];
        s += v[i];
    }
    long long total;
    long long run = block_excl_scan(s, &total) + tile_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int64_t idx = base + (int64_t)threadIdx.x * kItems + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
}

std::atomic<long long> g_launches{0};

}  // namespace

void phg::count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

extern "C" long long phfem_gpu_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" size_t phfem_gpu_scan_scratch(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return (size_t)(ntiles + 1) * sizeof(long long);
}

extern "C" int phfem_gpu_scan_i32(const int32_t* in, int64_t* out, int64_t n, void* scratch, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t ntiles = (n + kTile - 1) / kTile;
    long long* tile_sum = static_cast<long long*>(scratch);
    if (n > 0) {
        tile_reduce<<<(unsigned)ntiles, kThreads, 0, s>>>(in, n, tile_sum);
        phg::count_launches(3);
        scan_tile_sums<<<1, kThreads, 0, s>>>(tile_sum, ntiles, out + n);
        tile_scan<<<(unsigned)ntiles, kThreads, 0, s>>>(in, n, tile_sum, out);
    } else {
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
    }
    return (int)cudaGetLastError();
}
