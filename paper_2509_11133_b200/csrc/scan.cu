// Deterministic device-wide exclusive scans (counts -> int64 offsets), the
// "unique/scan" half of the numbering pipeline.
//
// Reduce-then-scan in three kernels, no inter-block waiting:
//   1. tile sums        (4096 items per 256-thread block, 16 B loads)
//   2. scan of the sums (one 1024-thread block)
//   3. tile scan        (offsets staged in shared memory and written out
//                        coalesced as 16 B stores)
// Integer sums: the result does not depend on the schedule.
#include <atomic>

#include <cuda_runtime.h>

#include "common.cuh"
#include "scan.cuh"

namespace {

using namespace phg;

// ------------------------------------------------------- generic int32 scan
__global__ void __launch_bounds__(kScanThreads) tile_sums_i32(const int32_t* __restrict__ in, int64_t n,
                                                             long long* __restrict__ sums) {
    const int64_t first = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long s = 0;
    if (first + kScanItems <= n) {
        const int4* p = reinterpret_cast<const int4*>(in + first);
#pragma unroll
        for (int i = 0; i < kScanItems / 4; ++i) {
            const int4 q = __ldg(p + i);
            s += (long long)q.x + q.y + q.z + q.w;
        }
    } else {
        for (int i = 0; i < kScanItems; ++i)
            if (first + i < n) s += in[first + i];
    }
    s = block_sum_ll<kScanThreads>(s);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kScanThreads) tile_scan_i32(const int32_t* __restrict__ in, int64_t n,
                                                             const long long* __restrict__ tile_off,
                                                             int64_t* __restrict__ out) {
    __shared__ long long stage[kScanTile + kScanTile / 16];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int64_t first = base + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    if (first + kScanItems <= n) {
        const int4* p = reinterpret_cast<const int4*>(in + first);
#pragma unroll
        for (int i = 0; i < kScanItems / 4; ++i) {
            const int4 q = __ldg(p + i);
            v[4 * i] = q.x;
            v[4 * i + 1] = q.y;
            v[4 * i + 2] = q.z;
            v[4 * i + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) v[i] = first + i < n ? in[first + i] : 0;
    }
    long long s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) s += v[i];
    long long run = block_excl_scan_ll<kScanThreads>(s) + tile_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        stage[scan_pad(threadIdx.x * kScanItems + i)] = run;
        run += v[i];
    }
    __syncthreads();
    store_tile_i64(stage, out, base, n);
}

// exclusive scan of the tile sums, 4 per thread per round, carried over
// rounds of 4096
__global__ void __launch_bounds__(1024) scan_sums_k(long long* __restrict__ sums, int64_t n,
                                                    int64_t* __restrict__ total) {
    long long carry = 0;
    for (int64_t b = 0; b < n; b += 4096) {
        const int64_t i0 = b + 4 * (int64_t)threadIdx.x;
        long long v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = i0 + k < n ? sums[i0 + k] : 0;
        long long round;
        long long run = carry + block_excl_scan_ll<1024>(v[0] + v[1] + v[2] + v[3], &round);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i0 + k < n) sums[i0 + k] = run;
            run += v[k];
        }
        carry += round;
    }
    if (threadIdx.x == 0) *total = carry;
}

std::atomic<long long> g_launches{0};

}  // namespace

void phg::count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void phg::scan_sums(long long* sums, int64_t n, int64_t* total, cudaStream_t s) {
    scan_sums_k<<<1, 1024, 0, s>>>(sums, n, total);
}

extern "C" long long phfem_gpu_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" size_t phfem_gpu_scan_scratch(int64_t n) {
    return (size_t)(phg::scan_tiles(n) + 1) * sizeof(long long);
}

extern "C" int phfem_gpu_scan_i32(const int32_t* in, int64_t* out, int64_t n, void* scratch, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n <= 0) {
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
        return (int)cudaGetLastError();
    }
    const int64_t ntiles = phg::scan_tiles(n);
    long long* sums = static_cast<long long*>(scratch);
    tile_sums_i32<<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, sums);
    phg::scan_sums(sums, ntiles, out + n, s);
    tile_scan_i32<<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, sums, out);
    phg::count_launches(3);
    return (int)cudaGetLastError();
}
