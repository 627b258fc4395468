// Mesh input path on the device: the n_x*n_y*n_z*6 Kuhn generator of the
// BASELINE.json configs (restated on the CPU by
// oracle/phfem_oracle.c:or_kuhn_mesh) and the mesh diameter (mesh.cpp:90-106).
// Coordinates use only correctly rounded +,*,/ so they are bit-identical to
// the CPU generator.
#include <algorithm>
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

using namespace phg;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform(uint64_t seed, uint64_t idx) {
    return __dmul_rn((double)(splitmix64(seed ^ idx) >> 11), 0x1.0p-53);
}

__global__ void kuhn_nodes(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                           uint64_t seed, double* __restrict__ coords) {
    const int64_t nnodes = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nnodes;
         n += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = n % (nx + 1);
        const int64_t j = (n / (nx + 1)) % (ny + 1);
        const int64_t k = n / ((int64_t)(nx + 1) * (ny + 1));
        double x = dvd(mul(lx, (double)i), (double)nx);
        double y = dvd(mul(ly, (double)j), (double)ny);
        double z = dvd(mul(lz, (double)k), (double)nz);
        if (jitter != 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
            const double hx = dvd(lx, (double)nx), hy = dvd(ly, (double)ny), hz = dvd(lz, (double)nz);
            x = add(x, mul(mul(sub(mul(2.0, uniform(seed, 3 * (uint64_t)n)), 1.0), jitter), hx));
            y = add(y, mul(mul(sub(mul(2.0, uniform(seed, 3 * (uint64_t)n + 1)), 1.0), jitter), hy));
            z = add(z, mul(mul(sub(mul(2.0, uniform(seed, 3 * (uint64_t)n + 2)), 1.0), jitter), hz));
        }
        coords[3 * n] = x;
        coords[3 * n + 1] = y;
        coords[3 * n + 2] = z;
    }
}

// path permutations of the Kuhn subdivision; odd ones swap the last two
// vertices to keep det[b-a, c-a, d-a] > 0
__device__ __forceinline__ void kuhn_tet(int nx, int ny, int nz, int64_t t, int64_t idx[4][3]) {
    const int64_t cell = t / 6;
    const int p = (int)(t % 6);
    const int64_t i = cell % nx, j = (cell / nx) % ny, k = cell / ((int64_t)nx * ny);
    const int perm0 = p < 2 ? 0 : (p < 4 ? 1 : 2);
    const int perm1 = (p == 0 || p == 5) ? 1 : ((p == 1 || p == 3) ? 2 : 0);
    int64_t a[3] = {i, j, k};
    for (int d = 0; d < 3; ++d) idx[0][d] = a[d];
    a[perm0] += 1;
    for (int d = 0; d < 3; ++d) idx[1][d] = a[d];
    a[perm1] += 1;
    for (int d = 0; d < 3; ++d) idx[2][d] = a[d];
    a[0] = i + 1; a[1] = j + 1; a[2] = k + 1;
    for (int d = 0; d < 3; ++d) idx[3][d] = a[d];
    const bool odd = (p == 1 || p == 2 || p == 5);
    if (odd)
        for (int d = 0; d < 3; ++d) {
            const int64_t tmp = idx[2][d];
            idx[2][d] = idx[3][d];
            idx[3][d] = tmp;
        }
}

// plane of local face f (0:x=0 1:x=max 2:y=0 3:y=max 4:z=0 5:z=max) or -1
__device__ __forceinline__ int face_plane(const int64_t idx[4][3], int f, int nx, int ny, int nz) {
    for (int d = 0; d < 3; ++d) {
        const int64_t c0 = idx[face_vert(f, 0)][d], c1 = idx[face_vert(f, 1)][d], c2 = idx[face_vert(f, 2)][d];
        const int64_t nmax = d == 0 ? nx : (d == 1 ? ny : nz);
        if (c0 == c1 && c1 == c2 && (c0 == 0 || c0 == nmax)) return 2 * d + (c0 == 0 ? 0 : 1);
    }
    return -1;
}

__global__ void kuhn_tets(int nx, int ny, int nz, uint32_t mask, int32_t* __restrict__ tets,
                          int32_t* __restrict__ bcount) {
    const int64_t ne = 6ll * nx * ny * nz;
    const int64_t sx = nx + 1, sy = ny + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t idx[4][3];
        kuhn_tet(nx, ny, nz, t, idx);
        int4 out;
        out.x = (int32_t)(idx[0][0] + sx * (idx[0][1] + sy * idx[0][2]));
        out.y = (int32_t)(idx[1][0] + sx * (idx[1][1] + sy * idx[1][2]));
        out.z = (int32_t)(idx[2][0] + sx * (idx[2][1] + sy * idx[2][2]));
        out.w = (int32_t)(idx[3][0] + sx * (idx[3][1] + sy * idx[3][2]));
        reinterpret_cast<int4*>(tets)[t] = out;
        int nd = 0, nn = 0;
        for (int f = 0; f < 4; ++f) {
            const int pl = face_plane(idx, f, nx, ny, nz);
            if (pl < 0) continue;
            if (mask & (1u << pl)) ++nd;
            else ++nn;
        }
        bcount[t] = nd | (nn << 8);
    }
}

__global__ void kuhn_boundary(int nx, int ny, int nz, uint32_t mask, const int32_t* __restrict__ tets,
                              const int64_t* __restrict__ dir_off, const int64_t* __restrict__ neu_off,
                              int32_t* __restrict__ db, int32_t* __restrict__ nb) {
    const int64_t ne = 6ll * nx * ny * nz;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        if (dir_off[t + 1] == dir_off[t] && neu_off[t + 1] == neu_off[t]) continue;
        int64_t idx[4][3];
        kuhn_tet(nx, ny, nz, t, idx);
        const int4 tt = ldtet(tets, t);
        int64_t d = dir_off[t], n = neu_off[t];
        for (int f = 0; f < 4; ++f) {
            const int pl = face_plane(idx, f, nx, ny, nz);
            if (pl < 0) continue;
            int32_t* dst = (mask & (1u << pl)) ? db + 3 * d++ : nb + 3 * n++;
            for (int v = 0; v < 3; ++v) dst[v] = tv(tt, face_vert(f, v));
        }
    }
}

__global__ void split_counts(const int32_t* __restrict__ packed, int32_t* __restrict__ dir,
                             int32_t* __restrict__ neu, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = packed[i];
        dir[i] = v & 0xff;
        neu[i] = (v >> 8) & 0xff;
    }
}

// elem_diameter / mesh_diameter (mesh.cpp:90-106): max over pairs of
// dot(d,d), sqrt, max over elements (order-free, so exact)
__global__ void diameter(const double* __restrict__ coords, const int32_t* __restrict__ tets, int64_t ne,
                         unsigned long long* __restrict__ out) {
    double best = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        double d2 = 0.0;
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j) {
                const V3 d = vsub(p[i], p[j]);
                d2 = fmax(d2, vdot(d, d));
            }
        best = fmax(best, __dsqrt_rn(d2));
    }
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

// index validation of uploaded tables (read_mesh's range check,
// mesh.cpp:151-158): out = first offending position, or all ones
__global__ void check_indices(const int32_t* __restrict__ a, int64_t n, int64_t nc, unsigned long long* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = a[i];
        if (v < 0 || v >= nc) atomicMin(out, (unsigned long long)i);
    }
}

// self-test of the shared-reciprocal division dq() against IEEE __ddiv_rn on
// random operands spanning the magnitudes the element kernels see (and the
// fallback window edges): counts mismatching quotients bit for bit
__global__ void division_selftest(int64_t n, uint64_t seed, unsigned long long* mismatches) {
    unsigned long long bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = splitmix64(seed ^ (2 * (uint64_t)i)), h2 = splitmix64(seed ^ (2 * (uint64_t)i + 1));
        // random significands, exponents in [-560, 560] (covers the window
        // edges at 2^+-500) with a bias towards the data range [-40, 10]
        const int e1 = (h1 >> 60) < 12 ? (int)((h1 >> 52) & 63) - 45 : (int)((h1 >> 52) & 1023) - 512 - 48;
        const int e2 = (h2 >> 60) < 12 ? (int)((h2 >> 52) & 63) - 45 : (int)((h2 >> 52) & 1023) - 512 - 48;
        double a = __longlong_as_double((long long)((h1 & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
        double b = __longlong_as_double((long long)((h2 & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
        a = ldexp(a, e1) * ((h1 & 1) ? -1.0 : 1.0);
        b = ldexp(b, e2) * ((h2 & 2) ? -1.0 : 1.0);
        if ((h1 & 0xff) == 7) a = 0.0;
        const double q1 = dq(a, make_div(b));
        const double q2 = __ddiv_rn(a, b);
        if (__double_as_longlong(q1) != __double_as_longlong(q2)) ++bad;
        // the constant divisors too
        if (__double_as_longlong(dq(a, kDiv3)) != __double_as_longlong(__ddiv_rn(a, 3.0))) ++bad;
        if (__double_as_longlong(dq(a, kDiv6)) != __double_as_longlong(__ddiv_rn(a, 6.0))) ++bad;
        if (__double_as_longlong(dq(a, kDiv20)) != __double_as_longlong(__ddiv_rn(a, 20.0))) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

// fp64 peak probe (roofline denominator of the fp64-bound assembly): 8
// independent FMA chains per thread, a full resident grid, nothing but DFMA
// in the loop
__global__ void __launch_bounds__(256) fp64_peak_k(int iters, double seed, double* sink) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + 1e-9 * (threadIdx.x + i);
    const double b = 1.0 - 1e-12, c = 1e-15;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 123.456) sink[0] = s;  // keeps the chains alive
}

}  // namespace

extern "C" int phfem_gpu_fp64_peak(int iters, double* sink, void* ev_begin, void* ev_end, double* flops,
                                   void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = 148 * 8, threads = 256;
    if (ev_begin) cudaEventRecord((cudaEvent_t)ev_begin, s);
    fp64_peak_k<<<blocks, threads, 0, s>>>(iters, 1.0, sink);
    if (ev_end) cudaEventRecord((cudaEvent_t)ev_end, s);
    phg::count_launches(1);
    if (flops) *flops = 2.0 * 8.0 * (double)iters * blocks * threads;
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_division_selftest(int64_t n, uint64_t seed, unsigned long long* mismatches, void* stream) {
    division_selftest<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(n, seed, mismatches);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

namespace {
struct WordPtrs {
    const unsigned long long* p[16];
};
__global__ void gather_words_k(WordPtrs s, int n, unsigned long long* dst) {
    const int i = threadIdx.x;
    if (i < n) dst[i] = *s.p[i];
    __threadfence_system();
}
}  // namespace

extern "C" int phfem_gpu_gather_words(const unsigned long long* const* src, int n, unsigned long long* dst,
                                      void* stream) {
    if (n <= 0) return 0;
    if (n > 16) return (int)cudaErrorInvalidValue;
    WordPtrs w{};
    for (int i = 0; i < n; ++i) w.p[i] = src[i];
    gather_words_k<<<1, 32, 0, (cudaStream_t)stream>>>(w, n, dst);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_check_indices(const int32_t* a, int64_t n, int64_t nc, unsigned long long* first_bad,
                                       void* stream) {
    if (n <= 0) return 0;
    const int g = std::min<int64_t>(grid_for(n, 256), 148 * 16);
    check_indices<<<g, 256, 0, (cudaStream_t)stream>>>(a, n, nc, first_bad);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_kuhn_nodes(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                                    uint64_t seed, double* coords, void* stream) {
    const int64_t n = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    kuhn_nodes<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, lx, ly, lz, jitter, seed, coords); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_kuhn_tets(int nx, int ny, int nz, uint32_t mask, int32_t* tets, int32_t* bcount,
                                   void* stream) {
    const int64_t ne = 6ll * nx * ny * nz;
    kuhn_tets<<<grid_for(ne, 256), 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, mask, tets, bcount); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_kuhn_boundary(int nx, int ny, int nz, uint32_t mask, const int32_t* tets,
                                       const int64_t* dir_off, const int64_t* neu_off, int32_t* db, int32_t* nb,
                                       void* stream) {
    const int64_t ne = 6ll * nx * ny * nz;
    kuhn_boundary<<<grid_for(ne, 256), 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, mask, tets, dir_off, neu_off,
                                                                         db, nb); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_split_counts(const int32_t* packed, int32_t* dir, int32_t* neu, int64_t n, void* stream) {
    split_counts<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(packed, dir, neu, n); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_diameter(const double* coords, const int32_t* tets, int64_t ne, double* out,
                                  double* partials, void* stream) {
    (void)partials;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(out, 0, sizeof(double), s);
    const int grid = (int)std::min<int64_t>(grid_for(ne, 256), 148 * 8);
    diameter<<<grid, 256, 0, s>>>(coords, tets, ne, reinterpret_cast<unsigned long long*>(out)); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" const char* phfem_gpu_error_string(int code) { return cudaGetErrorString((cudaError_t)code); }
