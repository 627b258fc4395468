// Shared device-side definitions of the phfem B200 path.
//
// All element arithmetic that must be bit-exact with the reference uses the
// explicitly rounded intrinsics below (no FMA contraction, true division), so
// the result does not depend on -fmad (SURVEY.md 8(a')).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "phfem_gpu.h"

// Checked builds (make EXTRA=-DPHG_CHECKS, tests/test_gpu_checked.py): device
// asserts on the indices the kernels compute (star positions, hash probes,
// first-occurrence slots, node / row ids).  compute-sanitizer is not
// available on the GPU pool; these bounds checks stand in for its memcheck.
#ifdef PHG_CHECKS
#include <cassert>
#define PHG_CHECK(cond) assert(cond)
#else
#define PHG_CHECK(cond) ((void)0)
#endif

namespace phg {

// ---------------------------------------------------------------- exact fp64
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded division by a divisor shared by several quotients:
// r = RN(1/b) once, then per quotient q0 = RN(a r), rem = a - b q0 (FMA,
// exact), q = RN(q0 + rem r) (Markstein's correction, correctly rounded in
// binary64 away from under/overflow).  Operands outside a safe exponent
// window fall back to __ddiv_rn, so the result always equals a / b; the
// GPU test test_division_matches_ieee checks this against __ddiv_rn.
struct Div {
    double b, r;
    bool safe;
};
__device__ __forceinline__ Div make_div(double b) {
    const double ab = fabs(b);
    return {b, __drcp_rn(b), ab > 0x1.0p-500 && ab < 0x1.0p+500};
}
// constant divisors of the reference formulas with r = RN(1/b)
static __device__ constexpr Div kDiv3 = {3.0, 0x1.5555555555555p-2, true};
static __device__ constexpr Div kDiv6 = {6.0, 0x1.5555555555555p-3, true};
static __device__ constexpr Div kDiv20 = {20.0, 0x1.999999999999ap-5, true};
static __device__ __noinline__ double div_slow(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dq(double a, const Div& d) {
    // |a|, |b| in [2^-500, 2^500]: q, a*r and the remainder stay normal
    const double aa = fabs(a);
    if (d.safe && aa < 0x1.0p+500) {
        if (aa > 0x1.0p-500) {
            const double q0 = __dmul_rn(a, d.r);
            const double rem = __fma_rn(-d.b, q0, a);
            return __fma_rn(rem, d.r, q0);
        }
        if (a == 0.0) return __dmul_rn(a, d.r);  // signed zero
    }
    return div_slow(a, d.b);
}

// Branch-free variant for straight-line element code: always takes the
// reciprocal path and clears `ok` when an operand is outside the window
// (zero numerators are fine); callers recompute the element with exact
// division when ok ends up false.
__device__ __forceinline__ bool dq_in_range(double a) {
    const unsigned hi = (unsigned)(__double_as_longlong(a) >> 32);
    const unsigned e = (hi >> 20) & 0x7FFu;  // biased exponent
    return (e - (1023u - 499u)) < 998u || a == 0.0;
}
__device__ __forceinline__ double dq_fast(double a, const Div& d, bool& ok) {
    ok = ok && dq_in_range(a);
    const double q0 = __dmul_rn(a, d.r);
    const double rem = __fma_rn(-d.b, q0, a);
    return __fma_rn(rem, d.r, q0);
}
__device__ __forceinline__ Div make_div_fast(double b, bool& ok) {
    ok = ok && dq_in_range(b) && b != 0.0;
    return {b, __drcp_rn(b), true};
}

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ V3 vmul(V3 a, double s) { return {mul(a.x, s), mul(a.y, s), mul(a.z, s)}; }
__device__ __forceinline__ V3 vdiv(V3 a, double s) { return {dvd(a.x, s), dvd(a.y, s), dvd(a.z, s)}; }
__device__ __forceinline__ V3 vdivq(V3 a, const Div& d) { return {dq(a.x, d), dq(a.y, d), dq(a.z, d)}; }
// dot(a,b) = (ax*bx + ay*by) + az*bz  (geom.hpp:22)
__device__ __forceinline__ double vdot(V3 a, V3 b) {
    return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z));
}
// cross (geom.hpp:25)
__device__ __forceinline__ V3 vcross(V3 a, V3 b) {
    return {sub(mul(a.y, b.z), mul(a.z, b.y)), sub(mul(a.z, b.x), mul(a.x, b.z)),
            sub(mul(a.x, b.y), mul(a.y, b.x))};
}
__device__ __forceinline__ V3 ldnode(const double* __restrict__ c, int32_t n) {
    const double* p = c + 3 * (int64_t)n;
    return {__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}

// local faces [abc],[acd],[adb],[dcb] (mesh.cpp:34-37, assembly.hpp:29)
static __constant__ int kFaceVerts[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {3, 2, 1}};
// local edge pairs (connectivity.cpp:15-18)
static __constant__ int kEdgeVerts[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

__device__ __forceinline__ int face_vert(int k, int j) {
    // kFaceVerts without a constant-memory lookup (divergent k)
    switch (k) {
        case 0: return j;                       // 0 1 2
        case 1: return j == 0 ? 0 : j + 1;      // 0 2 3
        case 2: return j == 0 ? 0 : (j == 1 ? 3 : 1);  // 0 3 1
        default: return 3 - j;                  // 3 2 1
    }
}
// local edge index of the pair (a, b) of local vertices, a != b
__device__ __forceinline__ int edge_index(int a, int b) {
    if (a > b) { const int t = a; a = b; b = t; }
    // (0,1)0 (0,2)1 (0,3)2 (1,2)3 (1,3)4 (2,3)5
    return a == 0 ? b - 1 : (a == 1 ? b + 1 : 5);
}

// Loads the compiler may not merge with an earlier load of the same
// address: re-reading a value from L1/L2 is cheaper than keeping it live
// across a register-hungry phase.
__device__ __forceinline__ double ld_fresh(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int4 ldtet(const int32_t* __restrict__ tets, int64_t t) {
    return __ldg(reinterpret_cast<const int4*>(tets) + t);
}
__device__ __forceinline__ int tv(const int4& t, int i) {
    return i == 0 ? t.x : (i == 1 ? t.y : (i == 2 ? t.z : t.w));
}

// Element-major Schur blocks (assemble.cu's SchurOut::st_val, read by the
// CG): S_T[r][q], r <= q, 10 values per element in 32-element AoSoA chunks.
__device__ __forceinline__ int64_t st_idx(int64_t t, int j) { return (t >> 5) * 320 + j * 32 + (t & 31); }
// (r, q), r <= q -> 0..9: (0,0..3) 0-3, (1,1..3) 4-6, (2,2..3) 7-8, (3,3) 9
__host__ __device__ constexpr int st_pair(int r, int q) { return r == 0 ? q : (r == 1 ? q + 3 : (r == 2 ? q + 5 : 9)); }

// ----------------------------------------------------------- error reporting
// Device error slots, each holding the minimum offending key (ULLONG_MAX =
// none); the host replays them in the reference's check order.
__device__ __forceinline__ void report(unsigned long long* err, int slot, unsigned long long key) {
    if (err) atomicMin(err + slot, key);
}

// ------------------------------------------------------------- launch sizes
constexpr int kSMs = 148;

// process-wide count of kernels launched by this library (bench.py's
// gpu_launches); defined in scan.cu
void count_launches(int n);
inline int grid_for(int64_t n, int block, int per_thread = 1) {
    int64_t g = (n + (int64_t)block * per_thread - 1) / ((int64_t)block * per_thread);
    if (g < 1) g = 1;
    if (g > 0x7fffffff) g = 0x7fffffff;
    return (int)g;
}

}  // namespace phg
