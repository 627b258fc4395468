// Device problem data: f, u_D, g and the exact solution of the six problem
// kinds (reference built-ins analysis.cpp:9-49 plus the config problems of
// BASELINE.json).  Same expression trees as the CPU restatement
// (oracle/problems.h) with explicitly rounded arithmetic, so the polynomial
// kinds are bit-identical to the reference; the transcendental kinds differ
// only by the libm-vs-libdevice ulp of sin/cos/exp.
#pragma once

#include "common.cuh"

namespace phg {

constexpr double kPi = 3.14159265358979323846;

struct Coef {
    double a0, a1, a2;  // diagonal diffusion
    double c;           // reaction
};

template <int KIND>
__device__ __forceinline__ double prob_u(double x, double y, double z) {
    if constexpr (KIND == 0) {
        return mul(mul(mul(mul(mul(x, x), y), y), z), z);
    } else if constexpr (KIND == 1) {
        return add(add(add(x, mul(2.0, y)), mul(3.0, z)), 4.0);
    } else if constexpr (KIND == 3) {
        return mul(mul(sin(mul(kPi, x)), sin(mul(kPi, y))), sin(mul(kPi, z)));
    } else if constexpr (KIND == 4) {
        return mul(mul(exp(x), cos(mul(kPi, y))), mul(z, z));
    } else if constexpr (KIND == 5) {
        return mul(mul(mul(x, sub(8.0, x)), sin(mul(kPi, y))), sin(mul(kPi, z)));
    } else {
        return 0.0;
    }
}

template <int KIND>
__device__ __forceinline__ V3 prob_grad(double x, double y, double z) {
    if constexpr (KIND == 0) {
        return {mul(mul(mul(mul(mul(2.0, x), y), y), z), z), mul(mul(mul(mul(mul(2.0, x), x), y), z), z),
                mul(mul(mul(mul(mul(2.0, x), x), y), y), z)};
    } else if constexpr (KIND == 1) {
        return {1.0, 2.0, 3.0};
    } else if constexpr (KIND == 3) {
        const double sx = sin(mul(kPi, x)), sy = sin(mul(kPi, y)), sz = sin(mul(kPi, z));
        const double cx = cos(mul(kPi, x)), cy = cos(mul(kPi, y)), cz = cos(mul(kPi, z));
        return {mul(mul(mul(kPi, cx), sy), sz), mul(mul(mul(kPi, sx), cy), sz), mul(mul(mul(kPi, sx), sy), cz)};
    } else if constexpr (KIND == 4) {
        const double ex = exp(x), cy = cos(mul(kPi, y)), sy = sin(mul(kPi, y));
        return {mul(mul(ex, cy), mul(z, z)), mul(mul(mul(-kPi, ex), sy), mul(z, z)), mul(mul(mul(2.0, ex), cy), z)};
    } else if constexpr (KIND == 5) {
        const double q = mul(x, sub(8.0, x));
        const double sy = sin(mul(kPi, y)), sz = sin(mul(kPi, z));
        const double cy = cos(mul(kPi, y)), cz = cos(mul(kPi, z));
        return {mul(mul(sub(8.0, mul(2.0, x)), sy), sz), mul(mul(mul(kPi, q), cy), sz), mul(mul(mul(kPi, q), sy), cz)};
    } else {
        return {0.0, 0.0, 0.0};
    }
}

// f = -div(A grad u) + c u
template <int KIND>
__device__ __forceinline__ double prob_f(double x, double y, double z, const Coef& k) {
    if constexpr (KIND == 0) {
        const double u = mul(mul(mul(mul(mul(x, x), y), y), z), z);
        const double yyzz = mul(mul(mul(y, y), z), z);
        const double xxzz = mul(mul(mul(x, x), z), z);
        const double xxyy = mul(mul(mul(x, x), y), y);
        return add(mul(-2.0, add(add(mul(k.a0, yyzz), mul(k.a1, xxzz)), mul(k.a2, xxyy))), mul(k.c, u));
    } else if constexpr (KIND == 1) {
        return mul(k.c, add(add(add(x, mul(2.0, y)), mul(3.0, z)), 4.0));
    } else if constexpr (KIND == 3) {
        const double u = mul(mul(sin(mul(kPi, x)), sin(mul(kPi, y))), sin(mul(kPi, z)));
        return mul(add(mul(mul(kPi, kPi), add(add(k.a0, k.a1), k.a2)), k.c), u);
    } else if constexpr (KIND == 4) {
        const double ex = exp(x), cy = cos(mul(kPi, y));
        const double u = mul(mul(ex, cy), mul(z, z));
        const double uxx = u, uyy = mul(-mul(kPi, kPi), u), uzz = mul(mul(2.0, ex), cy);
        return add(-add(add(mul(k.a0, uxx), mul(k.a1, uyy)), mul(k.a2, uzz)), mul(k.c, u));
    } else if constexpr (KIND == 5) {
        const double sy = sin(mul(kPi, y)), sz = sin(mul(kPi, z));
        const double u = mul(mul(mul(x, sub(8.0, x)), sy), sz);
        const double uxx = mul(mul(-2.0, sy), sz), uyy = mul(-mul(kPi, kPi), u);
        return add(-add(add(mul(k.a0, uxx), mul(k.a1, uyy)), mul(k.a2, uyy)), mul(k.c, u));
    } else {
        return 0.0;
    }
}

// Quadrature-loop version of f for the transcendental kinds: sinpi/cospi
// (no argument rounding of pi*x) and FMA.  These kinds cannot be bit-exact
// with the CPU's libm anyway; they stay within ~1e-15 relative of it, well
// inside the 1e-12 load-vector bar.  Polynomial kinds use prob_f.
template <int KIND>
__device__ __forceinline__ double prob_f_fast(double x, double y, double z, double cpre, const Coef& k) {
    if constexpr (KIND == 3) {
        return cpre * (sinpi(x) * sinpi(y) * sinpi(z));
    } else if constexpr (KIND == 4) {
        // -(a0 u + a1 (-pi^2) u + a2 (2 e^x cos)) + c u with u = e^x cos z^2
        const double ec = exp(x) * cospi(y);
        const double u = ec * (z * z);
        return fma(cpre, u, -(k.a2 * 2.0) * ec);
    } else if constexpr (KIND == 5) {
        const double s = sinpi(y) * sinpi(z);
        const double u = x * (8.0 - x) * s;
        return fma(cpre, u, 2.0 * k.a0 * s);
    } else {
        return prob_f<KIND>(x, y, z, k);
    }
}
// sin(pi x), cos(pi x) and e^x at the quadrature points of one element as a
// series around the centre of the element's range on each axis: with
// delta = l1 d1 + l2 d2 + l3 d3 (d_i = x_i - x0) and m = (min + max) / 2 of
// {0, d1, d2, d3}, x = x0 + m + (delta - m) and, with z = pi (delta - m)
// (trig) or z = delta - m (exp),
//   g(x0 + m + z') = sum_{n<=N} g^(n)(x0 + m)/n! * z^n,
// whose coefficients are formed once per element from sinpi/cospi/exp at
// x0 + m; one quadrature point then costs 1 + N FMA per axis (the argument
// is a fused chain l1 e1 + l2 e2 + l3 e3 - pi m).  |z| <= r = pi (max - min)/2,
// half the span of a series around a vertex, so a Kuhn element of config 4
// (r = pi/256) needs one order less.  All derivatives of these g are
// bounded by 1 (trig) or e^xc e^|z| (exp), so the truncation error of the
// plain series is below r^(N+1)/(N+1)!; the economised series below do
// better at one order less.  Elements with r > 0.12 keep the direct
// sinpi/cospi/exp evaluation.
enum { kTaySin = 0, kTayCos = 1, kTayExp = 2 };
template <int N>
struct AxisTaylor {
    double k[N + 1];
    double e1, e2, e3, em;  // z = l1 e1 + l2 e2 + l3 e3 + em
};
// half span of one axis (pi-scaled; also bounds the exp axis' |z|)
__device__ __forceinline__ double axis_r(double x0, double x1, double x2, double x3) {
    const double d1 = x1 - x0, d2 = x2 - x0, d3 = x3 - x0;
    const double lo = fmin(fmin(0.0, d1), fmin(d2, d3)), hi = fmax(fmax(0.0, d1), fmax(d2, d3));
    return kPi * 0.5 * (hi - lo);
}
// The series are Chebyshev-economised: the Taylor series one or two degrees
// higher with its top terms replaced through T_m on [-r, r] (the same
// magnitudes as 1/n! with tiny corrections; generated and checked by
// tools/econ_tables.py, tests/test_econ_tables.py).  Classes and their
// errors measured against mpmath over the interval (relative):
//   N = 5, |z| <= 0.0125: cos 2.2e-16, sin 4.7e-19, exp 2.3e-16
//   N = 6, |z| <= 0.028:  cos 1.5e-19, sin 4.2e-17, exp 5.0e-17
//   N = 7, |z| <= 0.05:   cos 1.5e-17, sin 5.4e-18, exp 1.9e-17
//   N = 9, |z| <= 0.12:   cos 7.7e-19, sin 1.9e-18, exp 2.4e-18
// N >= 6 stay below half an ulp, N = 5 within one ulp of 1 -- the
// libm-vs-libdevice difference of sin/cos/exp themselves, and four orders
// below the 1e-12 parity tolerance of the load vector (plain Taylor at
// these orders would leave up to ~3e-15).  Table entry n = |coefficient of
// z^n| (the sign comes from the derivative cycle of sin / cos; all positive
// for exp).
template <int N>
__device__ __forceinline__ double econ_trig(int n) {
    if constexpr (N == 5) {
        constexpr double c[6] = {0x1.fffffffffffffp-1, 0x1.fffffffffffffp-1, 0x1.ffffffffac1d3p-2,
                                 0x1.55555555300cfp-3, 0x1.5554a6921735fp-5, 0x1.11109c8ee7a6dp-7};
        return c[n];
    } else if constexpr (N == 6) {
        constexpr double c[7] = {1.0, 0x1.fffffffffffa2p-1, 0x1.fffffffffffcap-2, 0x1.55555551aab14p-3,
                                 0x1.55555552b6e02p-5, 0x1.110ec879513c9p-7, 0x1.6c142550f260ep-10};
        return c[n];
    } else if constexpr (N == 7) {
        constexpr double c[8] = {1.0, 1.0, 0x1.ffffffffff92fp-2, 0x1.5555555555555p-3, 0x1.5555553ab3ecdp-5,
                                 0x1.1111111111111p-7, 0x1.6c0e6efb6a97fp-10, 0x1.a01a01a01a01ap-13};
        return c[n];
    } else {
        constexpr double c[10] = {1.0, 1.0, 0x1.fffffffffffebp-2, 0x1.5555555555555p-3, 0x1.555555553eb70p-5,
                                  0x1.1111111111111p-7, 0x1.6c16bf4655446p-10, 0x1.a01a01a01a01ap-13,
                                  0x1.9fef65c59e4bfp-16, 0x1.71de3a556c734p-19};
        return c[n];
    }
}
template <int N>
__device__ __forceinline__ double econ_exp(int n) {
    if constexpr (N == 5) {
        constexpr double c[6] = {0x1.0000000000001p+0, 0x1.0000000000000p+0, 0x1.ffffffffac1d3p-2,
                                 0x1.5555555555555p-3, 0x1.555604189374cp-5, 0x1.1111111111111p-7};
        return c[n];
    } else if constexpr (N == 6) {
        constexpr double c[7] = {1.0, 0x1.000000000002fp+0, 0x1.0000000000000p-1, 0x1.55555551aab14p-3,
                                 0x1.5555555555555p-5, 0x1.111359a8d0e59p-7, 0x1.6c16c16c16c17p-10};
        return c[n];
    } else if constexpr (N == 7) {
        constexpr double c[8] = {1.0, 1.0, 0x1.0000000000369p-1, 0x1.5555555555555p-3, 0x1.5555553ab3ecdp-5,
                                 0x1.1111111111111p-7, 0x1.6c1f13dcc2eaep-10, 0x1.a01a01a01a01ap-13};
        return c[n];
    } else {
        constexpr double c[10] = {1.0, 1.0, 0x1.fffffffffffebp-2, 0x1.5555555555555p-3, 0x1.555555556bf3bp-5,
                                  0x1.1111111111111p-7, 0x1.6c16bf4655446p-10, 0x1.a01a01a01a01ap-13,
                                  0x1.a0449d7a95b75p-16, 0x1.71de3a556c734p-19};
        return c[n];
    }
}
// 0 = out of range (direct evaluation by sinpi / cospi / exp)
__device__ __forceinline__ int taylor_order(double r) {
    return r <= 0.0125 ? 5 : (r <= 0.028 ? 6 : (r <= 0.05 ? 7 : (r <= 0.12 ? 9 : 0)));
}
template <int N, int G>
__device__ __forceinline__ AxisTaylor<N> axis_taylor(double x0, double x1, double x2, double x3) {
    AxisTaylor<N> a;
    const double sc = G == kTayExp ? 1.0 : kPi;
    const double d1 = x1 - x0, d2 = x2 - x0, d3 = x3 - x0;
    const double lo = fmin(fmin(0.0, d1), fmin(d2, d3)), hi = fmax(fmax(0.0, d1), fmax(d2, d3));
    // the expansion point xc and the offset xc - x0 it really has
    const double xc = x0 + 0.5 * (lo + hi);
    a.e1 = sc * d1;
    a.e2 = sc * d2;
    a.e3 = sc * d3;
    a.em = -sc * (xc - x0);
    if constexpr (G == kTayExp) {
        const double e0 = exp(xc);
#pragma unroll
        for (int n = 0; n <= N; ++n) a.k[n] = e0 * econ_exp<N>(n);
    } else {
        double s0, c0;
        sincospi(xc, &s0, &c0);
        // derivative cycle of sin: s c -s -c; of cos: c -s -c s
        const double d[4] = {G == kTaySin ? s0 : c0, G == kTaySin ? c0 : -s0, G == kTaySin ? -s0 : -c0,
                             G == kTaySin ? -c0 : s0};
#pragma unroll
        for (int n = 0; n <= N; ++n) a.k[n] = d[n & 3] * econ_trig<N>(n);
    }
    return a;
}

// loop-invariant factor of prob_f_fast
template <int KIND>
__device__ __forceinline__ double prob_f_pre(const Coef& k) {
    constexpr double pi2 = kPi * kPi;
    if constexpr (KIND == 3) return pi2 * (k.a0 + k.a1 + k.a2) + k.c;
    if constexpr (KIND == 4) return -k.a0 + k.a1 * pi2 + k.c;
    if constexpr (KIND == 5) return (k.a1 + k.a2) * pi2 + k.c;
    return 0.0;
}

// g = (A grad u) . n
template <int KIND>
__device__ __forceinline__ double prob_g(double x, double y, double z, V3 n, const Coef& k) {
    const V3 g = prob_grad<KIND>(x, y, z);
    return add(add(mul(mul(k.a0, g.x), n.x), mul(mul(k.a1, g.y), n.y)), mul(mul(k.a2, g.z), n.z));
}

__device__ __forceinline__ Coef load_coef(const phg_problem& p, int64_t t) {
    Coef k;
    if (p.a_diag) {
        k.a0 = __ldg(p.a_diag + 3 * t);
        k.a1 = __ldg(p.a_diag + 3 * t + 1);
        k.a2 = __ldg(p.a_diag + 3 * t + 2);
    } else if (p.a_elem) {
        k.a0 = k.a1 = k.a2 = __ldg(p.a_elem + t);
    } else {
        k.a0 = k.a1 = k.a2 = 1.0;
    }
    k.c = p.c;
    return k;
}

// load_coef with loads that are not merged with earlier ones (ld_fresh)
__device__ __forceinline__ Coef load_coef_fresh(const phg_problem& p, int64_t t) {
    Coef k;
    if (p.a_diag) {
        k.a0 = ld_fresh(p.a_diag + 3 * t);
        k.a1 = ld_fresh(p.a_diag + 3 * t + 1);
        k.a2 = ld_fresh(p.a_diag + 3 * t + 2);
    } else if (p.a_elem) {
        k.a0 = k.a1 = k.a2 = ld_fresh(p.a_elem + t);
    } else {
        k.a0 = k.a1 = k.a2 = 1.0;
    }
    k.c = p.c;
    return k;
}

// -------------------------------------------------------------- element core

// Division policies of the element core.  ExactDiv gives IEEE quotients
// (dq: shared reciprocal + Markstein, IEEE fallback).  FastDiv is
// straight-line (no branches) and records in `ok` whether every operand was
// inside the window where that equals IEEE division; when it is not, the
// caller recomputes the element with ExactDiv.
struct ExactDiv {
    __device__ __forceinline__ bool good() const { return true; }
    __device__ __forceinline__ double div(double a, const Div& d) { return dq(a, d); }
    __device__ __forceinline__ Div make(double b) { return make_div(b); }
};
struct FastDiv {
    bool ok = true;
    __device__ __forceinline__ bool good() const { return ok; }
    __device__ __forceinline__ double div(double a, const Div& d) { return dq_fast(a, d, ok); }
    __device__ __forceinline__ Div make(double b) { return make_div_fast(b, ok); }
};

// local_stiffness_mass (assembly.cpp:7-33) with A_T = K(A) + c M
struct Local {
    double a[4][4];
    double vol;
    V3 g[4];
    bool degenerate;
};

template <class Dv>
__device__ __forceinline__ void local_matrices(const V3 p[4], const Coef& k, Local& L, Dv& dv) {
    const V3 d1 = vsub(p[1], p[0]), d2 = vsub(p[2], p[0]), d3 = vsub(p[3], p[0]);
    const double det = vdot(vcross(d1, d2), d3);
    L.degenerate = det == 0.0;
    L.vol = dv.div(fabs(det), kDiv6);
    const Div ddet = dv.make(det);
    const V3 c1 = vcross(d2, d3), c2 = vcross(d3, d1), c3 = vcross(d1, d2);
    L.g[1] = {dv.div(c1.x, ddet), dv.div(c1.y, ddet), dv.div(c1.z, ddet)};
    L.g[2] = {dv.div(c2.x, ddet), dv.div(c2.y, ddet), dv.div(c2.z, ddet)};
    L.g[3] = {dv.div(c3.x, ddet), dv.div(c3.y, ddet), dv.div(c3.z, ddet)};
    L.g[0] = vmul(vadd(vadd(L.g[1], L.g[2]), L.g[3]), -1.0);
    const double m20 = dv.div(L.vol, kDiv20);
    const double mdiag = mul(k.c, mul(m20, 2.0)), moff = mul(k.c, mul(m20, 1.0));
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const V3 gi = L.g[i], gj = L.g[j];
            const double d = add(add(mul(k.a0, mul(gi.x, gj.x)), mul(k.a1, mul(gi.y, gj.y))), mul(k.a2, mul(gi.z, gj.z)));
            L.a[i][j] = add(mul(L.vol, d), i == j ? mdiag : moff);
        }
}
__device__ __forceinline__ void local_matrices(const V3 p[4], const Coef& k, Local& L) {
    ExactDiv dv;
    local_matrices(p, k, L, dv);
}

// Mat4Lu::factor / solve (geom.hpp:48-87)
struct Lu4 {
    double lu[4][4];
    int perm[4];
    bool singular;
    Div piv[4];  // shared reciprocals of the pivots lu[i][i]
};

template <class Dv>
__device__ __forceinline__ void lu_factor(const double a[4][4], Lu4& f, Dv& dv) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f.perm[i] = i;
#pragma unroll
        for (int j = 0; j < 4; ++j) f.lu[i][j] = a[i][j];
    }
    f.singular = false;
#pragma unroll
    for (int col = 0; col < 4; ++col) {
        int piv = col;
        double best = fabs(f.lu[col][col]);
#pragma unroll
        for (int r = col + 1; r < 4; ++r) {
            const double v = fabs(f.lu[r][col]);
            if (v > best) { best = v; piv = r; }
        }
        if (best == 0.0) { f.singular = true; return; }
        if (piv != col) {
            // swap rows piv and col (register arrays: select instead of
            // dynamic indexing)
#pragma unroll
            for (int r = col + 1; r < 4; ++r) {
                if (r == piv) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const double t = f.lu[r][c];
                        f.lu[r][c] = f.lu[col][c];
                        f.lu[col][c] = t;
                    }
                    const int tp = f.perm[r];
                    f.perm[r] = f.perm[col];
                    f.perm[col] = tp;
                }
            }
        }
        f.piv[col] = dv.make(f.lu[col][col]);
#pragma unroll
        for (int r = col + 1; r < 4; ++r) {
            const double m = dv.div(f.lu[r][col], f.piv[col]);
            f.lu[r][col] = m;
#pragma unroll
            for (int c = col + 1; c < 4; ++c) f.lu[r][c] = sub(f.lu[r][c], mul(m, f.lu[col][c]));
        }
    }
}
__device__ __forceinline__ void lu_factor(const double a[4][4], Lu4& f) {
    ExactDiv dv;
    lu_factor(a, f, dv);
}

__device__ __forceinline__ double sel4(const double b[4], int i) {
    return i == 0 ? b[0] : (i == 1 ? b[1] : (i == 2 ? b[2] : b[3]));
}

template <class Dv>
__device__ __forceinline__ void lu_solve(const Lu4& f, const double b[4], double x[4], Dv& dv) {
    double y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double s = sel4(b, f.perm[i]);
#pragma unroll
        for (int j = 0; j < i; ++j) s = sub(s, mul(f.lu[i][j], y[j]));
        y[i] = s;
    }
#pragma unroll
    for (int i = 3; i >= 0; --i) {
        double s = y[i];
#pragma unroll
        for (int j = i + 1; j < 4; ++j) s = sub(s, mul(f.lu[i][j], x[j]));
        x[i] = dv.div(s, f.piv[i]);
    }
}
__device__ __forceinline__ void lu_solve(const Lu4& f, const double b[4], double x[4]) {
    ExactDiv dv;
    lu_solve(f, b, x, dv);
}

}  // namespace phg
