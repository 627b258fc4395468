/* Problem data of the hot path, shared by the CPU oracle (phfem_oracle.c) and
 * the reference driver (ref_driver.cpp).  TEST INFRASTRUCTURE: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use anything under
 * oracle/.
 *
 * Kinds 0..2 restate the reference's built-in problems exactly
 * (analysis.cpp:9-49: manufactured x^2y^2z^2, linear patch, zero).  Kinds 3..5
 * are the BASELINE.json config problems; the reference has no
 * coefficient support, so the coefficient extension is defined here so that
 * it reduces bit-exactly to the reference at A = I, c = 1:
 *   -div(A grad u) + c u = f,  A = diag(A0, A1, A2) per element,
 *   g = (A grad u) . n  on Neumann faces, u_D = u on Dirichlet faces.
 * Every expression keeps the reference's left-to-right evaluation order, and
 * coefficients enter as factors that are exact when equal to 1.
 */
#ifndef PHFEM_ORACLE_PROBLEMS_H
#define PHFEM_ORACLE_PROBLEMS_H

#include <math.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum {
    OR_PROBLEM_MANUFACTURED = 0, /* u = x^2 y^2 z^2            (analysis.cpp:9-25)  */
    OR_PROBLEM_LINEAR = 1,       /* u = x + 2y + 3z + 4        (analysis.cpp:27-38) */
    OR_PROBLEM_ZERO = 2,         /* f = u_D = g = 0            (analysis.cpp:40-49) */
    OR_PROBLEM_SIN3 = 3,         /* u = sin(pi x) sin(pi y) sin(pi z)   configs 1, 4 */
    OR_PROBLEM_EXPCOS = 4,       /* u = exp(x) cos(pi y) z^2            config 3 */
    OR_PROBLEM_POLYSIN = 5       /* u = x (8 - x) sin(pi y) sin(pi z)   config 5 */
};

static inline double orp_u(int kind, double x, double y, double z) {
    switch (kind) {
        case OR_PROBLEM_MANUFACTURED: return x * x * y * y * z * z;
        case OR_PROBLEM_LINEAR: return x + 2.0 * y + 3.0 * z + 4.0;
        case OR_PROBLEM_SIN3: return sin(M_PI * x) * sin(M_PI * y) * sin(M_PI * z);
        case OR_PROBLEM_EXPCOS: return exp(x) * cos(M_PI * y) * (z * z);
        case OR_PROBLEM_POLYSIN: return x * (8.0 - x) * sin(M_PI * y) * sin(M_PI * z);
        default: return 0.0;
    }
}

/* exact gradient (not A-weighted) */
static inline void orp_grad(int kind, double x, double y, double z, double g[3]) {
    switch (kind) {
        case OR_PROBLEM_MANUFACTURED:
            g[0] = 2.0 * x * y * y * z * z;
            g[1] = 2.0 * x * x * y * z * z;
            g[2] = 2.0 * x * x * y * y * z;
            return;
        case OR_PROBLEM_LINEAR: g[0] = 1.0; g[1] = 2.0; g[2] = 3.0; return;
        case OR_PROBLEM_SIN3: {
            const double sx = sin(M_PI * x), sy = sin(M_PI * y), sz = sin(M_PI * z);
            const double cx = cos(M_PI * x), cy = cos(M_PI * y), cz = cos(M_PI * z);
            g[0] = M_PI * cx * sy * sz;
            g[1] = M_PI * sx * cy * sz;
            g[2] = M_PI * sx * sy * cz;
            return;
        }
        case OR_PROBLEM_EXPCOS: {
            const double ex = exp(x), cy = cos(M_PI * y), sy = sin(M_PI * y);
            g[0] = ex * cy * (z * z);
            g[1] = -M_PI * ex * sy * (z * z);
            g[2] = 2.0 * ex * cy * z;
            return;
        }
        case OR_PROBLEM_POLYSIN: {
            const double q = x * (8.0 - x);
            const double sy = sin(M_PI * y), sz = sin(M_PI * z);
            const double cy = cos(M_PI * y), cz = cos(M_PI * z);
            g[0] = (8.0 - 2.0 * x) * sy * sz;
            g[1] = M_PI * q * cy * sz;
            g[2] = M_PI * q * sy * cz;
            return;
        }
        default: g[0] = g[1] = g[2] = 0.0; return;
    }
}

/* f = -div(A grad u) + c u.  Kind 0 at A = I, c = 1 is the reference's
 * `-2.0 * (y^2 z^2 + x^2 z^2 + x^2 y^2) + u(x)` (analysis.cpp:16-18). */
static inline double orp_f(int kind, double x, double y, double z, const double A[3], double c) {
    switch (kind) {
        case OR_PROBLEM_MANUFACTURED: {
            const double u = x * x * y * y * z * z;
            return -2.0 * (A[0] * (y * y * z * z) + A[1] * (x * x * z * z) + A[2] * (x * x * y * y)) +
                   c * u;
        }
        case OR_PROBLEM_LINEAR: return c * (x + 2.0 * y + 3.0 * z + 4.0);
        case OR_PROBLEM_SIN3: {
            const double u = sin(M_PI * x) * sin(M_PI * y) * sin(M_PI * z);
            return ((M_PI * M_PI) * (A[0] + A[1] + A[2]) + c) * u;
        }
        case OR_PROBLEM_EXPCOS: {
            const double ex = exp(x), cy = cos(M_PI * y);
            const double u = ex * cy * (z * z);
            const double uxx = u, uyy = -(M_PI * M_PI) * u, uzz = 2.0 * ex * cy;
            return -(A[0] * uxx + A[1] * uyy + A[2] * uzz) + c * u;
        }
        case OR_PROBLEM_POLYSIN: {
            const double sy = sin(M_PI * y), sz = sin(M_PI * z);
            const double u = x * (8.0 - x) * sy * sz;
            const double uxx = -2.0 * sy * sz, uyy = -(M_PI * M_PI) * u;
            return -(A[0] * uxx + A[1] * uyy + A[2] * uyy) + c * u;
        }
        default: return 0.0;
    }
}

/* Neumann flux g = (A grad u) . n; kind 0/1 at A = I is dot(grad(x), n)
 * (analysis.cpp:21, 34). */
static inline double orp_g(int kind, double x, double y, double z, const double n[3],
                           const double A[3]) {
    double g[3];
    orp_grad(kind, x, y, z, g);
    return (A[0] * g[0]) * n[0] + (A[1] * g[1]) * n[1] + (A[2] * g[2]) * n[2];
}

#endif
