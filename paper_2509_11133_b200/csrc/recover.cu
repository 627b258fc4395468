// Element-local primal recovery, the residual checks of verify_solution and
// the error norms, on the device.
//   recover     U_T = A_T^-1 (B_T + C_T' Lambda)        (solver.cpp:168-181)
//               + || A U - rhs - C' Lambda ||^2 partials  (solver.cpp:44-53)
//   constraint  r2 = C U - b_D per multiplier row          (solver.cpp:54-62)
//   errors      broken Y-norm, multiplier h-norm           (analysis.cpp:51-105)
//               and the L2 error (the north-star accuracy check)
// A_T and its LU are recomputed from the coordinates (cheaper than storing
// 136 B per element); B_T comes from the assembly.
#include <cuda_runtime.h>

#include "problems.cuh"

namespace phg {
// tet_rule(9) for the error norms (this translation unit's copy)
__constant__ double c_lam9[216 * 4];
__constant__ double c_w9[216];
}  // namespace phg

extern "C" int phfem_gpu_set_rules_errors(const double* lam9, const double* w9) {
    cudaMemcpyToSymbol(phg::c_lam9, lam9, sizeof(double) * 4 * 216);
    cudaMemcpyToSymbol(phg::c_w9, w9, sizeof(double) * 216);
    return (int)cudaGetLastError();
}

namespace {

using namespace phg;

constexpr int kThreads = 128;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    return s;
}
__device__ __forceinline__ double block_max(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, sh[i]);
    return s;
}

struct SlotInfo {
    int32_t row[4];
    double coef[4];
};

__device__ __forceinline__ void slot_info(int64_t t, const int32_t* __restrict__ face_of_slot,
                                          const int32_t* __restrict__ slot_mate, const int32_t* __restrict__ face_mrow,
                                          const double* __restrict__ face_area, SlotInfo& si) {
    const int4 mate4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
    const int4 fos4 = __ldg(reinterpret_cast<const int4*>(face_of_slot) + t);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int32_t s = (int32_t)(4 * t + q);
        const int32_t mate = tv(mate4, q);
        const int32_t f = tv(fos4, q);
        si.row[q] = __ldg(face_mrow + f);
        const double sg = (mate < 0 || mate > s) ? 1.0 : -1.0;
        si.coef[q] = dvd(mul(sg, __ldg(face_area + f)), 3.0);
    }
}

template <int KIND>
__global__ void __launch_bounds__(kThreads)
    recover_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
              const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
              const int32_t* __restrict__ face_mrow, const double* __restrict__ face_area,
              const double* __restrict__ rhs, const double* __restrict__ lambda, double* __restrict__ u,
              double* __restrict__ partials, unsigned long long* err) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        const Coef k = load_coef(prob, t);
        Local L;
        local_matrices(p, k, L);
        Lu4 lu;
        lu_factor(L.a, lu);
        if (L.degenerate || lu.singular) {
            report(err, PHG_ERR_SINGULAR, (unsigned long long)t);
            continue;
        }
        SlotInfo si;
        slot_info(t, face_of_slot, slot_mate, face_mrow, face_area, si);
        double b[4], bb[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = bb[v] = rhs[4 * t + v];
        double lam[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) lam[r] = si.row[r] >= 0 ? lambda[si.row[r]] : 0.0;
        // rhs[v] += coef_r * Lambda[row_r] over r, kFaceVerts order
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (si.row[r] < 0) continue;
            const double cl = mul(si.coef[r], lam[r]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int v = face_vert(r, j);
                bb[v] = add(bb[v], cl);
            }
        }
        double x[4];
        lu_solve(lu, bb, x);
        reinterpret_cast<double2*>(u)[2 * t] = make_double2(x[0], x[1]);
        reinterpret_cast<double2*>(u)[2 * t + 1] = make_double2(x[2], x[3]);
        // r1 = A U - rhs - C' Lambda; C' Lambda accumulates rows ascending
        // (multiply_transpose, sparse.cpp:54-58)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) s = add(s, mul(L.a[i][j], x[j]));
            double r1 = sub(s, b[i]);
            // the (up to 3) faces containing local vertex i, in row order
            int32_t rr[3];
            double cc[3];
            int n = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int opp = q == 0 ? 3 : (q == 3 ? 0 : q);
                if (opp == i || si.row[q] < 0) continue;
                rr[n] = si.row[q];
                cc[n] = mul(si.coef[q], lam[q]);
                ++n;
            }
            for (int a = 1; a < n; ++a)
                for (int c = a; c > 0 && rr[c - 1] > rr[c]; --c) {
                    const int32_t tr = rr[c]; rr[c] = rr[c - 1]; rr[c - 1] = tr;
                    const double tc = cc[c]; cc[c] = cc[c - 1]; cc[c - 1] = tc;
                }
            double ctl = 0.0;
            for (int a = 0; a < n; ++a) ctl = add(ctl, cc[a]);
            r1 = sub(r1, ctl);
            acc += r1 * r1;
        }
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads)
    constraint_k(int64_t l, const int32_t* __restrict__ row_face, const int32_t* __restrict__ face_slots,
                 const double* __restrict__ face_area, const double* __restrict__ u, const double* __restrict__ bd,
                 double* __restrict__ partials) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0, rmax = 0.0, bmax = 0.0;
    for (int64_t R = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; R < l; R += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = row_face[R];
        const int2 fs = reinterpret_cast<const int2*>(face_slots)[f];
        const double area = face_area[f];
        double cu = 0.0;
        for (int side = 0; side < 2; ++side) {
            const int32_t s = side == 0 ? fs.x : fs.y;
            if (s < 0) break;
            const int64_t t = s >> 2;
            const int k = s & 3;
            const double coef = dvd(mul(side == 0 ? 1.0 : -1.0, area), 3.0);
            // columns ascending: the face's local vertices sorted
            int v0 = face_vert(k, 0), v1 = face_vert(k, 1), v2 = face_vert(k, 2);
            if (v0 > v1) { const int tmp = v0; v0 = v1; v1 = tmp; }
            if (v1 > v2) { const int tmp = v1; v1 = v2; v2 = tmp; }
            if (v0 > v1) { const int tmp = v0; v0 = v1; v1 = tmp; }
            cu = add(cu, mul(coef, u[4 * t + v0]));
            cu = add(cu, mul(coef, u[4 * t + v1]));
            cu = add(cu, mul(coef, u[4 * t + v2]));
        }
        const double b = bd[R];
        const double r2 = sub(cu, b);
        acc += r2 * r2;
        rmax = fmax(rmax, fabs(r2));
        bmax = fmax(bmax, fabs(b));
    }
    const double s = block_sum(acc, sh);
    const double m1 = block_max(rmax, sh);
    const double m2 = block_max(bmax, sh);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = s;
        partials[3 * blockIdx.x + 1] = m1;
        partials[3 * blockIdx.x + 2] = m2;
    }
}

template <int KIND>
__global__ void __launch_bounds__(kThreads)
    errors_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
             const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
             const int32_t* __restrict__ face_mrow, const double* __restrict__ u, const double* __restrict__ lambda,
             double h, double* __restrict__ partials) {
    __shared__ double sh[kThreads / 32];
    const double inv_h2 = dvd(1.0, mul(h, h));
    double acc_y = 0.0, acc_k = 0.0, acc_l2 = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        const Coef k = load_coef(prob, t);
        Local L;
        local_matrices(p, k, L);
        double ut[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) ut[v] = u[4 * t + v];
        V3 guh = {0.0, 0.0, 0.0};
#pragma unroll
        for (int v = 0; v < 4; ++v) guh = vadd(guh, vmul(L.g[v], ut[v]));
        double ey = 0.0, el = 0.0;
        for (int q = 0; q < 216; ++q) {
            const double l0 = c_lam9[4 * q], l1 = c_lam9[4 * q + 1], l2 = c_lam9[4 * q + 2], l3 = c_lam9[4 * q + 3];
            const V3 x = vadd(vadd(vadd(vmul(p[0], l0), vmul(p[1], l1)), vmul(p[2], l2)), vmul(p[3], l3));
            double uh = 0.0;
            uh = add(uh, mul(l0, ut[0]));
            uh = add(uh, mul(l1, ut[1]));
            uh = add(uh, mul(l2, ut[2]));
            uh = add(uh, mul(l3, ut[3]));
            const V3 g = prob_grad<KIND>(x.x, x.y, x.z);
            const V3 dg = vsub(g, guh);
            const double dv = sub(prob_u<KIND>(x.x, x.y, x.z), uh);
            const double vw = mul(L.vol, c_w9[q]);
            ey += mul(vw, add(vdot(dg, dg), mul(mul(inv_h2, dv), dv)));
            el += mul(vw, mul(dv, dv));
        }
        acc_y += ey;
        acc_l2 += el;
        // multiplier h-norm over non-Neumann slots, edge-midpoint rule
        const int4 mate4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        const int4 fos4 = __ldg(reinterpret_cast<const int4*>(face_of_slot) + t);
        for (int kk = 0; kk < 4; ++kk) {
            const int32_t row = face_mrow[tv(fos4, kk)];
            if (row < 0) continue;
            const int32_t s = (int32_t)(4 * t + kk);
            const int32_t mate = tv(mate4, kk);
            const double sg = (mate < 0 || mate > s) ? 1.0 : -1.0;
            const V3 q0 = p[face_vert(kk, 0)], q1 = p[face_vert(kk, 1)], q2 = p[face_vert(kk, 2)];
            const V3 n = vcross(vsub(q2, q0), vsub(q1, q0));
            const double len = __dsqrt_rn(vdot(n, n));
            const double ar = mul(0.5, len);
            const V3 un = vdiv(n, len);
            const double kh = mul(sg, lambda[row]);
            const double w3 = dvd(1.0, 3.0);
            for (int qq = 0; qq < 3; ++qq) {
                const double a0 = qq == 1 ? 0.0 : 0.5, a1 = qq == 2 ? 0.0 : 0.5, a2 = qq == 0 ? 0.0 : 0.5;
                const V3 x = vadd(vadd(vmul(q0, a0), vmul(q1, a1)), vmul(q2, a2));
                const double diff = sub(prob_g<KIND>(x.x, x.y, x.z, un, k), kh);
                acc_k += mul(mul(mul(mul(h, ar), w3), diff), diff);
            }
        }
    }
    const double s0 = block_sum(acc_y, sh);
    const double s1 = block_sum(acc_k, sh);
    const double s2 = block_sum(acc_l2, sh);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = s0;
        partials[3 * blockIdx.x + 1] = s1;
        partials[3 * blockIdx.x + 2] = s2;
    }
}

// deterministic final reduction of NV-wide partials; mode bit i: max
__global__ void reduce_partials(const double* __restrict__ partials, int n, int nv, unsigned max_mask,
                                double* __restrict__ out) {
    __shared__ double sh[32];
    for (int i = 0; i < nv; ++i) {
        const bool is_max = (max_mask >> i) & 1u;
        double a = 0.0;
        for (int b = threadIdx.x; b < n; b += blockDim.x) {
            const double v = partials[nv * b + i];
            a = is_max ? fmax(a, v) : a + v;
        }
        const double s = is_max ? block_max(a, sh) : block_sum(a, sh);
        if (threadIdx.x == 0) out[i] = s;
        __syncthreads();
    }
}

__global__ void sell_row_nnz(int64_t l, const int32_t* __restrict__ col, int32_t* __restrict__ nnz) {
    for (int64_t R = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; R < l; R += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = (R >> 5) * (PHG_SELL_C * PHG_SELL_W) + (R & 31);
        int n = 1;
        for (int k = 1; k < PHG_SELL_W; ++k) n += col[base + k * PHG_SELL_C] != (int32_t)R;
        nnz[R] = n;
    }
}

__global__ void sell_to_csr(int64_t l, const int32_t* __restrict__ scol, const double* __restrict__ sval,
                            const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col, double* __restrict__ val) {
    for (int64_t R = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; R < l; R += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = (R >> 5) * (PHG_SELL_C * PHG_SELL_W) + (R & 31);
        int32_t c[PHG_SELL_W];
        double v[PHG_SELL_W];
        int n = 0;
        for (int k = 0; k < PHG_SELL_W; ++k) {
            const int32_t cc = scol[base + k * PHG_SELL_C];
            if (k > 0 && cc == (int32_t)R) continue;
            c[n] = cc;
            v[n] = sval[base + k * PHG_SELL_C];
            ++n;
        }
        for (int a = 1; a < n; ++a)
            for (int b = a; b > 0 && c[b - 1] > c[b]; --b) {
                const int32_t tc = c[b]; c[b] = c[b - 1]; c[b - 1] = tc;
                const double tv2 = v[b]; v[b] = v[b - 1]; v[b - 1] = tv2;
            }
        const int64_t o = row_ptr[R];
        for (int a = 0; a < n; ++a) {
            col[o + a] = c[a];
            val[o + a] = v[a];
        }
    }
}

inline int rgrid(int64_t n) {
    const int g = grid_for(n, kThreads);
    return g < kSMs * 16 ? g : kSMs * 16;
}

}  // namespace

extern "C" int phfem_gpu_recover(int64_t ne, const double* coords, const int32_t* tets, const phg_problem* prob,
                                 const int32_t* face_of_slot, const int32_t* slot_mate, const int32_t* face_mrow,
                                 const double* face_area, const double* rhs, const double* lambda, double* u,
                                 double* sums, double* partials, unsigned long long* err, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g = rgrid(ne);
    const phg_problem p = *prob;
#define PHG_REC(K) \
    recover_k<K><<<g, kThreads, 0, s>>>(ne, coords, tets, p, face_of_slot, slot_mate, face_mrow, face_area, rhs, \
                                        lambda, u, partials, err)
    switch (p.kind) {
        case 0: PHG_REC(0); break;
        case 1: PHG_REC(1); break;
        case 2: PHG_REC(2); break;
        case 3: PHG_REC(3); break;
        case 4: PHG_REC(4); break;
        case 5: PHG_REC(5); break;
        default: return (int)cudaErrorInvalidValue;
    }
#undef PHG_REC
    reduce_partials<<<1, 256, 0, s>>>(partials, g, 1, 0u, sums);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_constraint_residual(int64_t l, const int32_t* row_face, const int32_t* face_slots,
                                             const int32_t* slot_mate, const int32_t* face_of_slot,
                                             const double* face_area, const int32_t* tets, const double* u,
                                             const double* bd, double* out, double* partials, void* stream) {
    (void)slot_mate;
    (void)face_of_slot;
    (void)tets;
    cudaStream_t s = (cudaStream_t)stream;
    const int g = rgrid(l);
    constraint_k<<<g, kThreads, 0, s>>>(l, row_face, face_slots, face_area, u, bd, partials);
    reduce_partials<<<1, 256, 0, s>>>(partials, g, 3, 0x6u, out);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_errors(int64_t ne, const double* coords, const int32_t* tets, const phg_problem* prob,
                                const int32_t* face_of_slot, const int32_t* slot_mate, const int32_t* face_mrow,
                                const double* u, const double* lambda, double h, double* out, double* partials,
                                void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g = rgrid(ne);
    const phg_problem p = *prob;
#define PHG_ERRK(K) \
    errors_k<K><<<g, kThreads, 0, s>>>(ne, coords, tets, p, face_of_slot, slot_mate, face_mrow, u, lambda, h, partials)
    switch (p.kind) {
        case 0: PHG_ERRK(0); break;
        case 1: PHG_ERRK(1); break;
        case 2: PHG_ERRK(2); break;
        case 3: PHG_ERRK(3); break;
        case 4: PHG_ERRK(4); break;
        case 5: PHG_ERRK(5); break;
        default: return (int)cudaErrorInvalidValue;
    }
#undef PHG_ERRK
    reduce_partials<<<1, 256, 0, s>>>(partials, g, 3, 0u, out);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_sell_row_nnz(int64_t l, const int32_t* sell_col, int32_t* row_nnz, void* stream) {
    sell_row_nnz<<<rgrid(l), kThreads, 0, (cudaStream_t)stream>>>(l, sell_col, row_nnz);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_sell_to_csr(int64_t l, const int32_t* sell_col, const double* sell_val,
                                     const int64_t* row_ptr, int32_t* col, double* val, void* stream) {
    sell_to_csr<<<rgrid(l), kThreads, 0, (cudaStream_t)stream>>>(l, sell_col, sell_val, row_ptr, col, val);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}
