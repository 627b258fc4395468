// Assembly + element-local Schur condensation on the device
// (assemble_system, assembly.cpp:7-138, and the local part of build_schur,
// solver.cpp:90-127), scattering straight into the SELL-32 Schur matrix.
//
// Two element-parallel kernels, split by register footprint:
//   load     B_T = Gauss-64 load vector + Neumann terms (assembly.cpp:46-94),
//            the fp64-heavy part, at high occupancy (few live registers);
//   condense A_T = K_T(A) + c M_T, C_T rows sigma*|F|/3, Dirichlet data,
//            partial-pivot LU of A_T, S_T = C A^-1 C', r_T = C A^-1 B, and the
//            scatter of S_T and b_D - r_T into the face system.
// Everything the reference computes in these loops is replayed in its
// operation order without FMA, so A_T, C_T and S_T are bit-identical; the
// transcendental load data differ only by libm-vs-libdevice ulps.
//
// Scatter (each S entry has one contribution except interior diagonals,
// which have two; a two-term sum is order free, so atomics stay exact):
//   row R of face f, owner slot -> positions 0 (diag, atomic), 1-3
//   second slot               -> positions 0 (diag, atomic), 4-6
//   rhs_neg[R] = b_D - r_T (Dirichlet) or -(r_T1 + r_T2) via two atomics.
#include <cuda_runtime.h>

#include "problems.cuh"

namespace phg {
__constant__ double c_lam5[64 * 4];
__constant__ double c_w5[64];
}  // namespace phg

extern "C" int phfem_gpu_set_rules_errors(const double* lam9, const double* w9);

namespace {

using namespace phg;

constexpr int kLoadThreads = 128;
constexpr int kCondThreads = 128;

__device__ __forceinline__ int64_t sell_idx(int64_t row, int pos) {
    return (row >> 5) * (PHG_SELL_C * PHG_SELL_W) + pos * PHG_SELL_C + (row & 31);
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = add(s, sh[i]);
    return s;
}

struct Slots {
    int32_t row[4];
    int32_t face[4];
    bool owner[4], bnd[4];
};

__device__ __forceinline__ void load_slots(int64_t t, const int32_t* __restrict__ face_of_slot,
                                           const int32_t* __restrict__ slot_mate,
                                           const int32_t* __restrict__ face_mrow, Slots& s) {
    const int4 mate4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
    const int4 fos4 = __ldg(reinterpret_cast<const int4*>(face_of_slot) + t);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int32_t sl = (int32_t)(4 * t + q);
        const int32_t mate = tv(mate4, q);
        s.face[q] = tv(fos4, q);
        s.row[q] = __ldg(face_mrow + s.face[q]);
        s.owner[q] = mate < 0 || mate > sl;
        s.bnd[q] = mate < 0;
    }
}

// B_T: Gauss-64 load vector (assembly.cpp:64-78) + Neumann terms
// (assembly.cpp:81-94, face order == local slot order for one element),
// rhs = b + LN (assembly.cpp:135).
template <int KIND>
__global__ void __launch_bounds__(kLoadThreads)
    load_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
           const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
           const int32_t* __restrict__ face_mrow, double* __restrict__ rhs_out, double* __restrict__ partials,
           unsigned long long* err) {
    (void)face_of_slot;
    (void)slot_mate;
    (void)face_mrow;
    (void)partials;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        const Coef k = load_coef(prob, t);
        // elem_volume == local.volume (assembly.cpp:18, 47)
        const V3 d1 = vsub(p[1], p[0]), d2 = vsub(p[2], p[0]), d3 = vsub(p[3], p[0]);
        const double det = vdot(vcross(d1, d2), d3);
        if (det == 0.0) {
            report(err, PHG_ERR_ZERO_VOLUME, (unsigned long long)t);
            continue;
        }
        const double vol = dq(fabs(det), kDiv6);
        double b[4] = {0.0, 0.0, 0.0, 0.0};
        if constexpr (KIND <= 2) {
            // polynomial data: the reference's exact operation order
#pragma unroll 2
            for (int qp = 0; qp < 64; ++qp) {
                const double l0 = c_lam5[4 * qp], l1 = c_lam5[4 * qp + 1], l2 = c_lam5[4 * qp + 2],
                             l3 = c_lam5[4 * qp + 3];
                const V3 x = vadd(vadd(vadd(vmul(p[0], l0), vmul(p[1], l1)), vmul(p[2], l2)), vmul(p[3], l3));
                const double fw = mul(mul(vol, c_w5[qp]), prob_f<KIND>(x.x, x.y, x.z, k));
                b[0] = add(b[0], mul(fw, l0));
                b[1] = add(b[1], mul(fw, l1));
                b[2] = add(b[2], mul(fw, l2));
                b[3] = add(b[3], mul(fw, l3));
            }
        } else {
            const double cpre = prob_f_pre<KIND>(k);
            // trig factors by angle addition from vertex 0 when the element
            // is small enough (problems.cuh: axis_sincos), else sinpi/cospi
            const AxisTrig ax = axis_trig(p[0].x, p[1].x, p[2].x, p[3].x);
            const AxisTrig ay = axis_trig(p[0].y, p[1].y, p[2].y, p[3].y);
            const AxisTrig az = axis_trig(p[0].z, p[1].z, p[2].z, p[3].z);
            const double zmax = fmax(axis_zmax(ax), fmax(axis_zmax(ay), axis_zmax(az)));
            if (zmax <= 0.25) {
                const double e0 = KIND == 4 ? exp(p[0].x) : 0.0;
#pragma unroll 2
                for (int qp = 0; qp < 64; ++qp) {
                    const double l0 = c_lam5[4 * qp], l1 = c_lam5[4 * qp + 1], l2 = c_lam5[4 * qp + 2],
                                 l3 = c_lam5[4 * qp + 3];
                    double f;
                    if constexpr (KIND == 3) {
                        double sx, cx, sy, cy, sz, cz;
                        axis_sincos(ax, l1, l2, l3, sx, cx);
                        axis_sincos(ay, l1, l2, l3, sy, cy);
                        axis_sincos(az, l1, l2, l3, sz, cz);
                        f = cpre * (sx * sy * sz);
                    } else if constexpr (KIND == 4) {
                        const double dx = fma(l3, ax.d3, fma(l2, ax.d2, l1 * ax.d1));
                        const double z = fma(p[3].z, l3, fma(p[2].z, l2, fma(p[1].z, l1, p[0].z * l0)));
                        double sy, cy;
                        axis_sincos(ay, l1, l2, l3, sy, cy);
                        const double ec = (e0 * exp_small(dx)) * cy;
                        f = fma(cpre, ec * (z * z), -(k.a2 * 2.0) * ec);
                    } else {
                        const double x = fma(p[3].x, l3, fma(p[2].x, l2, fma(p[1].x, l1, p[0].x * l0)));
                        double sy, cy, sz, cz;
                        axis_sincos(ay, l1, l2, l3, sy, cy);
                        axis_sincos(az, l1, l2, l3, sz, cz);
                        const double s = sy * sz;
                        f = fma(cpre, x * (8.0 - x) * s, 2.0 * k.a0 * s);
                    }
                    const double fw = (vol * c_w5[qp]) * f;
                    b[0] = fma(fw, l0, b[0]);
                    b[1] = fma(fw, l1, b[1]);
                    b[2] = fma(fw, l2, b[2]);
                    b[3] = fma(fw, l3, b[3]);
                }
            } else {
#pragma unroll 2
            for (int qp = 0; qp < 64; ++qp) {
                const double l0 = c_lam5[4 * qp], l1 = c_lam5[4 * qp + 1], l2 = c_lam5[4 * qp + 2],
                             l3 = c_lam5[4 * qp + 3];
                const double x = fma(p[3].x, l3, fma(p[2].x, l2, fma(p[1].x, l1, p[0].x * l0)));
                const double y = fma(p[3].y, l3, fma(p[2].y, l2, fma(p[1].y, l1, p[0].y * l0)));
                const double z = fma(p[3].z, l3, fma(p[2].z, l2, fma(p[1].z, l1, p[0].z * l0)));
                const double fw = (vol * c_w5[qp]) * prob_f_fast<KIND>(x, y, z, cpre, k);
                b[0] = fma(fw, l0, b[0]);
                b[1] = fma(fw, l1, b[1]);
                b[2] = fma(fw, l2, b[2]);
                b[3] = fma(fw, l3, b[3]);
            }
            }
        }
        // b only; condense_k adds the Neumann terms (rhs = b + LN)
        reinterpret_cast<double2*>(rhs_out)[2 * t] = make_double2(b[0], b[1]);
        reinterpret_cast<double2*>(rhs_out)[2 * t + 1] = make_double2(b[2], b[3]);
    }
}

template <int KIND>
__global__ void __launch_bounds__(kCondThreads, 4)
    condense_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
               const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
               const int32_t* __restrict__ face_mrow, const double* __restrict__ face_area,
               double* __restrict__ rhs_in, int32_t* __restrict__ sell_col, double* __restrict__ sell_val,
               double* __restrict__ rhs_neg, double* __restrict__ bd, double* __restrict__ a_blocks,
               double* __restrict__ slot_coef, int32_t* __restrict__ slot_mrow, double* __restrict__ partials,
               unsigned long long* err) {
    __shared__ double sh[kCondThreads / 32];
    double acc_bd = 0.0, acc_rhs = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        const Coef k = load_coef(prob, t);
        Slots sl;
        load_slots(t, face_of_slot, slot_mate, face_mrow, sl);
        // boundary data first, while only the coordinates are live:
        // Neumann terms (assembly.cpp:81-94; this element's Neumann faces in
        // face order == local slot order) and Dirichlet traces b_D = |F|
        // u_D(centroid) (assembly.cpp:96-104; stored tuple = owner slot)
        double ln[4] = {0.0, 0.0, 0.0, 0.0};
        double bdv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!sl.bnd[q]) continue;
            const int i0 = face_vert(q, 0), i1 = face_vert(q, 1), i2 = face_vert(q, 2);
            const V3 q0 = p[i0], q1 = p[i1], q2 = p[i2];
            const V3 cen = vdivq(vadd(vadd(q0, q1), q2), kDiv3);
            if (sl.row[q] >= 0) {
                bdv[q] = mul(__ldg(face_area + sl.face[q]), prob_u<KIND>(cen.x, cen.y, cen.z));
                continue;
            }
            const V3 n = vcross(vsub(q2, q0), vsub(q1, q0));
            const double len = __dsqrt_rn(vdot(n, n));
            const double ar = mul(0.5, len);
            const V3 un = vdivq(n, make_div(len));
            const double gc = prob_g<KIND>(cen.x, cen.y, cen.z, un, k);
            const double contrib = dq(mul(ar, gc), kDiv3);
            ln[i0] = add(ln[i0], contrib);
            ln[i1] = add(ln[i1], contrib);
            ln[i2] = add(ln[i2], contrib);
        }
        Local L;
        local_matrices(p, k, L);  // local_stiffness_mass (assembly.cpp:7-33)
        if (L.degenerate) continue;  // reported by load_k
        double coef[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // slot_coef = sigma*|F|/3 (assembly.cpp:125)
            const double sg = sl.owner[q] ? 1.0 : -1.0;
            coef[q] = dq(mul(sg, __ldg(face_area + sl.face[q])), kDiv3);
        }
        if (a_blocks) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) a_blocks[16 * t + 4 * i + j] = L.a[i][j];
        }
        if (slot_coef) {
#pragma unroll
            for (int q = 0; q < 4; ++q) slot_coef[4 * t + q] = coef[q];
        }
        if (slot_mrow) {
#pragma unroll
            for (int q = 0; q < 4; ++q) slot_mrow[4 * t + q] = sl.row[q];
        }
        const double2 r01 = reinterpret_cast<const double2*>(rhs_in)[2 * t];
        const double2 r23 = reinterpret_cast<const double2*>(rhs_in)[2 * t + 1];
        const double rhs[4] = {add(r01.x, ln[0]), add(r01.y, ln[1]), add(r23.x, ln[2]), add(r23.y, ln[3])};
        reinterpret_cast<double2*>(const_cast<double*>(rhs_in))[2 * t] = make_double2(rhs[0], rhs[1]);
        reinterpret_cast<double2*>(const_cast<double*>(rhs_in))[2 * t + 1] = make_double2(rhs[2], rhs[3]);
        acc_rhs = add(acc_rhs, add(add(add(mul(rhs[0], rhs[0]), mul(rhs[1], rhs[1])), mul(rhs[2], rhs[2])),
                                   mul(rhs[3], rhs[3])));

        // local Schur complement (solver.cpp:101-127)
        Lu4 lu;
        lu_factor(L.a, lu);
        if (lu.singular) {
            report(err, PHG_ERR_SINGULAR, (unsigned long long)t);
            continue;
        }
        // local C rows c[r][v] = coef_r on the face's vertices, 0 on the
        // opposite one and on Neumann faces (local_c_rows, solver.cpp:33-40)
        auto cr = [&](int r, int v) -> double {
            const bool on = sl.row[r] >= 0 && v != (r == 0 ? 3 : (r == 3 ? 0 : r));
            return on ? coef[r] : 0.0;
        };
        // one solved column x = A^-1 c_q at a time: S_T[r][q] for all r,
        // accumulated over p = 0..3 exactly as solver.cpp:121-125
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (sl.row[q] < 0) {
                // Neumann column: padding in the rows of the other faces
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r == q || sl.row[r] < 0) continue;
                    const int64_t R = sl.row[r];
                    const int64_t ix = sell_idx(R, (sl.owner[r] ? 0 : 3) + 1 + (q < r ? q : q - 1));
                    sell_col[ix] = (int32_t)R;
                    sell_val[ix] = 0.0;
                }
                continue;
            }
            const double cq[4] = {cr(q, 0), cr(q, 1), cr(q, 2), cr(q, 3)};
            double x[4];
            lu_solve(lu, cq, x);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (sl.row[r] < 0) continue;
                double s = 0.0;
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) s = add(s, mul(cr(r, pp), x[pp]));
                const int64_t R = sl.row[r];
                if (q == r) {
                    atomicAdd(sell_val + sell_idx(R, 0), s);
                    sell_col[sell_idx(R, 0)] = (int32_t)R;
                } else {
                    const int64_t ix = sell_idx(R, (sl.owner[r] ? 0 : 3) + 1 + (q < r ? q : q - 1));
                    sell_col[ix] = sl.row[q];
                    sell_val[ix] = s;
                }
            }
        }
        double ainv_b[4];
        lu_solve(lu, rhs, ainv_b);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (sl.row[r] < 0) continue;
            double rb = 0.0;
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) rb = add(rb, mul(cr(r, pp), ainv_b[pp]));
            const int64_t R = sl.row[r];
            if (sl.bnd[r]) {
#pragma unroll
                for (int pos = 4; pos < 7; ++pos) {
                    sell_col[sell_idx(R, pos)] = (int32_t)R;
                    sell_val[sell_idx(R, pos)] = 0.0;
                }
                // rhs_neg = b_D - r_T (solver.cpp:131-138), single contributor
                rhs_neg[R] = sub(bdv[r], rb);
                bd[R] = bdv[r];
                acc_bd = add(acc_bd, mul(bdv[r], bdv[r]));
            } else {
                atomicAdd(rhs_neg + R, -rb);
            }
        }
    }
    const double s0 = block_sum(acc_rhs, sh);
    const double s1 = block_sum(acc_bd, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = s0;
        partials[2 * blockIdx.x + 1] = s1;
    }
}

__global__ void __launch_bounds__(1024) reduce_pairs(const double* __restrict__ partials, int n,
                                                     double* __restrict__ out) {
    __shared__ double sh[32];
    // fixed-shape tree: 4 independent strided chains per thread, then the
    // block tree; deterministic for a given n
    double a4[4] = {0.0, 0.0, 0.0, 0.0}, b4[4] = {0.0, 0.0, 0.0, 0.0};
    const double2* pp = reinterpret_cast<const double2*>(partials);
    int i = threadIdx.x;
    for (; i + 3 * (int)blockDim.x < n; i += 4 * blockDim.x) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2 v = pp[i + u * blockDim.x];
            a4[u] = add(a4[u], v.x);
            b4[u] = add(b4[u], v.y);
        }
    }
    for (; i < n; i += blockDim.x) {
        const double2 v = pp[i];
        a4[0] = add(a4[0], v.x);
        b4[0] = add(b4[0], v.y);
    }
    double a = add(add(a4[0], a4[1]), add(a4[2], a4[3]));
    double b = add(add(b4[0], b4[1]), add(b4[2], b4[3]));
    a = block_sum(a, sh);
    b = block_sum(b, sh);
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
    }
}

}  // namespace

extern "C" int phfem_gpu_set_rules(const double* lam5, const double* w5, int n5, const double* lam9, const double* w9,
                                   int n9) {
    if (n5 != 64 || n9 != 216) return (int)cudaErrorInvalidValue;
    cudaMemcpyToSymbol(phg::c_lam5, lam5, sizeof(double) * 4 * 64);
    cudaMemcpyToSymbol(phg::c_w5, w5, sizeof(double) * 64);
    const int rc = (int)cudaGetLastError();
    return rc ? rc : phfem_gpu_set_rules_errors(lam9, w9);
}

// One element per thread, blocks in element order: the elements in flight
// (and so the S rows they scatter into) stay within an L2-resident window;
// a grid-stride loop spread them over ~600k elements and turned the
// scattered SELL writes into DRAM read-modify-writes (ncu, profiles/).
extern "C" int phfem_gpu_assemble_grid(int64_t ne) {
    return grid_for(ne, kLoadThreads);
}

extern "C" int phfem_gpu_assemble_condense(int64_t ne, const double* coords, const int32_t* tets,
                                           const phg_problem* prob, const int32_t* face_of_slot,
                                           const int32_t* slot_mate, const int32_t* face_mrow,
                                           const double* face_area, int32_t* sell_col, double* sell_val,
                                           double* rhs_neg, double* bd, double* rhs, double* a_blocks,
                                           double* slot_coef, int32_t* slot_mrow, double* norms, double* partials,
                                           unsigned long long* err, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = phfem_gpu_assemble_grid(ne);
    const phg_problem p = *prob;
#define PHG_ASM(K)                                                                                                  \
    load_k<K><<<grid, kLoadThreads, 0, s>>>(ne, coords, tets, p, face_of_slot, slot_mate, face_mrow, rhs, partials,  \
                                            err);                                                                   \
    condense_k<K><<<grid, kCondThreads, 0, s>>>(ne, coords, tets, p, face_of_slot, slot_mate, face_mrow, face_area, \
                                                rhs, sell_col, sell_val, rhs_neg, bd, a_blocks, slot_coef,         \
                                                slot_mrow, partials, err)
    switch (p.kind) {
        case 0: PHG_ASM(0); break;
        case 1: PHG_ASM(1); break;
        case 2: PHG_ASM(2); break;
        case 3: PHG_ASM(3); break;
        case 4: PHG_ASM(4); break;
        case 5: PHG_ASM(5); break;
        default: return (int)cudaErrorInvalidValue;
    }
#undef PHG_ASM
    reduce_pairs<<<1, 1024, 0, s>>>(partials, grid, norms);
    phg::count_launches(3);
    return (int)cudaGetLastError();
}
