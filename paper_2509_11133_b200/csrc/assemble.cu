// Assembly + element-local Schur condensation on the device
// (assemble_system, assembly.cpp:7-138, and the local part of build_schur,
// solver.cpp:90-127), scattering straight into the SELL-32 Schur matrix.
//
// One fused element-parallel kernel per problem kind: the fp64-heavy
// Gauss-64 load vector (assembly.cpp:46-78) and the latency-bound gathers /
// scatter of the condensation overlap across the warps of an SM.  Per
// element: B_T = b + Neumann terms, A_T = K_T(A) + c M_T, C_T rows
// sigma*|F|/3, Dirichlet data, partial-pivot LU of A_T, S_T = C A^-1 C',
// r_T = C A^-1 B, streamed into the face system as they are formed.
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
// the same rule in its collapsed-product structure (quadrature.cpp:47-59):
// point 16a + 4b + c has lambda1 = c_l1[a], lambda2 = c_l2[4a + b],
// lambda3 = c_l3[16a + 4b + c]
__constant__ double c_l1[4];
__constant__ double c_l2[16];
__constant__ double c_l3[64];
__constant__ double c_l0[64];  // lambda0 of each point, as the rule stores it
}  // namespace phg

extern "C" int phfem_gpu_set_rules_errors(const double* lam9, const double* w9);

namespace {

using namespace phg;

constexpr int kCondThreads = 128;
#ifndef PHG_COND_MINB
#define PHG_COND_MINB 4  // resident blocks per SM the register budget is sized for
#endif

__device__ __forceinline__ int64_t sell_idx(int64_t row, int pos) {
    return (row >> 5) * (PHG_SELL_C * PHG_SELL_W) + pos * PHG_SELL_C + (row & 31);
}

// Where the condensed operator goes.  SELL (exports, the C++ API's S): the
// reference's S row by row, both triangles as build_schur computes them.
// Element-major (the solve path): per element the upper triangle of S_T,
// S_T[r][q] for r <= q as solver.cpp:121-125 computes it (10 values,
// 32-element AoSoA chunks), rows = slot_mrow, and the assembled diagonal
// (two-term sums, so the atomics are order-free); S = sum_T S_T exactly as
// from_triplets sums it, minus the lower triangle's last-bit differences.
struct SchurOut {
    int32_t* sell_col;
    double* sell_val;
    double* st_val;  // [10 x ne], element-major
    double* diag;    // [l], element-major
    // element-major with halves: the second element's diagonal and rhs_neg
    // terms of each interior row go to diag2 / rhs2 [l] with plain stores
    // (the owner's to diag / rhs_neg), summed when a solve needs S
    // (sum_halves_k): no clearing pass, no atomics.  NULL: atomics on
    // cleared rows.
    double* diag2;
    double* rhs2;
};

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

// cp.async (LDGSTS): a gather that lands in shared memory without holding a
// register or a scoreboard; waited for with cp_async_wait_all
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Per-thread staging (structure of arrays over the block's threads: a warp's
// accesses to one field are consecutive words) of what the condensation
// needs after the load vector: the coordinates, and the face-side gathers
// face_mrow / face_area / face_bval of the element's four faces, issued
// before the load vector so their latency hides under it.
struct Stage {
    double xyz[12][kCondThreads];
    double area[4][kCondThreads];
    double bval[4][kCondThreads];
    int32_t row[4][kCondThreads];
    int32_t face[4][kCondThreads];
    int32_t mate[4][kCondThreads];
};

// Gauss-64 load vector of the transcendental kinds with the trig / exp
// factors as order-N economised series around the element's centre
// (problems.cuh),
// walking the rule in its collapsed-product order (a, b, c):
//   z = lambda1 e1 + lambda2 e2 + lambda3 e3 + em = A(a, b) + lambda3 e3,
//       A(a, b) = fma(lambda2, e2, fma(lambda1, e1, em)) once per (a, b): the
//       same operations as the per-point fma chain, a third of the cost;
//   b1 = sum_a lambda1(a) T_a, b2 = sum_ab lambda2(a, b) U_ab with the
//       partial sums U_ab = sum_c w f, T_a = sum_b U_ab, b3 and b0 per point
//       (b0 accumulates w f lambda0 itself, as assembly.cpp:75 does: forming
//       it as S - b1 - b2 - b3 cancels where f changes sign in the element).
template <int N>
__device__ __forceinline__ double horner(const AxisTaylor<N>& t, double z) {
    double r = t.k[N];
#pragma unroll
    for (int n = N - 1; n >= 0; --n) r = fma(r, z, t.k[n]);
    return r;
}
template <int KIND, int N>
__device__ __forceinline__ void load_taylor(const V3 p[4], double cpre, const Coef& k, double vol, double b[4]) {
    const int GX = KIND == 3 ? kTaySin : kTayExp;
    const int GY = KIND == 4 ? kTayCos : kTaySin;
    const AxisTaylor<N> tx = axis_taylor<N, GX>(p[0].x, p[1].x, p[2].x, p[3].x);
    const AxisTaylor<N> ty = axis_taylor<N, GY>(p[0].y, p[1].y, p[2].y, p[3].y);
    const AxisTaylor<N> tz = axis_taylor<N, kTaySin>(p[0].z, p[1].z, p[2].z, p[3].z);
    (void)tz;
    (void)tx;
    // the coordinate entering f polynomially: z (kind 4) or x (kind 5)
    const double c0 = KIND == 4 ? p[0].z : p[0].x;
    const double d1 = (KIND == 4 ? p[1].z : p[1].x) - c0, d2 = (KIND == 4 ? p[2].z : p[2].x) - c0,
                 d3 = (KIND == 4 ? p[3].z : p[3].x) - c0;
    // two b3 / b0 accumulators and a pairwise U keep the per-(a, b)
    // dependency chains at depth 2 (the loop is short of independent work
    // otherwise)
    double b0 = 0.0, b0o = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0, b3o = 0.0;
    for (int a = 0; a < 4; ++a) {
        const double l1 = c_l1[a];
        double T = 0.0;
#pragma unroll 1
        for (int bb = 0; bb < 4; ++bb) {
            const double l2 = c_l2[4 * a + bb];
            const double ax = fma(l2, tx.e2, fma(l1, tx.e1, tx.em)), ay = fma(l2, ty.e2, fma(l1, ty.e1, ty.em)),
                         az = fma(l2, tz.e2, fma(l1, tz.e1, tz.em)), al = fma(l2, d2, fma(l1, d1, c0));
            double fw[4];
            // the 12 (kind 3) or 8 series of the four points in lockstep:
            // independent FMA chains side by side for the dependent-issue
            // latency
            double hx[4], hy[4], hz[4], zx[4], zy[4], zz[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double l3 = c_l3[16 * a + 4 * bb + c];
                zx[c] = fma(l3, tx.e3, ax);
                zy[c] = fma(l3, ty.e3, ay);
                zz[c] = fma(l3, tz.e3, az);
                hx[c] = tx.k[N];
                hy[c] = ty.k[N];
                hz[c] = tz.k[N];
            }
#pragma unroll
            for (int n = N - 1; n >= 0; --n) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (KIND != 5) hx[c] = fma(hx[c], zx[c], tx.k[n]);
                    hy[c] = fma(hy[c], zy[c], ty.k[n]);
                    if (KIND != 4) hz[c] = fma(hz[c], zz[c], tz.k[n]);
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int qp = 16 * a + 4 * bb + c;
                const double l3 = c_l3[qp];
                double f;
                if constexpr (KIND == 3) {
                    f = hx[c] * hy[c] * hz[c];
                } else if constexpr (KIND == 4) {
                    const double zc = fma(l3, d3, al);
                    const double ec = hx[c] * hy[c];
                    f = fma(cpre, ec * (zc * zc), -(k.a2 * 2.0) * ec);
                } else {
                    const double xc = fma(l3, d3, al);
                    const double sv = hy[c] * hz[c];
                    f = fma(cpre, xc * (8.0 - xc) * sv, 2.0 * k.a0 * sv);
                }
                fw[c] = c_w5[qp] * f;
            }
            const int q0 = 16 * a + 4 * bb;
            b3 = fma(fw[2], c_l3[q0 + 2], fma(fw[0], c_l3[q0], b3));
            b3o = fma(fw[3], c_l3[q0 + 3], fma(fw[1], c_l3[q0 + 1], b3o));
            b0 = fma(fw[2], c_l0[q0 + 2], fma(fw[0], c_l0[q0], b0));
            b0o = fma(fw[3], c_l0[q0 + 3], fma(fw[1], c_l0[q0 + 1], b0o));
            const double U = (fw[0] + fw[1]) + (fw[2] + fw[3]);
            T += U;
            b2 = fma(U, l2, b2);
        }
        b1 = fma(T, l1, b1);
    }
    b3 += b3o;
    b0 += b0o;
    const double sc = KIND == 3 ? vol * cpre : vol;
    b[0] = b0 * sc;
    b[1] = b1 * sc;
    b[2] = b2 * sc;
    b[3] = b3 * sc;
}

// Gauss-64 load vector b_T (assembly.cpp:64-78) of one element with
// volume vol.
template <int KIND>
__device__ __forceinline__ void load_vector(const V3 p[4], const Coef& k, double vol, double b[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 0.0;
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
        // series around the centre of the element's span when the element
        // is small enough (problems.cuh: axis_taylor), else sinpi/cospi/exp
        const double r = fmax(axis_r(p[0].x, p[1].x, p[2].x, p[3].x),
                              fmax(axis_r(p[0].y, p[1].y, p[2].y, p[3].y), axis_r(p[0].z, p[1].z, p[2].z, p[3].z)));
        switch (taylor_order(r)) {
            case 5: load_taylor<KIND, 5>(p, cpre, k, vol, b); break;
            case 6: load_taylor<KIND, 6>(p, cpre, k, vol, b); break;
            case 7: load_taylor<KIND, 7>(p, cpre, k, vol, b); break;
            case 9: load_taylor<KIND, 9>(p, cpre, k, vol, b); break;
            default:
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
}

// face-side inputs of one element
struct FaceIn {
    const int32_t* __restrict__ face_of_slot;
    const int32_t* __restrict__ slot_mate;
    const int32_t* __restrict__ face_mrow;
    const double* __restrict__ face_area;
    const double* __restrict__ face_bval;  // boundary_terms_k, boundary faces only
};

// One element's assembly and condensation, streamed straight into the face
// system (assembly.cpp:7-138, solver.cpp:101-145).  Every output except the
// two-contributor sums (S diagonal and rhs_neg of interior rows) has a
// single writer and is a plain store made as soon as it is known; those
// atomics are issued only at the end, once dv.good() is known.  An element
// whose FastDiv operands left the exact window returns 1 without any atomic:
// its plain stores are garbage that the ExactDiv redo pass overwrites.
// Returns 0 done, 1 redo, 2 singular block, 3 zero volume.
//
// Row R of face r: owner slot -> positions 0 (atomic diagonal) and 1-3,
// second slot -> 0 and 4-6; padding col = R, val = 0.
template <int KIND, bool ELEM, class Dv>
__device__ __forceinline__ int assemble_elem(int64_t t, const double* __restrict__ coords,
                                             const int32_t* __restrict__ tets, const phg_problem& prob,
                                             const FaceIn& fin, double* __restrict__ a_blocks, const SchurOut& so,
                                             double* __restrict__ rhs_neg, double* __restrict__ bd,
                                             double* __restrict__ rhs, double* __restrict__ slot_coef,
                                             int32_t* __restrict__ slot_mrow, Dv& dv) {
    // elem_volume == local.volume (assembly.cpp:18, 47)
    double bt[4];
    __shared__ Stage stg;
    const int tid = threadIdx.x;
    {
        const int4 e = ldtet(tets, t);
        const int4 mate4 = __ldg(reinterpret_cast<const int4*>(fin.slot_mate) + t);
        const int4 fos4 = __ldg(reinterpret_cast<const int4*>(fin.face_of_slot) + t);
        const V3 p0[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int32_t f = tv(fos4, q), mate = tv(mate4, q);
            cp_async4(&stg.row[q][tid], fin.face_mrow + f);
            cp_async8(&stg.area[q][tid], fin.face_area + f);
            if (mate < 0) cp_async8(&stg.bval[q][tid], fin.face_bval + f);
            stg.face[q][tid] = f;
            stg.mate[q][tid] = mate;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            stg.xyz[3 * i][tid] = p0[i].x;
            stg.xyz[3 * i + 1][tid] = p0[i].y;
            stg.xyz[3 * i + 2][tid] = p0[i].z;
        }
        const double det = vdot(vcross(vsub(p0[1], p0[0]), vsub(p0[2], p0[0])), vsub(p0[3], p0[0]));
        if (det == 0.0) {
            cp_async_wait_all();
            return 3;
        }
        load_vector<KIND>(p0, load_coef(prob, t), dq(fabs(det), kDiv6), bt);
    }
    cp_async_wait_all();
    V3 p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = {stg.xyz[3 * i][tid], stg.xyz[3 * i + 1][tid], stg.xyz[3 * i + 2][tid]};
    const Coef k = load_coef_fresh(prob, t);
    Slots sl;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int32_t mate = stg.mate[q][tid];
        sl.face[q] = stg.face[q][tid];
        sl.row[q] = stg.row[q][tid];
        sl.owner[q] = mate < 0 || mate > (int32_t)(4 * t + q);
        sl.bnd[q] = mate < 0;
    }
    double area[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) area[q] = stg.area[q][tid];
    // boundary data (boundary_terms_k): Neumann terms (assembly.cpp:81-94;
    // this element's Neumann faces in face order == local slot order) and
    // Dirichlet traces b_D = |F| u_D(centroid) (assembly.cpp:96-104)
    double ln[4] = {0.0, 0.0, 0.0, 0.0};
    double bdv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        bdv[q] = 0.0;
        if (!sl.bnd[q]) continue;
        const double v = stg.bval[q][tid];
        if (sl.row[q] >= 0) {
            bdv[q] = v;
            continue;
        }
        const int i0 = face_vert(q, 0), i1 = face_vert(q, 1), i2 = face_vert(q, 2);
        ln[i0] = add(ln[i0], v);
        ln[i1] = add(ln[i1], v);
        ln[i2] = add(ln[i2], v);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) bt[v] = add(bt[v], ln[v]);  // B_T = b + LN (assembly.cpp:135)
    reinterpret_cast<double2*>(rhs)[2 * t] = make_double2(bt[0], bt[1]);
    reinterpret_cast<double2*>(rhs)[2 * t + 1] = make_double2(bt[2], bt[3]);
    double coef[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // slot_coef = sigma*|F|/3 (assembly.cpp:125)
        const double sg = sl.owner[q] ? 1.0 : -1.0;
        coef[q] = dv.div(mul(sg, area[q]), kDiv3);
    }
    if (slot_coef) {
#pragma unroll
        for (int q = 0; q < 4; ++q) slot_coef[4 * t + q] = coef[q];
    }
    if (slot_mrow) {
#pragma unroll
        for (int q = 0; q < 4; ++q) slot_mrow[4 * t + q] = sl.row[q];
    }
    Lu4 lu;
    {
        Local L;
        local_matrices(p, k, L, dv);  // local_stiffness_mass (assembly.cpp:7-33)
        if (a_blocks) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) a_blocks[16 * t + 4 * i + j] = L.a[i][j];
        }
        lu_factor(L.a, lu, dv);  // local Schur complement (solver.cpp:101-127)
    }
    // only the exact pass may call a block singular: FastDiv pivots outside
    // the exact window are not trusted (-> redo)
    if (lu.singular) return dv.good() ? 2 : 1;
    // local C rows c[r][v] = coef_r on the face's vertices, 0 on the
    // opposite one and on Neumann faces (local_c_rows, solver.cpp:33-40)
    auto cr = [&](int r, int v) -> double {
        const bool on = sl.row[r] >= 0 && v != (r == 0 ? 3 : (r == 3 ? 0 : r));
        return on ? coef[r] : 0.0;
    };
    // r_T = C A^-1 B_T; Dirichlet rows get b_D - r_T and b_D (single
    // contributor), interior rows keep -r_T for the final atomic
    double nrb[4];
    {
        double ainv_b[4];
        lu_solve(lu, bt, ainv_b, dv);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            nrb[r] = 0.0;
            if (sl.row[r] < 0) continue;
            double rb = 0.0;
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) rb = add(rb, mul(cr(r, pp), ainv_b[pp]));
            const int64_t R = sl.row[r];
            if (!ELEM) so.sell_col[sell_idx(R, 0)] = (int32_t)R;
            if (sl.bnd[r]) {
                rhs_neg[R] = sub(bdv[r], rb);
                bd[R] = bdv[r];
                if (!ELEM) {
#pragma unroll
                    for (int pos = 4; pos < 7; ++pos) {
                        so.sell_col[sell_idx(R, pos)] = (int32_t)R;
                        so.sell_val[sell_idx(R, pos)] = 0.0;
                    }
                }
            } else {
                bd[R] = 0.0;
                nrb[r] = -rb;
            }
        }
    }
    // one solved column x = A^-1 c_q at a time; S_T[r][q] accumulated over
    // p = 0..3 exactly as solver.cpp:121-125, stored at once (r != q)
    double sdiag[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double x[4] = {0.0, 0.0, 0.0, 0.0};
        const bool real = sl.row[q] >= 0;
        if (real) {
            const double cq[4] = {cr(q, 0), cr(q, 1), cr(q, 2), cr(q, 3)};
            lu_solve(lu, cq, x, dv);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (ELEM && r > q) continue;  // the upper triangle only
            // element-major: every pair is stored, 0 where a slot has no row
            if (!ELEM && sl.row[r] < 0) continue;
            double s = 0.0;
            if (real && sl.row[r] >= 0) {
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) s = add(s, mul(cr(r, pp), x[pp]));
            }
            if (r == q) {
                sdiag[r] = s;
                if (ELEM) so.st_val[st_idx(t, st_pair(r, r))] = s;
                continue;
            }
            if (ELEM) {
                so.st_val[st_idx(t, st_pair(r, q))] = s;
                continue;
            }
            const int64_t ix = sell_idx(sl.row[r], (sl.owner[r] ? 1 : 4) + (q < r ? q : q - 1));
            so.sell_col[ix] = real ? sl.row[q] : sl.row[r];
            so.sell_val[ix] = real ? s : 0.0;
        }
    }
    if (!dv.good()) return 1;
    if (ELEM && so.diag2) {
        // single writers: the owner slot writes the row's first half (and
        // zero second halves on a boundary row), the second slot the second
        // half of an interior row (a boundary row's rhs_neg was stored above)
        double* const d2 = so.diag2;
        double* const r2 = so.rhs2;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (sl.row[r] < 0) continue;
            const int64_t R = sl.row[r];
            if (sl.owner[r]) {
                so.diag[R] = sdiag[r];
                if (sl.bnd[r]) {
                    d2[R] = 0.0;
                    r2[R] = 0.0;
                } else {
                    rhs_neg[R] = nrb[r];
                }
            } else {
                d2[R] = sdiag[r];
                r2[R] = nrb[r];
            }
        }
        return 0;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (sl.row[r] < 0) continue;
        const int64_t R = sl.row[r];
        atomicAdd(ELEM ? so.diag + R : so.sell_val + sell_idx(R, 0), sdiag[r]);
        if (!sl.bnd[r]) atomicAdd(rhs_neg + R, nrb[r]);
    }
    return 0;
}

// Boundary terms, one thread per boundary list entry (db then nb, mapped to
// faces by the classification), computed as the element loop of
// assembly.cpp does from the owner element's local vertex order, with IEEE
// division (the values are the ones the element kernel would form):
//   Dirichlet: |F| u_D(centroid)                       (assembly.cpp:96-104)
//   Neumann:   0.5 |n| g(centroid, n / |n|) / 3, n = (q2 - q0) x (q1 - q0)
//                                                      (assembly.cpp:81-94)
// Kept out of assemble_k: its code (u, g with their transcendentals) ran in
// ~1 warp in 9 with a few lanes active and crowded the instruction cache.
template <int KIND>
__global__ void __launch_bounds__(128)
    boundary_terms_k(int64_t nd, int64_t nn, const int32_t* __restrict__ entry_face,
                     const int32_t* __restrict__ face_slots, const double* __restrict__ coords,
                     const int32_t* __restrict__ tets, phg_problem prob, const double* __restrict__ face_area,
                     double* __restrict__ face_bval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd + nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = entry_face[i];
        if (f < 0) continue;  // reported by the classification
        const int32_t slot = face_slots[2 * (int64_t)f];
        const int64_t t = slot >> 2;
        const int q = slot & 3;
        const int4 e = ldtet(tets, t);
        const int i0 = face_vert(q, 0), i1 = face_vert(q, 1), i2 = face_vert(q, 2);
        const V3 q0 = ldnode(coords, tv(e, i0)), q1 = ldnode(coords, tv(e, i1)), q2 = ldnode(coords, tv(e, i2));
        ExactDiv dv;
        const V3 s3 = vadd(vadd(q0, q1), q2);
        const V3 cen = {dv.div(s3.x, kDiv3), dv.div(s3.y, kDiv3), dv.div(s3.z, kDiv3)};
        if (i < nd) {
            face_bval[f] = mul(face_area[f], prob_u<KIND>(cen.x, cen.y, cen.z));
            continue;
        }
        const Coef k = load_coef(prob, t);
        const V3 n = vcross(vsub(q2, q0), vsub(q1, q0));
        const double len = __dsqrt_rn(vdot(n, n));
        const double ar = mul(0.5, len);
        const Div dl = dv.make(len);
        const V3 un = {dv.div(n.x, dl), dv.div(n.y, dl), dv.div(n.z, dl)};
        const double gc = prob_g<KIND>(cen.x, cen.y, cen.z, un, k);
        face_bval[f] = dv.div(mul(ar, gc), kDiv3);
    }
}

// Fast pass: one element per thread, blocks in element order (the elements
// in flight and the S rows they scatter into stay in an L2-resident window),
// FastDiv division.  Elements whose operands left the exact window are
// appended to redo_list.
// One red refinement of element t written by the assembly kernel itself
// (refine.cu's refine_staged per-parent body, refine.cpp:16-74): the
// element's nodes and coordinates are what the assembly loads anyway, and
// its 12 children (192 B) and new nodes are plain stores that the
// fp64-bound kernel issues beside its arithmetic, instead of a separate
// HBM-bound pass re-reading the mesh and the edge tables.  Children 1..11
// go to ne + 11 t + k as in refine_staged, one 176-byte run per thread (L2
// merges the lanes' partial sectors).
struct RefineOut {
    int64_t nc;                        // parent nodes (child ids start there)
    const int32_t* edge_first;         // 6 per element: first-occurrence slot
    const int32_t* edge_of_slot;       // 6 per element: edge id
    const int64_t* edge_off;           // low word: edges first seen before t
    double* coords_out;                // child coordinates (parents copied)
    int32_t* tets_out;                 // 12 ne child rows
};
__device__ __forceinline__ void refine_elem(int64_t t, int64_t ne, const double* __restrict__ coords,
                                            const int32_t* __restrict__ tets, const RefineOut& ro) {
    const int2* ef2 = reinterpret_cast<const int2*>(ro.edge_first) + 3 * t;
    const int2* eo2 = reinterpret_cast<const int2*>(ro.edge_of_slot) + 3 * t;
    const int2 f01 = __ldg(ef2), f23 = __ldg(ef2 + 1), f45 = __ldg(ef2 + 2);
    const int2 o01 = __ldg(eo2), o23 = __ldg(eo2 + 1), o45 = __ldg(eo2 + 2);
    const int64_t c = ro.nc + t + (uint32_t)__ldg(ro.edge_off + t);
    const int4 e = ldtet(tets, t);
    const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
    const V3 ct = vdiv(vadd(vadd(vadd(p[0], p[1]), p[2]), p[3]), 4.0);  // refine.cpp:33-34
    double* const co = ro.coords_out;
    co[3 * c] = ct.x;
    co[3 * c + 1] = ct.y;
    co[3 * c + 2] = ct.z;
    const int32_t fs[6] = {f01.x, f01.y, f23.x, f23.y, f45.x, f45.y};
    const int32_t os[6] = {o01.x, o01.y, o23.x, o23.y, o45.x, o45.y};
    int32_t mid[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const int64_t sl = 6 * t + k;
        const int64_t node = ro.nc + fs[k] / 6 + 1 + os[k];
        PHG_CHECK(fs[k] >= 0 && fs[k] <= (int32_t)sl && os[k] >= 0 && node < c + 7);
        mid[k] = (int32_t)node;
        if (fs[k] == (int32_t)sl) {
            const int a = k < 3 ? 0 : (k < 5 ? 1 : 2);
            const int b = k < 3 ? k + 1 : (k < 5 ? k - 1 : 3);
            const V3 pm = vdiv(vadd(p[a], p[b]), 2.0);  // refine.cpp:43
            co[3 * node] = pm.x;
            co[3 * node + 1] = pm.y;
            co[3 * node + 2] = pm.z;
        }
    }
    const int32_t i = e.x, j = e.y, k = e.z, l = e.w;
    const int32_t ij = mid[0], ik = mid[1], il = mid[2], jk = mid[3], jl = mid[4], kl = mid[5];
    const int32_t cc = (int32_t)c;
    int4* const out = reinterpret_cast<int4*>(ro.tets_out);
#ifdef PHG_REFINE_CS
#define PHG_ST4(p, v) __stcs(p, v)
#else
#define PHG_ST4(p, v) (*(p) = (v))
#endif
    PHG_ST4(out + t, make_int4(i, ij, ik, il));  // child 0 keeps slot t
    int4* const rest = out + ne + 11 * t;  // refine.cpp:58-61
    PHG_ST4(rest + 0, make_int4(j, jk, ij, jl));
    PHG_ST4(rest + 1, make_int4(k, ik, jk, kl));
    PHG_ST4(rest + 2, make_int4(l, kl, jl, il));
    PHG_ST4(rest + 3, make_int4(ij, ik, il, cc));
    PHG_ST4(rest + 4, make_int4(jk, ij, jl, cc));
    PHG_ST4(rest + 5, make_int4(ik, jk, kl, cc));
    PHG_ST4(rest + 6, make_int4(kl, jl, il, cc));
    PHG_ST4(rest + 7, make_int4(ij, jk, ik, cc));
    PHG_ST4(rest + 8, make_int4(ik, kl, il, cc));
    PHG_ST4(rest + 9, make_int4(ij, il, jl, cc));
    PHG_ST4(rest + 10, make_int4(kl, jk, jl, cc));
#undef PHG_ST4
}

template <int KIND, bool ELEM>
#ifdef PHG_COND_MAXREG
__global__ void __maxnreg__(PHG_COND_MAXREG)
#else
__global__ void __launch_bounds__(kCondThreads, PHG_COND_MINB)
#endif
    assemble_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
               const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
               const int32_t* __restrict__ face_mrow, const double* __restrict__ face_area,
               const double* __restrict__ face_bval, double* __restrict__ rhs, SchurOut so,
               double* __restrict__ rhs_neg, double* __restrict__ bd, double* __restrict__ a_blocks,
               double* __restrict__ slot_coef, int32_t* __restrict__ slot_mrow, int32_t* __restrict__ redo_list,
               int32_t* __restrict__ redo_count, unsigned long long* err, RefineOut ro) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ne) return;
#ifndef PHG_REFINE_AT_END
    if (ro.tets_out) refine_elem(t, ne, coords, tets, ro);
#endif
    FastDiv fd;
    const int st = assemble_elem<KIND, ELEM>(t, coords, tets, prob,
                                             {face_of_slot, slot_mate, face_mrow, face_area, face_bval}, a_blocks, so,
                                             rhs_neg, bd, rhs, slot_coef, slot_mrow, fd);
#ifdef PHG_REFINE_AT_END
    if (ro.tets_out) refine_elem(t, ne, coords, tets, ro);
#endif
    if (st == 1) redo_list[atomicAdd(redo_count, 1)] = (int32_t)t;
    // "degenerate element block" (solver.cpp:103-109)
    if (st == 2) report(err, PHG_ERR_SINGULAR, (unsigned long long)t);
    // "degenerate element (zero volume)" (assembly.cpp:13-14)
    if (st == 3) report(err, PHG_ERR_ZERO_VOLUME, (unsigned long long)t);
}

// Exact pass over the listed elements (IEEE division throughout).
template <int KIND, bool ELEM>
__global__ void __launch_bounds__(kCondThreads)
    assemble_redo_k(const int32_t* __restrict__ redo_list, const int32_t* __restrict__ redo_count,
                    const double* __restrict__ coords, const int32_t* __restrict__ tets, phg_problem prob,
                    const int32_t* __restrict__ face_of_slot, const int32_t* __restrict__ slot_mate,
                    const int32_t* __restrict__ face_mrow, const double* __restrict__ face_area,
                    const double* __restrict__ face_bval, double* __restrict__ rhs, SchurOut so,
                    double* __restrict__ rhs_neg, double* __restrict__ bd, double* __restrict__ a_blocks,
                    double* __restrict__ slot_coef, int32_t* __restrict__ slot_mrow, unsigned long long* err) {
    const int32_t n = *redo_count;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t t = redo_list[i];
        ExactDiv ed;
        if (assemble_elem<KIND, ELEM>(t, coords, tets, prob, {face_of_slot, slot_mate, face_mrow, face_area, face_bval},
                                      a_blocks, so, rhs_neg, bd, rhs, slot_coef, slot_mrow, ed) == 2)
            report(err, PHG_ERR_SINGULAR, (unsigned long long)t);
    }
}

// clear the two-contributor accumulators (S diagonal, rhs_neg) of rows 0..l-1
__global__ void __launch_bounds__(256) zero_rows_k(int64_t l, SchurOut so, double* __restrict__ rhs_neg) {
    // two rows per thread and step (16 B stores; rows 2i, 2i+1 share a slice)
    const double2 z = make_double2(0.0, 0.0);
    const int64_t l2 = l / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l2; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t R = 2 * i;
        reinterpret_cast<double2*>(so.diag ? so.diag + R : so.sell_val + sell_idx(R, 0))[0] = z;
        reinterpret_cast<double2*>(rhs_neg)[i] = z;
    }
    if ((l & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        (so.diag ? so.diag[l - 1] : so.sell_val[sell_idx(l - 1, 0)]) = 0.0;
        rhs_neg[l - 1] = 0.0;
    }
}

// SELL rows from the element-major S (the positions assemble_elem's SELL
// mode uses: owner slot -> 0 and 1-3, second slot -> 4-6, boundary rows
// padded with col = R, val = 0), one thread per element; the diagonal
// (position 0) by the row's owner slot
__global__ void __launch_bounds__(256)
    elem_to_sell_k(int64_t ne, const double* __restrict__ st_val, const int32_t* __restrict__ slot_mrow,
                   const int32_t* __restrict__ slot_mate, const double* __restrict__ diag,
                   int32_t* __restrict__ sell_col, double* __restrict__ sell_val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 rw4 = __ldg(reinterpret_cast<const int4*>(slot_mrow) + t);
        const int4 m4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        const int32_t rw[4] = {rw4.x, rw4.y, rw4.z, rw4.w}, mt[4] = {m4.x, m4.y, m4.z, m4.w};
        double sv[10];
#pragma unroll
        for (int j = 0; j < 10; ++j) sv[j] = __ldg(st_val + st_idx(t, j));
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (rw[r] < 0) continue;
            const int64_t R = rw[r];
            const bool owner = mt[r] < 0 || mt[r] > (int32_t)(4 * t + r);
            const int base = owner ? 1 : 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q == r) continue;
                const int64_t ix = sell_idx(R, base + (q < r ? q : q - 1));
                const bool real = rw[q] >= 0;
                sell_col[ix] = real ? rw[q] : (int32_t)R;
                sell_val[ix] = real ? sv[r < q ? st_pair(r, q) : st_pair(q, r)] : 0.0;
            }
            if (owner) {
                sell_col[sell_idx(R, 0)] = (int32_t)R;
                sell_val[sell_idx(R, 0)] = __ldg(diag + R);
            }
            if (mt[r] < 0) {
#pragma unroll
                for (int pos = 4; pos < 7; ++pos) {
                    sell_col[sell_idx(R, pos)] = (int32_t)R;
                    sell_val[sell_idx(R, pos)] = 0.0;
                }
            }
        }
    }
}

// deterministic sums of squares of B_T and b_D (fixed grid, fixed order)
__global__ void __launch_bounds__(256) sumsq2_k(const double* __restrict__ a, int64_t na, const double* __restrict__ b,
                                                int64_t nb, double* __restrict__ partials) {
    __shared__ double sh[8];
    double sa = 0.0, sb = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na; i += (int64_t)gridDim.x * blockDim.x)
        sa = fma(a[i], a[i], sa);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x)
        sb = fma(b[i], b[i], sb);
    sa = block_sum(sa, sh);
    sb = block_sum(sb, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = sa;
        partials[2 * blockIdx.x + 1] = sb;
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
    // collapsed-product structure of the degree-5 rule (4 x 4 x 4 points)
    double l0[64], l1[4], l2[16], l3[64];
    for (int a = 0; a < 4; ++a) {
        l1[a] = lam5[4 * (16 * a) + 1];
        for (int b = 0; b < 4; ++b) {
            l2[4 * a + b] = lam5[4 * (16 * a + 4 * b) + 2];
            for (int c = 0; c < 4; ++c) {
                const int q = 16 * a + 4 * b + c;
                l3[q] = lam5[4 * q + 3];
                l0[q] = lam5[4 * q];
                if (lam5[4 * q + 1] != l1[a] || lam5[4 * q + 2] != l2[4 * a + b]) return (int)cudaErrorInvalidValue;
            }
        }
    }
    cudaMemcpyToSymbol(phg::c_l1, l1, sizeof(l1));
    cudaMemcpyToSymbol(phg::c_l2, l2, sizeof(l2));
    cudaMemcpyToSymbol(phg::c_l3, l3, sizeof(l3));
    cudaMemcpyToSymbol(phg::c_l0, l0, sizeof(l0));
    const int rc = (int)cudaGetLastError();
    return rc ? rc : phfem_gpu_set_rules_errors(lam9, w9);
}

// One element per thread, blocks in element order: the elements in flight
// (and so the S rows they scatter into) stay within an L2-resident window;
// a grid-stride loop spread them over ~600k elements and turned the
// scattered SELL writes into DRAM read-modify-writes (ncu, profiles/).
// partial-sum slots used by the deterministic norm reduction
constexpr int kNormGrid = kSMs * 8;
extern "C" int phfem_gpu_assemble_grid(int64_t ne) {
    (void)ne;
    return kNormGrid;
}

extern "C" int phfem_gpu_assemble_condense(int64_t ne, int64_t l, const double* coords, const int32_t* tets,
                                           const phg_problem* prob, const int32_t* face_of_slot,
                                           const int32_t* slot_mate, const int32_t* face_mrow,
                                           const double* face_area, int64_t nd, int64_t nn,
                                           const int32_t* entry_face, const int32_t* face_slots, double* face_bval,
                                           int32_t* sell_col, double* sell_val, double* st_val, double* diag,
                                           double* rhs_neg, double* bd, double* rhs, double* a_blocks,
                                           double* slot_coef, int32_t* slot_mrow, int32_t* redo, double* halves,
                                           unsigned long long* err, const phg_refine_out* refine, void* ev_begin,
                                           void* ev_end, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    RefineOut ro{0, nullptr, nullptr, nullptr, nullptr, nullptr};
    if (refine) {
        ro = {refine->nc, refine->edge_first, refine->edge_of_slot, refine->edge_off, refine->coords_out,
              refine->tets_out};
        cudaMemcpyAsync(refine->coords_out, coords, (size_t)(3 * refine->nc) * sizeof(double),
                        cudaMemcpyDeviceToDevice, s);
    }
    if (ne == 0) {
        // nothing to assemble; the caller's events still bracket the (empty) kernel
        if (ev_begin) cudaEventRecord((cudaEvent_t)ev_begin, s);
        if (ev_end) cudaEventRecord((cudaEvent_t)ev_end, s);
        return (int)cudaGetLastError();
    }
    const unsigned grid = (unsigned)((ne + kCondThreads - 1) / kCondThreads);
    const phg_problem p = *prob;
    cudaMemsetAsync(redo, 0, sizeof(int32_t), s);
    // element-major when st_val is given (diag and slot_mrow required), else
    // SELL rows (sell_col / sell_val: NULL when there are no rows, L = 0)
    const bool elem = st_val != nullptr;
    if (elem && ((!diag && l > 0) || !slot_mrow)) return (int)cudaErrorInvalidValue;
    const bool split = elem && halves != nullptr;
    const SchurOut so{sell_col, sell_val, elem ? st_val : nullptr, elem ? diag : nullptr,
                      split ? halves : nullptr, split ? halves + l : nullptr};
    if (!split) zero_rows_k<<<kSMs * 8, 256, 0, s>>>(l, so, rhs_neg);
#define PHG_ASM(K, E)                                                                                                \
    assemble_k<K, E><<<grid, kCondThreads, 0, s>>>(ne, coords, tets, p, face_of_slot, slot_mate, face_mrow,          \
                                                   face_area, face_bval, rhs, so, rhs_neg, bd, a_blocks, slot_coef,  \
                                                   slot_mrow, redo + 1, redo, err, ro);                              \
    if (ev_end) cudaEventRecord((cudaEvent_t)ev_end, s);                                                             \
    assemble_redo_k<K, E><<<kSMs, kCondThreads, 0, s>>>(redo + 1, redo, coords, tets, p, face_of_slot, slot_mate,    \
                                                        face_mrow, face_area, face_bval, rhs, so, rhs_neg, bd,       \
                                                        a_blocks, slot_coef, slot_mrow, err)
#define PHG_KIND(K)                                                                                                  \
    if (nd + nn > 0)                                                                                                 \
        boundary_terms_k<K><<<(unsigned)((nd + nn + 127) / 128), 128, 0, s>>>(nd, nn, entry_face, face_slots, coords, \
                                                                             tets, p, face_area, face_bval);        \
    if (ev_begin) cudaEventRecord((cudaEvent_t)ev_begin, s);                                                         \
    if (elem) {                                                                                                      \
        PHG_ASM(K, true);                                                                                            \
    } else {                                                                                                         \
        PHG_ASM(K, false);                                                                                           \
    }
    switch (p.kind) {
        case 0: PHG_KIND(0); break;
        case 1: PHG_KIND(1); break;
        case 2: PHG_KIND(2); break;
        case 3: PHG_KIND(3); break;
        case 4: PHG_KIND(4); break;
        case 5: PHG_KIND(5); break;
        default: return (int)cudaErrorInvalidValue;
    }
#undef PHG_KIND
#undef PHG_ASM
    phg::count_launches(split ? 3 : 4);
    return (int)cudaGetLastError();
}

// diag = (0 + diag) + diag2, rhs_neg = (0 + rhs_neg) + rhs2: the value the
// atomics on cleared rows give (a two-term sum is order free)
__global__ void __launch_bounds__(256) sum_halves_k(int64_t l, double* __restrict__ diag,
                                                    double* __restrict__ rhs_neg, const double* __restrict__ halves) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
        diag[i] = (0.0 + diag[i]) + halves[i];
        rhs_neg[i] = (0.0 + rhs_neg[i]) + halves[l + i];
    }
}

extern "C" int phfem_gpu_sum_halves(int64_t l, double* diag, double* rhs_neg, const double* halves, void* stream) {
    if (l == 0) return 0;
    sum_halves_k<<<grid_for(l, 256), 256, 0, (cudaStream_t)stream>>>(l, diag, rhs_neg, halves);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

// ||B||^2, ||b_D||^2 for inner_cg_options (solver.cpp:78-86): computed when a
// solve asks for them, as the reference does, not inside the assembly
extern "C" int phfem_gpu_sumsq2(const double* rhs, int64_t n, const double* bd, int64_t l, double* partials,
                                double* norms, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    sumsq2_k<<<kNormGrid, 256, 0, s>>>(rhs, n, bd, l, partials);
    reduce_pairs<<<1, 1024, 0, s>>>(partials, kNormGrid, norms);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_elem_to_sell(int64_t ne, int64_t l, const double* st_val, const int32_t* slot_mrow,
                                      const int32_t* slot_mate, const double* diag, int32_t* sell_col,
                                      double* sell_val, void* stream) {
    (void)l;
    if (ne == 0) return 0;
    elem_to_sell_k<<<grid_for(ne, 256), 256, 0, (cudaStream_t)stream>>>(ne, st_val, slot_mrow, slot_mate, diag,
                                                                        sell_col, sell_val);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}
