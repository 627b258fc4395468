// Device kernels behind the reference's C++ API (include/phfem_cxx/*.hpp,
// implemented in cxx_api.cpp).  The C ABI pipeline never needs these: they
// serve the value-returning host API, whose inputs are host structs that may
// not come from a device mesh (a LinearSystem, a CsrMatrix, triplets):
//
//   * segmented sort: group items by a segment id (count, scan, scatter),
//     then sort each segment by (minor key, item index); the building block
//     of the E2T map (connectivity.cpp:46-70), CsrMatrix::from_triplets
//     (sparse.cpp:12-44), transpose (68-87) and spgemm (122-149), each of
//     which the reference defines through a (stable) sort;
//   * CSR kernels with the reference's summation order (multiply 46-52,
//     diagonal 60-66), so products are bit-identical to it;
//   * element-local condensation from given blocks (build_schur,
//     solver.cpp:90-147), recovery and verify residuals (44-76, 168-181);
//   * tabulated problem data: evaluation points for host callbacks and the
//     entries formed from the tabulated values (load_vector, neumann_vector,
//     dirichlet_vector, assembly.cpp:46-104; y_norm_error and
//     multiplier_norm_error, analysis.cpp:51-105).
// Arithmetic that the reference fixes is replayed with explicitly rounded
// intrinsics (common.cuh); one thread owns each sequential sum.
#include <cuda_runtime.h>

#include "problems.cuh"

namespace {

using namespace phg;

constexpr int kT = 256;

inline unsigned blocks_for(int64_t n) { return (unsigned)grid_for(n, kT); }

// --------------------------------------------------------- segmented sort

__global__ void seg_count_k(int64_t n, const int64_t* __restrict__ seg, int32_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + seg[i], 1);
}

__global__ void seg_scatter_k(int64_t n, const int64_t* __restrict__ seg, const int64_t* __restrict__ ptr,
                              int32_t* __restrict__ cursor, int64_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = seg[i];
        const int32_t k = atomicAdd(cursor + s, 1);
        PHG_CHECK(ptr[s] + k < ptr[s + 1]);
        perm[ptr[s] + k] = i;
    }
}

__device__ __forceinline__ bool item_less(const int64_t* minor, int64_t a, int64_t b) {
    const int64_t ka = minor[a], kb = minor[b];
    return ka != kb ? ka < kb : a < b;
}

// one thread per segment: insertion sort for short segments, bottom-up merge
// sort (through tmp) for long ones; keys (minor, index) are distinct, so
// the order is total
__global__ void seg_sort_k(int64_t nseg, const int64_t* __restrict__ ptr, const int64_t* __restrict__ minor,
                           int64_t* __restrict__ perm, int64_t* __restrict__ tmp) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = ptr[s], n = ptr[s + 1] - b;
        int64_t* a = perm + b;
        if (n <= 32) {
            for (int64_t i = 1; i < n; ++i) {
                const int64_t v = a[i];
                int64_t j = i - 1;
                while (j >= 0 && item_less(minor, v, a[j])) {
                    a[j + 1] = a[j];
                    --j;
                }
                a[j + 1] = v;
            }
            continue;
        }
        int64_t* src = a;
        int64_t* dst = tmp + b;
        for (int64_t w = 1; w < n; w *= 2) {
            for (int64_t lo = 0; lo < n; lo += 2 * w) {
                const int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
                int64_t i = lo, j = mid, k = lo;
                while (i < mid && j < hi) dst[k++] = item_less(minor, src[j], src[i]) ? src[j++] : src[i++];
                while (i < mid) dst[k++] = src[i++];
                while (j < hi) dst[k++] = src[j++];
            }
            int64_t* t = src;
            src = dst;
            dst = t;
        }
        if (src != a)
            for (int64_t i = 0; i < n; ++i) a[i] = src[i];
    }
}

__global__ void iota_k(int64_t n, int64_t* __restrict__ a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = i;
}

// -------------------------------------------------------------- E2T map

// entries of element m in the reference's order: for each oriented face
// [x y z] (local faces kFaceVerts) the keys (e_yz, e_xy), (e_zx, e_yz),
// (e_xy, e_zx) (connectivity.cpp:51-61)
// The reference's key of entry (from, to) is from * ned + to in uint64
// arithmetic, where pair_to_edge gives -1 for a pair of equal node ids
// (connectivity.hpp:25-30): such keys wrap.  Each entry is stored as the
// (segment, minor) pair the sort orders by: (K / ned, K % ned) for K < ned^2,
// else the extra segment ned with minor K + ned + 1 (K >= 2^64 - ned - 1
// there), so sorting by (segment, minor, entry) orders the reference's keys
// as its std::sort of (key, element) pairs does.
__device__ __forceinline__ void e2t_put(int64_t ned, int32_t f, int32_t t, int64_t* from, int64_t* to) {
    const unsigned long long K = (unsigned long long)(long long)f * (unsigned long long)ned +
                                 (unsigned long long)(long long)t;
    const unsigned long long lim = (unsigned long long)ned * (unsigned long long)ned;
    if (K < lim) {
        *from = (int64_t)(K / (unsigned long long)ned);
        *to = (int64_t)(K % (unsigned long long)ned);
    } else {
        *from = ned;
        *to = (int64_t)(K + (unsigned long long)ned + 1ull);
    }
}

__global__ void e2t_entries_k(int64_t ne, int64_t ned, const int32_t* __restrict__ edge_of_slot,
                              const int32_t* __restrict__ edge_nodes, int64_t* __restrict__ from,
                              int64_t* __restrict__ to) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < ne; m += (int64_t)gridDim.x * blockDim.x) {
        int32_t e[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            e[k] = edge_of_slot[6 * m + k];
            // pair_to_edge(a, a) == -1 (an element with a repeated node id)
            if (edge_nodes && e[k] >= 0 && edge_nodes[2 * (int64_t)e[k]] == edge_nodes[2 * (int64_t)e[k] + 1]) e[k] = -1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int x = face_vert(k, 0), y = face_vert(k, 1), z = face_vert(k, 2);
            const int32_t exy = e[edge_index(x, y)], eyz = e[edge_index(y, z)], ezx = e[edge_index(z, x)];
            const int64_t o = 12 * m + 3 * k;
            e2t_put(ned, eyz, exy, from + o, to + o);
            e2t_put(ned, ezx, eyz, from + o + 1, to + o + 1);
            e2t_put(ned, exy, ezx, from + o + 2, to + o + 2);
        }
    }
}

// sorted entries + the first duplicate key in sorted order (the pair the
// reference's error message names, connectivity.cpp:62-68)
__global__ void e2t_finish_k(int64_t n, int64_t ned, const int64_t* __restrict__ perm,
                             const int64_t* __restrict__ from, const int64_t* __restrict__ to,
                             unsigned long long* __restrict__ key, int32_t* __restrict__ elem,
                             unsigned long long* __restrict__ first_dup) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm[j];
        const unsigned long long k =
            from[i] < ned ? (unsigned long long)from[i] * (unsigned long long)ned + (unsigned long long)to[i]
                          : (unsigned long long)to[i] - (unsigned long long)ned - 1ull;
        key[j] = k;
        elem[j] = (int32_t)(i / 12);
        if (j > 0) {
            const int64_t ip = perm[j - 1];
            if (from[ip] == from[i] && to[ip] == to[i]) atomicMin(first_dup, (unsigned long long)j);
        }
    }
}

// ------------------------------------------------------------------ CSR

__global__ void widen_k(int64_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// per row of the row-sorted triplets: number of distinct columns
__global__ void csr_unique_k(int64_t rows, const int64_t* __restrict__ ptr, const int64_t* __restrict__ perm,
                             const int64_t* __restrict__ col, int32_t* __restrict__ cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = 0;
        int64_t prev = -1;
        for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
            const int64_t cj = col[perm[j]];
            if (j == ptr[r] || cj != prev) ++c;
            prev = cj;
        }
        cnt[r] = c;
    }
}

// duplicates summed in insertion order: v = first; v += next (sparse.cpp:31-33)
__global__ void csr_write_k(int64_t rows, const int64_t* __restrict__ ptr, const int64_t* __restrict__ perm,
                            const int64_t* __restrict__ col, const double* __restrict__ val,
                            const int64_t* __restrict__ out_ptr, int32_t* __restrict__ out_col,
                            double* __restrict__ out_val) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = out_ptr[r] - 1;
        int64_t prev = -1;
        for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
            const int64_t i = perm[j];
            const int64_t cj = col[i];
            if (j == ptr[r] || cj != prev) {
                ++o;
                out_col[o] = (int32_t)cj;
                out_val[o] = val[i];
            } else {
                out_val[o] = add(out_val[o], val[i]);
            }
            prev = cj;
        }
    }
}

// y = A x, s = 0; s += a x per row in storage order (sparse.cpp:46-52)
__global__ void csr_spmv_k(int64_t rows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) s = add(s, mul(val[k], x[col[k]]));
        y[r] = s;
    }
}

// diagonal (sparse.cpp:60-66)
__global__ void csr_diag_k(int64_t rows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, double* __restrict__ d) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k)
            if (col[k] == r) s = add(s, val[k]);
        d[r] = s;
    }
}

// row index of every stored entry
__global__ void csr_rowof_k(int64_t rows, const int64_t* __restrict__ ptr, int64_t* __restrict__ rowof) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) rowof[k] = r;
}

// transpose from the column-grouped permutation (entries of a column in
// storage order = ascending row, sparse.cpp:68-87)
__global__ void csr_transpose_k(int64_t nnz, const int64_t* __restrict__ perm, const int64_t* __restrict__ rowof,
                                const double* __restrict__ val, int32_t* __restrict__ tcol,
                                double* __restrict__ tval) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = perm[j];
        tcol[j] = (int32_t)rowof[k];
        tval[j] = val[k];
    }
}

// spgemm: products per row of A (count, then fill in the reference's
// accumulation order: A's row order, then B's row order)
__global__ void spgemm_count_k(int64_t rows, const int64_t* __restrict__ aptr, const int32_t* __restrict__ acol,
                               const int64_t* __restrict__ bptr, int32_t* __restrict__ cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int64_t k = aptr[r]; k < aptr[r + 1]; ++k) c += bptr[acol[k] + 1] - bptr[acol[k]];
        cnt[r] = (int32_t)c;
    }
}

__global__ void spgemm_fill_k(int64_t rows, const int64_t* __restrict__ aptr, const int32_t* __restrict__ acol,
                              const double* __restrict__ aval, const int64_t* __restrict__ bptr,
                              const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                              const int64_t* __restrict__ pptr, int64_t* __restrict__ pcol,
                              double* __restrict__ pval) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = pptr[r];
        for (int64_t k = aptr[r]; k < aptr[r + 1]; ++k) {
            const int32_t mid = acol[k];
            const double av = aval[k];
            for (int64_t kb = bptr[mid]; kb < bptr[mid + 1]; ++kb) {
                pcol[o] = bcol[kb];
                pval[o] = mul(av, bval[kb]);
                ++o;
            }
        }
    }
}

// acc[c] = 0.0; acc[c] += product, per distinct column in accumulation
// order (sparse.cpp:133-145)
__global__ void spgemm_write_k(int64_t rows, const int64_t* __restrict__ pptr, const int64_t* __restrict__ perm,
                               const int64_t* __restrict__ pcol, const double* __restrict__ pval,
                               const int64_t* __restrict__ out_ptr, int32_t* __restrict__ out_col,
                               double* __restrict__ out_val) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = out_ptr[r] - 1;
        int64_t prev = -1;
        for (int64_t j = pptr[r]; j < pptr[r + 1]; ++j) {
            const int64_t i = perm[j];
            if (j == pptr[r] || pcol[i] != prev) {
                ++o;
                out_col[o] = (int32_t)pcol[i];
                out_val[o] = add(0.0, pval[i]);
            } else {
                out_val[o] = add(out_val[o], pval[i]);
            }
            prev = pcol[i];
        }
    }
}

// --------------------------------------------------- block condensation

__device__ __forceinline__ void load_block(const double* __restrict__ a, int64_t t, double A[4][4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) A[i][j] = a[16 * t + 4 * i + j];
}

// local C rows c[r][v] = coef_r on face r's vertices, 0 on Neumann faces
// (local_c_rows, solver.cpp:33-40)
__device__ __forceinline__ void c_rows(const double* coef, const int32_t* mrow, int64_t t, double c[4][4]) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int v = 0; v < 4; ++v) c[r][v] = 0.0;
        if (mrow[4 * t + r] < 0) continue;
#pragma unroll
        for (int j = 0; j < 3; ++j) c[r][face_vert(r, j)] = coef[4 * t + r];
    }
}

// build_schur's element part (solver.cpp:101-127): LU, S_T, r_T
__global__ void condense_k(int64_t ne, const double* __restrict__ a_blocks, const double* __restrict__ coef,
                           const int32_t* __restrict__ mrow, const double* __restrict__ rhs,
                           double* __restrict__ lu_out, int32_t* __restrict__ perm_out,
                           uint8_t* __restrict__ singular, double* __restrict__ s_loc, double* __restrict__ r_loc,
                           unsigned long long* __restrict__ first_singular) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double A[4][4];
        load_block(a_blocks, t, A);
        Lu4 lu;
        lu_factor(A, lu);
        singular[t] = lu.singular ? 1 : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            perm_out[4 * t + i] = lu.perm[i];
#pragma unroll
            for (int j = 0; j < 4; ++j) lu_out[16 * t + 4 * i + j] = lu.lu[i][j];
        }
        if (lu.singular) {
            atomicMin(first_singular, (unsigned long long)t);
#pragma unroll
            for (int i = 0; i < 16; ++i) s_loc[16 * t + i] = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) r_loc[4 * t + i] = 0.0;
            continue;
        }
        double c[4][4], x[4][4], b[4], xb[4];
        c_rows(coef, mrow, t, c);
#pragma unroll
        for (int r = 0; r < 4; ++r) lu_solve(lu, c[r], x[r]);
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = rhs[4 * t + i];
        lu_solve(lu, b, xb);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double rb = 0.0;
#pragma unroll
            for (int p = 0; p < 4; ++p) rb = add(rb, mul(c[r][p], xb[p]));
            r_loc[4 * t + r] = rb;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double s = 0.0;
#pragma unroll
                for (int p = 0; p < 4; ++p) s = add(s, mul(c[r][p], x[q][p]));
                s_loc[16 * t + 4 * r + q] = s;
            }
        }
    }
}

__device__ __forceinline__ int rows_of(const int32_t* __restrict__ mrow, int64_t t) {
    return (mrow[4 * t] >= 0) + (mrow[4 * t + 1] >= 0) + (mrow[4 * t + 2] >= 0) + (mrow[4 * t + 3] >= 0);
}

// triplet counts per element: S (nr^2) and rhs_neg (nr)
__global__ void schur_counts_k(int64_t ne, const int32_t* __restrict__ mrow, int32_t* __restrict__ cs,
                               int32_t* __restrict__ cr) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int nr = rows_of(mrow, t);
        cs[t] = nr * nr;
        cr[t] = nr;
    }
}

// the reference's triplet stream (solver.cpp:131-145): element order, then
// r, then q over the non-Neumann rows
__global__ void schur_triplets_k(int64_t ne, const int32_t* __restrict__ mrow, const double* __restrict__ s_loc,
                                 const double* __restrict__ r_loc, const int64_t* __restrict__ os,
                                 const int64_t* __restrict__ orr, int64_t* __restrict__ trow,
                                 int64_t* __restrict__ tcol, double* __restrict__ tval,
                                 int64_t* __restrict__ rrow, double* __restrict__ rval) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = os[t], p = orr[t];
        for (int r = 0; r < 4; ++r) {
            const int32_t row = mrow[4 * t + r];
            if (row < 0) continue;
            rrow[p] = row;
            rval[p++] = r_loc[4 * t + r];
            for (int q = 0; q < 4; ++q) {
                const int32_t cq = mrow[4 * t + q];
                if (cq < 0) continue;
                trow[o] = row;
                tcol[o] = cq;
                tval[o++] = s_loc[16 * t + 4 * r + q];
            }
        }
    }
}

// rhs_neg = b_D; rhs_neg[row] -= r_T in triplet order (solver.cpp:133-138)
__global__ void rhs_neg_k(int64_t l, const int64_t* __restrict__ ptr, const int64_t* __restrict__ perm,
                          const double* __restrict__ rval, const double* __restrict__ bd, double* __restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < l; r += (int64_t)gridDim.x * blockDim.x) {
        double v = bd[r];
        for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) v = sub(v, rval[perm[j]]);
        out[r] = v;
    }
}

// recovery U_T = A_T^-1 (B_T + C_T' Lambda_T) (solver.cpp:168-181) and the
// element part of verify_solution's r1 = A U - B (solver.cpp:45-50)
__global__ void recover_blocks_k(int64_t ne, const double* __restrict__ a_blocks, const double* __restrict__ coef,
                                 const int32_t* __restrict__ mrow, const double* __restrict__ rhs,
                                 const double* __restrict__ lambda, double* __restrict__ u,
                                 double* __restrict__ r1) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double A[4][4];
        load_block(a_blocks, t, A);
        Lu4 lu;
        lu_factor(A, lu);
        double b[4], x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = rhs[4 * t + i];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int32_t row = mrow[4 * t + r];
            if (row < 0) continue;
            const double cl = mul(coef[4 * t + r], lambda[row]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int v = face_vert(r, j);
                b[v] = add(b[v], cl);
            }
        }
        lu_solve(lu, b, x);
#pragma unroll
        for (int i = 0; i < 4; ++i) u[4 * t + i] = x[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) s = add(s, mul(A[i][j], x[j]));
            r1[4 * t + i] = sub(s, rhs[4 * t + i]);
        }
    }
}

__global__ void axpy_sub_k(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = sub(a[i], b[i]);
}

// deterministic [sum x^2, max |x|] over a vector (fixed grid, fixed tree)
constexpr int kRedGrid = 296;
__global__ void __launch_bounds__(kT) sumsq_max_k(int64_t n, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double ss[kT], sm[kT];
    double s = 0.0, m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        s = add(s, mul(x[i], x[i]));
        m = fmax(m, fabs(x[i]));
    }
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            ss[threadIdx.x] = add(ss[threadIdx.x], ss[threadIdx.x + w]);
            sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ss[0];
        part[2 * blockIdx.x + 1] = sm[0];
    }
}
__global__ void sumsq_max_finish_k(int nb, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    double s = 0.0, m = 0.0;
    for (int b = 0; b < nb; ++b) {
        s = add(s, part[2 * b]);
        m = fmax(m, part[2 * b + 1]);
    }
    out[0] = s;
    out[1] = m;
}

// ------------------------------------------------------- tabulated data

__device__ __forceinline__ V3 node3(const double* __restrict__ c, int32_t n) {
    return {c[3 * (int64_t)n], c[3 * (int64_t)n + 1], c[3 * (int64_t)n + 2]};
}

// elem_volume (mesh.cpp:39-49) and the evaluation points of the load rule:
//   Gauss: x_q = ((p0 l0 + p1 l1) + p2 l2) + p3 l3 (assembly.cpp:72-73)
//   FaceCentroid: ((pa + pb) + pc) / 3 of local face k (assembly.cpp:53-55)
__global__ void load_points_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                              int rule, int nq, const double* __restrict__ lam, double* __restrict__ vol,
                              double* __restrict__ pts) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        vol[t] = dvd(fabs(vdot(vcross(vsub(p[1], p[0]), vsub(p[2], p[0])), vsub(p[3], p[0]))), 6.0);
        if (rule == 0) {
            for (int q = 0; q < nq; ++q) {
                const double* L = lam + 4 * q;
                const V3 x = vadd(vadd(vadd(vmul(p[0], L[0]), vmul(p[1], L[1])), vmul(p[2], L[2])), vmul(p[3], L[3]));
                double* o = pts + 3 * (nq * t + q);
                o[0] = x.x;
                o[1] = x.y;
                o[2] = x.z;
            }
        } else {
            for (int k = 0; k < 4; ++k) {
                const V3 x = vdiv(vadd(vadd(p[face_vert(k, 0)], p[face_vert(k, 1)]), p[face_vert(k, 2)]), 3.0);
                double* o = pts + 3 * (4 * t + k);
                o[0] = x.x;
                o[1] = x.y;
                o[2] = x.z;
            }
        }
    }
}

// load vector from tabulated f (assembly.cpp:46-79)
__global__ void load_tab_k(int64_t ne, int rule, int nq, const double* __restrict__ lam, const double* __restrict__ w,
                           const double* __restrict__ vol, const double* __restrict__ fv, double* __restrict__ b) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double V = vol[t];
        if (rule == 0) {
            for (int q = 0; q < nq; ++q) {
                const double fw = mul(mul(V, w[q]), fv[nq * t + q]);
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[v] = add(acc[v], mul(fw, lam[4 * q + v]));
            }
        } else {
            const double v12 = dvd(V, 12.0);
            for (int k = 0; k < 4; ++k) {
                const double c = mul(v12, fv[4 * t + k]);
                for (int j = 0; j < 3; ++j) {
                    const int v = face_vert(k, j);
                    acc[v] = add(acc[v], c);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) b[4 * t + v] = acc[v];
    }
}

// face_area_and_normal + face_centroid of listed faces (mesh.cpp:76-88):
// out[7 i] = area, unit normal (3), centroid (3); degenerate faces reported
__global__ void face_geom_k(int64_t n, const int32_t* __restrict__ ids, const int32_t* __restrict__ faces,
                            const double* __restrict__ coords, double* __restrict__ out,
                            unsigned long long* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = ids ? ids[i] : i;
        const V3 p0 = node3(coords, faces[3 * f]), p1 = node3(coords, faces[3 * f + 1]),
                 p2 = node3(coords, faces[3 * f + 2]);
        const V3 nrm = vcross(vsub(p2, p0), vsub(p1, p0));
        const double len = __dsqrt_rn(vdot(nrm, nrm));
        if (len == 0.0) atomicMin(bad, (unsigned long long)i);
        const V3 un = vdiv(nrm, len);
        const V3 c = vdiv(vadd(vadd(p0, p1), p2), 3.0);
        double* o = out + 7 * i;
        o[0] = mul(0.5, len);
        o[1] = un.x;
        o[2] = un.y;
        o[3] = un.z;
        o[4] = c.x;
        o[5] = c.y;
        o[6] = c.z;
    }
}

// Neumann terms (assembly.cpp:81-94) per element over its Neumann slots in
// local order (= ascending face id for faces_up numbering), then rhs = b + LN
__global__ void neumann_tab_k(int64_t ne, const int32_t* __restrict__ slot_to_face,
                              const uint8_t* __restrict__ face_class, const int64_t* __restrict__ face_slots,
                              const int32_t* __restrict__ geo_of_face, const double* __restrict__ geo,
                              const double* __restrict__ gv, double* __restrict__ ln) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < 4; ++k) {
            const int32_t f = slot_to_face[4 * t + k];
            if (face_class[f] != 2 || face_slots[2 * (int64_t)f] != 4 * t + k) continue;
            const int32_t g = geo_of_face[f];
            const double term = dvd(mul(geo[7 * (int64_t)g], gv[g]), 3.0);
            for (int j = 0; j < 3; ++j) {
                const int v = face_vert(k, j);
                acc[v] = add(acc[v], term);
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) ln[4 * t + v] = acc[v];
    }
}

// ---------------------------------------------------------- error norms

// tet_rule(9) points per element (analysis.cpp:62-63)
__global__ void ynorm_points_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                               int nq, const double* __restrict__ lam, double* __restrict__ pts) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        for (int q = 0; q < nq; ++q) {
            const double* L = lam + 4 * q;
            const V3 x = vadd(vadd(vadd(vmul(p[0], L[0]), vmul(p[1], L[1])), vmul(p[2], L[2])), vmul(p[3], L[3]));
            double* o = pts + 3 * ((int64_t)nq * t + q);
            o[0] = x.x;
            o[1] = x.y;
            o[2] = x.z;
        }
    }
}

// per-element y-norm sum from tabulated exact u, grad u (analysis.cpp:51-76)
__global__ void ynorm_elem_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                             const double* __restrict__ u, int nq, const double* __restrict__ lam,
                             const double* __restrict__ w, const double* __restrict__ ex, double inv_h2,
                             double* __restrict__ acc) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        Local L;
        const Coef k1 = {1.0, 1.0, 1.0, 1.0};
        local_matrices(p, k1, L);
        V3 gh = {0.0, 0.0, 0.0};
#pragma unroll
        for (int v = 0; v < 4; ++v) gh = vadd(gh, vmul(L.g[v], u[4 * t + v]));
        double s = 0.0;
        for (int q = 0; q < nq; ++q) {
            double uh = 0.0;
#pragma unroll
            for (int v = 0; v < 4; ++v) uh = add(uh, mul(lam[4 * q + v], u[4 * t + v]));
            const double* e = ex + 4 * ((int64_t)nq * t + q);
            const V3 dg = vsub(V3{e[1], e[2], e[3]}, gh);
            const double dv = sub(e[0], uh);
            s = add(s, mul(mul(L.vol, w[q]), add(vdot(dg, dg), mul(mul(inv_h2, dv), dv))));
        }
        acc[t] = s;
    }
}

// the three edge midpoints of each element's oriented faces (analysis.cpp:
// 94-99, tri_midpoint_rule); Neumann slots are skipped by the reducer
__global__ void kappa_points_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                               double* __restrict__ pts) {
    const double ml[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        for (int k = 0; k < 4; ++k) {
            const V3 a = p[face_vert(k, 0)], b = p[face_vert(k, 1)], c = p[face_vert(k, 2)];
            for (int q = 0; q < 3; ++q) {
                const V3 x = vadd(vadd(vmul(a, ml[q][0]), vmul(b, ml[q][1])), vmul(c, ml[q][2]));
                double* o = pts + 3 * (12 * t + 3 * k + q);
                o[0] = x.x;
                o[1] = x.y;
                o[2] = x.z;
            }
        }
    }
}

__global__ void kappa_elem_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                             const int32_t* __restrict__ slot_to_face, const double* __restrict__ sigma,
                             const uint8_t* __restrict__ face_class, const int32_t* __restrict__ mult,
                             const double* __restrict__ lambda, const double* __restrict__ gr, double h,
                             double* __restrict__ acc) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        double s = 0.0;
        for (int k = 0; k < 4; ++k) {
            const int64_t slot = 4 * t + k;
            const int32_t f = slot_to_face[slot];
            if (face_class[f] == 2) continue;
            const V3 a = p[face_vert(k, 0)], b = p[face_vert(k, 1)], c = p[face_vert(k, 2)];
            const V3 nrm = vcross(vsub(c, a), vsub(b, a));
            const double len = __dsqrt_rn(vdot(nrm, nrm));
            const V3 un = vdiv(nrm, len);
            const double area = mul(0.5, len);
            const double kh = mul(sigma[slot], lambda[mult[f]]);
            for (int q = 0; q < 3; ++q) {
                const double* g = gr + 3 * (12 * t + 3 * k + q);
                const double diff = sub(vdot(V3{g[0], g[1], g[2]}, un), kh);
                s = add(s, mul(mul(mul(mul(h, area), 1.0 / 3.0), diff), diff));
            }
        }
        acc[t] = s;
    }
}

// assemble_system's element part (assembly.cpp:115-130) from the mesh and a
// given face table: A_T = K_T + M_T, slot_mrow, slot_coef = (sigma |F|) / 3
__global__ void element_blocks_k(int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                                 const int32_t* __restrict__ slot_to_face, const double* __restrict__ sigma,
                                 const double* __restrict__ area, const int32_t* __restrict__ mult,
                                 double* __restrict__ a, double* __restrict__ coef, int32_t* __restrict__ mrow,
                                 unsigned long long* __restrict__ bad) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        V3 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = node3(coords, tets[4 * t + i]);
        Local L;
        const Coef k1 = {1.0, 1.0, 1.0, 1.0};
        local_matrices(p, k1, L);
        if (L.degenerate) atomicMin(bad, (unsigned long long)t);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[16 * t + 4 * i + j] = L.a[i][j];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t f = slot_to_face[4 * t + k];
            mrow[4 * t + k] = mult[f];
            coef[4 * t + k] = dvd(mul(sigma[4 * t + k], area[f]), 3.0);
        }
    }
}

// C triplets (row, 4t + v, coef) in element / slot / face-vertex order
// (assembly.cpp:121-130) at offsets 3 orr[t]
__global__ void c_triplets_k(int64_t ne, const int32_t* __restrict__ mrow, const double* __restrict__ coef,
                             const int64_t* __restrict__ orr, int64_t* __restrict__ trow, int64_t* __restrict__ tcol,
                             double* __restrict__ tval) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = 3 * orr[t];
        for (int k = 0; k < 4; ++k) {
            const int32_t r = mrow[4 * t + k];
            if (r < 0) continue;
            for (int j = 0; j < 3; ++j) {
                trow[o] = r;
                tcol[o] = 4 * t + face_vert(k, j);
                tval[o++] = coef[4 * t + k];
            }
        }
    }
}

// solve_direct's A^-1 (solver.cpp:203-212): Mat4Lu::inverse per element
__global__ void block_inverse_k(int64_t ne, const double* __restrict__ a, double* __restrict__ inv,
                                unsigned long long* __restrict__ first_singular) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double A[4][4];
        load_block(a, t, A);
        Lu4 lu;
        lu_factor(A, lu);
        if (lu.singular) {
            atomicMin(first_singular, (unsigned long long)t);
            continue;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double e[4] = {0.0, 0.0, 0.0, 0.0}, x[4];
            e[c] = 1.0;
            lu_solve(lu, e, x);
#pragma unroll
            for (int r = 0; r < 4; ++r) inv[16 * t + 4 * r + c] = x[r];
        }
    }
}

__global__ void block_pattern_k(int64_t ne, int64_t* __restrict__ row, int64_t* __restrict__ col) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 16 * ne; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i >> 4, ij = i & 15;
        row[i] = 4 * t + (ij >> 2);
        col[i] = 4 * t + (ij & 3);
    }
}

// u_T = Mat4Lu::factor(A_T).solve(b_T) (solver.cpp:235-239)
__global__ void block_solve_k(int64_t ne, const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ u) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        double A[4][4], bb[4], x[4];
        load_block(a, t, A);
        Lu4 lu;
        lu_factor(A, lu);
#pragma unroll
        for (int i = 0; i < 4; ++i) bb[i] = b[4 * t + i];
        lu_solve(lu, bb, x);
#pragma unroll
        for (int i = 0; i < 4; ++i) u[4 * t + i] = x[i];
    }
}

// r1 = A U - B per element (solver.cpp:45-50)
__global__ void block_residual_k(int64_t ne, const double* __restrict__ a, const double* __restrict__ u,
                                 const double* __restrict__ rhs, double* __restrict__ r1) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) s = add(s, mul(a[16 * t + 4 * i + j], u[4 * t + j]));
            r1[4 * t + i] = sub(s, rhs[4 * t + i]);
        }
    }
}

__global__ void add_inplace_k(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = add(a[i], b[i]);
}

// a = b - a (rhs_neg = b_D - C A^-1 B, solver.cpp:220)
__global__ void rsub_inplace_k(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = sub(b[i], a[i]);
}

// deterministic plain sum (fixed grid, fixed tree)
__global__ void __launch_bounds__(kT) sum_k(int64_t n, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double ss[kT];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s = add(s, x[i]);
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) ss[threadIdx.x] = add(ss[threadIdx.x], ss[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = ss[0];
}
__global__ void sum_finish_k(int nb, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s = add(s, part[b]);
    out[0] = s;
}

// refine_boundary_faces' 4-way split (refine.cpp:88-94) from the three
// midpoint ids of each face (m12, m23, m13)
__global__ void split_boundary_k(int64_t nf, const int32_t* __restrict__ in, const int32_t* __restrict__ mid,
                                 int32_t* __restrict__ out) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t n1 = in[3 * f], n2 = in[3 * f + 1], n3 = in[3 * f + 2];
        const int32_t m12 = mid[3 * f], m23 = mid[3 * f + 1], m13 = mid[3 * f + 2];
        int32_t* o = out + 3 * f;
        o[0] = n1, o[1] = m12, o[2] = m13;
        o = out + 3 * (nf + 3 * f);
        o[0] = n2, o[1] = m23, o[2] = m12;
        o[3] = n3, o[4] = m13, o[5] = m23;
        o[6] = m12, o[7] = m23, o[8] = m13;
    }
}

__global__ void refine_parent_k(int64_t ne, int32_t* __restrict__ parent) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < 12 * ne; c += (int64_t)gridDim.x * blockDim.x)
        parent[c] = (int32_t)(c < ne ? c : (c - ne) / 11);
}

}  // namespace

// ======================================================================

extern "C" int phfem_gpu_seg_sort(int64_t n, int64_t nseg, const int64_t* seg, const int64_t* minor,
                                  int64_t* seg_ptr, int64_t* perm, int32_t* cnt, int64_t* tmp, void* scan_scratch,
                                  void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nseg > 0 ? nseg : 1), s);
    if (n > 0) seg_count_k<<<blocks_for(n), kT, 0, s>>>(n, seg, cnt);
    int rc = phfem_gpu_scan_i32(cnt, seg_ptr, nseg, scan_scratch, stream);
    if (rc) return rc;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nseg > 0 ? nseg : 1), s);
    if (n > 0) {
        seg_scatter_k<<<blocks_for(n), kT, 0, s>>>(n, seg, seg_ptr, cnt, perm);
        seg_sort_k<<<blocks_for(nseg), kT, 0, s>>>(nseg, seg_ptr, minor, perm, tmp);
    }
    phg::count_launches(3);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_sort_within(int64_t n, int64_t nseg, const int64_t* seg_ptr, const int64_t* minor,
                                     int64_t* perm, int64_t* tmp, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n > 0) {
        iota_k<<<blocks_for(n), kT, 0, s>>>(n, perm);
        seg_sort_k<<<blocks_for(nseg), kT, 0, s>>>(nseg, seg_ptr, minor, perm, tmp);
    }
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_e2t_entries(int64_t ne, int64_t ned, const int32_t* edge_of_slot, const int32_t* edge_nodes,
                                     int64_t* from, int64_t* to, void* stream) {
    if (ne > 0)
        e2t_entries_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, ned, edge_of_slot, edge_nodes, from, to);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_e2t_finish(int64_t n, int64_t ned, const int64_t* perm, const int64_t* from,
                                    const int64_t* to, unsigned long long* key, int32_t* elem,
                                    unsigned long long* first_dup, void* stream) {
    if (n > 0)
        e2t_finish_k<<<blocks_for(n), kT, 0, (cudaStream_t)stream>>>(n, ned, perm, from, to, key, elem, first_dup);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_widen(int64_t n, const int32_t* a, int64_t* b, void* stream) {
    if (n > 0) widen_k<<<blocks_for(n), kT, 0, (cudaStream_t)stream>>>(n, a, b);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_unique(int64_t rows, const int64_t* ptr, const int64_t* perm, const int64_t* col,
                                    int32_t* cnt, void* stream) {
    if (rows > 0) csr_unique_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, perm, col, cnt);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_write(int64_t rows, const int64_t* ptr, const int64_t* perm, const int64_t* col,
                                   const double* val, const int64_t* out_ptr, int32_t* out_col, double* out_val,
                                   void* stream) {
    if (rows > 0)
        csr_write_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, perm, col, val, out_ptr, out_col,
                                                                       out_val);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_spmv(int64_t rows, const int64_t* ptr, const int32_t* col, const double* val,
                                  const double* x, double* y, void* stream) {
    if (rows > 0) csr_spmv_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, col, val, x, y);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_diag(int64_t rows, const int64_t* ptr, const int32_t* col, const double* val, double* d,
                                  void* stream) {
    if (rows > 0) csr_diag_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, col, val, d);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_rowof(int64_t rows, const int64_t* ptr, int64_t* rowof, void* stream) {
    if (rows > 0) csr_rowof_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, rowof);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_csr_transpose(int64_t nnz, const int64_t* perm, const int64_t* rowof, const double* val,
                                       int32_t* tcol, double* tval, void* stream) {
    if (nnz > 0) csr_transpose_k<<<blocks_for(nnz), kT, 0, (cudaStream_t)stream>>>(nnz, perm, rowof, val, tcol, tval);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_spgemm_count(int64_t rows, const int64_t* aptr, const int32_t* acol, const int64_t* bptr,
                                      int32_t* cnt, void* stream) {
    if (rows > 0) spgemm_count_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, aptr, acol, bptr, cnt);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_spgemm_fill(int64_t rows, const int64_t* aptr, const int32_t* acol, const double* aval,
                                     const int64_t* bptr, const int32_t* bcol, const double* bval,
                                     const int64_t* pptr, int64_t* pcol, double* pval, void* stream) {
    if (rows > 0)
        spgemm_fill_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, aptr, acol, aval, bptr, bcol, bval, pptr,
                                                                         pcol, pval);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_spgemm_write(int64_t rows, const int64_t* pptr, const int64_t* perm, const int64_t* pcol,
                                      const double* pval, const int64_t* out_ptr, int32_t* out_col, double* out_val,
                                      void* stream) {
    if (rows > 0)
        spgemm_write_k<<<blocks_for(rows), kT, 0, (cudaStream_t)stream>>>(rows, pptr, perm, pcol, pval, out_ptr,
                                                                          out_col, out_val);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_condense_blocks(int64_t ne, const double* a_blocks, const double* coef, const int32_t* mrow,
                                         const double* rhs, double* lu, int32_t* perm, uint8_t* singular,
                                         double* s_loc, double* r_loc, unsigned long long* first_singular,
                                         void* stream) {
    if (ne > 0)
        condense_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, a_blocks, coef, mrow, rhs, lu, perm, singular,
                                                                    s_loc, r_loc, first_singular);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_schur_counts(int64_t ne, const int32_t* mrow, int32_t* cs, int32_t* cr, void* stream) {
    if (ne > 0) schur_counts_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, mrow, cs, cr);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_schur_triplets(int64_t ne, const int32_t* mrow, const double* s_loc, const double* r_loc,
                                        const int64_t* os, const int64_t* orr, int64_t* trow, int64_t* tcol,
                                        double* tval, int64_t* rrow, double* rval, void* stream) {
    if (ne > 0)
        schur_triplets_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, mrow, s_loc, r_loc, os, orr, trow, tcol,
                                                                           tval, rrow, rval);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_rhs_neg(int64_t l, const int64_t* ptr, const int64_t* perm, const double* rval,
                                 const double* bd, double* out, void* stream) {
    if (l > 0) rhs_neg_k<<<blocks_for(l), kT, 0, (cudaStream_t)stream>>>(l, ptr, perm, rval, bd, out);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_recover_blocks(int64_t ne, const double* a_blocks, const double* coef, const int32_t* mrow,
                                        const double* rhs, const double* lambda, double* u, double* r1,
                                        void* stream) {
    if (ne > 0)
        recover_blocks_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, a_blocks, coef, mrow, rhs, lambda, u, r1);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_sub_inplace(int64_t n, double* a, const double* b, void* stream) {
    if (n > 0) axpy_sub_k<<<blocks_for(n), kT, 0, (cudaStream_t)stream>>>(n, a, b);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_sumsq_max_partials(void) { return kRedGrid; }

extern "C" int phfem_gpu_sumsq_max(int64_t n, const double* x, double* partials, double* out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    sumsq_max_k<<<kRedGrid, kT, 0, s>>>(n, x, partials);
    sumsq_max_finish_k<<<1, 32, 0, s>>>(kRedGrid, partials, out);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_load_points(int64_t ne, const double* coords, const int32_t* tets, int rule, int nq,
                                     const double* lam, double* vol, double* pts, void* stream) {
    if (ne > 0)
        load_points_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, coords, tets, rule, nq, lam, vol, pts);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_load_tab(int64_t ne, int rule, int nq, const double* lam, const double* w, const double* vol,
                                  const double* fv, double* b, void* stream) {
    if (ne > 0) load_tab_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, rule, nq, lam, w, vol, fv, b);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_face_geom(int64_t n, const int32_t* ids, const int32_t* faces, const double* coords,
                                   double* out, unsigned long long* bad, void* stream) {
    if (n > 0) face_geom_k<<<blocks_for(n), kT, 0, (cudaStream_t)stream>>>(n, ids, faces, coords, out, bad);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_neumann_tab(int64_t ne, const int32_t* slot_to_face, const uint8_t* face_class,
                                     const int64_t* face_slots, const int32_t* geo_of_face, const double* geo,
                                     const double* gv, double* ln, void* stream) {
    if (ne > 0)
        neumann_tab_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, slot_to_face, face_class, face_slots,
                                                                       geo_of_face, geo, gv, ln);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_ynorm_points(int64_t ne, const double* coords, const int32_t* tets, int nq,
                                      const double* lam, double* pts, void* stream) {
    if (ne > 0) ynorm_points_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, coords, tets, nq, lam, pts);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_ynorm_elem(int64_t ne, const double* coords, const int32_t* tets, const double* u, int nq,
                                    const double* lam, const double* w, const double* ex, double inv_h2, double* acc,
                                    void* stream) {
    if (ne > 0)
        ynorm_elem_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, coords, tets, u, nq, lam, w, ex, inv_h2, acc);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_kappa_points(int64_t ne, const double* coords, const int32_t* tets, double* pts,
                                      void* stream) {
    if (ne > 0) kappa_points_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, coords, tets, pts);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_kappa_elem(int64_t ne, const double* coords, const int32_t* tets,
                                    const int32_t* slot_to_face, const double* sigma, const uint8_t* face_class,
                                    const int32_t* mult, const double* lambda, const double* gr, double h,
                                    double* acc, void* stream) {
    if (ne > 0)
        kappa_elem_k<<<blocks_for(ne), kT, 0, (cudaStream_t)stream>>>(ne, coords, tets, slot_to_face, sigma, face_class,
                                                                      mult, lambda, gr, h, acc);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

#define PHG_API_LAUNCH(n, kernel, ...)                                                      \
    do {                                                                                    \
        if ((n) > 0) kernel<<<blocks_for(n), kT, 0, (cudaStream_t)stream>>>(__VA_ARGS__); \
        phg::count_launches(1);                                                             \
        return (int)cudaGetLastError();                                                     \
    } while (0)

extern "C" int phfem_gpu_element_blocks(int64_t ne, const double* coords, const int32_t* tets,
                                        const int32_t* slot_to_face, const double* sigma, const double* area,
                                        const int32_t* mult, double* a, double* coef, int32_t* mrow,
                                        unsigned long long* bad, void* stream) {
    PHG_API_LAUNCH(ne, element_blocks_k, ne, coords, tets, slot_to_face, sigma, area, mult, a, coef, mrow, bad);
}

extern "C" int phfem_gpu_c_triplets(int64_t ne, const int32_t* mrow, const double* coef, const int64_t* orr,
                                    int64_t* trow, int64_t* tcol, double* tval, void* stream) {
    PHG_API_LAUNCH(ne, c_triplets_k, ne, mrow, coef, orr, trow, tcol, tval);
}

extern "C" int phfem_gpu_block_inverses(int64_t ne, const double* a, double* inv, unsigned long long* first_singular,
                                        void* stream) {
    PHG_API_LAUNCH(ne, block_inverse_k, ne, a, inv, first_singular);
}

extern "C" int phfem_gpu_block_pattern(int64_t ne, int64_t* row, int64_t* col, void* stream) {
    PHG_API_LAUNCH(16 * ne, block_pattern_k, ne, row, col);
}

extern "C" int phfem_gpu_block_solve(int64_t ne, const double* a, const double* b, double* u, void* stream) {
    PHG_API_LAUNCH(ne, block_solve_k, ne, a, b, u);
}

extern "C" int phfem_gpu_block_residual(int64_t ne, const double* a, const double* u, const double* rhs, double* r1,
                                        void* stream) {
    PHG_API_LAUNCH(ne, block_residual_k, ne, a, u, rhs, r1);
}

extern "C" int phfem_gpu_add_inplace(int64_t n, double* a, const double* b, void* stream) {
    PHG_API_LAUNCH(n, add_inplace_k, n, a, b);
}

extern "C" int phfem_gpu_rsub_inplace(int64_t n, double* a, const double* b, void* stream) {
    PHG_API_LAUNCH(n, rsub_inplace_k, n, a, b);
}

extern "C" int phfem_gpu_sum(int64_t n, const double* x, double* partials, double* out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    sum_k<<<kRedGrid, kT, 0, s>>>(n, x, partials);
    sum_finish_k<<<1, 32, 0, s>>>(kRedGrid, partials, out);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_split_boundary(int64_t nf, const int32_t* in, const int32_t* mid, int32_t* out,
                                        void* stream) {
    if (nf > 0) split_boundary_k<<<blocks_for(nf), kT, 0, (cudaStream_t)stream>>>(nf, in, mid, out);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_refine_parents(int64_t ne, int32_t* parent, void* stream) {
    if (ne > 0) refine_parent_k<<<blocks_for(12 * ne), kT, 0, (cudaStream_t)stream>>>(ne, parent);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}
