// Jacobi-preconditioned CG on the SELL-32 Schur matrix (pcg_jacobi,
// sparse.cpp:163-212, with the stopping rule of inner_cg_options,
// solver.cpp:78-86).  Three kernels per iteration:
//   spmv   q = S p, partial p.q; last block: alpha = rz / pq
//   update r -= alpha q, z = d r, partials r.r, r.z;
//          last block: stop test, beta = rz'/rz
//   pdir   x += alpha p, p = d r + beta p
// The reference's x += alpha p (before the stop test) runs in pdir, which
// reads p anyway: one vector pass fewer per iteration, the same arithmetic
// (on the stopping iteration pdir updates x only).
// Scalars live in device memory (phg_cg_state); kernels become no-ops once
// `done` is set, so the host can enqueue batches of iterations (captured in
// a CUDA graph) and poll rarely.  Every reduction is a fixed-shape tree over
// fixed-grid block partials finished by the last block to arrive, so the
// iterates are bit-reproducible run to run.
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

using namespace phg;

constexpr int kThreads = 256;

inline int cg_grid(int64_t l) {
    const int g = grid_for(l, kThreads);
    return g < kSMs * 8 ? g : kSMs * 8;
}

__device__ __forceinline__ int64_t sell_idx(int64_t row, int pos) {
    return (row >> 5) * (PHG_SELL_C * PHG_SELL_W) + pos * PHG_SELL_C + (row & 31);
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block sum, valid in thread 0
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[kThreads / 32];
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < kThreads / 32 ? sh[threadIdx.x] : 0.0;
        s = warp_sum(s);
    }
    return s;
}

// Writes the block partials of NV values and returns true in every thread
// of the last block to finish; that block then has the totals in tot[].
template <int NV>
__device__ __forceinline__ bool finish(const double (&v)[NV], double* partials, unsigned* counter, double (&tot)[NV]) {
    __shared__ bool last;
    __shared__ double shtot[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double s = block_sum(v[i]);
        if (threadIdx.x == 0) partials[NV * blockIdx.x + i] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return false;
    __threadfence();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += __ldcg(partials + NV * b + i);
        s = block_sum(s);
        if (threadIdx.x == 0) shtot[i] = s;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = shtot[i];
    if (threadIdx.x == 0) *counter = 0;
    return true;
}

// the diagonal of S: SELL position 0, or the CSR row's entries on the
// diagonal summed in storage order (CsrMatrix::diagonal, sparse.cpp:60-66)
struct SellDiag {
    const double* sell_val;
    __device__ __forceinline__ double operator()(int64_t i) const { return sell_val[sell_idx(i, 0)]; }
};
struct ArrDiag {
    const double* diag;
    __device__ __forceinline__ double operator()(int64_t i) const { return diag[i]; }
};
struct CsrDiag {
    const int64_t* ptr;
    const int32_t* col;
    const double* val;
    __device__ __forceinline__ double operator()(int64_t i) const {
        double s = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
            if (col[k] == i) s = __dadd_rn(s, val[k]);
        return s;
    }
};

template <class Diag>
__global__ void __launch_bounds__(kThreads)
    cg_init(int64_t l, Diag diag_of, const double* __restrict__ b, double* __restrict__ x,
            double* __restrict__ r, double* __restrict__ p, double* __restrict__ d, double tol, double abs_tol,
            long long max_iter, phg_cg_state* st, double* partials) {
    double acc[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
        const double diag = diag_of(i);
        const double di = diag != 0.0 ? 1.0 / diag : 1.0;
        const double bi = b[i];
        d[i] = di;
        x[i] = 0.0;
        r[i] = bi;
        const double z = di * bi;
        p[i] = z;
        acc[0] += bi * bi;
        acc[1] += bi * z;
    }
    double tot[2];
    if (!finish<2>(acc, partials, &st->counter[0], tot)) return;
    if (threadIdx.x == 0) {
        const double bnorm = sqrt(tot[0]);
        st->bnorm = bnorm;
        st->rz = tot[1];
        st->it = 0;
        st->max_iter = max_iter;
        st->converged = 0;
        st->not_spd = 0;
        st->rel_residual = 1.0;
        st->rnorm = bnorm;
        const double rel = tol * bnorm;
        st->stop = abs_tol > 0.0 ? fmin(rel, abs_tol) : rel;
        if (bnorm == 0.0) {  // sparse.cpp:168: zero rhs, zero solution
            st->done = 1;
            st->converged = 1;
            st->rel_residual = 0.0;
        } else {
            st->done = 0;
        }
    }
}

__global__ void __launch_bounds__(kThreads)
    cg_spmv(int64_t l, const int32_t* __restrict__ sell_col, const double* __restrict__ sell_val,
            const double* __restrict__ p, double* __restrict__ q, phg_cg_state* st, double* partials) {
    if (st->done) {
        // the stopping iteration's pdir has run: nothing pending for x
        if (blockIdx.x == 0 && threadIdx.x == 0) st->x_pending = 0;
        return;
    }
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = (i >> 5) * (PHG_SELL_C * PHG_SELL_W) + (i & 31);
        // position 0 is the diagonal: its column is the row itself
        const double pi = __ldg(p + i);
        double s = __ldg(sell_val + base) * pi;
#pragma unroll
        for (int k = 1; k < PHG_SELL_W; ++k) {
            const int32_t c = __ldg(sell_col + base + k * PHG_SELL_C);
            PHG_CHECK(c >= 0 && c < l);
            const double v = __ldg(sell_val + base + k * PHG_SELL_C);
            s += v * __ldg(p + c);
        }
        q[i] = s;
        acc[0] += pi * s;
    }
    double tot[1];
    if (!finish<1>(acc, partials, &st->counter[1], tot)) return;
    if (threadIdx.x == 0) {
        st->pq = tot[0];
        if (tot[0] <= 0.0) {  // sparse.cpp:185
            st->not_spd = 1;
            st->done = 1;
        } else {
            st->alpha = st->rz / tot[0];
        }
    }
}

// q = S p straight from the element-major blocks (the pipeline's system):
// row R is the face of slots (s1 = owner, s2 = second or -1), and its
// entries are S_T[r][q] of those slots' elements, q over the element's other
// faces in increasing order, owner first -- the SELL row of elem_to_sell_k,
// summed in the same order with the same padding (0 * p[R] for a slot
// without a row, three of them for a face with one element), so the
// iterates are those of the SELL path bit for bit.  Per row 8 bytes of slots
// + 8 of diagonal instead of 84 bytes of SELL columns and values; the
// element's 6 off-diagonal values and its 4 row ids (64 bytes) are gathered
// by its faces' rows, which run close together (owner rows are consecutive,
// L2 holds the second elements' blocks in between).
// pair index (st_pair) of the k-th other face of local face r, 4 bits per
// (r, k): r = 0: (0,1) (0,2) (0,3); 1: (0,1) (1,2) (1,3); 2: (0,2) (1,2)
// (2,3); 3: (0,3) (1,3) (2,3)
constexpr unsigned long long kEmPairs = 0x321ull | 0x651ull << 12 | 0x852ull << 24 | 0x863ull << 36;
__device__ __forceinline__ double em_slot(int32_t slot, double s, double pi, const double* __restrict__ st_val,
                                          const int32_t* __restrict__ slot_mrow, const double* __restrict__ p,
                                          int64_t l) {
    const int64_t t = slot >> 2;
    const int r = slot & 3;
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(slot_mrow) + t);
    // the other three rows in local order
    const int32_t c[3] = {r == 0 ? m4.y : m4.x, r <= 1 ? m4.z : m4.y, r <= 2 ? m4.w : m4.z};
    const double* base = st_val + ((t >> 5) * 320 + (t & 31));
    const unsigned pairs = (unsigned)(kEmPairs >> (12 * r));
    double v[3], pc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        PHG_CHECK(c[k] < l);
        v[k] = c[k] >= 0 ? __ldg(base + 32 * ((pairs >> (4 * k)) & 15u)) : 0.0;
        pc[k] = c[k] >= 0 ? __ldg(p + c[k]) : pi;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) s += v[k] * pc[k];
    return s;
}

__global__ void __launch_bounds__(kThreads)
    cg_spmv_em(int64_t l, const int2* __restrict__ row_slots, const double* __restrict__ st_val,
               const int32_t* __restrict__ slot_mrow, const double* __restrict__ diag, const double* __restrict__ p,
               double* __restrict__ q, phg_cg_state* st, double* partials) {
    if (st->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->x_pending = 0;
        return;
    }
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
        const int2 rs = __ldg(row_slots + i);
        const double pi = __ldg(p + i);
        double s = __ldg(diag + i) * pi;
        s = em_slot(rs.x, s, pi, st_val, slot_mrow, p, l);
        if (rs.y >= 0) {
            s = em_slot(rs.y, s, pi, st_val, slot_mrow, p, l);
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) s += 0.0 * pi;  // SELL padding
        }
        q[i] = s;
        acc[0] += pi * s;
    }
    double tot[1];
    if (!finish<1>(acc, partials, &st->counter[1], tot)) return;
    if (threadIdx.x == 0) {
        st->pq = tot[0];
        if (tot[0] <= 0.0) {  // sparse.cpp:185
            st->not_spd = 1;
            st->done = 1;
        } else {
            st->alpha = st->rz / tot[0];
        }
    }
}

// row R -> (owner slot, second slot or -1), from the element-major rows
__global__ void __launch_bounds__(256)
    em_row_slots_k(int64_t ne, const int32_t* __restrict__ slot_mrow, const int32_t* __restrict__ slot_mate,
                   int2* __restrict__ row_slots) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 rw4 = __ldg(reinterpret_cast<const int4*>(slot_mrow) + t);
        const int4 m4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        const int32_t rw[4] = {rw4.x, rw4.y, rw4.z, rw4.w}, mt[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (rw[r] < 0) continue;
            const int32_t slot = (int32_t)(4 * t + r);
            const bool owner = mt[r] < 0 || mt[r] > slot;
            if (owner) row_slots[rw[r]] = make_int2(slot, mt[r] < 0 ? -1 : mt[r]);
        }
    }
}

// q = A p for a general CSR matrix (the C++ API's pcg_jacobi on a host
// CsrMatrix): one row per thread, entries in storage order
__global__ void __launch_bounds__(kThreads)
    cg_spmv_csr(int64_t l, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ p, double* __restrict__ q,
                phg_cg_state* st, double* partials) {
    if (st->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->x_pending = 0;
        return;
    }
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * __ldg(p + col[k]);
        q[i] = s;
        acc[0] += p[i] * s;
    }
    double tot[1];
    if (!finish<1>(acc, partials, &st->counter[1], tot)) return;
    if (threadIdx.x == 0) {
        st->pq = tot[0];
        if (tot[0] <= 0.0) {
            st->not_spd = 1;
            st->done = 1;
        } else {
            st->alpha = st->rz / tot[0];
        }
    }
}

__global__ void __launch_bounds__(kThreads)
    cg_update(int64_t l, double* __restrict__ r, const double* __restrict__ q, const double* __restrict__ d,
              phg_cg_state* st, double* partials) {
    if (st->done) return;
    const double alpha = st->alpha;
    double acc[2] = {0.0, 0.0};
    // two rows per thread and step (16 B accesses: twice the bytes in flight)
    const int64_t l2 = l / 2;
    const double2 *q2 = reinterpret_cast<const double2*>(q), *d2 = reinterpret_cast<const double2*>(d);
    double2* r2 = reinterpret_cast<double2*>(r);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l2; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 qi = q2[i], di = d2[i], ri = r2[i];
        const double ra = ri.x - alpha * qi.x, rb = ri.y - alpha * qi.y;
        r2[i] = make_double2(ra, rb);
        acc[0] += ra * ra;
        acc[0] += rb * rb;
        acc[1] += ra * (di.x * ra);
        acc[1] += rb * (di.y * rb);
    }
    if ((l & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail row
        const int64_t i = l - 1;
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        acc[0] += ri * ri;
        acc[1] += ri * (d[i] * ri);
    }
    double tot[2];
    if (!finish<2>(acc, partials, &st->counter[2], tot)) return;
    if (threadIdx.x == 0) {
        const long long it = st->it + 1;
        st->it = it;
        const double rnorm = sqrt(tot[0]);
        st->rnorm = rnorm;
        st->rel_residual = rnorm / st->bnorm;
        if (rnorm <= st->stop) {
            st->converged = 1;
            st->done = 1;
            st->x_pending = 1;
        } else if (it >= st->max_iter) {
            st->done = 1;
            st->x_pending = 1;
        } else {
            st->beta = tot[1] / st->rz;
            st->rz = tot[1];
        }
    }
}

__global__ void __launch_bounds__(kThreads)
    cg_pdir(int64_t l, double* __restrict__ x, const double* __restrict__ r, double* __restrict__ p,
            const double* __restrict__ d, const phg_cg_state* st) {
    if (st->done && !st->x_pending) return;
    const bool last = st->done;  // the stopping iteration: x only
    const double alpha = st->alpha, beta = st->beta;
    const int64_t l2 = l / 2;
    const double2 *r2 = reinterpret_cast<const double2*>(r), *d2 = reinterpret_cast<const double2*>(d);
    double2 *p2 = reinterpret_cast<double2*>(p), *x2 = reinterpret_cast<double2*>(x);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l2; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 pi = p2[i];
        double2 xi = x2[i];
        xi.x += alpha * pi.x;
        xi.y += alpha * pi.y;
        x2[i] = xi;
        if (!last) {
            const double2 ri = r2[i], di = d2[i];
            p2[i] = make_double2(di.x * ri.x + beta * pi.x, di.y * ri.y + beta * pi.y);
        }
    }
    if ((l & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = l - 1;
        x[i] += alpha * p[i];
        if (!last) p[i] = d[i] * r[i] + beta * p[i];
    }
}

}  // namespace

extern "C" int phfem_gpu_cg_init(int64_t l, const int32_t* sell_col, const double* sell_val, const double* b,
                                 double* x, double* r, double* p, double* d, double tol, double abs_tol,
                                 long long max_iter, phg_cg_state* st, double* partials, void* stream) {
    (void)sell_col;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(st, 0, sizeof(phg_cg_state), s);
    cg_init<<<cg_grid(l), kThreads, 0, s>>>(l, SellDiag{sell_val}, b, x, r, p, d, tol, abs_tol, max_iter, st, partials);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_cgcsr_init(int64_t l, const int64_t* ptr, const int32_t* col, const double* val,
                                    const double* b, double* x, double* r, double* p, double* d, double tol,
                                    double abs_tol, long long max_iter, phg_cg_state* st, double* partials,
                                    void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(st, 0, sizeof(phg_cg_state), s);
    cg_init<<<cg_grid(l), kThreads, 0, s>>>(l, CsrDiag{ptr, col, val}, b, x, r, p, d, tol, abs_tol, max_iter, st,
                                            partials);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_cgcsr_iterations(int n, int64_t l, const int64_t* ptr, const int32_t* col, const double* val,
                                          double* x, double* r, double* p, double* q, const double* d,
                                          phg_cg_state* st, double* partials, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g = cg_grid(l);
    for (int i = 0; i < n; ++i) {
        cg_spmv_csr<<<g, kThreads, 0, s>>>(l, ptr, col, val, p, q, st, partials);
        cg_update<<<g, kThreads, 0, s>>>(l, r, q, d, st, partials);
        cg_pdir<<<g, kThreads, 0, s>>>(l, x, r, p, d, st);
    }
    phg::count_launches(3 * n);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_cg_iterations(int n, int64_t l, const int32_t* sell_col, const double* sell_val, double* x,
                                       double* r, double* p, double* q, const double* d, phg_cg_state* st,
                                       double* partials, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g = cg_grid(l);
    for (int i = 0; i < n; ++i) {
        cg_spmv<<<g, kThreads, 0, s>>>(l, sell_col, sell_val, p, q, st, partials); phg::count_launches(1);
        cg_update<<<g, kThreads, 0, s>>>(l, r, q, d, st, partials); phg::count_launches(1);
        cg_pdir<<<g, kThreads, 0, s>>>(l, x, r, p, d, st); phg::count_launches(1);
    }
    return (int)cudaGetLastError();
}


extern "C" int phfem_gpu_cg_em_rows(int64_t ne, const int32_t* slot_mrow, const int32_t* slot_mate, int32_t* row_slots,
                                    void* stream) {
    if (ne == 0) return 0;
    em_row_slots_k<<<grid_for(ne, 256), 256, 0, (cudaStream_t)stream>>>(ne, slot_mrow, slot_mate,
                                                                        reinterpret_cast<int2*>(row_slots));
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_cg_em_init(int64_t l, const double* diag, const double* b, double* x, double* r, double* p,
                                    double* d, double tol, double abs_tol, long long max_iter, phg_cg_state* st,
                                    double* partials, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(st, 0, sizeof(phg_cg_state), s);
    cg_init<<<cg_grid(l), kThreads, 0, s>>>(l, ArrDiag{diag}, b, x, r, p, d, tol, abs_tol, max_iter, st, partials);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_cg_em_iterations(int n, int64_t l, const int32_t* row_slots, const double* st_val,
                                          const int32_t* slot_mrow, const double* diag, double* x, double* r,
                                          double* p, double* q, const double* d, phg_cg_state* st, double* partials,
                                          void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g = cg_grid(l);
    for (int i = 0; i < n; ++i) {
        cg_spmv_em<<<g, kThreads, 0, s>>>(l, reinterpret_cast<const int2*>(row_slots), st_val, slot_mrow, diag, p, q,
                                          st, partials);
        cg_update<<<g, kThreads, 0, s>>>(l, r, q, d, st, partials);
        cg_pdir<<<g, kThreads, 0, s>>>(l, x, r, p, d, st);
    }
    phg::count_launches(3 * n);
    return (int)cudaGetLastError();
}
