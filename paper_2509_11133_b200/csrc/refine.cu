// Uniform 12-way red refinement on the device (refine.cpp:16-96), one thread
// per parent element.
//
// The reference creates new nodes sequentially in first-occurrence order
// (per element: centroid, then the midpoints of edges not seen before).  With
// the first-occurrence edge numbering that order has a closed form, so every
// parent writes its own nodes independently:
//   centroid(t)  = nC + t + E_t          (E_t = edges first seen before t)
//   midpoint(e)  = nC + firstElem(e) + 1 + e
// Coordinates are ((c0+c1)+c2)+c3)/4 and (a+b)/2: additions and exact
// divisions by powers of two only, hence bit-identical to the CPU.
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

using namespace phg;

// A block owns kRefBlock consecutive parents, whose children 1..11 form one
// contiguous run of 11*kRefBlock rows: they are assembled in shared memory
// and streamed out with coalesced 16-byte stores.  The new nodes' 24-byte
// coordinates are stored directly (staging them too halved the occupancy).
constexpr int kRefBlock = 128;

__global__ void __launch_bounds__(kRefBlock)
    refine_staged(int64_t nc, int64_t ne, const double* __restrict__ coords, const int32_t* __restrict__ tets,
                  const int32_t* __restrict__ edge_first, const int32_t* __restrict__ edge_of_slot,
                  const int64_t* __restrict__ edge_off, double* __restrict__ coords_out,
                  int32_t* __restrict__ tets_out, int32_t* __restrict__ midpoint_node,
                  int32_t* __restrict__ centroid_node) {
    __shared__ int4 s_child[11 * kRefBlock];
    const int64_t t0 = (int64_t)blockIdx.x * kRefBlock;
    const int64_t t = t0 + threadIdx.x;
    const int64_t tend = t0 + kRefBlock < ne ? t0 + kRefBlock : ne;
    if (t < ne) {
        const int4 e = ldtet(tets, t);
        const V3 p[4] = {ldnode(coords, e.x), ldnode(coords, e.y), ldnode(coords, e.z), ldnode(coords, e.w)};
        const int64_t c = nc + t + (uint32_t)edge_off[t];  // low word: the offset
        const V3 ct = vdiv(vadd(vadd(vadd(p[0], p[1]), p[2]), p[3]), 4.0);  // refine.cpp:33-34
        coords_out[3 * c] = ct.x;
        coords_out[3 * c + 1] = ct.y;
        coords_out[3 * c + 2] = ct.z;
        if (centroid_node) centroid_node[t] = (int32_t)c;
        int32_t mid[6];
        const int2* ef2 = reinterpret_cast<const int2*>(edge_first) + 3 * t;
        const int2* eo2 = reinterpret_cast<const int2*>(edge_of_slot) + 3 * t;
        const int2 f01 = __ldg(ef2), f23 = __ldg(ef2 + 1), f45 = __ldg(ef2 + 2);
        const int2 o01 = __ldg(eo2), o23 = __ldg(eo2 + 1), o45 = __ldg(eo2 + 2);
        const int32_t fs[6] = {f01.x, f01.y, f23.x, f23.y, f45.x, f45.y};
        const int32_t os[6] = {o01.x, o01.y, o23.x, o23.y, o45.x, o45.y};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int64_t s = 6 * t + k;
            const int32_t first = fs[k];
            const int32_t id = os[k];
            const int64_t node = nc + first / 6 + 1 + id;
            PHG_CHECK(first >= 0 && first <= (int32_t)s && id >= 0 && node < nc + t + 1 + (uint32_t)edge_off[t] + 6);
            mid[k] = (int32_t)node;
            if (first == (int32_t)s) {
                const int a = k < 3 ? 0 : (k < 5 ? 1 : 2);
                const int b = k < 3 ? k + 1 : (k < 5 ? k - 1 : 3);
                const V3 pm = vdiv(vadd(p[a], p[b]), 2.0);  // refine.cpp:43
                coords_out[3 * node] = pm.x;
                coords_out[3 * node + 1] = pm.y;
                coords_out[3 * node + 2] = pm.z;
                if (midpoint_node) midpoint_node[id] = (int32_t)node;
            }
        }
        const int32_t i = e.x, j = e.y, k = e.z, l = e.w;
        const int32_t ij = mid[0], ik = mid[1], il = mid[2], jk = mid[3], jl = mid[4], kl = mid[5];
        const int32_t cc = (int32_t)c;
        reinterpret_cast<int4*>(tets_out)[t] = make_int4(i, ij, ik, il);  // child 0 keeps slot t
        int4* rest = s_child + 11 * threadIdx.x;  // refine.cpp:58-61
        rest[0] = make_int4(j, jk, ij, jl);
        rest[1] = make_int4(k, ik, jk, kl);
        rest[2] = make_int4(l, kl, jl, il);
        rest[3] = make_int4(ij, ik, il, cc);
        rest[4] = make_int4(jk, ij, jl, cc);
        rest[5] = make_int4(ik, jk, kl, cc);
        rest[6] = make_int4(kl, jl, il, cc);
        rest[7] = make_int4(ij, jk, ik, cc);
        rest[8] = make_int4(ik, kl, il, cc);
        rest[9] = make_int4(ij, il, jl, cc);
        rest[10] = make_int4(kl, jk, jl, cc);
    }
    __syncthreads();
    const int nrows = 11 * (int)(tend - t0);
    int4* dst = reinterpret_cast<int4*>(tets_out) + ne + 11 * t0;
    for (int r = threadIdx.x; r < nrows; r += kRefBlock) dst[r] = s_child[r];
}

// midpoint node of the mesh edge (a, b) through the star of min(a, b), or -1
__device__ int32_t edge_midpoint(int32_t a, int32_t b, int64_t nc, const int64_t* __restrict__ star_ptr,
                                 const int32_t* __restrict__ star, const int32_t* __restrict__ tets,
                                 const int32_t* __restrict__ edge_first, const int32_t* __restrict__ edge_of_slot) {
    if (a == b) return -1;
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    for (int64_t i = star_ptr[lo]; i < star_ptr[lo + 1]; ++i) {
        const int32_t inc = star[i];
        const int64_t t = inc >> 2;
        const int4 tet = ldtet(tets, t);
        for (int w = 0; w < 4; ++w) {
            if (tv(tet, w) != hi) continue;
            const int64_t s = 6 * t + edge_index(inc & 3, w);
            return (int32_t)(nc + edge_first[s] / 6 + 1 + edge_of_slot[s]);
        }
    }
    return -1;
}

__global__ void refine_boundary_k(int64_t nf, const int32_t* __restrict__ faces, int64_t list_base, int64_t nc,
                                  const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                                  const int32_t* __restrict__ tets, const int32_t* __restrict__ edge_first,
                                  const int32_t* __restrict__ edge_of_slot, int32_t* __restrict__ out,
                                  unsigned long long* err) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t n1 = faces[3 * f], n2 = faces[3 * f + 1], n3 = faces[3 * f + 2];
        const int32_t pr[3][2] = {{n1, n2}, {n2, n3}, {n1, n3}};
        int32_t m[3];
        bool ok = true;
        for (int q = 0; q < 3 && ok; ++q) {
            m[q] = edge_midpoint(pr[q][0], pr[q][1], nc, star_ptr, star, tets, edge_first, edge_of_slot);
            if (m[q] < 0) {
                report(err, PHG_ERR_BOUNDARY_EDGE, (unsigned long long)(list_base + f) << 2 | (unsigned)q);
                ok = false;
            }
        }
        if (!ok) continue;
        const int32_t m12 = m[0], m23 = m[1], m13 = m[2];
        int32_t* o = out + 3 * f;
        o[0] = n1; o[1] = m12; o[2] = m13;
        o = out + 3 * (nf + 3 * f);
        o[0] = n2; o[1] = m23; o[2] = m12;
        o[3] = n3; o[4] = m13; o[5] = m23;
        o[6] = m12; o[7] = m23; o[8] = m13;
    }
}


// The same split for a mesh whose classification is done: each entry's face
// is entry_face[list_base + f], owned by the slot (t, k), and the three
// midpoints follow from t's edge slots (no star search).  The entries are
// faces of the mesh, so no boundary-edge error can arise.
__global__ void refine_boundary_owned_k(int64_t nf, const int32_t* __restrict__ faces, int64_t list_base,
                                        int64_t nc, const int32_t* __restrict__ entry_face,
                                        const int32_t* __restrict__ face_slots, const int32_t* __restrict__ tets,
                                        const int32_t* __restrict__ edge_first,
                                        const int32_t* __restrict__ edge_of_slot, int32_t* __restrict__ out) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t n1 = faces[3 * f], n2 = faces[3 * f + 1], n3 = faces[3 * f + 2];
        const int32_t fid = __ldg(entry_face + list_base + f);
        PHG_CHECK(fid >= 0);
        const int64_t t = __ldg(face_slots + 2 * (int64_t)fid) >> 2;
        const int4 tet = ldtet(tets, t);
        const int l1 = tet.x == n1 ? 0 : (tet.y == n1 ? 1 : (tet.z == n1 ? 2 : 3));
        const int l2 = tet.x == n2 ? 0 : (tet.y == n2 ? 1 : (tet.z == n2 ? 2 : 3));
        const int l3 = tet.x == n3 ? 0 : (tet.y == n3 ? 1 : (tet.z == n3 ? 2 : 3));
        auto mid = [&](int a, int b) {
            const int64_t s = 6 * t + edge_index(a, b);
            return (int32_t)(nc + __ldg(edge_first + s) / 6 + 1 + __ldg(edge_of_slot + s));
        };
        const int32_t m12 = mid(l1, l2), m23 = mid(l2, l3), m13 = mid(l1, l3);
        int32_t* o = out + 3 * f;
        o[0] = n1; o[1] = m12; o[2] = m13;
        o = out + 3 * (nf + 3 * f);
        o[0] = n2; o[1] = m23; o[2] = m12;
        o[3] = n3; o[4] = m13; o[5] = m23;
        o[6] = m12; o[7] = m23; o[8] = m13;
    }
}

}  // namespace

extern "C" int phfem_gpu_refine(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                                const int32_t* edge_first, const int32_t* edge_of_slot, const int64_t* edge_off,
                                double* coords_out, int32_t* tets_out, int32_t* midpoint_node, int32_t* centroid_node,
                                void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemcpyAsync(coords_out, coords, (size_t)(3 * nc) * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (ne == 0) return (int)cudaGetLastError();
    refine_staged<<<(unsigned)((ne + kRefBlock - 1) / kRefBlock), kRefBlock, 0, s>>>(nc, ne, coords, tets, edge_first,
                                                                                   edge_of_slot, edge_off, coords_out,
                                               tets_out, midpoint_node, centroid_node); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_refine_boundary(int64_t nf, const int32_t* faces, int64_t list_base, int64_t nc,
                                         const int64_t* star_ptr, const int32_t* star, const int32_t* tets,
                                         const int32_t* edge_first, const int32_t* edge_of_slot, int32_t* out,
                                         unsigned long long* err, void* stream) {
    if (nf == 0) return 0;
    refine_boundary_k<<<grid_for(nf, 128), 128, 0, (cudaStream_t)stream>>>(nf, faces, list_base, nc, star_ptr, star,
                                                                           tets, edge_first, edge_of_slot, out, err); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_refine_boundary_owned(int64_t nf, const int32_t* faces, int64_t list_base, int64_t nc,
                                               const int32_t* entry_face, const int32_t* face_slots,
                                               const int32_t* tets, const int32_t* edge_first,
                                               const int32_t* edge_of_slot, int32_t* out, void* stream) {
    if (nf == 0) return 0;
    refine_boundary_owned_k<<<grid_for(nf, 128), 128, 0, (cudaStream_t)stream>>>(
        nf, faces, list_base, nc, entry_face, face_slots, tets, edge_first, edge_of_slot, out);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}
