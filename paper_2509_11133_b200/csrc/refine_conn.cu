// Connectivity of a red-refined mesh in closed form from its parent's tables
// (no vertex star, no hashing): the child's first-occurrence edge slots
// (edge_first), face mates (slot_mate) and per-element first/owner masks
// with the offsets' tile sums, one thread per parent element writing the 12
// children's 72 edge and 48 face slots (refined_groups_k); the child's
// boundary classification from the parent's (refined_classify_k).  The
// offsets' scan and the ids / tables (`number`) are the generic pipeline's.
//
// Children of parent t = (i, j, k, l) with midpoints m_ab and centroid c
// (refine.cpp:58-61): C0 = (i ij ik il) at index t, C1..C11 at
// nE + 11 t + q - 1.  Child edges are of three kinds:
//   V  (a, m_ab): only in the corner children at a.  First occurrence: C0 of
//      the first parent containing edge ab whose vertex 0 is a (A0 table),
//      else the corner child at a of the first parent containing ab (the
//      parent's first-occurrence element of ab);
//   F  (m_ab, m_ac) inside parent face abc: C0 of the first of the face's
//      (one or two) parents whose vertex 0 is a, else the corner child at a
//      of the face's owner (lower) parent;
//   C  (m_ab, c): only in t's centroid children, first in C4 / C5 / C6.
// Child faces are either shared by two children of the same parent (fixed
// table) or sub-triangles of a parent face, whose mate is the corresponding
// child of the parent across that face (or none on the boundary).
// tools/refined_conn_proto.py states the same rules in Python and checks
// them against the generic path; the tables below were generated from it.
#include <climits>
#include <cuda_runtime.h>

#include "common.cuh"
#include "scan.cuh"

namespace {

using namespace phg;

// [q][kk] = {kind, a, b, c}: kind 0 V (corner a, other end b), 1 F (shared
// corner a, other corners b, c), 2 C (first in child a, local edge b)
__device__ constexpr signed char kREdge[12][6][4] = {
    {{0, 0, 1, 0}, {0, 0, 2, 0}, {0, 0, 3, 0}, {1, 0, 1, 2}, {1, 0, 1, 3}, {1, 0, 2, 3}},
    {{0, 1, 2, 0}, {0, 1, 0, 0}, {0, 1, 3, 0}, {1, 1, 2, 0}, {1, 1, 2, 3}, {1, 1, 0, 3}},
    {{0, 2, 0, 0}, {0, 2, 1, 0}, {0, 2, 3, 0}, {1, 2, 0, 1}, {1, 2, 0, 3}, {1, 2, 1, 3}},
    {{0, 3, 2, 0}, {0, 3, 1, 0}, {0, 3, 0, 0}, {1, 3, 2, 1}, {1, 3, 2, 0}, {1, 3, 1, 0}},
    {{1, 0, 1, 2}, {1, 0, 1, 3}, {2, 4, 2, 0}, {1, 0, 2, 3}, {2, 4, 4, 0}, {2, 4, 5, 0}},
    {{1, 1, 2, 0}, {1, 1, 2, 3}, {2, 5, 2, 0}, {1, 1, 0, 3}, {2, 4, 2, 0}, {2, 5, 5, 0}},
    {{1, 2, 0, 1}, {1, 2, 0, 3}, {2, 4, 4, 0}, {1, 2, 1, 3}, {2, 5, 2, 0}, {2, 6, 5, 0}},
    {{1, 3, 2, 1}, {1, 3, 2, 0}, {2, 6, 5, 0}, {1, 3, 1, 0}, {2, 5, 5, 0}, {2, 4, 5, 0}},
    {{1, 1, 0, 2}, {1, 0, 1, 2}, {2, 4, 2, 0}, {1, 2, 1, 0}, {2, 5, 2, 0}, {2, 4, 4, 0}},
    {{1, 2, 0, 3}, {1, 0, 2, 3}, {2, 4, 4, 0}, {1, 3, 2, 0}, {2, 6, 5, 0}, {2, 4, 5, 0}},
    {{1, 0, 1, 3}, {1, 1, 0, 3}, {2, 4, 2, 0}, {1, 3, 0, 1}, {2, 4, 5, 0}, {2, 5, 5, 0}},
    {{1, 2, 3, 1}, {1, 3, 2, 1}, {2, 6, 5, 0}, {1, 1, 2, 3}, {2, 5, 2, 0}, {2, 5, 5, 0}}};

// [q][kf] = {kind, a, b}: kind 0 shared inside the parent with child a,
// local face b; 1 corner sub-triangle at corner a of parent face b; 2 middle
// sub-triangle of parent face a
__device__ constexpr signed char kRFace[12][4][4] = {
    {{1, 0, 0, 0}, {1, 0, 1, 0}, {1, 0, 2, 0}, {0, 4, 0, 0}},
    {{1, 1, 0, 0}, {1, 1, 2, 0}, {1, 1, 3, 0}, {0, 5, 0, 0}},
    {{1, 2, 0, 0}, {1, 2, 3, 0}, {1, 2, 1, 0}, {0, 6, 0, 0}},
    {{1, 3, 3, 0}, {1, 3, 2, 0}, {1, 3, 1, 0}, {0, 7, 0, 0}},
    {{0, 0, 3, 0}, {0, 10, 2, 0}, {0, 8, 1, 0}, {0, 9, 1, 0}},
    {{0, 1, 3, 0}, {0, 11, 3, 0}, {0, 8, 2, 0}, {0, 10, 1, 0}},
    {{0, 2, 3, 0}, {0, 9, 2, 0}, {0, 8, 3, 0}, {0, 11, 2, 0}},
    {{0, 3, 3, 0}, {0, 9, 3, 0}, {0, 11, 1, 0}, {0, 10, 3, 0}},
    {{2, 0, 0, 0}, {0, 4, 2, 0}, {0, 5, 2, 0}, {0, 6, 2, 0}},
    {{2, 1, 0, 0}, {0, 4, 3, 0}, {0, 6, 1, 0}, {0, 7, 1, 0}},
    {{2, 2, 0, 0}, {0, 5, 3, 0}, {0, 4, 1, 0}, {0, 7, 3, 0}},
    {{2, 3, 0, 0}, {0, 7, 2, 0}, {0, 6, 3, 0}, {0, 5, 1, 0}}};

// position of midpoint m_qx in corner child q (x != q):
// {{-1, 1, 2, 3}, {2, -1, 1, 3}, {1, 2, -1, 3}, {3, 2, 1, -1}}, packed + 1 in
// nibbles (runtime indices without a memory table)
__device__ __forceinline__ int rpos(int q, int x) {
    return (int)((0x234403242034320ull >> (4 * (4 * q + x))) & 0xFu) - 1;
}

// local face k excludes local vertex kExcl[k]; the same map sends a vertex
// to the face that excludes it
__device__ __forceinline__ int excl(int k) { return k == 0 ? 3 : (k == 3 ? 0 : k); }

// A0 entries start as 0x7f7f7f7f (byte memset): no parent with that vertex 0
constexpr int32_t kNoParent = 0x7f7f7f7f;

__device__ __forceinline__ int64_t child(int64_t t, int q, int64_t n) { return q == 0 ? t : n + 11 * t + q - 1; }

__device__ __forceinline__ int idx_of(const int4& p, int32_t g) {
    return p.x == g ? 0 : (p.y == g ? 1 : (p.z == g ? 2 : 3));
}

__device__ __forceinline__ int ledge(int a, int b) { return edge_index(a, b); }

// A0[2e + w]: the first parent with vertex 0 = the smaller (w = 0) / larger
// (w = 1) endpoint of edge e, from the slots (t, k < 3) whose local pair
// contains vertex 0
__global__ void a0_k(int64_t ne, const int32_t* __restrict__ tets, const int32_t* __restrict__ edge_of_slot,
                     int32_t* __restrict__ a0) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 p = ldtet(tets, t);
        const int32_t o[3] = {p.y, p.z, p.w};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int32_t e = edge_of_slot[6 * t + k];
            PHG_CHECK(e >= 0);
            atomicMin(a0 + 2 * (int64_t)e + (p.x < o[k] ? 0 : 1), (int32_t)t);
        }
    }
}

// The 12 children's rows are staged in shared memory and written out
// coalesced: the block's C1..C11 rows are one contiguous range (nE + 11 t0
// ...), its C0 rows another (t0 ...).  Row r of the stage is C(q) of local
// parent lt at r = 11 lt + q - 1 (q >= 1) or 11 kRgBlock + lt (q = 0).
constexpr int kRgBlock = 64;

__device__ __forceinline__ int stage_row(int lt, int q) { return q == 0 ? 11 * kRgBlock + lt : 11 * lt + q - 1; }

__global__ void __launch_bounds__(kRgBlock)
    refined_groups_k(int64_t n, const int32_t* __restrict__ tets, const int32_t* __restrict__ edge_of_slot,
                     const int32_t* __restrict__ edge_first, const int32_t* __restrict__ slot_mate,
                     const int32_t* __restrict__ a0, int32_t* __restrict__ ef_out, int32_t* __restrict__ sm_out,
                     uint16_t* __restrict__ masks, long long* __restrict__ tile_sums) {
    // one stage buffer, the edge rows then the face rows
    __shared__ int4 s_buf[12 * kRgBlock * 6 / 4];
    __shared__ uint16_t s_mask[12 * kRgBlock];
    int2* s_ef = reinterpret_cast<int2*>(s_buf);
    int4* s_sm = s_buf;
    const int64_t t0 = (int64_t)blockIdx.x * kRgBlock;
    const int lt = threadIdx.x;
    const int64_t t = t0 + lt;
    const int nb = (int)(n - t0 < kRgBlock ? n - t0 : kRgBlock);
    // mates of the sub-triangles of parent face k: FM[k][a] at corner a,
    // MM[k] the middle one (kept in registers across the edge-row stage)
    int32_t FM[4][4], MM[4];
    // 32-bit ids: 6 x 12 nE < 2^31 (refine_mesh checks it)
    const int32_t n32 = (int32_t)n, t32 = (int32_t)t;
    auto ch = [n32](int32_t tt, int q) { return q == 0 ? tt : n32 + 11 * tt + q - 1; };
    if (lt < nb) {
        const int4 pt = ldtet(tets, t);
        const int32_t pv[4] = {pt.x, pt.y, pt.z, pt.w};
        int32_t ef[6];
        int2 a0p[6];  // both A0 entries of each edge
        {
            const int2* eo2 = reinterpret_cast<const int2*>(edge_of_slot) + 3 * t;
            const int2* ef2 = reinterpret_cast<const int2*>(edge_first) + 3 * t;
            const int2 e01 = __ldg(eo2), e23 = __ldg(eo2 + 1), e45 = __ldg(eo2 + 2);
            const int2 f01 = __ldg(ef2), f23 = __ldg(ef2 + 1), f45 = __ldg(ef2 + 2);
            const int32_t eos[6] = {e01.x, e01.y, e23.x, e23.y, e45.x, e45.y};
            ef[0] = f01.x; ef[1] = f01.y; ef[2] = f23.x; ef[3] = f23.y; ef[4] = f45.x; ef[5] = f45.y;
#pragma unroll
            for (int k = 0; k < 6; ++k) a0p[k] = __ldg(reinterpret_cast<const int2*>(a0) + eos[k]);
        }
        const int4 sm4 = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        const int32_t sm[4] = {sm4.x, sm4.y, sm4.z, sm4.w};
        // the parent across each face and the positions there of the face's
        // three corners (mp[k][j] for corner face_vert(k, j))
        int mp[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int4 m4 = sm[k] >= 0 ? ldtet(tets, sm[k] >> 2) : make_int4(-1, -1, -1, -1);
#pragma unroll
            for (int j = 0; j < 3; ++j) mp[k][j] = idx_of(m4, pv[face_vert(k, j)]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t ms = sm[k];
            const int32_t t2 = ms >> 2;
            const int k2 = ms & 3;
            MM[k] = ms < 0 ? -1 : 4 * ch(t2, 8 + k2);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int a2 = mp[k][j];
                FM[k][face_vert(k, j)] = ms < 0 ? -1 : 4 * ch(t2, a2) + excl(rpos(a2, excl(k2)));
            }
        }
        // The distinct child edges once each (the 72 slots repeat them):
        // V[a][b] for the half-edge (a, m_ab), F[k][a] for the edge
        // (m_ab, m_ac) inside parent face k at its corner a; the C edges are
        // closed-form.  All table indices are compile-time constants after
        // unrolling; where the first parent is t itself the positions are too.
        int32_t V[4][4], F[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                if (a == b) continue;
                const int32_t ga = pv[a], gb = pv[b];
                const int le = ledge(a, b);
                const int32_t ts = ga < gb ? a0p[le].x : a0p[le].y;
                int32_t first;
                if (ts == t32) {
                    first = 6 * t32 + b - 1;  // C0 of t (vertex 0 = a)
                } else if (ts != kNoParent) {
                    first = 6 * ts + idx_of(ldtet(tets, ts), gb) - 1;
                } else {
                    const int32_t t1 = ef[le] / 6;
                    if (t1 == t32) {
                        first = 6 * ch(t32, a) + rpos(a, b) - 1;
                    } else {
                        const int4 p1 = ldtet(tets, t1);
                        const int qa = idx_of(p1, ga), qb = idx_of(p1, gb);
                        first = 6 * ch(t1, qa) + rpos(qa, qb) - 1;
                    }
                }
                V[a][b] = first;
            }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // parent face k and the parent across it: the first of the two
            // whose vertex 0 is the corner, else the lower one's corner child
            const int32_t ms = sm[k];
            const int32_t t2 = ms >> 2;
            const bool t_first = ms < 0 || t32 < t2;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int a = face_vert(k, j), b = face_vert(k, (j + 1) % 3), c = face_vert(k, (j + 2) % 3);
                const int ma = mp[k][j], mb = mp[k][(j + 1) % 3], mc = mp[k][(j + 2) % 3];
                const int32_t own0 = 6 * t32 + ledge(b, c);                          // t, vertex 0 = a
                const int32_t own = 6 * ch(t32, a) + ledge(rpos(a, b), rpos(a, c));  // t's corner child
                int32_t first;
                if (t_first) {
                    if (a == 0) first = own0;
                    else if (ms >= 0 && ma == 0) first = 6 * t2 + ledge(mb, mc);
                    else first = own;
                } else {
                    if (ma == 0) first = 6 * t2 + ledge(mb, mc);
                    else if (a == 0) first = own0;
                    else first = 6 * ch(t2, ma) + ledge(rpos(ma, mb), rpos(ma, mc));
                }
                F[k][a] = first;
            }
        }
#pragma unroll
        for (int q = 0; q < 12; ++q) {
            int32_t out[6];
#pragma unroll
            for (int kk = 0; kk < 6; ++kk) {
                const int kind = kREdge[q][kk][0], a = kREdge[q][kk][1], b = kREdge[q][kk][2], c = kREdge[q][kk][3];
                if (kind == 2) out[kk] = 6 * ch(t32, a) + b;
                else if (kind == 0) out[kk] = V[a][b];
                else out[kk] = F[excl(6 - a - b - c)][a];
            }
#pragma unroll
            for (int kk = 0; kk < 6; ++kk) PHG_CHECK(out[kk] >= 0 && out[kk] <= 6 * ch(t32, q) + kk);
            int2* o2 = s_ef + 3 * stage_row(lt, q);
            o2[0] = make_int2(out[0], out[1]);
            o2[1] = make_int2(out[2], out[3]);
            o2[2] = make_int2(out[4], out[5]);
            // first-occurrence slots of the child (offsets_count_k's bits 0-5)
            const int32_t base = 6 * ch(t32, q);
            uint32_t m = 0;
#pragma unroll
            for (int kk = 0; kk < 6; ++kk) m |= (uint32_t)(out[kk] == base + kk) << kk;
            s_mask[stage_row(lt, q)] = (uint16_t)m;
        }
    }
    __syncthreads();
    // C1..C11: rows nE + 11 t0 + [0, 11 nb); C0: rows t0 + [0, nb)
    {
        int2* e1 = reinterpret_cast<int2*>(ef_out) + 3 * (n + 11 * t0);
        for (int i = lt; i < 33 * nb; i += kRgBlock) e1[i] = s_ef[i];
        int2* e0 = reinterpret_cast<int2*>(ef_out) + 3 * t0;
        for (int i = lt; i < 3 * nb; i += kRgBlock) e0[i] = s_ef[33 * kRgBlock + i];
    }
    if (sm_out) {
        __syncthreads();
        if (lt < nb) {
#pragma unroll
            for (int q = 0; q < 12; ++q) {
                int32_t fo[4];
#pragma unroll
                for (int kf = 0; kf < 4; ++kf) {
                    const int kind = kRFace[q][kf][0], a = kRFace[q][kf][1], b = kRFace[q][kf][2];
                    fo[kf] = kind == 0 ? 4 * ch(t32, a) + b : (kind == 1 ? FM[b][a] : MM[a]);
                }
#pragma unroll
                for (int kf = 0; kf < 4; ++kf) PHG_CHECK(fo[kf] >= -1 && fo[kf] < 48 * n32 && fo[kf] != 4 * ch(t32, q) + kf);
                s_sm[stage_row(lt, q)] = make_int4(fo[0], fo[1], fo[2], fo[3]);
                // owned face slots (bits 6-9)
                const int32_t sl = 4 * ch(t32, q);
                uint32_t m = 0;
#pragma unroll
                for (int kf = 0; kf < 4; ++kf) m |= (uint32_t)(fo[kf] < 0 || fo[kf] > sl + kf) << (6 + kf);
                s_mask[stage_row(lt, q)] |= (uint16_t)m;
            }
        }
        __syncthreads();
        int4* f1 = reinterpret_cast<int4*>(sm_out) + n + 11 * t0;
        for (int i = lt; i < 11 * nb; i += kRgBlock) f1[i] = s_sm[i];
        int4* f0 = reinterpret_cast<int4*>(sm_out) + t0;
        for (int i = lt; i < nb; i += kRgBlock) f0[i] = s_sm[11 * kRgBlock + i];
    }
    // the masks and this block's share of the offsets' tile sums (packed
    // edges << 31 | faces, offsets_count_k's format): C0 rows lie in one
    // tile, the C1..C11 range in at most two
    const int64_t c1 = n + 11 * t0;
    const int64_t tile1 = c1 / kScanTile;
    long long s0 = 0, s1 = 0, s2 = 0;
    for (int i = lt; i < 11 * nb; i += kRgBlock) {
        const uint32_t m = s_mask[i];
        masks[c1 + i] = (uint16_t)m;
        const long long v = (long long)__popc(m & 63u) << 31 | __popc(m >> 6);
        if ((c1 + i) / kScanTile == tile1) s1 += v;
        else s2 += v;
    }
    if (lt < nb) {
        const uint32_t m = s_mask[11 * kRgBlock + lt];
        masks[t0 + lt] = (uint16_t)m;
        s0 = (long long)__popc(m & 63u) << 31 | __popc(m >> 6);
    }
    s0 = block_sum_ll<kRgBlock>(s0);
    __syncthreads();
    s1 = block_sum_ll<kRgBlock>(s1);
    __syncthreads();
    s2 = block_sum_ll<kRgBlock>(s2);
    if (lt == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(tile_sums + t0 / kScanTile), (unsigned long long)s0);
        atomicAdd(reinterpret_cast<unsigned long long*>(tile_sums + tile1), (unsigned long long)s1);
        if (s2) atomicAdd(reinterpret_cast<unsigned long long*>(tile_sums + tile1 + 1), (unsigned long long)s2);
    }
}

// Classification of a refined mesh's boundary lists, which refine_mesh built
// from the parent's (refine.cpp:88-94: row j = the corner triangle at n1,
// rows nL + 3 j + 0/1/2 = the corner triangles at n2, n3 and the middle
// one): parent entry j lies on the parent face entry_face[j], owned by the
// parent slot (t, k); its four sub-triangles are faces of t's children at
// fixed local faces (corner child a: the face without m_ad, d the vertex of t
// off the face; middle: child 8 + k, face 0).  One thread per parent entry
// writes the child entries' face ids and claims, as classify does.
__global__ void refined_classify_k(int64_t nd, int64_t nn, const int32_t* __restrict__ db,
                                   const int32_t* __restrict__ nb, const int32_t* __restrict__ p_entry_face,
                                   const int32_t* __restrict__ p_face_slots, const int32_t* __restrict__ p_tets,
                                   int64_t n, const int32_t* __restrict__ face_of_slot,
                                   const int32_t* __restrict__ face_slots, uint32_t* __restrict__ claim,
                                   int32_t* __restrict__ entry_face, uint8_t* __restrict__ face_class,
                                   unsigned long long* err) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nd + nn; j += (int64_t)gridDim.x * blockDim.x) {
        const bool dir = j < nd;
        const int64_t jl = dir ? j : j - nd, nl = dir ? nd : nn, base = dir ? 0 : 4 * nd;
        const int32_t* tri = (dir ? db : nb) + 3 * jl;
        const int32_t pf = __ldg(p_entry_face + j);
        const int64_t t = __ldg(p_face_slots + 2 * (int64_t)pf) >> 2;
        const int4 pt = ldtet(p_tets, t);
        const int a1 = idx_of(pt, __ldg(tri)), a2 = idx_of(pt, __ldg(tri + 1)), a3 = idx_of(pt, __ldg(tri + 2));
        const int d = 6 - a1 - a2 - a3;
        const int64_t rows[4] = {base + jl, base + nl + 3 * jl, base + nl + 3 * jl + 1, base + nl + 3 * jl + 2};
        const int64_t slots[4] = {4 * child(t, a1, n) + excl(rpos(a1, d)), 4 * child(t, a2, n) + excl(rpos(a2, d)),
                                  4 * child(t, a3, n) + excl(rpos(a3, d)), 4 * child(t, 8 + excl(d), n)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int32_t f = __ldg(face_of_slot + slots[q]);
            PHG_CHECK(f >= 0);
            entry_face[rows[q]] = f;
            atomicMin(claim + f, (uint32_t)rows[q]);
            if (face_class) face_class[f] = dir ? 1 : 2;
            if (__ldg(face_slots + 2 * (int64_t)f + 1) >= 0)
                report(err, PHG_ERR_CLASSIFY, (unsigned long long)rows[q] << 2 | 2);
        }
    }
}

}  // namespace

extern "C" int phfem_gpu_refined_groups(int64_t n, const int32_t* tets, const int32_t* edge_of_slot,
                                        const int32_t* edge_first, const int32_t* slot_mate, int64_t ned,
                                        int32_t* a0, int32_t* ef_out, int32_t* sm_out, uint16_t* masks,
                                        void* scratch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) return 0;
    long long* sums = static_cast<long long*>(scratch);
    cudaMemsetAsync(sums, 0, sizeof(long long) * (size_t)scan_tiles(12 * n), s);
    cudaMemsetAsync(a0, 0x7f, sizeof(int32_t) * 2 * (size_t)(ned > 0 ? ned : 1), s);
    a0_k<<<grid_for(n, 256), 256, 0, s>>>(n, tets, edge_of_slot, a0);
    refined_groups_k<<<grid_for(n, kRgBlock), kRgBlock, 0, s>>>(n, tets, edge_of_slot, edge_first, slot_mate, a0,
                                                                ef_out, sm_out, masks, sums);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_refined_classify(int64_t nd, int64_t nn, const int32_t* db, const int32_t* nb,
                                          const int32_t* p_entry_face, const int32_t* p_face_slots,
                                          const int32_t* p_tets, int64_t n, const int32_t* face_of_slot,
                                          const int32_t* face_slots, uint32_t* claim, int32_t* entry_face,
                                          uint8_t* face_class, unsigned long long* err, void* stream) {
    if (nd + nn == 0) return 0;
    refined_classify_k<<<grid_for(nd + nn, 128), 128, 0, (cudaStream_t)stream>>>(
        nd, nn, db, nb, p_entry_face, p_face_slots, p_tets, n, face_of_slot, face_slots, claim, entry_face,
        face_class, err);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}
