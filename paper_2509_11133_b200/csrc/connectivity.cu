// Edge and face connectivity on the device, bit-exact with the reference's
// num_edges / edge_pairs_to_elems / faces_up / full_face_table
// (connectivity.cpp:22-203).
//
// The reference numbers edges and faces by first occurrence over the
// element-major slot sequence.  Here that order is reproduced without a hash
// map or a global sort:
//   1. vertex star: CSR of (element, local vertex) incidences by vertex;
//   2. per vertex v, the edges (v,b) with b>v and the faces whose smallest
//      vertex is v are grouped in a small shared-memory hash table; the group
//      minimum is the first occurrence (edges) or the owner slot (faces: the
//      lower element, i.e. the slot faces_up emits) and the other face slot is
//      the neighbour across it;
//   3. ids = exclusive scan over elements of the first-occurrence / owner
//      counts (scan.cu), assigned in local slot order;
//   4. the remaining slots copy the id of their group's first slot.
// The directed edge-pair map (E2T) is never materialised; its only check
// (two elements claiming the same oriented face) is the orientation test in 2.
#include <climits>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "scan.cuh"

namespace {

using namespace phg;

// The star of v holds the incidences (t, lv) whose vertex v is not t's
// largest: every edge and face is grouped at its smallest vertex, and no
// candidate of an element's largest vertex lies above it, so that incidence
// would contribute nothing (3 incidences per element instead of 4).
// top = the local vertex with the largest id (the first of equal ones).
__device__ __forceinline__ int top_vertex(const int4& e) {
    int k = 0;
    int32_t m = e.x;
    if (e.y > m) { k = 1; m = e.y; }
    if (e.z > m) { k = 2; m = e.z; }
    if (e.w > m) k = 3;
    return k;
}

__device__ __forceinline__ bool repeats_id(const int4& e) {
    return e.x == e.y || e.x == e.z || e.x == e.w || e.y == e.z || e.y == e.w || e.z == e.w;
}

__global__ void star_count(const int32_t* __restrict__ tets, int64_t ne, int32_t* __restrict__ count,
                           int32_t* __restrict__ repeated) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        if (repeated && repeats_id(e)) *repeated = 1;
        const int top = top_vertex(e);
        if (top != 0) atomicAdd(count + e.x, 1);
        if (top != 1) atomicAdd(count + e.y, 1);
        if (top != 2) atomicAdd(count + e.z, 1);
        if (top != 3) atomicAdd(count + e.w, 1);
    }
}

// position = segment start + the count left after a 32-bit decrement
__global__ void star_fill(const int32_t* __restrict__ tets, int64_t ne, const int64_t* __restrict__ star_ptr,
                          int32_t* __restrict__ count, int32_t* __restrict__ star) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ne; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 e = ldtet(tets, t);
        const int top = top_vertex(e);
        const int32_t base = (int32_t)(4 * t);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k == top) continue;
            const int32_t v = tv(e, k);
            const int32_t c = atomicSub(count + v, 1);
            PHG_CHECK(c >= 1 && c <= star_ptr[v + 1] - star_ptr[v]);
            star[__ldg(star_ptr + v) + c - 1] = base + k;
        }
    }
}

// ------------------------------------------------------------ star groups

struct FaceTab {
    unsigned long long* key;
    int32_t* lo;
    int32_t* hi;
    int32_t* cnt;  // count << 2 | orientation bits
};

__device__ __forceinline__ unsigned hash32(uint32_t k) { return k * 0x9E3779B1u; }
// table slot from the HIGH bits of a multiplicative hash: the low bits of
// k * odd depend only on the low bits of k, and structured meshes have
// neighbour ids that agree there (v + 1, v + (n+1), v + (n+1)^2, ...)
__device__ __forceinline__ unsigned bucket(unsigned h, unsigned mask) { return __umulhi(h, mask + 1); }
__device__ __forceinline__ unsigned hash64(unsigned long long k) {
    k ^= k >> 29;
    k *= 0xBF58476D1CE4E5B9ull;
    return (unsigned)(k >> 32);
}

__device__ __forceinline__ int edge_slot_insert(int32_t* key, unsigned mask, int32_t b) {
    unsigned h = bucket(hash32((uint32_t)b), mask);
    for (unsigned probe = 0;; ++probe) {
        PHG_CHECK(probe <= mask);
        const int32_t old = atomicCAS(key + h, -1, b);
        if (old == -1 || old == b) return (int)h;
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ int edge_slot_find(const int32_t* key, unsigned mask, int32_t b) {
    unsigned h = bucket(hash32((uint32_t)b), mask);
    while (key[h] != b) h = (h + 1) & mask;
    return (int)h;
}
__device__ __forceinline__ int face_slot_insert(unsigned long long* key, unsigned mask, unsigned long long k) {
    unsigned h = bucket(hash64(k), mask);
    for (unsigned probe = 0;; ++probe) {
        PHG_CHECK(probe <= mask);
        const unsigned long long old = atomicCAS(key + h, ~0ull, k);
        if (old == ~0ull || old == k) return (int)h;
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ int face_slot_find(const unsigned long long* key, unsigned mask, unsigned long long k) {
    unsigned h = bucket(hash64(k), mask);
    while (key[h] != k) h = (h + 1) & mask;
    return (int)h;
}

// Face candidate of incidence (t, lv) and local face k containing lv:
// the two other vertices x (following v in the oriented cycle) and y.
__device__ __forceinline__ void face_other(const int4& tet, int k, int lv, int32_t& x, int32_t& y) {
    int j = 0;
    while (face_vert(k, j) != lv) ++j;
    x = tv(tet, face_vert(k, (j + 1) % 3));
    y = tv(tet, face_vert(k, (j + 2) % 3));
}
// the local face opposite local vertex lv
__device__ __forceinline__ int opposite_face(int lv) { return lv == 0 ? 3 : (lv == 3 ? 0 : lv); }

// Elements with a repeated node id (the reference accepts them up to the
// face table).  Their edge (v, v) is an edge like any other
// (connectivity.cpp:22-37 keys it (v, v)): it is grouped at v and listed
// from the incidence with the larger local index of the pair, which is in
// the star whenever the pair holds the element's largest id.  A face with a
// repeated id matches only itself in the E2T map, so faces_up never lists it
// (connectivity.cpp:78-84) and full_face_table fails on it (:140-143); so
// does a face whose two sides are faces of one element.  Such a slot gets
// the mate kDegenerate (not an owner, no face id) and is reported.
constexpr int32_t kDegenerate = -2;
__device__ __forceinline__ bool edge_here(int32_t b, int32_t v, int w, int lv) {
    return b > v || (b == v && w < lv);
}
__device__ __forceinline__ void mark_degenerate(int32_t* slot_mate, int32_t slot, unsigned long long* err) {
    slot_mate[slot] = kDegenerate;
    report(err, PHG_ERR_DEGEN_FACE, (unsigned long long)slot);
}

// One group (a warp, or a whole block for big stars) processes vertex v.
template <int NT, typename Sync>
__device__ void group_vertex(int32_t v, int64_t beg, int m, int rank, const int32_t* __restrict__ star,
                             const int32_t* __restrict__ tets, int32_t* __restrict__ edge_first,
                             int32_t* __restrict__ slot_mate, int32_t* ekey, int32_t* eval, FaceTab ft,
                             unsigned mask, unsigned cap, unsigned long long* err, Sync sync) {
    if (edge_first) {
        for (unsigned i = rank; i < cap; i += NT) {
            ekey[i] = -1;
            eval[i] = INT_MAX;
        }
        sync();
        for (int e = rank; e < m; e += NT) {
            const int32_t inc = star[beg + e];
            const int64_t t = inc >> 2;
            const int lv = inc & 3;
            const int4 tet = ldtet(tets, t);
            for (int w = 0; w < 4; ++w) {
                const int32_t b = tv(tet, w);
                if (w == lv || !edge_here(b, v, w, lv)) continue;
                const int h = edge_slot_insert(ekey, mask, b);
                atomicMin(eval + h, (int32_t)(6 * t + edge_index(lv, w)));
            }
        }
        sync();
        for (int e = rank; e < m; e += NT) {
            const int32_t inc = star[beg + e];
            const int64_t t = inc >> 2;
            const int lv = inc & 3;
            const int4 tet = ldtet(tets, t);
            for (int w = 0; w < 4; ++w) {
                const int32_t b = tv(tet, w);
                if (w == lv || !edge_here(b, v, w, lv)) continue;
                edge_first[6 * t + edge_index(lv, w)] = eval[edge_slot_find(ekey, mask, b)];
            }
        }
        sync();
    }
    if (slot_mate) {
        for (unsigned i = rank; i < cap; i += NT) {
            ft.key[i] = ~0ull;
            ft.lo[i] = INT_MAX;
            ft.hi[i] = -1;
            ft.cnt[i] = 0;
        }
        sync();
        for (int e = rank; e < m; e += NT) {
            const int32_t inc = star[beg + e];
            const int64_t t = inc >> 2;
            const int lv = inc & 3;
            const int4 tet = ldtet(tets, t);
            const int opp = opposite_face(lv);
            for (int k = 0; k < 4; ++k) {
                if (k == opp) continue;
                int32_t x, y;
                face_other(tet, k, lv, x, y);
                if (x == v || y == v || x == y) {
                    mark_degenerate(slot_mate, (int32_t)(4 * t + k), err);
                    continue;
                }
                if (x < v || y < v) continue;
                const unsigned long long key = x < y ? ((unsigned long long)x << 32 | (uint32_t)y)
                                                     : ((unsigned long long)y << 32 | (uint32_t)x);
                const int h = face_slot_insert(ft.key, mask, key);
                const int32_t slot = (int32_t)(4 * t + k);
                atomicMin(ft.lo + h, slot);
                atomicMax(ft.hi + h, slot);
                atomicAdd(ft.cnt + h, 4);
                atomicOr(ft.cnt + h, x < y ? 1 : 2);
            }
        }
        sync();
        for (int e = rank; e < m; e += NT) {
            const int32_t inc = star[beg + e];
            const int64_t t = inc >> 2;
            const int lv = inc & 3;
            const int4 tet = ldtet(tets, t);
            const int opp = opposite_face(lv);
            for (int k = 0; k < 4; ++k) {
                if (k == opp) continue;
                int32_t x, y;
                face_other(tet, k, lv, x, y);
                if (x <= v || y <= v || x == y) continue;
                const unsigned long long key = x < y ? ((unsigned long long)x << 32 | (uint32_t)y)
                                                     : ((unsigned long long)y << 32 | (uint32_t)x);
                const int h = face_slot_find(ft.key, mask, key);
                const int32_t slot = (int32_t)(4 * t + k);
                const int32_t c = ft.cnt[h];
                const int32_t lo = ft.lo[h], hi = ft.hi[h];
                const int count = c >> 2;
                if (count > 2 || (count == 2 && (c & 3) != 3)) {
                    // same orientation twice: "elements A and B claim the
                    // same oriented face" (connectivity.cpp:62-68)
                    const unsigned long long a = (unsigned long long)(lo >> 2), b = (unsigned long long)(hi >> 2);
                    report(err, PHG_ERR_DUP_ORIENT, a << 32 | b);
                }
                if (count == 2 && lo >> 2 == hi >> 2)
                    mark_degenerate(slot_mate, slot, err);  // both sides in one element
                else
                    slot_mate[slot] = count >= 2 ? (slot == lo ? hi : lo) : -1;
            }
        }
        sync();
    }
}

// ------------------------------------------- warp paths: stars of <= 64

constexpr int kFastWarps = 4;

// Local tables of the candidate generation in star_groups_warp, per local
// vertex lv of an incidence (faces [abc],[acd],[adb],[dcb]):
//   neighbour i (i < 3) = the i-th other local vertex in ascending order;
//   edge ids  0xb15663088 >> 9 lv, 3 bits per i: local edge (lv, neighbour i)
//             in the (0,1)(0,2)(0,3)(1,2)(1,3)(2,3) order;
//   faces     the face containing lv but not neighbour i is local face k,
//             0x9c72c9 >> 6 lv, 2 bits per i; its other vertices are
//             neighbours i+1, i+2 (mod 3), the first of them following lv
//             in the face's oriented cycle for even lv, the second for odd.

// E incidences per lane: E = 1 handles stars of <= 32 incidences (all Kuhn
// vertices), E = 2 those of <= 64 (refined meshes reach 36).  Vertices come
// from `list` (or 0..n-1) with n = *count (or nv); larger stars are appended
// to defer_list for the next pass.  No host round trip between passes.
//
// Work compaction: of the 6 candidates per incidence (3 edges, 3 faces) only
// those whose other vertices are all above v belong to v (about 60 of 144
// for a Kuhn vertex).  They are first appended to per-warp lists in shared
// memory (ballot + popc positions), and the hash inserts / read-backs /
// resets then run over the lists with all 32 lanes busy: 2-3 rounds per
// vertex instead of 6 mostly idle ones.
template <int E>
__global__ void __launch_bounds__(32 * kFastWarps)
    star_groups_warp(int64_t nv, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                     const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                     const int32_t* __restrict__ tets, int32_t* __restrict__ edge_first,
                     int32_t* __restrict__ slot_mate, int32_t* __restrict__ defer_list,
                     int32_t* __restrict__ defer_count, unsigned long long* err) {
    // E = 1: lists of 64 candidates (a Kuhn vertex has ~36 edge and ~24 face
    // candidates; a vertex with more is deferred to the E = 2 pass) and
    // tables of 64 (keys <= list entries, so an insert always finds a slot);
    // the small footprint keeps ~2x the warps resident.  E = 2: 3 candidates
    // per incidence always fit.
    constexpr int CAP = E == 1 ? 64 : 256;
    constexpr unsigned mask = CAP - 1;
    constexpr int LCAP = E == 1 ? 64 : 192;
    constexpr int R = LCAP / 32;  // rounds of 32 over a full list
    __shared__ int32_t s_ekey[kFastWarps][CAP], s_eval[kFastWarps][CAP];
    __shared__ unsigned long long s_fkey[kFastWarps][CAP];
    // face groups: count << 2 | orientation bits, and the (at most two,
    // else an error) slots in arrival order -- one atomic per candidate
    __shared__ int32_t s_fcnt[kFastWarps][CAP];
    __shared__ int2 s_fsl[kFastWarps][CAP];
    __shared__ int2 s_el[kFastWarps][LCAP];  // (b, edge slot)
    __shared__ int4 s_fl[kFastWarps][LCAP];  // (lo, hi, face slot, count increment)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int32_t* ekey = s_ekey[warp];
    int32_t* eval = s_eval[warp];
    unsigned long long* fkey = s_fkey[warp];
    int32_t* fcnt = s_fcnt[warp];
    int32_t* fsl = reinterpret_cast<int32_t*>(s_fsl[warp]);
    int2* el = s_el[warp];
    int4* fl = s_fl[warp];
    for (int i = lane; i < CAP; i += 32) {
        ekey[i] = -1;
        eval[i] = INT_MAX;
        fkey[i] = ~0ull;
        fcnt[i] = 0;
    }
    __syncwarp();
    const bool do_faces = slot_mate != nullptr;
    const int64_t n = count ? (int64_t)*count : nv;
    const int64_t nwarps = (int64_t)gridDim.x * kFastWarps;
    // Software pipeline over this warp's vertices: the dependent loads
    // star_ptr -> star -> tets of the next vertices are issued one and two
    // iterations ahead, so their latency overlaps the current vertex.
    // (no arithmetic on a loaded value in the stage that loads it: that
    // would wait for the load right there)
    struct Ptr {
        int32_t v;
        int64_t beg, end;
    };
    auto load_ptr = [&](int64_t i) -> Ptr {
        Ptr P{-1, 0, 0};
        if (i < n) {
            P.v = list ? list[i] : (int32_t)i;
            P.beg = star_ptr[P.v];
            P.end = star_ptr[P.v + 1];
        }
        return P;
    };
    auto load_inc = [&](const Ptr& P, int32_t (&inc)[E]) {
        const int64_t m = P.end - P.beg;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int e = lane + 32 * u;
            inc[u] = -1;
            if (e < m && m <= 32 * E) inc[u] = __ldg(star + P.beg + e);
        }
    };
    auto load_tet = [&](const int32_t (&inc)[E], int4 (&tt)[E]) {
#pragma unroll
        for (int u = 0; u < E; ++u) {
            tt[u] = make_int4(0, 0, 0, 0);
            if (inc[u] >= 0) tt[u] = ldtet(tets, inc[u] >> 2);
        }
    };
    const int64_t it0 = (int64_t)blockIdx.x * kFastWarps + warp;
    Ptr P1 = load_ptr(it0), P2 = load_ptr(it0 + nwarps);
    int32_t I1[E], I2[E];
    int4 T1[E];
    load_inc(P1, I1);
    load_tet(I1, T1);
    load_inc(P2, I2);
    Ptr P3 = load_ptr(it0 + 2 * nwarps);
    for (int64_t it = it0; it < n; it += nwarps) {
        // stages for it + nwarps (tets) and it + 2 nwarps (incidences, ptrs);
        // the pointer loads go first: issued after the 16-byte tet loads they
        // waited for those loads to release their address registers
        const Ptr P4 = load_ptr(it + 3 * nwarps);
        int32_t I3[E];
        load_inc(P3, I3);
        int4 T2[E];
        load_tet(I2, T2);
        const int32_t v = P1.v;
        const int m = (int)(P1.end - P1.beg);
        const bool deferred = m > 32 * E;
        if (deferred && lane == 0) defer_list[atomicAdd(defer_count, 1)] = v;
        if (!deferred) {
        // 1. candidates of v -> lists
        int ne_l = 0, nf_l = 0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int e = lane + 32 * u;
            const bool valid = e < m;
            const int32_t t = valid ? I1[u] >> 2 : 0;
            const int lv = valid ? I1[u] & 3 : 0;
            const int4 tet = T1[u];
            // the other three vertices in local order (= nbr_of(lv, i)), their
            // local edge ids and, for face i containing lv, its local face k
            // and the positions of x, y (the vertices following lv in the
            // oriented cycle) among them; 3-bit / 6-bit packed per lv
            const int32_t o[3] = {lv == 0 ? tet.y : tet.x, lv <= 1 ? tet.z : tet.y, lv <= 2 ? tet.w : tet.z};
            const unsigned etab = (unsigned)(0xb15663088ull >> (9 * lv));
            const unsigned ktab = (unsigned)(0x9c72c9u >> (6 * lv)) & 63u;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int32_t b = o[i];
                const bool q = valid && (b > v || (b == v && i < lv));
                const unsigned bal = __ballot_sync(0xffffffffu, q);
                const int pe = ne_l + __popc(bal & lt);
                if (q && pe < LCAP) el[pe] = make_int2(b, 6 * t + (int)((etab >> (3 * i)) & 7u));
                ne_l += __popc(bal);
                if (do_faces) {
                    // the face of lv without neighbour i: the other two
                    // neighbours a, b; the vertex following lv in its
                    // oriented cycle is a for even lv, b for odd lv
                    const int32_t a = o[(i + 1) % 3], b = o[(i + 2) % 3];
                    const int32_t lo = min(a, b), hi = max(a, b);
                    if (valid && (lo == v || a == b)) mark_degenerate(slot_mate, 4 * t + (int)((ktab >> (2 * i)) & 3u), err);
                    const bool qf = valid && lo > v && a != b;
                    const unsigned balf = __ballot_sync(0xffffffffu, qf);
                    // count in bits 2+, orientation (x < y: 1, else 2) below:
                    // exactly one slot of each orientation sums to 11
                    const bool xy = (lv & 1) ? b < a : a < b;
                    const int pf = nf_l + __popc(balf & lt);
                    if (qf && pf < LCAP) fl[pf] = make_int4(lo, hi, 4 * t + (int)((ktab >> (2 * i)) & 3u), xy ? 5 : 6);
                    nf_l += __popc(balf);
                }
            }
        }
        __syncwarp();
        const int nl_max = max(ne_l, nf_l);
        if (ne_l > LCAP || nf_l > LCAP) {  // too many candidates for this pass
            if (lane == 0) defer_list[atomicAdd(defer_count, 1)] = v;
        } else {
        // 2. inserts over the lists, all lanes busy
        int eh[R], fh[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (E > 1 && 32 * r >= nl_max) break;  // warp-uniform: only the rounds in use
            eh[r] = fh[r] = -1;
            const int j = lane + 32 * r;
            if (j < ne_l) {
                const int2 c = el[j];
                unsigned h = bucket(hash32((uint32_t)c.x), mask);
                for (unsigned probe = 0;; ++probe) {
                    PHG_CHECK(probe <= mask);
                    const int32_t old = atomicCAS(ekey + h, -1, c.x);
                    if (old == -1 || old == c.x) break;
                    h = (h + 1) & mask;
                }
                eh[r] = (int)h;
                atomicMin(eval + h, c.y);
            }
            if (j < nf_l) {
                const int4 c = fl[j];
                const unsigned long long key = (unsigned long long)c.x << 32 | (uint32_t)c.y;
                unsigned h = bucket(hash64(key), mask);
                for (unsigned probe = 0;; ++probe) {
                    PHG_CHECK(probe <= mask);
                    const unsigned long long old = atomicCAS(fkey + h, ~0ull, key);
                    if (old == ~0ull || old == key) break;
                    h = (h + 1) & mask;
                }
                fh[r] = (int)h;
                const int pos = atomicAdd(fcnt + h, c.w) >> 2;
                if (pos < 2) fsl[2 * h + pos] = c.z;
            }
        }
        __syncwarp();
        // 3. read-back: every listed slot gets its group's result
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (E > 1 && 32 * r >= nl_max) break;  // warp-uniform: only the rounds in use
            const int j = lane + 32 * r;
            if (eh[r] >= 0) {
                PHG_CHECK(eval[eh[r]] <= el[j].y && eval[eh[r]] >= 0);  // the first occurrence is not later
                edge_first[el[j].y] = eval[eh[r]];
            }
            if (fh[r] >= 0) {
                const int h = fh[r];
                const int32_t slot = fl[j].z;
                const int32_t c = fcnt[h];
                const int cnt = c >> 2;
                const int2 pr = s_fsl[warp][h];
                const int32_t lo = min(pr.x, pr.y), hi = max(pr.x, pr.y);
                if (cnt > 2 || (cnt == 2 && c != 11)) {
                    // same orientation twice: "elements A and B claim the
                    // same oriented face" (connectivity.cpp:62-68)
                    const unsigned long long a = (unsigned long long)(lo >> 2), b = (unsigned long long)(hi >> 2);
                    report(err, PHG_ERR_DUP_ORIENT, a << 32 | b);
                }
                if (cnt == 2 && pr.x >> 2 == pr.y >> 2)
                    mark_degenerate(slot_mate, slot, err);  // both sides in one element
                else
                    slot_mate[slot] = cnt >= 2 ? (slot == pr.x ? pr.y : pr.x) : -1;
            }
        }
        __syncwarp();
        // 4. reset the touched table entries
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (E > 1 && 32 * r >= nl_max) break;  // warp-uniform: only the rounds in use
            if (eh[r] >= 0) {
                ekey[eh[r]] = -1;
                eval[eh[r]] = INT_MAX;
            }
            if (fh[r] >= 0) {
                fkey[fh[r]] = ~0ull;
                fcnt[fh[r]] = 0;
            }
        }
        __syncwarp();
        }
        }
        P1 = P2;
        P2 = P3;
        P3 = P4;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            I1[u] = I2[u];
            I2[u] = I3[u];
            T1[u] = T2[u];
        }
    }
}

// The first pass without hash tables: stars of <= 32 incidences, one per
// lane.  A vertex's edge candidates go to two lists by one hash bit of the
// other vertex b (so equal keys share a list) and its face candidates to a
// third; with every list <= 32 entries, one warp-wide match per list groups
// equal keys (__match_any_sync), the group minimum is a warp reduction
// (__reduce_min_sync) and a face's mate the other lane of its pair
// (__shfl_sync) -- no shared-memory table to probe, fill or reset.  A vertex
// with a longer list is deferred to the hashing pass (star_groups_warp<2>).
constexpr int kMatchWarps = 8;
#ifndef PHG_MATCH_MINB
#define PHG_MATCH_MINB 1
#endif
__global__ void __launch_bounds__(32 * kMatchWarps, PHG_MATCH_MINB)
    star_groups_match(int64_t nv, const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                      const int32_t* __restrict__ tets, int32_t* __restrict__ edge_first,
                      int32_t* __restrict__ slot_mate, int32_t* __restrict__ defer_list,
                      int32_t* __restrict__ defer_count, const int32_t* __restrict__ repeated,
                      unsigned long long* err) {
    __shared__ int2 s_e[kMatchWarps][2][32];  // (b, edge slot) by hash bit of b
    // an element repeats a node id somewhere (star_count): check every star
    const bool any_rep = repeated == nullptr || *repeated != 0;
    __shared__ int4 s_f[kMatchWarps][32];     // (lo, hi, face slot, orientation)
    __shared__ int32_t s_min[kMatchWarps][32];  // edge group minimum at the group's first lane
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* gmin = s_min[warp];
    const unsigned lt = (1u << lane) - 1u;
    int2* e0 = s_e[warp][0];
    int2* e1 = s_e[warp][1];
    int4* fl = s_f[warp];
    const bool do_faces = slot_mate != nullptr;
    const int64_t nwarps = (int64_t)gridDim.x * kMatchWarps;
    // software pipeline of the dependent loads star_ptr -> star -> tets, as
    // in star_groups_warp
    struct Ptr {
        int32_t v;
        int64_t beg, end;
    };
    auto load_ptr = [&](int64_t i) -> Ptr {
        Ptr P{-1, 0, 0};
        if (i < nv) {
            P.v = (int32_t)i;
            P.beg = star_ptr[i];
            P.end = star_ptr[i + 1];
        }
        return P;
    };
    auto load_inc = [&](const Ptr& P) -> int32_t {
        const int64_t m = P.end - P.beg;
        return lane < m && m <= 32 ? __ldg(star + P.beg + lane) : -1;
    };
    auto load_tet = [&](int32_t inc) -> int4 { return inc >= 0 ? ldtet(tets, inc >> 2) : make_int4(0, 0, 0, 0); };
    const int64_t it0 = (int64_t)blockIdx.x * kMatchWarps + warp;
    Ptr P1 = load_ptr(it0), P2 = load_ptr(it0 + nwarps);
    int32_t I1 = load_inc(P1);
    int4 T1 = load_tet(I1);
    int32_t I2 = load_inc(P2);
    Ptr P3 = load_ptr(it0 + 2 * nwarps);
    for (int64_t it = it0; it < nv; it += nwarps) {
        const Ptr P4 = load_ptr(it + 3 * nwarps);
        const int32_t I3 = load_inc(P3);
        const int4 T2 = load_tet(I2);
        const int32_t v = P1.v;
        const int m = (int)(P1.end - P1.beg);
        // a star with an element that repeats a node id goes to the hashing
        // pass, which handles edges (a, a) and faces without a mate
        bool defer = m > 32;
        if (any_rep) defer = defer || __any_sync(0xffffffffu, lane < m && repeats_id(T1));
        if (!defer) {
            const bool valid = lane < m;
            const int32_t t = valid ? I1 >> 2 : 0;
            const int lv = valid ? I1 & 3 : 0;
            const int4 tet = T1;
            const int32_t o[3] = {lv == 0 ? tet.y : tet.x, lv <= 1 ? tet.z : tet.y, lv <= 2 ? tet.w : tet.z};
            const unsigned etab = (unsigned)(0xb15663088ull >> (9 * lv));
            const unsigned ktab = (unsigned)(0x9c72c9u >> (6 * lv)) & 63u;
            int n0 = 0, n1 = 0, nf = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int32_t b = o[i];
                const bool q = valid && b > v;
                const bool hb = (hash32((uint32_t)b) >> 31) != 0;
                const unsigned bal0 = __ballot_sync(0xffffffffu, q && !hb), bal1 = __ballot_sync(0xffffffffu, q && hb);
                const int pe = (hb ? n1 + __popc(bal1 & lt) : n0 + __popc(bal0 & lt));
                if (q && pe < 32) (hb ? e1 : e0)[pe] = make_int2(b, 6 * t + (int)((etab >> (3 * i)) & 7u));
                n0 += __popc(bal0);
                n1 += __popc(bal1);
                if (do_faces) {
                    const int32_t a = o[(i + 1) % 3], c = o[(i + 2) % 3];
                    const int32_t lo = min(a, c), hi = max(a, c);
                    const bool qf = valid && lo > v;
                    const unsigned balf = __ballot_sync(0xffffffffu, qf);
                    const bool xy = (lv & 1) ? c < a : a < c;
                    const int pf = nf + __popc(balf & lt);
                    if (qf && pf < 32) fl[pf] = make_int4(lo, hi, 4 * t + (int)((ktab >> (2 * i)) & 3u), xy ? 1 : 0);
                    nf += __popc(balf);
                }
            }
            __syncwarp();
            defer = n0 > 32 || n1 > 32 || nf > 32;
            if (!defer) {
                // one match per list over its own lanes (match_any costs
                // grow with the distinct keys among the participating lanes:
                // padding lanes with unique keys made it 1.7x slower)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = h ? n1 : n0;
                    if (lane < n) {
                        const int2 c = (h ? e1 : e0)[lane];
                        const unsigned mk = n == 32 ? 0xffffffffu : (1u << n) - 1u;
                        const unsigned g = __match_any_sync(mk, c.x);
                        // the group minimum through a shared-memory min at the
                        // group's first lane (__reduce_min_sync over the
                        // warp's distinct group masks ran as a loop, a
                        // quarter of the kernel)
                        const int lead = __ffs(g) - 1;
                        gmin[lane] = INT_MAX;
                        __syncwarp(mk);
                        atomicMin(gmin + lead, c.y);
                        __syncwarp(mk);
                        const int32_t first = gmin[lead];
                        PHG_CHECK(first <= c.y && first >= 0);
                        edge_first[c.y] = first;
                    }
                    __syncwarp();
                }
                if (lane < nf) {
                    const int4 c = fl[lane];
                    const unsigned mk = nf == 32 ? 0xffffffffu : (1u << nf) - 1u;
                    const unsigned long long key = (unsigned long long)c.x << 32 | (uint32_t)c.y;
                    const unsigned g = __match_any_sync(mk, key);
                    const unsigned others = g & ~(1u << lane);
                    const int src = others ? __ffs(others) - 1 : lane;
                    const int32_t oslot = __shfl_sync(mk, c.z, src);
                    const int32_t ow = __shfl_sync(mk, c.w, src);
                    const int cnt = __popc(g);
                    if (cnt > 2 || (cnt == 2 && ow == c.w)) {
                        // same orientation twice: "elements A and B claim the
                        // same oriented face" (connectivity.cpp:62-68; the
                        // host names the reference's pair from the E2T)
                        const unsigned long long a = (unsigned long long)(min(c.z, oslot) >> 2),
                                                 b = (unsigned long long)(max(c.z, oslot) >> 2);
                        report(err, PHG_ERR_DUP_ORIENT, a << 32 | b);
                    }
                    slot_mate[c.z] = cnt >= 2 ? oslot : -1;
                }
            }
            __syncwarp();
        }
        if (defer && lane == 0) defer_list[atomicAdd(defer_count, 1)] = v;
        P1 = P2;
        P2 = P3;
        P3 = P4;
        I1 = I2;
        I2 = I3;
        T1 = T2;
    }
}

struct WarpSync {
    __device__ void operator()() const { __syncwarp(); }
};
struct BlockSync {
    __device__ void operator()() const { __syncthreads(); }
};

// stars of more than 64 incidences: one block per vertex, tables in dynamic
// shared memory of capacity `cap` (> 3 m), vertices from list[0..*count)
__global__ void __launch_bounds__(256)
    star_groups_big(const int32_t* __restrict__ big_list, const int32_t* __restrict__ big_count,
                    const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                    const int32_t* __restrict__ tets, int32_t* __restrict__ edge_first,
                    int32_t* __restrict__ slot_mate, unsigned cap, int32_t* __restrict__ huge_list,
                    int32_t* __restrict__ huge_count, unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int32_t n = *big_count;
    for (int32_t it = blockIdx.x; it < n; it += gridDim.x) {
        const int32_t v = big_list[it];
        const int64_t beg = star_ptr[v];
        const int m = (int)(star_ptr[v + 1] - beg);
        if ((unsigned)(3 * m) >= cap) {
            // too large for shared memory: placeholders that keep the
            // numbering kernels in bounds (own slot as first occurrence, no
            // mate), and the vertex goes to the global-memory pass the host
            // runs when PHG_ERR_VALENCE is set (star_groups_global)
            for (int e = threadIdx.x; e < m; e += blockDim.x) {
                const int32_t inc = star[beg + e];
                const int64_t t = inc >> 2;
                const int lv = inc & 3;
                const int4 tet = ldtet(tets, t);
                for (int w = 0; w < 4; ++w) {
                    if (w == lv || tv(tet, w) <= v) continue;
                    if (edge_first) edge_first[6 * t + edge_index(lv, w)] = (int32_t)(6 * t + edge_index(lv, w));
                }
                if (!slot_mate) continue;
                const int opp = opposite_face(lv);
                for (int k = 0; k < 4; ++k) {
                    if (k == opp) continue;
                    int32_t x, y;
                    face_other(tet, k, lv, x, y);
                    if (x > v && y > v) slot_mate[4 * t + k] = -1;
                }
            }
            if (threadIdx.x == 0) {
                report(err, PHG_ERR_VALENCE, (unsigned long long)v);
                huge_list[atomicAdd(huge_count, 1)] = v;
            }
            __syncthreads();
            continue;
        }
        int32_t* ekey = reinterpret_cast<int32_t*>(dsm);
        int32_t* eval = ekey + cap;
        FaceTab ft;
        ft.key = reinterpret_cast<unsigned long long*>(dsm);
        ft.lo = reinterpret_cast<int32_t*>(dsm + (size_t)cap * 8);
        ft.hi = ft.lo + cap;
        ft.cnt = ft.hi + cap;
        group_vertex<256>(v, beg, m, threadIdx.x, star, tets, edge_first, slot_mate, ekey, eval, ft, cap - 1, cap,
                          err, BlockSync{});
        __syncthreads();
    }
}

// Stars too large for the shared-memory tables (more than ~2730
// incidences; the reference has no valence limit): one block, hash tables of
// capacity `cap` (a power of two > 3 m) in global scratch memory.  Run by the
// host only when star_groups_big listed such a vertex.
__global__ void __launch_bounds__(256)
    star_groups_global(int32_t v, const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                       const int32_t* __restrict__ tets, int32_t* __restrict__ edge_first,
                       int32_t* __restrict__ slot_mate, unsigned char* __restrict__ scratch, unsigned cap,
                       unsigned long long* err) {
    const int64_t beg = star_ptr[v];
    const int m = (int)(star_ptr[v + 1] - beg);
    int32_t* ekey = reinterpret_cast<int32_t*>(scratch);
    int32_t* eval = ekey + cap;
    FaceTab ft;
    ft.key = reinterpret_cast<unsigned long long*>(scratch);
    ft.lo = reinterpret_cast<int32_t*>(scratch + (size_t)cap * 8);
    ft.hi = ft.lo + cap;
    ft.cnt = ft.hi + cap;
    group_vertex<256>(v, beg, m, threadIdx.x, star, tets, edge_first, slot_mate, ekey, eval, ft, cap - 1, cap, err,
                      BlockSync{});
}

// -------------------------------------------------------------- numbering

__device__ __forceinline__ bool face_owner(int32_t s, int32_t mate) { return mate == -1 || mate > s; }

// Per-element masks of first-occurrence edge slots (bits 0-5) and owned face
// slots (bits 6-9) and the exclusive offsets edge_off / face_off [ne + 1] of
// their popcounts, reduce-then-scan (scan.cuh):
//   offsets_count_k  masks + tile sums, both counts packed in one int64
//                    (edges << 31 | faces; 6 nE < 2^31 is enforced at
//                    upload, so no carry)
//   scan_sums        the tile sums
//   offsets_scan_k   16 elements per thread from 32 B of masks; writes
//                    edge_off[t] = offset | edge mask << 32 and
//                    face_off[t] = offset | face mask << 32
// number() ranks non-first slots in their group's first element from that
// one 8-byte word (offset + mask in a single gather).
__device__ __forceinline__ uint32_t elem_mask(int64_t t, const int32_t* e6, const int4* mate) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) m |= (uint32_t)(e6[k] == (int32_t)(6 * t + k)) << k;
    if (mate) {
        const int4 q = *mate;
        const int32_t sl = (int32_t)(4 * t);
        m |= (uint32_t)face_owner(sl, q.x) << 6 | (uint32_t)face_owner(sl + 1, q.y) << 7 |
             (uint32_t)face_owner(sl + 2, q.z) << 8 | (uint32_t)face_owner(sl + 3, q.w) << 9;
    }
    return m;
}

__global__ void __launch_bounds__(kScanThreads)
    offsets_count_k(int64_t ne, const int32_t* __restrict__ edge_first, const int32_t* __restrict__ slot_mate,
                    uint16_t* __restrict__ masks, long long* __restrict__ sums) {
    // striped over the tile (element base + i * kScanThreads + thread): the
    // 24 B of edge_first and 16 B of slot_mate per element load coalesced,
    // and the tile sum does not depend on the order
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    long long se = 0, sf = 0;
#pragma unroll 4
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t t = base + i * kScanThreads + threadIdx.x;
        if (t >= ne) break;
        const int2* ef2 = reinterpret_cast<const int2*>(edge_first) + 3 * t;
        const int2 a01 = __ldg(ef2), a23 = __ldg(ef2 + 1), a45 = __ldg(ef2 + 2);
        const int32_t e[6] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y};
        int4 q;
        if (slot_mate) q = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        const uint32_t m = elem_mask(t, e, slot_mate ? &q : nullptr);
        masks[t] = (uint16_t)m;
        se += __popc(m & 63u);
        sf += __popc(m >> 6);
    }
    const long long s = block_sum_ll<kScanThreads>(se << 31 | sf);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kScanThreads)
    offsets_scan_k(int64_t ne, const uint16_t* __restrict__ masks, const long long* __restrict__ tile_off,
                   int64_t* __restrict__ edge_off, int64_t* __restrict__ face_off) {
    __shared__ long long stage[kScanTile + kScanTile / 16];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int64_t first = base + (int64_t)threadIdx.x * kScanItems;
    uint16_t mk[kScanItems];
    if (first + kScanItems <= ne) {
        const uint4* p = reinterpret_cast<const uint4*>(masks + first);
        const uint4 q0 = __ldg(p), q1 = __ldg(p + 1);
        const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) mk[i] = (uint16_t)(w[i / 2] >> (16 * (i % 2)));
    } else {
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) mk[i] = first + i < ne ? masks[first + i] : (uint16_t)0;
    }
    uint8_t ce[kScanItems], cf[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        ce[i] = (uint8_t)__popc(mk[i] & 63u);
        cf[i] = (uint8_t)__popc((uint32_t)mk[i] >> 6);
    }
    long long se = 0, sf = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        se += ce[i];
        sf += cf[i];
    }
    const long long packed = block_excl_scan_ll<kScanThreads>(se << 31 | sf) + tile_off[blockIdx.x];
    long long run = packed >> 31;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        stage[scan_pad(threadIdx.x * kScanItems + i)] = run | (long long)(mk[i] & 63u) << 32;
        run += ce[i];
    }
    __syncthreads();
    store_tile_i64(stage, edge_off, base, ne);
    if (!face_off) return;
    __syncthreads();
    run = packed & 0x7fffffffll;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        stage[scan_pad(threadIdx.x * kScanItems + i)] = run | (long long)((uint32_t)mk[i] >> 6) << 32;
        run += cf[i];
    }
    __syncthreads();
    store_tile_i64(stage, face_off, base, ne);
}

__global__ void __launch_bounds__(256) face_rows_identity_k(int64_t nf, int32_t* __restrict__ mrow,
                                                             int32_t* __restrict__ row_face) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        mrow[f] = (int32_t)f;
        row_face[f] = (int32_t)f;
    }
}

// grand totals edge_off[ne], face_off[ne] from the packed total
__global__ void offsets_total_k(const int64_t* __restrict__ packed_total, int64_t ne, int64_t* __restrict__ edge_off,
                                int64_t* __restrict__ face_off) {
    const long long p = *packed_total;
    edge_off[ne] = p >> 31;
    if (face_off) face_off[ne] = p & 0x7fffffffll;
}

// Ids of all slots of one element (one thread per element, blocks in element
// order).  Own first-occurrence edge slots and owned face slots get
// E_t + rank / F_t + rank; the others find their group's first element g < t
// through edge_first / slot_mate and rank there, so every id is written once,
// in full 16-24 byte rows (no second pass over the slots).
__global__ void __launch_bounds__(256)
    number(int64_t ne, const int32_t* __restrict__ tets, const double* __restrict__ coords,
           const int32_t* __restrict__ edge_first, const int64_t* __restrict__ edge_off,
           int32_t* __restrict__ edge_of_slot, int32_t* __restrict__ edge_nodes,
           const int32_t* __restrict__ slot_mate, const int64_t* __restrict__ face_off,
           int32_t* __restrict__ face_of_slot, int8_t* __restrict__ sigma, int32_t* __restrict__ faces,
           int32_t* __restrict__ face_slots, double* __restrict__ face_area, unsigned long long* err) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ne) return;
    const int4 tet = ldtet(tets, t);
    if (edge_first) {
        const int2* ef2 = reinterpret_cast<const int2*>(edge_first) + 3 * t;
        const int2 a01 = __ldg(ef2), a23 = __ldg(ef2 + 1), a45 = __ldg(ef2 + 2);
        const int32_t ef[6] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y};
        int64_t id = (uint32_t)edge_off[t];
        int32_t ids[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int64_t s = 6 * t + k;
            const int32_t f = ef[k];
            if (f == (int32_t)s) {
                ids[k] = (int32_t)id;
                int32_t a = tv(tet, k < 3 ? 0 : (k < 5 ? 1 : 2));
                int32_t b = tv(tet, k < 3 ? k + 1 : (k < 5 ? k - 1 : 3));
                if (a > b) { const int32_t tmp = a; a = b; b = tmp; }
                reinterpret_cast<int2*>(edge_nodes)[id] = make_int2(a, b);
                ++id;
            } else {
                // rank of slot f among the first-occurrence slots of its element
                PHG_CHECK(f >= 0 && f < (int32_t)s);
                const int64_t g = f / 6;
                const uint32_t below = (1u << (f - 6 * g)) - 1u;
                const unsigned long long w = (unsigned long long)__ldg(edge_off + g);
                ids[k] = (int32_t)((uint32_t)w + __popc((uint32_t)(w >> 32) & below));
            }
        }
        int2* eo = reinterpret_cast<int2*>(edge_of_slot) + 3 * t;
        eo[0] = make_int2(ids[0], ids[1]);
        eo[1] = make_int2(ids[2], ids[3]);
        eo[2] = make_int2(ids[4], ids[5]);
    }
    if (slot_mate) {
        // the element's four nodes once (owned faces' areas), not per face
        const V3 pn[4] = {ldnode(coords, tet.x), ldnode(coords, tet.y), ldnode(coords, tet.z), ldnode(coords, tet.w)};
        int64_t id = (uint32_t)face_off[t];
        const int4 m = __ldg(reinterpret_cast<const int4*>(slot_mate) + t);
        int32_t fid[4];
        int sg[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t s = (int32_t)(4 * t + k);
            const int32_t mate = tv(m, k);
            if (face_owner(s, mate)) {
                fid[k] = (int32_t)id;
                sg[k] = 1;
                const int32_t f0 = tv(tet, face_vert(k, 0)), f1 = tv(tet, face_vert(k, 1)), f2 = tv(tet, face_vert(k, 2));
                faces[3 * id] = f0;
                faces[3 * id + 1] = f1;
                faces[3 * id + 2] = f2;
                reinterpret_cast<int2*>(face_slots)[id] = make_int2(s, mate);
                // face_area_and_normal (mesh.cpp:76-84): area = 0.5*|(z-x)x(y-x)|
                const V3 p0 = pn[face_vert(k, 0)], p1 = pn[face_vert(k, 1)], p2 = pn[face_vert(k, 2)];
                const V3 n = vcross(vsub(p2, p0), vsub(p1, p0));
                const double len = __dsqrt_rn(vdot(n, n));
                if (len == 0.0) report(err, PHG_ERR_FACE, (unsigned long long)id << 2 | 0);
                face_area[id] = mul(0.5, len);
                ++id;
            } else if (mate == kDegenerate) {
                // a face with a repeated node id: no face (the pass reports it)
                fid[k] = -1;
                sg[k] = 0;
            } else {
                // the owner is slot `mate` of an earlier element g: its rank
                // among g's owned slots (sigma = -1: opposite orientation,
                // checked in star_groups)
                PHG_CHECK(mate >= 0 && mate < s);
                const int64_t g = mate >> 2;
                const uint32_t below = (1u << (mate & 3)) - 1u;
                const unsigned long long w = (unsigned long long)__ldg(face_off + g);
                fid[k] = (int32_t)((uint32_t)w + __popc((uint32_t)(w >> 32) & below));
                sg[k] = -1;
            }
        }
        reinterpret_cast<int4*>(face_of_slot)[t] = make_int4(fid[0], fid[1], fid[2], fid[3]);
        reinterpret_cast<char4*>(sigma)[t] = make_char4((signed char)sg[0], (signed char)sg[1], (signed char)sg[2],
                                                        (signed char)sg[3]);
    }
}

// ---------------------------------------------------------- classification

// Face id of the element face with vertex set {a,b,c}, searched through the
// star of its smallest vertex, or -1.
__device__ int32_t find_face(int32_t a, int32_t b, int32_t c, const int64_t* __restrict__ star_ptr,
                             const int32_t* __restrict__ star, const int32_t* __restrict__ tets,
                             const int32_t* __restrict__ face_of_slot) {
    int32_t lo = a, mid = b, hi = c;
    if (lo > mid) { const int32_t t = lo; lo = mid; mid = t; }
    if (mid > hi) { const int32_t t = mid; mid = hi; hi = t; }
    if (lo > mid) { const int32_t t = lo; lo = mid; mid = t; }
    if (lo == mid || mid == hi) return -1;
    const int64_t beg = star_ptr[lo], end = star_ptr[lo + 1];
    for (int64_t i = beg; i < end; ++i) {
        const int32_t inc = star[i];
        const int64_t t = inc >> 2;
        const int4 tet = ldtet(tets, t);
        int pos_mid = -1, pos_hi = -1;
        for (int w = 0; w < 4; ++w) {
            if (tv(tet, w) == mid) pos_mid = w;
            if (tv(tet, w) == hi) pos_hi = w;
        }
        if (pos_mid < 0 || pos_hi < 0) continue;
        const int lv = inc & 3;
        const int opp = 6 - lv - pos_mid - pos_hi;  // the fourth local vertex
        return face_of_slot[4 * t + opposite_face(opp)];
    }
    return -1;
}

__global__ void classify(int64_t nd, const int32_t* __restrict__ db, int64_t nn, const int32_t* __restrict__ nb,
                         const int64_t* __restrict__ star_ptr, const int32_t* __restrict__ star,
                         const int32_t* __restrict__ tets, const int32_t* __restrict__ face_of_slot,
                         const int32_t* __restrict__ face_slots, uint32_t* __restrict__ claim,
                         int32_t* __restrict__ entry_face, unsigned long long* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd + nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* tri = i < nd ? db + 3 * i : nb + 3 * (i - nd);
        const int32_t f = find_face(tri[0], tri[1], tri[2], star_ptr, star, tets, face_of_slot);
        entry_face[i] = f;
        if (f < 0) {
            report(err, PHG_ERR_CLASSIFY, (unsigned long long)i << 2 | 0);
            continue;
        }
        atomicMin(claim + f, (uint32_t)i);
        if (face_slots[2 * (int64_t)f + 1] >= 0) report(err, PHG_ERR_CLASSIFY, (unsigned long long)i << 2 | 2);
    }
}

__global__ void classify_check(int64_t nd, int64_t nn, const int32_t* __restrict__ entry_face,
                               const uint32_t* __restrict__ claim, unsigned long long* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd + nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = entry_face[i];
        if (f >= 0 && claim[f] != (uint32_t)i) report(err, PHG_ERR_CLASSIFY, (unsigned long long)i << 2 | 1);
    }
}

// Face classes and multiplier rows, reduce-then-scan over tiles of
// kScanTile faces (scan.cuh), thread i of a tile owning faces
// [16 i, 16 i + 16):
//   face_class_k  class (0 interior, 1 Dirichlet, 2 Neumann) per face, the
//                 tile's count of row faces (non-Neumann) and the class counts
//   scan_sums     the tile counts
//   face_rows_k   rows = rank among the row faces, and the inverse map
__device__ __forceinline__ uint8_t face_class_of(int64_t f, uint32_t cl, int32_t mate, int64_t nd,
                                                 unsigned long long* err) {
    uint8_t cls = 0;
    if (cl != 0xffffffffu) cls = (int64_t)cl < nd ? 1 : 2;
    else if (mate < 0) report(err, PHG_ERR_FACE, (unsigned long long)f << 2 | 1);
    return cls;
}

__global__ void __launch_bounds__(kScanThreads)
    face_class_k(int64_t nf, int64_t nd, const uint32_t* __restrict__ claim, const int32_t* __restrict__ face_slots,
                 uint8_t* __restrict__ face_class, long long* __restrict__ sums, unsigned long long* __restrict__ counts,
                 unsigned long long* err) {
    // striped groups of four faces: 16 B loads / 4 B stores, coalesced
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    int c[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < kScanItems / 4; ++i) {
        const int64_t f = base + 4 * (i * kScanThreads + (int64_t)threadIdx.x);
        if (f + 4 <= nf) {
            const uint4 cl = __ldg(reinterpret_cast<const uint4*>(claim + f));
            const int4 s01 = __ldg(reinterpret_cast<const int4*>(face_slots + 2 * f));
            const int4 s23 = __ldg(reinterpret_cast<const int4*>(face_slots + 2 * f) + 1);
            const uint8_t k0 = face_class_of(f, cl.x, s01.y, nd, err), k1 = face_class_of(f + 1, cl.y, s01.w, nd, err),
                          k2 = face_class_of(f + 2, cl.z, s23.y, nd, err),
                          k3 = face_class_of(f + 3, cl.w, s23.w, nd, err);
            reinterpret_cast<uchar4*>(face_class + f)[0] = make_uchar4(k0, k1, k2, k3);
            ++c[k0];
            ++c[k1];
            ++c[k2];
            ++c[k3];
        } else {
            for (int j = 0; j < 4 && f + j < nf; ++j) {
                const uint8_t k = face_class_of(f + j, claim[f + j], face_slots[2 * (f + j) + 1], nd, err);
                face_class[f + j] = k;
                ++c[k];
            }
        }
    }
    // rows: interior + Dirichlet faces; one atomic triple per block
    const long long rows = block_sum_ll<kScanThreads>(c[0] + c[1]);
    if (threadIdx.x == 0) sums[blockIdx.x] = rows;
    __shared__ int sc[3];
    if (threadIdx.x < 3) sc[threadIdx.x] = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) {
        c[0] += __shfl_xor_sync(0xffffffffu, c[0], o);
        c[1] += __shfl_xor_sync(0xffffffffu, c[1], o);
        c[2] += __shfl_xor_sync(0xffffffffu, c[2], o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sc + 0, c[0]);
        atomicAdd(sc + 1, c[1]);
        atomicAdd(sc + 2, c[2]);
    }
    __syncthreads();
    if (threadIdx.x < 3) atomicAdd(counts + threadIdx.x, (unsigned long long)sc[threadIdx.x]);
}

// the tile row counts alone, from classes already written (refined meshes)
__global__ void __launch_bounds__(kScanThreads)
    face_tile_rows_k(int64_t nf, const uint8_t* __restrict__ face_class, long long* __restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    int rows = 0;
#pragma unroll
    for (int i = 0; i < kScanItems / 4; ++i) {
        const int64_t f = base + 4 * (i * kScanThreads + (int64_t)threadIdx.x);
        if (f + 4 <= nf) {
            const uchar4 k = __ldg(reinterpret_cast<const uchar4*>(face_class + f));
            rows += (k.x != 2) + (k.y != 2) + (k.z != 2) + (k.w != 2);
        } else {
            for (int j = 0; j < 4 && f + j < nf; ++j) rows += face_class[f + j] != 2;
        }
    }
    const long long tot = block_sum_ll<kScanThreads>(rows);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// classes staged in shared memory (striped in, blocked for the scan), rows
// staged again and written out striped, with the row -> face list
__global__ void __launch_bounds__(kScanThreads)
    face_rows_k(int64_t nf, const uint8_t* __restrict__ face_class, const long long* __restrict__ tile_off,
                int32_t* __restrict__ face_mrow, int32_t* __restrict__ row_face) {
    __shared__ __align__(16) uint8_t s_cls[kScanTile];
    __shared__ int32_t s_row[kScanTile + kScanTile / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int nt = (int)(nf - base < kScanTile ? nf - base : kScanTile);
    if (nt == kScanTile) {
        reinterpret_cast<uint4*>(s_cls)[threadIdx.x] = __ldg(reinterpret_cast<const uint4*>(face_class + base) + threadIdx.x);
    } else {
        for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) s_cls[i] = i < nt ? face_class[base + i] : 2;
    }
    __syncthreads();
    const uint4 q = reinterpret_cast<const uint4*>(s_cls)[threadIdx.x];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    int n = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) n += ((w[i / 4] >> (8 * (i % 4))) & 0xffu) != 2;
    int r = (int)block_excl_scan_ll<kScanThreads>(n);
    const long long off = tile_off[blockIdx.x];
    // local index i of the tile lives at s_row[i + i / 32] (one pad word per
    // 32: blocked writes of 16 consecutive words stay conflict-light)
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int li = threadIdx.x * kScanItems + i;
        const bool row = ((w[i / 4] >> (8 * (i % 4))) & 0xffu) != 2;
        s_row[li + (li >> 5)] = row ? (int32_t)(off + r) : -1;
        r += row;
    }
    __syncthreads();
    if (nt == kScanTile) {
#pragma unroll
        for (int k = 0; k < kScanItems / 4; ++k) {
            const int i = 4 * (k * kScanThreads + threadIdx.x);  // 4 consecutive, same pad group
            const int p = i + (i >> 5);
            reinterpret_cast<int4*>(face_mrow + base)[k * kScanThreads + threadIdx.x] =
                make_int4(s_row[p], s_row[p + 1], s_row[p + 2], s_row[p + 3]);
        }
    } else {
        for (int i = threadIdx.x; i < nt; i += kScanThreads) face_mrow[base + i] = s_row[i + (i >> 5)];
    }
    // the inverse map, striped over the tile: a warp's rows are consecutive
    // apart from the Neumann faces it skips
    for (int i = threadIdx.x; i < nt; i += kScanThreads) {
        const int32_t row = s_row[i + (i >> 5)];
        if (row >= 0) row_face[row] = (int32_t)(base + i);
    }
}

inline int grid_cap(int64_t n, int block) {
    const int g = grid_for(n, block);
    return g < kSMs * 32 ? g : kSMs * 32;
}

}  // namespace

extern "C" int phfem_gpu_star_count(const int32_t* tets, int64_t ne, int32_t* count, int32_t* repeated,
                                    void* stream) {
    star_count<<<grid_cap(ne, 256), 256, 0, (cudaStream_t)stream>>>(tets, ne, count, repeated);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_star_fill(const int32_t* tets, int64_t ne, const int64_t* star_ptr, int32_t* count,
                                   int32_t* star, void* stream) {
    star_fill<<<grid_cap(ne, 256), 256, 0, (cudaStream_t)stream>>>(tets, ne, star_ptr, count, star);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_star_groups(int64_t nc, const int64_t* star_ptr, const int32_t* star, const int32_t* tets,
                                     int32_t* edge_first, int32_t* slot_mate, int32_t* defer_list,
                                     int32_t* defer_count, unsigned long long* err, const int32_t* repeated,
                                     void* stream) {
    // pass 1: all vertices, stars <= 32 (warp, one incidence per lane)
    // pass 2: deferred stars <= 64 (warp, two per lane)
    // pass 3: anything larger (block per vertex); counts stay on the device
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(defer_count, 0, 3 * sizeof(int32_t), s);
    // one full wave of resident blocks (grid-stride over the vertices)
    static int resident = 0, resident_m = 0, use_match = -1;
    if (use_match < 0) {
        const char* e = getenv("PHFEM_GROUPS_HASH");
        use_match = e && atoi(e) != 0 ? 0 : 1;
    }
    if (resident == 0) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, star_groups_warp<1>, 32 * kFastWarps, 0);
        resident = (per_sm > 0 ? per_sm : 8) * kSMs;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, star_groups_match, 32 * kMatchWarps, 0);
        resident_m = (per_sm > 0 ? per_sm : 4) * kSMs;
    }
    if (use_match) {
        const int64_t blocks = (nc + kMatchWarps - 1) / kMatchWarps;
        const int grid = (int)(blocks < resident_m ? blocks : resident_m);
        star_groups_match<<<grid, 32 * kMatchWarps, 0, s>>>(nc, star_ptr, star, tets, edge_first, slot_mate,
                                                            defer_list, defer_count, repeated, err);
    } else {
        const int64_t blocks = (nc + kFastWarps - 1) / kFastWarps;
        const int grid = (int)(blocks < resident ? blocks : resident);
        star_groups_warp<1><<<grid, 32 * kFastWarps, 0, s>>>(nc, nullptr, nullptr, star_ptr, star, tets, edge_first,
                                                             slot_mate, defer_list, defer_count, err);
    }
    star_groups_warp<2><<<kSMs * 4, 32 * kFastWarps, 0, s>>>(0, defer_list, defer_count, star_ptr, star, tets,
                                                             edge_first, slot_mate, defer_list + nc,
                                                             defer_count + 1, err);
    constexpr unsigned cap = 8192;  // stars up to 2730 incidences
    const size_t bytes = (size_t)cap * 20;
    cudaFuncSetAttribute(star_groups_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    star_groups_big<<<kSMs, 256, bytes, s>>>(defer_list + nc, defer_count + 1, star_ptr, star, tets, edge_first,
                                             slot_mate, cap, defer_list + 2 * nc, defer_count + 2, err);
    phg::count_launches(3);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_star_groups_global(int32_t v, const int64_t* star_ptr, const int32_t* star,
                                            const int32_t* tets, int32_t* edge_first, int32_t* slot_mate,
                                            void* scratch, unsigned cap, unsigned long long* err, void* stream) {
    star_groups_global<<<1, 256, 0, (cudaStream_t)stream>>>(v, star_ptr, star, tets, edge_first, slot_mate,
                                                           static_cast<unsigned char*>(scratch), cap, err);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" size_t phfem_gpu_element_offsets_scratch(int64_t ne) {
    // tile sums + packed total
    return (size_t)(scan_tiles(ne) + 2) * sizeof(long long);
}

extern "C" int phfem_gpu_element_offsets(int64_t ne, const int32_t* edge_first, const int32_t* slot_mate,
                                         uint16_t* masks, int64_t* edge_off, int64_t* face_off, void* scratch,
                                         void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ne <= 0) {
        // (no slots: slot_mate may be NULL even when faces are asked for)
        cudaMemsetAsync(edge_off, 0, sizeof(int64_t), s);
        if (face_off) cudaMemsetAsync(face_off, 0, sizeof(int64_t), s);
        return (int)cudaGetLastError();
    }
    const int64_t ntiles = scan_tiles(ne);
    long long* sums = static_cast<long long*>(scratch);
    int64_t* total = reinterpret_cast<int64_t*>(sums + ntiles);
    offsets_count_k<<<(unsigned)ntiles, kScanThreads, 0, s>>>(ne, edge_first, slot_mate, masks, sums);
    scan_sums(sums, ntiles, total, s);
    offsets_scan_k<<<(unsigned)ntiles, kScanThreads, 0, s>>>(ne, masks, sums, edge_off, slot_mate ? face_off : nullptr);
    offsets_total_k<<<1, 1, 0, s>>>(total, ne, edge_off, slot_mate ? face_off : nullptr);
    phg::count_launches(4);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_element_offsets_scan(int64_t ne, const uint16_t* masks, bool faces, int64_t* edge_off,
                                              int64_t* face_off, void* scratch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ne <= 0) return phfem_gpu_element_offsets(ne, nullptr, nullptr, nullptr, edge_off, face_off, scratch, stream);
    const int64_t ntiles = scan_tiles(ne);
    long long* sums = static_cast<long long*>(scratch);
    int64_t* total = reinterpret_cast<int64_t*>(sums + ntiles);
    scan_sums(sums, ntiles, total, s);
    offsets_scan_k<<<(unsigned)ntiles, kScanThreads, 0, s>>>(ne, masks, sums, edge_off, faces ? face_off : nullptr);
    offsets_total_k<<<1, 1, 0, s>>>(total, ne, edge_off, faces ? face_off : nullptr);
    phg::count_launches(3);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_number(int64_t ne, const int32_t* tets, const double* coords, const int32_t* edge_first,
                                const int64_t* edge_off, int32_t* edge_of_slot,
                                int32_t* edge_nodes,
                                const int32_t* slot_mate, const int64_t* face_off, int32_t* face_of_slot,
                                int8_t* sigma, int32_t* faces, int32_t* face_slots, double* face_area,
                                unsigned long long* err, void* stream) {
    if (ne == 0) return 0;
    number<<<(unsigned)((ne + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        ne, tets, coords, edge_first, edge_off, edge_of_slot, edge_nodes, slot_mate, face_off, face_of_slot, sigma,
        faces, face_slots, face_area, err);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_classify(int64_t nd, const int32_t* db, int64_t nn, const int32_t* nb,
                                  const int64_t* star_ptr, const int32_t* star, const int32_t* tets,
                                  const int32_t* face_of_slot, const int32_t* face_slots, uint32_t* claim,
                                  int32_t* entry_face, unsigned long long* err, void* stream) {
    if (nd + nn == 0) return 0;
    classify<<<grid_cap(nd + nn, 128), 128, 0, (cudaStream_t)stream>>>(nd, db, nn, nb, star_ptr, star, tets,
                                                                      face_of_slot, face_slots, claim, entry_face,
                                                                      err); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_classify_check(int64_t nd, int64_t nn, const int32_t* entry_face, const uint32_t* claim,
                                        unsigned long long* err, void* stream) {
    if (nd + nn == 0) return 0;
    classify_check<<<grid_cap(nd + nn, 256), 256, 0, (cudaStream_t)stream>>>(nd, nn, entry_face, claim, err); phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" size_t phfem_gpu_face_rows_scratch(int64_t nf) {
    return (size_t)(scan_tiles(nf) + 1) * sizeof(long long);
}

extern "C" int phfem_gpu_face_class(int64_t nf, int64_t nd, const uint32_t* claim, const int32_t* face_slots,
                                    uint8_t* face_class, unsigned long long* counts, void* scratch, int64_t* n_rows,
                                    unsigned long long* err, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (nf <= 0) {
        cudaMemsetAsync(n_rows, 0, sizeof(int64_t), s);
        return (int)cudaGetLastError();
    }
    const int64_t ntiles = scan_tiles(nf);
    long long* sums = static_cast<long long*>(scratch);
    face_class_k<<<(unsigned)ntiles, kScanThreads, 0, s>>>(nf, nd, claim, face_slots, face_class, sums, counts, err);
    scan_sums(sums, ntiles, n_rows, s);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_face_rows(int64_t nf, const uint8_t* face_class, const void* scratch, int32_t* face_mrow,
                                   int32_t* row_face, void* stream) {
    if (nf <= 0) return 0;
    face_rows_k<<<(unsigned)scan_tiles(nf), kScanThreads, 0, (cudaStream_t)stream>>>(
        nf, face_class, static_cast<const long long*>(scratch), face_mrow, row_face);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_face_rows_identity(int64_t nf, int32_t* face_mrow, int32_t* row_face, void* stream) {
    if (nf == 0) return 0;
    face_rows_identity_k<<<grid_cap(nf, 256), 256, 0, (cudaStream_t)stream>>>(nf, face_mrow, row_face);
    phg::count_launches(1);
    return (int)cudaGetLastError();
}

extern "C" int phfem_gpu_face_tile_rows(int64_t nf, const uint8_t* face_class, void* scratch, int64_t* n_rows,
                                        void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (nf <= 0) {
        cudaMemsetAsync(n_rows, 0, sizeof(int64_t), s);
        return (int)cudaGetLastError();
    }
    const int64_t ntiles = scan_tiles(nf);
    long long* sums = static_cast<long long*>(scratch);
    face_tile_rows_k<<<(unsigned)ntiles, kScanThreads, 0, s>>>(nf, face_class, sums);
    scan_sums(sums, ntiles, n_rows, s);
    phg::count_launches(2);
    return (int)cudaGetLastError();
}
