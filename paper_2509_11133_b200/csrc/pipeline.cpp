// Stage orchestration of the hot path: connectivity, refinement, fused
// assembly + condensation.  Device-only sizes (nEd, nF, L) are read back once
// per stage; device error slots are replayed in the reference's check order
// so the same exception and message shape surface.  All transient buffers
// live in the owner's Work so repeated passes reuse device memory.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "runtime.hpp"

namespace phb {

namespace {

constexpr unsigned long long kNone = ~0ull;

void reset_err(Work& w) {
    w.err.alloc(PHG_ERR_COUNT);
    w.err.fill_bytes(0xff);
}

// read several device scalars with one synchronisation (read_words)
template <class T, size_t N>
std::array<T, N> read_many(const std::array<const T*, N>& src) {
    static_assert(sizeof(T) == 8 && N <= 16, "8-byte words, at most 16");
    const unsigned long long* p[N];
    for (size_t i = 0; i < N; ++i) p[i] = reinterpret_cast<const unsigned long long*>(src[i]);
    unsigned long long w[N];
    read_words(p, (int)N, w);
    std::array<T, N> out;
    for (size_t i = 0; i < N; ++i) std::memcpy(&out[i], &w[i], sizeof(T));
    return out;
}

std::string tri_str(const int32_t* f) {
    return "[" + std::to_string(f[0] + 1) + " " + std::to_string(f[1] + 1) + " " + std::to_string(f[2] + 1) + "]";
}

void fetch_tri(const int32_t* dev, int64_t i, int32_t out[3]) {
    check(cudaMemcpyAsync(out, dev + 3 * i, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
}

// connectivity.cpp:62-68, 156-194 and mesh.cpp:80-82, in that order; `upto`
// stops after the checks the stage that ran owns (1: edges, which the
// reference's num_edges never fails; 2: + the E2T duplicate-orientation
// check; 3: everything)
void replay_connectivity_errors(const std::vector<unsigned long long>& e, const MeshData& m, const Connectivity& c,
                                int upto = 3) {
    // (PHG_ERR_VALENCE is not an error: those stars took the global path)
    if (upto < 2) return;
    const bool degen = e[PHG_ERR_DEGEN_FACE] != kNone;
    if (e[PHG_ERR_DUP_ORIENT] != kNone || degen) {
        // the reference names the first repeated key of its sorted E2T
        // entries: build that map on this error path to name the same pair
        // (faces with a repeated node id register their own keys there, so
        // their elements are checked the same way)
        const unsigned long long k = e[PHG_ERR_DUP_ORIENT];
        int32_t a = (int32_t)(k >> 32), b = (int32_t)(k & 0xffffffffull);
        if (e2t_first_duplicate(m, c, a, b) || !degen)
            throw MeshError("inconsistent mesh: elements " + std::to_string(a + 1) + " and " + std::to_string(b + 1) +
                            " claim the same oriented face");
    }
    if (upto < 3) return;
    if (degen) {
        // full_face_table's element loop (connectivity.cpp:136-143): the
        // first slot whose oriented face is not in faces_up's list is the
        // first face with a repeated node id
        const int64_t slot = (int64_t)e[PHG_ERR_DEGEN_FACE];
        const int64_t t = slot >> 2;
        const int k = (int)(slot & 3);
        int32_t tet[4];
        check(cudaMemcpyAsync(tet, m.tets.p + 4 * t, sizeof tet, cudaMemcpyDeviceToHost, S()), "D2H");
        sync();
        static const int fv[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {3, 2, 1}};  // elem_oriented_faces
        const int32_t f[3] = {tet[fv[k][0]], tet[fv[k][1]], tet[fv[k][2]]};
        throw MeshError("inconsistent mesh: face " + tri_str(f) + " of element " + std::to_string(t + 1) +
                        " matches no unique face");
    }
    if (e[PHG_ERR_CLASSIFY] != kNone) {
        const int64_t i = (int64_t)(e[PHG_ERR_CLASSIFY] >> 2);
        const int kind = (int)(e[PHG_ERR_CLASSIFY] & 3);
        int32_t tri[3];
        const bool dir = i < m.nd;
        fetch_tri(dir ? m.db.p : m.nb.p, dir ? i : i - m.nd, tri);
        const std::string what = dir ? "Dirichlet" : "Neumann";
        if (kind == 0) throw MeshError("inconsistent mesh: " + what + " face " + tri_str(tri) + " matches no element face");
        if (kind == 1) throw MeshError("inconsistent mesh: boundary face " + tri_str(tri) + " listed twice");
        throw MeshError("inconsistent mesh: " + what + " face " + tri_str(tri) + " is interior");
    }
    if (e[PHG_ERR_FACE] != kNone) {
        const int64_t f = (int64_t)(e[PHG_ERR_FACE] >> 2);
        const int kind = (int)(e[PHG_ERR_FACE] & 3);
        int32_t tri[3];
        fetch_tri(c.faces.p, f, tri);
        if (kind == 0) throw MeshError("degenerate face with collinear nodes " + tri_str(tri));
        throw MeshError("inconsistent mesh: boundary face " + tri_str(tri) +
                        " is in neither the Dirichlet nor the Neumann list");
    }
}

// Stars above the shared-memory capacity of star_groups_big (listed at
// big_list + 2 nC): grouped one by one with global-memory tables, then the
// valence flag is cleared.  Rare (no such vertex in any config here), so the
// host loop and its reads are off the normal path.
void group_huge_stars(const MeshData& m, Connectivity& c, bool faces) {
    Work& w = c.w;
    const int64_t nc = m.nc;
    int32_t n = 0;
    check(cudaMemcpyAsync(&n, w.big_count.p + 2, sizeof n, cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
    std::vector<int32_t> list(n);
    if (n) check(cudaMemcpyAsync(list.data(), w.big_list.p + 2 * nc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, S()),
                 "D2H");
    sync();
    DBuf<unsigned char> scratch;
    for (const int32_t v : list) {
        int64_t se[2];
        check(cudaMemcpyAsync(se, c.star_ptr.p + v, sizeof se, cudaMemcpyDeviceToHost, S()), "D2H");
        sync();
        unsigned cap = 16;
        while (cap <= 3 * (uint64_t)(se[1] - se[0])) cap <<= 1;
        scratch.alloc((int64_t)cap * 20);
        check(phfem_gpu_star_groups_global(v, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                           faces ? c.slot_mate.p : nullptr, scratch.p, cap, w.err.p, SV()),
              "star groups (global)");
    }
    check(cudaMemsetAsync(w.err.p + PHG_ERR_VALENCE, 0xff, sizeof(unsigned long long), S()), "memset");
}

}  // namespace

// ------------------------------------------------------------ connectivity

void build_star(const MeshData& m, Connectivity& c, Stages* st) {
    Work& w = c.w;
    cudaEvent_t t0 = st ? st->mark() : nullptr;
    if (w.scratch.cap < (int64_t)phfem_gpu_scan_scratch(m.nc)) w.scratch.alloc((int64_t)phfem_gpu_scan_scratch(m.nc));
    // counts, then one word set when an element repeats a node id (read by
    // the star grouping)
    w.cnt.alloc(m.nc + 1);
    w.cnt.zero();
    check(phfem_gpu_star_count(m.tets.p, m.ne, w.cnt.p, w.cnt.p + m.nc, SV()), "star count");
    c.star_ptr.alloc(m.nc + 1);
    check(phfem_gpu_scan_i32(w.cnt.p, c.star_ptr.p, m.nc, w.scratch.p, SV()), "star scan");
    c.star.alloc(3 * m.ne);  // no incidence of an element's largest vertex
    check(phfem_gpu_star_fill(m.tets.p, m.ne, c.star_ptr.p, w.cnt.p, c.star.p, SV()), "star fill");
    if (st) st->span(&st->star, t0);
    c.has_star = true;
}

void build_connectivity(const MeshData& m, Connectivity& c, bool faces, Stages* st, bool classify) {
    const int64_t nc = m.nc, ne = m.ne;
    Work& w = c.w;
    cudaEvent_t t0 = nullptr;
    const auto w0 = std::chrono::steady_clock::now();
    reset_err(w);
    w.scratch.alloc((int64_t)std::max(phfem_gpu_scan_scratch(std::max<int64_t>({nc, ne, 4 * ne})),
                                      phfem_gpu_element_offsets_scratch(ne)));
    // a child of a red refinement whose parent kept its full tables: the
    // grouping (and, with faces, the classification) in closed form
    // (refine_conn.cu), else per-vertex hashing through the star
    const Connectivity* pc = m.parent_conn.get();
    const MeshData* pm = m.parent_mesh.get();
    const bool refined = pc && pm && pc->has_faces && 12 * pm->ne == ne;
    const bool refined_cls = refined && faces && classify && m.nd == 4 * pm->nd && m.nn == 4 * pm->nn;
    // 1. vertex star (CSR by vertex)
    c.has_star = false;
    if (!refined_cls) build_star(m, c, st);
    // 2. per-vertex grouping of edges and faces
    if (st) t0 = st->mark();
    c.edge_first.alloc(6 * ne);
    if (faces) c.slot_mate.alloc(4 * ne);
    w.big_list.alloc(3 * (nc > 0 ? nc : 1));
    w.big_count.alloc(3);
    c.edge_off.alloc(ne + 1);
    if (faces) w.face_off.alloc(ne + 1);
    w.masks.alloc(ne + 8);
    if (refined) {
        // also the per-element masks and tile sums: the offsets need only
        // their scan (no offsets_count_k pass over the slots)
        w.a0.alloc(2 * pc->ned + 2);
        check(phfem_gpu_refined_groups(pm->ne, pm->tets.p, pc->edge_of_slot.p, pc->edge_first.p, pc->slot_mate.p,
                                       pc->ned, w.a0.p, c.edge_first.p, faces ? c.slot_mate.p : nullptr, w.masks.p,
                                       w.scratch.p, SV()),
              "refined groups");
    } else {
        check(phfem_gpu_star_groups(nc, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                    faces ? c.slot_mate.p : nullptr, w.big_list.p, w.big_count.p, w.err.p,
                                    w.cnt.p + nc, SV()),
              "star groups");
    }
    if (st) st->span(&st->groups, t0);
    // 3. numbering: per-element counts, scans, ids, remaining slots
    if (st) t0 = st->mark();
    if (refined)
        check(phfem_gpu_element_offsets_scan(ne, w.masks.p, faces, c.edge_off.p, faces ? w.face_off.p : nullptr,
                                             w.scratch.p, SV()),
              "element offsets");
    else
        check(phfem_gpu_element_offsets(ne, c.edge_first.p, faces ? c.slot_mate.p : nullptr, w.masks.p,
                                        c.edge_off.p, faces ? w.face_off.p : nullptr, w.scratch.p, SV()),
              "element offsets");
    // the totals, and whether a star was too large for the shared-memory
    // tables (the reference has no valence limit): then the global-memory
    // pass groups those vertices and the offsets are redone
    for (int pass = 0;; ++pass) {
        const auto tot = read_many<int64_t, 3>({c.edge_off.p + ne, faces ? w.face_off.p + ne : c.edge_off.p + ne,
                                                reinterpret_cast<const int64_t*>(w.err.p + PHG_ERR_VALENCE)});
        c.ned = tot[0];
        c.nf = faces ? tot[1] : 0;
        if ((unsigned long long)tot[2] == kNone || pass > 0) break;
        group_huge_stars(m, c, faces);
        check(phfem_gpu_element_offsets(ne, c.edge_first.p, faces ? c.slot_mate.p : nullptr, w.masks.p,
                                        c.edge_off.p, faces ? w.face_off.p : nullptr, w.scratch.p, SV()),
              "element offsets");
    }
    c.edge_of_slot.alloc(6 * ne);
    c.edge_nodes.alloc(2 * c.ned);
    if (faces) {
        c.face_of_slot.alloc(4 * ne);
        c.sigma.alloc(4 * ne);
        c.faces.alloc(3 * c.nf);
        c.face_slots.alloc(2 * c.nf);
        c.face_area.alloc(c.nf);
    }
    check(phfem_gpu_number(ne, m.tets.p, m.coords.p, c.edge_first.p, c.edge_off.p, c.edge_of_slot.p,
                           c.edge_nodes.p,
                           faces ? c.slot_mate.p : nullptr, faces ? w.face_off.p : nullptr,
                           faces ? c.face_of_slot.p : nullptr, faces ? c.sigma.p : nullptr,
                           faces ? c.faces.p : nullptr, faces ? c.face_slots.p : nullptr,
                           faces ? c.face_area.p : nullptr, w.err.p, SV()),
          "number");
    if (st) st->span(&st->number, t0);
    c.has_edges = true;
    c.has_faces = false;
    c.t_edges = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    if (!faces || !classify) {
        replay_connectivity_errors(w.err.download(), m, c, faces ? 2 : 1);
        return;
    }
    // 4. boundary classification and multiplier rows
    const auto w1 = std::chrono::steady_clock::now();
    if (st) t0 = st->mark();
    const int64_t nf = c.nf;
    w.claim.alloc(nf);
    w.claim.fill_bytes(0xff);
    c.entry_face.alloc(m.nd + m.nn);
    // A refined child's boundary faces are exactly the sub-triangles of its
    // parent's classified boundary faces, each listed once in the child's
    // lists: the classes are written by the refined classification, the
    // class counts follow from the list sizes, and without Neumann faces
    // every face is a multiplier row (rows = face ids).
    const bool closed_rows = refined_cls;
    if (closed_rows) {
        c.face_class.alloc(nf + 16);
        c.face_class.zero();
    }
    if (refined_cls) {
        check(phfem_gpu_refined_classify(pm->nd, pm->nn, pm->db.p, pm->nb.p, pc->entry_face.p, pc->face_slots.p,
                                         pm->tets.p, pm->ne, c.face_of_slot.p, c.face_slots.p, w.claim.p,
                                         c.entry_face.p, closed_rows ? c.face_class.p : nullptr, w.err.p, SV()),
              "refined classify");
    } else {
        check(phfem_gpu_classify(m.nd, m.db.p, m.nn, m.nb.p, c.star_ptr.p, c.star.p, m.tets.p, c.face_of_slot.p,
                                 c.face_slots.p, w.claim.p, c.entry_face.p, w.err.p, SV()),
              "classify");
    }
    check(phfem_gpu_classify_check(m.nd, m.nn, c.entry_face.p, w.claim.p, w.err.p, SV()), "classify check");
    if (closed_rows) {
        static_assert(PHG_ERR_COUNT == 8, "error slots");
        const auto e = read_many<unsigned long long, 8>(
            {w.err.p, w.err.p + 1, w.err.p + 2, w.err.p + 3, w.err.p + 4, w.err.p + 5, w.err.p + 6, w.err.p + 7});
        replay_connectivity_errors(std::vector<unsigned long long>(e.begin(), e.end()), m, c);
        c.n_dir = m.nd;
        c.n_neu = m.nn;
        c.n_int = nf - m.nd - m.nn;
        c.l = nf - m.nn;
        c.face_mrow.alloc(nf);
        c.row_face.alloc(c.l);
        if (m.nn == 0) {
            check(phfem_gpu_face_rows_identity(nf, c.face_mrow.p, c.row_face.p, SV()), "face rows");
        } else {
            w.counts.alloc(4);
            w.scratch.alloc((int64_t)phfem_gpu_face_rows_scratch(nf));
            check(phfem_gpu_face_tile_rows(nf, c.face_class.p, w.scratch.p, reinterpret_cast<int64_t*>(w.counts.p + 3),
                                           SV()),
                  "face rows");
            check(phfem_gpu_face_rows(nf, c.face_class.p, w.scratch.p, c.face_mrow.p, c.row_face.p, SV()),
                  "face rows");
        }
        if (st) st->span(&st->classify, t0);
        c.has_faces = true;
        c.t_faces = std::chrono::duration<double>(std::chrono::steady_clock::now() - w1).count();
        return;
    }
    c.face_class.alloc(nf + 16);
    w.counts.alloc(4);
    w.counts.zero();
    w.scratch.alloc((int64_t)phfem_gpu_face_rows_scratch(nf));
    check(phfem_gpu_face_class(nf, m.nd, w.claim.p, c.face_slots.p, c.face_class.p, w.counts.p, w.scratch.p,
                               reinterpret_cast<int64_t*>(w.counts.p + 3), w.err.p, SV()),
          "face class");
    // the class counts and every connectivity error slot in one read (face
    // rows below report nothing)
    static_assert(PHG_ERR_COUNT == 8, "error slots");
    const auto cnt = read_many<unsigned long long, 12>(
        {w.counts.p, w.counts.p + 1, w.counts.p + 2, w.counts.p + 3, w.err.p, w.err.p + 1, w.err.p + 2,
         w.err.p + 3, w.err.p + 4, w.err.p + 5, w.err.p + 6, w.err.p + 7});
    replay_connectivity_errors(std::vector<unsigned long long>(cnt.begin() + 4, cnt.end()), m, c);
    c.n_int = (int64_t)cnt[0];
    c.n_dir = (int64_t)cnt[1];
    c.n_neu = (int64_t)cnt[2];
    c.l = (int64_t)cnt[3];
    c.face_mrow.alloc(nf);
    c.row_face.alloc(c.l);
    check(phfem_gpu_face_rows(nf, c.face_class.p, w.scratch.p, c.face_mrow.p, c.row_face.p, SV()), "face rows");
    if (st) st->span(&st->classify, t0);
    c.has_faces = true;
    c.t_faces = std::chrono::duration<double>(std::chrono::steady_clock::now() - w1).count();
}

// -------------------------------------------------------------- refinement

std::shared_ptr<MeshData> prepare_child(const MeshData& m, const Connectivity& c, std::shared_ptr<MeshData> into) {
    if (!c.has_edges) throw MeshError("refine_mesh: edge table missing");
    const int64_t nc2 = m.nc + c.ned + m.ne;
    const int64_t ne2 = 12 * m.ne;
    if (nc2 >= (int64_t)INT32_MAX || 6 * ne2 >= (int64_t)INT32_MAX)
        throw MeshError("out of memory while refining to level " + std::to_string(m.level + 1) +
                        ": 32-bit node/element ids exhausted");
    auto out = into ? into : std::make_shared<MeshData>();
    out->nc = nc2;
    out->ne = ne2;
    out->nd = 4 * m.nd;
    out->nn = 4 * m.nn;
    out->level = m.level + 1;
    out->coords.alloc(3 * nc2);
    out->tets.alloc(4 * ne2);
    out->db.alloc(3 * out->nd);
    out->nb.alloc(3 * out->nn);
    return out;
}

std::shared_ptr<MeshData> refine_mesh(const MeshData& m, Connectivity& c, RefineMap* map, Stages* st,
                                      std::shared_ptr<MeshData> into, bool elements_written) {
    if (elements_written && (map || !into)) throw InvalidArgument("refine_mesh: fused elements need the prepared child");
    cudaEvent_t t0 = st ? st->mark() : nullptr;
    auto out = elements_written ? into : prepare_child(m, c, into);
    if (map) {
        map->midpoint.alloc(c.ned);
        map->centroid.alloc(m.ne);
    }
    Work& w = c.w;
    reset_err(w);
    if (!elements_written)
        check(phfem_gpu_refine(m.nc, m.ne, m.coords.p, m.tets.p, c.edge_first.p, c.edge_of_slot.p, c.edge_off.p,
                               out->coords.p, out->tets.p, map ? map->midpoint.p : nullptr,
                               map ? map->centroid.p : nullptr, SV()),
              "refine");
    if (c.has_faces) {
        // classified: each list entry's face and its owner element are known
        check(phfem_gpu_refine_boundary_owned(m.nd, m.db.p, 0, m.nc, c.entry_face.p, c.face_slots.p, m.tets.p,
                                              c.edge_first.p, c.edge_of_slot.p, out->db.p, SV()),
              "refine boundary");
        check(phfem_gpu_refine_boundary_owned(m.nn, m.nb.p, m.nd, m.nc, c.entry_face.p, c.face_slots.p, m.tets.p,
                                              c.edge_first.p, c.edge_of_slot.p, out->nb.p, SV()),
              "refine boundary");
    } else {
        if (!c.has_star) build_star(m, c, nullptr);
        check(phfem_gpu_refine_boundary(m.nd, m.db.p, 0, m.nc, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                        c.edge_of_slot.p, out->db.p, w.err.p, SV()),
              "refine boundary");
        check(phfem_gpu_refine_boundary(m.nn, m.nb.p, m.nd, m.nc, c.star_ptr.p, c.star.p, m.tets.p,
                                        c.edge_first.p, c.edge_of_slot.p, out->nb.p, w.err.p, SV()),
              "refine boundary");
    }
    if (st) st->span(&st->refine, t0);
    auto replay = [&m](const unsigned long long* e) {
        if (e[PHG_ERR_BOUNDARY_EDGE] != kNone) {
            const int64_t i = (int64_t)(e[PHG_ERR_BOUNDARY_EDGE] >> 2);
            const int q = (int)(e[PHG_ERR_BOUNDARY_EDGE] & 3);
            int32_t tri[3];
            const bool dir = i < m.nd;
            fetch_tri(dir ? m.db.p : m.nb.p, dir ? i : i - m.nd, tri);
            const int32_t a = q == 1 ? tri[1] : tri[0], b = q == 0 ? tri[1] : tri[2];
            throw MeshError("inconsistent mesh: boundary face edge (" + std::to_string(a + 1) + "," +
                            std::to_string(b + 1) + ") is not an element edge");
        }
    };
    if (st && st->defer) {
        st->defer_errors(w.err.p, replay);  // m outlives the pass (the caller's mesh)
    } else {
        const auto e = w.err.download();
        replay(e.data());
    }
    return out;
}

// ------------------------------------------------------ assembly + Schur

phg_problem device_problem(const Coefs& k, int problem) {
    phg_problem p;
    p.kind = problem;
    p.c = k.c;
    p.a_elem = k.has_elem ? k.a_elem.p : nullptr;
    p.a_diag = k.has_diag ? k.a_diag.p : nullptr;
    return p;
}

void System::finish() const {
    if (!split) return;
    check(phfem_gpu_sum_halves(l, const_cast<double*>(diag.p), const_cast<double*>(rhs_neg.p), halves.p, SV()),
          "sum halves");
    split = false;
}

void assemble_system(const MeshData& m, const Coefs& k, const Connectivity& c, int problem, System& sys,
                     bool debug_views, Stages* st, const phg_refine_out* refine) {
    if (!c.has_faces) throw MeshError("assemble: face table missing");
    if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
    cudaEvent_t t0 = st ? st->mark() : nullptr;
    sys.problem = problem;
    sys.coef_version = k.version;
    sys.n = 4 * m.ne;
    sys.l = c.l;
    // S in SELL-32 when the views are exported (the reference's rows, both
    // triangles), else element-major for the solve (half the bytes per CG
    // iteration and per assembly)
    sys.elem = !debug_views;
    sys.nchunks = (c.l + PHG_SELL_C - 1) / PHG_SELL_C;
    if (sys.elem) {
        sys.sell_col.release();
        sys.sell_val.release();
        sys.st_val.alloc(10 * ((m.ne + 31) / 32) * 32);
        sys.diag.alloc(c.l);
        sys.halves.alloc(2 * c.l);
    } else {
        const int64_t width = PHG_SELL_C * PHG_SELL_W;
        sys.sell_col.alloc(sys.nchunks * width);
        sys.sell_val.alloc(sys.nchunks * width);
        sys.st_val.release();
        sys.diag.release();
        sys.halves.release();
    }
    // the S diagonal, rhs_neg and b_D are cleared by the assembly kernel
    // itself (row owners), every other SELL slot is written exactly once
    sys.rhs_neg.alloc(c.l);
    sys.bd.alloc(c.l);
    sys.rhs.alloc(4 * m.ne);
    if (debug_views) {
        sys.a_blocks.alloc(16 * m.ne);
        sys.slot_coef.alloc(4 * m.ne);
    } else {
        sys.a_blocks.release();
        sys.slot_coef.release();
    }
    sys.slot_mrow.alloc(4 * m.ne);
    Work& w = sys.w;
    w.redo.alloc(m.ne + 1);
    reset_err(w);
    const phg_problem p = device_problem(k, problem);
    // the main kernel alone
    cudaEvent_t ka = st ? st->event() : nullptr, kb = st ? st->event() : nullptr;
    w.face_bval.alloc(c.nf);
    check(phfem_gpu_assemble_condense(m.ne, c.l, m.coords.p, m.tets.p, &p, c.face_of_slot.p, c.slot_mate.p,
                                      c.face_mrow.p, c.face_area.p, m.nd, m.nn, c.entry_face.p, c.face_slots.p,
                                      w.face_bval.p, sys.elem ? nullptr : sys.sell_col.p,
                                      sys.elem ? nullptr : sys.sell_val.p, sys.elem ? sys.st_val.p : nullptr,
                                      sys.elem ? sys.diag.p : nullptr, sys.rhs_neg.p, sys.bd.p, sys.rhs.p,
                                      debug_views ? sys.a_blocks.p : nullptr, debug_views ? sys.slot_coef.p : nullptr,
                                      sys.slot_mrow.p, w.redo.p, sys.elem ? sys.halves.p : nullptr, w.err.p, refine,
                                      ka, kb, SV()),
          "assemble");
    sys.split = sys.elem;
    if (st) {
        st->span(&st->assemble, t0);
        st->span(&st->assemble_kernel, ka, kb);
    }
    // assembly.cpp:13-14 (first element in order), then solver.cpp:128-129
    auto replay = [](const unsigned long long* e) {
        if (e[PHG_ERR_ZERO_VOLUME] != kNone)
            throw MeshError("degenerate element " + std::to_string(e[PHG_ERR_ZERO_VOLUME] + 1) + " (zero volume)");
        if (e[PHG_ERR_SINGULAR] != kNone)
            throw MeshError("degenerate element block " + std::to_string(e[PHG_ERR_SINGULAR] + 1));
    };
    if (st && st->defer) {
        st->defer_errors(w.err.p, replay);
    } else {
        const auto e = w.err.download();
        replay(e.data());
    }
}

}  // namespace phb
