// Host runtime: stage orchestration of the device pipeline.  Sizes that only
// the device knows (nEd, nF, L) are read back once per stage; everything else
// stays on the stream.  Device error slots are replayed in the reference's
// check order so the same exception (and message shape) surfaces.
#include "runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace phb {

// ------------------------------------------------------------------ basics

void check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw MeshError("out of memory");
    }
    throw MeshError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void tet_rule(int degree, std::vector<double>& lam, std::vector<double>& w);

Runtime::Runtime() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw MeshError(std::string("no CUDA device available for the B200 path: ") +
                        (e != cudaSuccess ? cudaGetErrorString(e) : "device count 0"));
    check(cudaGetDevice(&device), "get device");
    check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "create stream");
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    std::vector<double> l5, w5, l9, w9;
    tet_rule(5, l5, w5);
    tet_rule(9, l9, w9);
    check(phfem_gpu_set_rules(l5.data(), w5.data(), (int)w5.size(), l9.data(), w9.data(), (int)w9.size()),
          "upload quadrature");
}

Runtime& rt() {
    static Runtime r;
    return r;
}

void sync() { check(cudaStreamSynchronize(S()), "synchronize"); }

Timer::Timer() {
    check(cudaEventCreate(&a), "event");
    check(cudaEventCreate(&b), "event");
}
Timer::~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}
void Timer::start() { check(cudaEventRecord(a, S()), "event record"); }
double Timer::stop_ms() {
    check(cudaEventRecord(b, S()), "event record");
    check(cudaEventSynchronize(b), "event sync");
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, a, b), "event time");
    return ms;
}

// ------------------------------------------------------------- quadrature
// gauss_legendre / tet_rule, quadrature.cpp:9-62 (the host builds the
// tables exactly like the reference; the device receives them verbatim).

static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1.0, p1 = t;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (t * p1 - p0) / (t * t - 1.0);
            const double dt = p1 / dp;
            t -= dt;
            if (std::fabs(dt) < 1e-15) break;
        }
        x[n - 1 - i] = 0.5 * (1.0 + t);
        w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

void tet_rule(int degree, std::vector<double>& lam, std::vector<double>& w) {
    const int n = (degree + 3 + 1) / 2;
    std::vector<double> gx, gw;
    gauss_legendre(n, gx, gw);
    lam.clear();
    w.clear();
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            for (int c = 0; c < n; ++c) {
                const double u = gx[a], v = gx[b], ww = gx[c];
                const double x = u;
                const double y = v * (1.0 - u);
                const double z = ww * (1.0 - u) * (1.0 - v);
                const double jac = (1.0 - u) * (1.0 - u) * (1.0 - v);
                lam.push_back(1.0 - x - y - z);
                lam.push_back(x);
                lam.push_back(y);
                lam.push_back(z);
                w.push_back(6.0 * gw[a] * gw[b] * gw[c] * jac);
            }
}

std::string format_double(double v) {  // mesh.cpp:108-115
    char buf[40];
    for (int prec = 15; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    return buf;
}

// ----------------------------------------------------------------- meshes

std::shared_ptr<MeshData> upload_mesh(const double* coords, int64_t nc, const int32_t* tets, int64_t ne,
                                      const int32_t* db, int64_t nd, const int32_t* nb, int64_t nn, int level) {
    if (nc < 0 || ne < 0 || nd < 0 || nn < 0) throw InvalidArgument("negative mesh size");
    if (6 * ne >= (int64_t)INT32_MAX) throw MeshError("mesh too large: 6 nE must stay below 2^31");
    auto m = std::make_shared<MeshData>();
    m->nc = nc;
    m->ne = ne;
    m->nd = nd;
    m->nn = nn;
    m->level = level;
    m->coords.upload(coords, 3 * nc);
    m->tets.upload(tets, 4 * ne);
    m->db.upload(db, 3 * nd);
    m->nb.upload(nb, 3 * nn);
    sync();
    return m;
}

std::shared_ptr<MeshData> kuhn_mesh(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                                    uint64_t seed, uint32_t mask) {
    if (nx < 1 || ny < 1 || nz < 1) throw InvalidArgument("kuhn mesh needs at least one cell per axis");
    auto m = std::make_shared<MeshData>();
    m->nc = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    m->ne = 6ll * nx * ny * nz;
    if (6 * m->ne >= (int64_t)INT32_MAX) throw MeshError("mesh too large: 6 nE must stay below 2^31");
    m->coords.alloc(3 * m->nc);
    m->tets.alloc(4 * m->ne);
    check(phfem_gpu_kuhn_nodes(nx, ny, nz, lx, ly, lz, jitter, seed, m->coords.p, SV()), "kuhn nodes");
    DBuf<int32_t> packed(m->ne), cd(m->ne), cn(m->ne);
    check(phfem_gpu_kuhn_tets(nx, ny, nz, mask, m->tets.p, packed.p, SV()), "kuhn tets");
    check(phfem_gpu_split_counts(packed.p, cd.p, cn.p, m->ne, SV()), "kuhn counts");
    DBuf<int64_t> od(m->ne + 1), on(m->ne + 1);
    DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(m->ne));
    check(phfem_gpu_scan_i32(cd.p, od.p, m->ne, scratch.p, SV()), "scan");
    check(phfem_gpu_scan_i32(cn.p, on.p, m->ne, scratch.p, SV()), "scan");
    m->nd = read_scalar(od.p + m->ne);
    m->nn = read_scalar(on.p + m->ne);
    m->db.alloc(3 * m->nd);
    m->nb.alloc(3 * m->nn);
    check(phfem_gpu_kuhn_boundary(nx, ny, nz, mask, m->tets.p, od.p, on.p, m->db.p, m->nb.p, SV()), "kuhn boundary");
    sync();
    return m;
}

// ----------------------------------------------------------- error replay

namespace {

constexpr unsigned long long kNone = ~0ull;

struct ErrVec {
    DBuf<unsigned long long> d;
    ErrVec() : d(PHG_ERR_COUNT) { d.fill_bytes(0xff); }
    std::vector<unsigned long long> get() const { return d.download(); }
};

std::string tri_str(const int32_t* f) {
    return "[" + std::to_string(f[0] + 1) + " " + std::to_string(f[1] + 1) + " " + std::to_string(f[2] + 1) + "]";
}

void fetch_tri(const int32_t* dev, int64_t i, int32_t out[3]) {
    check(cudaMemcpyAsync(out, dev + 3 * i, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
}

// connectivity.cpp:62-68, 156-194 and mesh.cpp:80-82, in that order
void replay_connectivity_errors(const std::vector<unsigned long long>& e, const MeshData& m, const Connectivity& c) {
    if (e[PHG_ERR_VALENCE] != kNone)
        throw MeshError("vertex " + std::to_string(e[PHG_ERR_VALENCE] + 1) +
                        " is shared by more elements than the connectivity kernels support");
    if (e[PHG_ERR_DUP_ORIENT] != kNone) {
        const unsigned long long k = e[PHG_ERR_DUP_ORIENT];
        throw MeshError("inconsistent mesh: elements " + std::to_string((k >> 32) + 1) + " and " +
                        std::to_string((k & 0xffffffffull) + 1) + " claim the same oriented face");
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

}  // namespace

// ------------------------------------------------------------ connectivity

void build_connectivity(const MeshData& m, Connectivity& c, bool faces, Stages* st) {
    const int64_t nc = m.nc, ne = m.ne;
    Timer tm;
    const auto w0 = std::chrono::steady_clock::now();
    ErrVec err;
    // 1. vertex star (CSR by vertex)
    tm.start();
    {
        DBuf<int32_t> cnt(nc);
        cnt.zero();
        check(phfem_gpu_star_count(m.tets.p, ne, cnt.p, SV()), "star count");
        c.star_ptr.alloc(nc + 1);
        DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(nc));
        check(phfem_gpu_scan_i32(cnt.p, c.star_ptr.p, nc, scratch.p, SV()), "star scan");
        DBuf<int64_t> cursor(nc);
        if (nc) check(cudaMemcpyAsync(cursor.p, c.star_ptr.p, sizeof(int64_t) * nc, cudaMemcpyDeviceToDevice, S()), "D2D");
        c.star.alloc(4 * ne);
        check(phfem_gpu_star_fill(m.tets.p, ne, cursor.p, c.star.p, SV()), "star fill");
    }
    if (st) st->star += tm.stop_ms();
    // 2. per-vertex grouping of edges and faces
    tm.start();
    c.edge_first.alloc(6 * ne);
    if (faces) c.slot_mate.alloc(4 * ne);
    {
        DBuf<int32_t> big_list(nc > 0 ? nc : 1), big_count(1);
        big_count.zero();
        check(phfem_gpu_star_groups(nc, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                    faces ? c.slot_mate.p : nullptr, big_list.p, big_count.p, err.d.p, SV()),
              "star groups");
        const int32_t n_big = read_scalar(big_count.p);
        if (n_big > 0) {
            std::vector<int32_t> big((size_t)n_big);
            check(cudaMemcpyAsync(big.data(), big_list.p, sizeof(int32_t) * n_big, cudaMemcpyDeviceToHost, S()), "D2H");
            const std::vector<int64_t> ptr = c.star_ptr.download();
            int max_star = 0;
            for (int32_t v : big) max_star = std::max<int>(max_star, (int)(ptr[v + 1] - ptr[v]));
            check(phfem_gpu_star_groups_big(n_big, big_list.p, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                            faces ? c.slot_mate.p : nullptr, max_star, err.d.p, SV()),
                  "star groups (big)");
        }
    }
    if (st) st->groups += tm.stop_ms();
    // 3. numbering: element scans, ids, remaining slots
    tm.start();
    c.edge_off.alloc(ne + 1);
    DBuf<int64_t> face_off;
    {
        DBuf<int32_t> ecount(ne), fcount(faces ? ne : 0);
        check(phfem_gpu_element_counts(ne, c.edge_first.p, faces ? c.slot_mate.p : nullptr, ecount.p,
                                       faces ? fcount.p : nullptr, SV()),
              "element counts");
        DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(ne));
        check(phfem_gpu_scan_i32(ecount.p, c.edge_off.p, ne, scratch.p, SV()), "edge scan");
        if (faces) {
            face_off.alloc(ne + 1);
            check(phfem_gpu_scan_i32(fcount.p, face_off.p, ne, scratch.p, SV()), "face scan");
        }
        c.ned = read_scalar(c.edge_off.p + ne);
        if (faces) c.nf = read_scalar(face_off.p + ne);
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
    check(phfem_gpu_number(ne, m.tets.p, m.coords.p, c.edge_first.p, c.edge_off.p, c.edge_of_slot.p, c.edge_nodes.p,
                           faces ? c.slot_mate.p : nullptr, faces ? face_off.p : nullptr,
                           faces ? c.face_of_slot.p : nullptr, faces ? c.sigma.p : nullptr,
                           faces ? c.faces.p : nullptr, faces ? c.face_slots.p : nullptr,
                           faces ? c.face_area.p : nullptr, err.d.p, SV()),
          "number");
    check(phfem_gpu_fill_slots(ne, c.edge_first.p, c.edge_of_slot.p, faces ? c.slot_mate.p : nullptr,
                               faces ? c.face_of_slot.p : nullptr, faces ? c.sigma.p : nullptr, SV()),
          "fill slots");
    if (st) st->number += tm.stop_ms();
    c.has_edges = true;
    c.t_edges = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    if (!faces) {
        const auto e = err.get();
        replay_connectivity_errors(e, m, c);
        return;
    }
    // 4. boundary classification and multiplier rows
    const auto w1 = std::chrono::steady_clock::now();
    tm.start();
    {
        const int64_t nf = c.nf;
        DBuf<uint32_t> claim(nf);
        claim.fill_bytes(0xff);
        check(phfem_gpu_classify(m.nd, m.db.p, m.nn, m.nb.p, c.star_ptr.p, c.star.p, m.tets.p, c.face_of_slot.p,
                                 c.face_slots.p, claim.p, err.d.p, SV()),
              "classify");
        check(phfem_gpu_classify_check(m.nd, m.db.p, m.nn, m.nb.p, c.star_ptr.p, c.star.p, m.tets.p,
                                       c.face_of_slot.p, claim.p, err.d.p, SV()),
              "classify check");
        c.face_class.alloc(nf);
        DBuf<int32_t> is_row(nf);
        DBuf<unsigned long long> counts(3);
        counts.zero();
        check(phfem_gpu_face_class(nf, m.nd, claim.p, c.face_slots.p, c.face_area.p, c.face_class.p, is_row.p,
                                   counts.p, err.d.p, SV()),
              "face class");
        DBuf<int64_t> row_off(nf + 1);
        DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(nf));
        check(phfem_gpu_scan_i32(is_row.p, row_off.p, nf, scratch.p, SV()), "row scan");
        const std::vector<unsigned long long> cnt = counts.download();
        c.l = read_scalar(row_off.p + nf);
        c.n_int = (int64_t)cnt[0];
        c.n_dir = (int64_t)cnt[1];
        c.n_neu = (int64_t)cnt[2];
        c.face_mrow.alloc(nf);
        c.row_face.alloc(c.l);
        check(phfem_gpu_face_rows(nf, c.face_class.p, row_off.p, c.face_mrow.p, c.row_face.p, SV()), "face rows");
    }
    if (st) st->classify += tm.stop_ms();
    const auto e = err.get();
    replay_connectivity_errors(e, m, c);
    c.has_faces = true;
    c.t_faces = std::chrono::duration<double>(std::chrono::steady_clock::now() - w1).count();
}

// -------------------------------------------------------------- refinement

std::shared_ptr<MeshData> refine_mesh(const MeshData& m, const Connectivity& c, RefineMap* map, Stages* st) {
    if (!c.has_edges) throw MeshError("refine_mesh: edge table missing");
    const int64_t nc2 = m.nc + c.ned + m.ne;
    const int64_t ne2 = 12 * m.ne;
    if (nc2 >= (int64_t)INT32_MAX || 6 * ne2 >= (int64_t)INT32_MAX)
        throw MeshError("out of memory while refining to level " + std::to_string(m.level + 1) +
                        ": 32-bit node/element ids exhausted");
    Timer tm;
    tm.start();
    auto out = std::make_shared<MeshData>();
    out->nc = nc2;
    out->ne = ne2;
    out->nd = 4 * m.nd;
    out->nn = 4 * m.nn;
    out->level = m.level + 1;
    out->coords.alloc(3 * nc2);
    out->tets.alloc(4 * ne2);
    out->db.alloc(3 * out->nd);
    out->nb.alloc(3 * out->nn);
    if (map) {
        map->midpoint.alloc(c.ned);
        map->centroid.alloc(m.ne);
    }
    ErrVec err;
    check(phfem_gpu_refine(m.nc, m.ne, m.coords.p, m.tets.p, c.edge_first.p, c.edge_of_slot.p, c.edge_off.p,
                           out->coords.p, out->tets.p, map ? map->midpoint.p : nullptr,
                           map ? map->centroid.p : nullptr, SV()),
          "refine");
    check(phfem_gpu_refine_boundary(m.nd, m.db.p, 0, m.nc, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                    c.edge_of_slot.p, out->db.p, err.d.p, SV()),
          "refine boundary");
    check(phfem_gpu_refine_boundary(m.nn, m.nb.p, m.nd, m.nc, c.star_ptr.p, c.star.p, m.tets.p, c.edge_first.p,
                                    c.edge_of_slot.p, out->nb.p, err.d.p, SV()),
          "refine boundary");
    const double ms = tm.stop_ms();
    if (st) st->refine += ms;
    const auto e = err.get();
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

void assemble_system(const MeshData& m, const Coefs& k, const Connectivity& c, int problem, System& sys,
                     bool debug_views, Stages* st) {
    if (!c.has_faces) throw MeshError("assemble: face table missing");
    if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
    Timer tm;
    tm.start();
    sys.problem = problem;
    sys.coef_version = k.version;
    sys.n = 4 * m.ne;
    sys.l = c.l;
    sys.nchunks = (c.l + PHG_SELL_C - 1) / PHG_SELL_C;
    const int64_t width = PHG_SELL_C * PHG_SELL_W;
    sys.sell_col.alloc(sys.nchunks * width);
    sys.sell_val.alloc(sys.nchunks * width);
    if (sys.nchunks)
        check(cudaMemset2DAsync(sys.sell_val.p, width * sizeof(double), 0, PHG_SELL_C * sizeof(double),
                                (size_t)sys.nchunks, S()),
              "memset diag");
    sys.rhs_neg.alloc(c.l);
    sys.rhs_neg.zero();
    sys.bd.alloc(c.l);
    sys.bd.zero();
    sys.rhs.alloc(4 * m.ne);
    if (debug_views) {
        sys.a_blocks.alloc(16 * m.ne);
        sys.slot_coef.alloc(4 * m.ne);
        sys.slot_mrow.alloc(4 * m.ne);
    } else {
        sys.a_blocks.release();
        sys.slot_coef.release();
        sys.slot_mrow.release();
    }
    const int grid = phfem_gpu_assemble_grid(m.ne);
    DBuf<double> partials(2 * (int64_t)grid), norms(2);
    ErrVec err;
    const phg_problem p = device_problem(k, problem);
    check(phfem_gpu_assemble_condense(m.ne, m.coords.p, m.tets.p, &p, c.face_of_slot.p, c.slot_mate.p,
                                      c.face_mrow.p, c.face_area.p, sys.sell_col.p, sys.sell_val.p, sys.rhs_neg.p,
                                      sys.bd.p, sys.rhs.p, debug_views ? sys.a_blocks.p : nullptr,
                                      debug_views ? sys.slot_coef.p : nullptr,
                                      debug_views ? sys.slot_mrow.p : nullptr, norms.p, partials.p, err.d.p, SV()),
          "assemble");
    const double ms = tm.stop_ms();
    if (st) st->assemble += ms;
    const std::vector<double> nv = norms.download();
    sys.sum_rhs2 = nv[0];
    sys.sum_bd2 = nv[1];
    const auto e = err.get();
    // assembly.cpp:13-14 (first element in order), then solver.cpp:128-129
    if (e[PHG_ERR_ZERO_VOLUME] != kNone)
        throw MeshError("degenerate element " + std::to_string(e[PHG_ERR_ZERO_VOLUME] + 1) + " (zero volume)");
    if (e[PHG_ERR_SINGULAR] != kNone)
        throw MeshError("degenerate element block " + std::to_string(e[PHG_ERR_SINGULAR] + 1));
}

// ------------------------------------------------------------------- solve

void solve_schur(const MeshData& m, const Coefs& k, const Connectivity& c, const System& sys, int problem,
                 double tol, int64_t max_iter, const std::string& method, SolveResult& out) {
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t l = sys.l;
    const double nrm_rhs = std::sqrt(sys.sum_rhs2), nrm_bd = std::sqrt(sys.sum_bd2);
    // inner_cg_options, solver.cpp:78-86
    const double abs_tol = 0.2 * tol * std::hypot(nrm_rhs, nrm_bd);
    const long long mi = max_iter > 0 ? max_iter : 10 * std::max<int64_t>(l, 1);
    out.lambda.alloc(l);
    DBuf<double> r(l), p(l), q(l), d(l);
    DBuf<phg_cg_state> state(1);
    DBuf<double> partials(2 * 148 * 8 + 64);
    Timer tm;
    tm.start();
    check(phfem_gpu_cg_init(l, sys.sell_col.p, sys.sell_val.p, sys.rhs_neg.p, out.lambda.p, r.p, p.p, d.p, tol,
                            abs_tol, mi, state.p, partials.p, SV()),
          "cg init");
    phg_cg_state hs{};
    phg_cg_state* pinned = nullptr;
    check(cudaMallocHost(reinterpret_cast<void**>(&pinned), sizeof(phg_cg_state)), "pinned alloc");
    const int batch = l < 200000 ? 32 : 16;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    try {
        check(cudaMemcpyAsync(pinned, state.p, sizeof(phg_cg_state), cudaMemcpyDeviceToHost, S()), "D2H");
        sync();
        hs = *pinned;
        if (!hs.done) {
            check(cudaStreamBeginCapture(S(), cudaStreamCaptureModeThreadLocal), "capture");
            phfem_gpu_cg_iterations(batch, l, sys.sell_col.p, sys.sell_val.p, out.lambda.p, r.p, p.p, q.p, d.p,
                                    state.p, partials.p, SV());
            check(cudaStreamEndCapture(S(), &graph), "capture end");
            check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
            for (;;) {
                check(cudaGraphLaunch(exec, S()), "graph launch");
                check(cudaMemcpyAsync(pinned, state.p, sizeof(phg_cg_state), cudaMemcpyDeviceToHost, S()), "D2H");
                sync();
                hs = *pinned;
                if (hs.done) break;
            }
        }
    } catch (...) {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        cudaFreeHost(pinned);
        throw;
    }
    out.cg_ms = tm.stop_ms();
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaFreeHost(pinned);
    out.iterations = hs.it;
    out.converged = hs.converged != 0;
    if (hs.not_spd) throw SolverError("pcg: operator is not positive definite");
    if (!hs.converged) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "%f", hs.rel_residual);
        throw SolverError("schur: conjugate gradients stalled at relative residual " + std::string(buf) + " after " +
                          std::to_string(hs.it) + " iterations");
    }
    // recovery + verify_solution (solver.cpp:44-76, 168-181)
    out.u.alloc(4 * m.ne);
    const phg_problem pr = device_problem(k, problem);
    DBuf<double> rpart(148 * 16 * 3 + 64), sums(1), cres(3);
    ErrVec err;
    check(phfem_gpu_recover(m.ne, m.coords.p, m.tets.p, &pr, c.face_of_slot.p, c.slot_mate.p, c.face_mrow.p,
                            c.face_area.p, sys.rhs.p, out.lambda.p, out.u.p, sums.p, rpart.p, err.d.p, SV()),
          "recover");
    const std::vector<double> s1 = sums.download();
    check(phfem_gpu_constraint_residual(l, c.row_face.p, c.face_slots.p, c.slot_mate.p, c.face_of_slot.p,
                                        c.face_area.p, m.tets.p, out.u.p, sys.bd.p, cres.p, rpart.p, SV()),
          "constraint residual");
    const std::vector<double> s2 = cres.download();
    const double r1 = std::sqrt(s1[0]), r2 = std::sqrt(s2[0]);
    const double rhs_norm = std::hypot(nrm_rhs, nrm_bd);
    const double res_norm = std::hypot(r1, r2);
    out.residual = rhs_norm > 0.0 ? res_norm / rhs_norm : res_norm;
    out.constraint_residual = s2[1] / (1.0 + s2[2]);
    const bool ok = out.residual <= tol && r1 <= tol * std::max(nrm_rhs, 1e-300) && r2 <= tol * (1.0 + nrm_bd);
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!ok) {
        char buf[200];
        std::snprintf(buf, sizeof buf, "solver '%s' missed the residual target: %g > %g", method.c_str(),
                      out.residual, tol);
        throw SolverError(buf);
    }
}

// ------------------------------------------------------------------ norms

double mesh_diameter(const MeshData& m) {
    if (m.ne == 0) throw MeshError("mesh_diameter on empty mesh");
    DBuf<double> h(1);
    check(phfem_gpu_diameter(m.coords.p, m.tets.p, m.ne, h.p, nullptr, SV()), "diameter");
    return h.download()[0];
}

void error_norms(const MeshData& m, const Coefs& k, const Connectivity& c, int problem, const double* u,
                 const double* lambda, double out[3]) {
    const double h = mesh_diameter(m);
    DBuf<double> partials(148 * 16 * 3 + 64), res(3);
    const phg_problem p = device_problem(k, problem);
    check(phfem_gpu_errors(m.ne, m.coords.p, m.tets.p, &p, c.face_of_slot.p, c.slot_mate.p, c.face_mrow.p, u, lambda,
                           h, res.p, partials.p, SV()),
          "errors");
    const std::vector<double> v = res.download();
    for (int i = 0; i < 3; ++i) out[i] = std::sqrt(v[i]);
}

}  // namespace phb
