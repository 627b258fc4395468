// The reference's value-returning C++ API (namespace phfem, declared in
// include/phfem_cxx/*.hpp, the drop-in for /root/reference/proj/src/*.hpp)
// over the B200 runtime.  Host structs go up, the sm_100a kernels do the
// batched work (runtime.cpp / pipeline.cpp for the connectivity and
// refinement the C ABI also uses, api.cu for the operations that start from
// host structs), results come back by D2H copies.  What stays on the host:
// single-element / single-face geometry queries, the text and VTK writers,
// the quadrature tables, evaluating the caller's std::function data at
// device-computed points, and filling the host-side lookup structures the
// API exposes as fields (EdgeTable::pair_map).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <fstream>
#include <numeric>
#include <ostream>
#include <sstream>

#include "phfem_cxx/analysis.hpp"
#include "phfem_cxx/assembly.hpp"
#include "phfem_cxx/connectivity.hpp"
#include "phfem_cxx/mesh.hpp"
#include "phfem_cxx/quadrature.hpp"
#include "phfem_cxx/refine.hpp"
#include "phfem_cxx/solver.hpp"
#include "phfem_cxx/sparse.hpp"
#include "phfem_cxx/vtk.hpp"
#include "runtime.hpp"

namespace phfem {

namespace {

using phb::DBuf;
using phb::check;

constexpr unsigned long long kNone = ULLONG_MAX;

static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
static_assert(sizeof(Tet4) == 4 * sizeof(int32_t) && sizeof(Tri3) == 3 * sizeof(int32_t), "packed index tuples");

const double* flat(const std::vector<Vec3>& v) { return v.empty() ? nullptr : &v[0].x; }
const int32_t* flat(const std::vector<Tet4>& v) { return v.empty() ? nullptr : v[0].data(); }
const int32_t* flat(const std::vector<Tri3>& v) { return v.empty() ? nullptr : v[0].data(); }

std::shared_ptr<phb::MeshData> upload(const Mesh& m) {
    return phb::upload_mesh(flat(m.coords), m.num_nodes(), flat(m.tetra), m.num_elems(), flat(m.dirichlet_faces),
                            (int64_t)m.dirichlet_faces.size(), flat(m.neumann_faces),
                            (int64_t)m.neumann_faces.size(), m.level);
}

template <class T>
void put(DBuf<T>& d, const T* h, int64_t n) {
    d.alloc(n > 0 ? n : 1);
    if (n > 0) check(cudaMemcpyAsync(d.p, h, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, phb::S()), "H2D");
}
template <class T>
void get(const DBuf<T>& d, T* h, int64_t n) {
    if (n > 0) d.download_to(h, n);
}
template <class T>
T get1(const T* dptr) {
    T v;
    check(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, phb::S()), "D2H");
    phb::sync();
    return v;
}

void* scan_scratch(DBuf<unsigned char>& s, int64_t n) {
    s.alloc((int64_t)phfem_gpu_scan_scratch(n > 0 ? n : 1));
    return s.p;
}

// Device CSR: row_ptr int64, col int32, val double
struct DCsr {
    int64_t rows = 0, cols = 0, nnz = 0;
    DBuf<int64_t> ptr;
    DBuf<int32_t> col;
    DBuf<double> val;
};

void up(const CsrMatrix& a, DCsr& d) {
    d.rows = a.n_rows;
    d.cols = a.n_cols;
    d.nnz = a.nnz();
    if ((int64_t)a.row_ptr.size() != a.n_rows + 1) throw InvalidArgument("CsrMatrix: row_ptr size must be n_rows + 1");
    put(d.ptr, a.row_ptr.data(), a.n_rows + 1);
    put(d.col, a.col.data(), d.nnz);
    put(d.val, a.val.data(), d.nnz);
}

CsrMatrix down(const DCsr& d) {
    CsrMatrix a;
    a.n_rows = d.rows;
    a.n_cols = d.cols;
    a.row_ptr.resize(d.rows + 1);
    a.col.resize(d.nnz);
    a.val.resize(d.nnz);
    get(d.ptr, a.row_ptr.data(), d.rows + 1);
    get(d.col, a.col.data(), d.nnz);
    get(d.val, a.val.data(), d.nnz);
    phb::sync();
    return a;
}

// from_triplets on the device (sparse.cpp:12-44): group by row, sort each
// row by (column, insertion index), sum duplicates in insertion order
void triplets_to_csr(int64_t rows, int64_t cols, int64_t n, const DBuf<int64_t>& trow, const DBuf<int64_t>& tcol,
                     const DBuf<double>& tval, DCsr& out) {
    DBuf<int64_t> seg_ptr(rows + 1), perm(n > 0 ? n : 1), tmp(n > 0 ? n : 1);
    DBuf<int32_t> cnt(rows > 0 ? rows : 1);
    DBuf<unsigned char> ss;
    check(phfem_gpu_seg_sort(n, rows, trow.p, tcol.p, seg_ptr.p, perm.p, cnt.p, tmp.p, scan_scratch(ss, rows), phb::SV()),
          "triplet sort");
    check(phfem_gpu_csr_unique(rows, seg_ptr.p, perm.p, tcol.p, cnt.p, phb::SV()), "triplet unique");
    out.rows = rows;
    out.cols = cols;
    out.ptr.alloc(rows + 1);
    check(phfem_gpu_scan_i32(cnt.p, out.ptr.p, rows, scan_scratch(ss, rows), phb::SV()), "triplet scan");
    out.nnz = get1(out.ptr.p + rows);
    out.col.alloc(out.nnz > 0 ? out.nnz : 1);
    out.val.alloc(out.nnz > 0 ? out.nnz : 1);
    check(phfem_gpu_csr_write(rows, seg_ptr.p, perm.p, tcol.p, tval.p, out.ptr.p, out.col.p, out.val.p, phb::SV()),
          "triplet write");
}

void transpose_dev(const DCsr& a, DCsr& t) {
    DBuf<int64_t> rowof(a.nnz > 0 ? a.nnz : 1), idx(a.nnz > 0 ? a.nnz : 1), colw(a.nnz > 0 ? a.nnz : 1);
    DBuf<int64_t> perm(a.nnz > 0 ? a.nnz : 1), tmp(a.nnz > 0 ? a.nnz : 1);
    DBuf<int32_t> cnt(a.cols > 0 ? a.cols : 1);
    DBuf<unsigned char> ss;
    check(phfem_gpu_csr_rowof(a.rows, a.ptr.p, rowof.p, phb::SV()), "rowof");
    check(phfem_gpu_widen(a.nnz, a.col.p, colw.p, phb::SV()), "widen");
    // minor key = the entry index: a column's entries keep storage order
    std::vector<int64_t> iota((size_t)a.nnz);
    std::iota(iota.begin(), iota.end(), 0);
    put(idx, iota.data(), a.nnz);
    t.rows = a.cols;
    t.cols = a.rows;
    t.nnz = a.nnz;
    t.ptr.alloc(a.cols + 1);
    check(phfem_gpu_seg_sort(a.nnz, a.cols, colw.p, idx.p, t.ptr.p, perm.p, cnt.p, tmp.p, scan_scratch(ss, a.cols),
                             phb::SV()),
          "transpose sort");
    t.col.alloc(a.nnz > 0 ? a.nnz : 1);
    t.val.alloc(a.nnz > 0 ? a.nnz : 1);
    check(phfem_gpu_csr_transpose(a.nnz, perm.p, rowof.p, a.val.p, t.col.p, t.val.p, phb::SV()), "transpose");
}

void spgemm_dev(const DCsr& a, const DCsr& b, DCsr& c) {
    if (a.cols != b.rows) throw InvalidArgument("spgemm: dimension mismatch");
    DBuf<int32_t> cnt(a.rows > 0 ? a.rows : 1);
    DBuf<int64_t> pptr(a.rows + 1);
    DBuf<unsigned char> ss;
    check(phfem_gpu_spgemm_count(a.rows, a.ptr.p, a.col.p, b.ptr.p, cnt.p, phb::SV()), "spgemm count");
    check(phfem_gpu_scan_i32(cnt.p, pptr.p, a.rows, scan_scratch(ss, a.rows), phb::SV()), "spgemm scan");
    const int64_t np = get1(pptr.p + a.rows);
    DBuf<int64_t> pcol(np > 0 ? np : 1), perm(np > 0 ? np : 1), tmp(np > 0 ? np : 1);
    DBuf<double> pval(np > 0 ? np : 1);
    check(phfem_gpu_spgemm_fill(a.rows, a.ptr.p, a.col.p, a.val.p, b.ptr.p, b.col.p, b.val.p, pptr.p, pcol.p, pval.p,
                                phb::SV()),
          "spgemm fill");
    check(phfem_gpu_sort_within(np, a.rows, pptr.p, pcol.p, perm.p, tmp.p, phb::SV()), "spgemm sort");
    check(phfem_gpu_csr_unique(a.rows, pptr.p, perm.p, pcol.p, cnt.p, phb::SV()), "spgemm unique");
    c.rows = a.rows;
    c.cols = b.cols;
    c.ptr.alloc(a.rows + 1);
    check(phfem_gpu_scan_i32(cnt.p, c.ptr.p, a.rows, scan_scratch(ss, a.rows), phb::SV()), "spgemm scan");
    c.nnz = get1(c.ptr.p + a.rows);
    c.col.alloc(c.nnz > 0 ? c.nnz : 1);
    c.val.alloc(c.nnz > 0 ? c.nnz : 1);
    check(phfem_gpu_spgemm_write(a.rows, pptr.p, perm.p, pcol.p, pval.p, c.ptr.p, c.col.p, c.val.p, phb::SV()),
          "spgemm write");
}

// deterministic device sum of a vector (sum of the per-element partials)
double sumsq_sum(const double* dx, int64_t n) {
    DBuf<double> part(2 * phfem_gpu_sumsq_max_partials()), out(1);
    check(phfem_gpu_sum(n, dx, part.p, out.p, phb::SV()), "sum");
    return get1(out.p);
}

// deterministic device sum of squares and max |x|
std::pair<double, double> sumsq_max(const double* dx, int64_t n) {
    DBuf<double> part(2 * phfem_gpu_sumsq_max_partials()), out(2);
    check(phfem_gpu_sumsq_max(n, dx, part.p, out.p, phb::SV()), "norm");
    double h[2];
    out.download_to(h, 2);
    phb::sync();
    return {h[0], h[1]};
}

// Jacobi-PCG on a device CSR matrix (pcg_jacobi, sparse.cpp:163-212): the
// SELL path's vector kernels with a CSR SpMV; batches of iterations in a
// CUDA graph, the stop flag polled once per batch
CgResult pcg_dev(const DCsr& a, const double* db, double* dx, const CgOptions& opt) {
    const int64_t n = a.rows;
    const long long mi = opt.max_iter > 0 ? opt.max_iter : 10 * n;
    DBuf<double> r(n > 0 ? n : 1), p(n > 0 ? n : 1), q(n > 0 ? n : 1), d(n > 0 ? n : 1);
    DBuf<phg_cg_state> st(1);
    DBuf<double> partials(2 * 148 * 8 + 64);
    check(phfem_gpu_cgcsr_init(n, a.ptr.p, a.col.p, a.val.p, db, dx, r.p, p.p, d.p, opt.tol, opt.abs_tol, mi, st.p,
                               partials.p, phb::SV()),
          "cg init");
    phg_cg_state hs = get1(st.p);
    const int batch = 16;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    try {
        if (!hs.done) {
            check(cudaStreamBeginCapture(phb::S(), cudaStreamCaptureModeThreadLocal), "capture");
            phfem_gpu_cgcsr_iterations(batch, n, a.ptr.p, a.col.p, a.val.p, dx, r.p, p.p, q.p, d.p, st.p, partials.p,
                                       phb::SV());
            check(cudaStreamEndCapture(phb::S(), &graph), "capture end");
            check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
            while (!hs.done) {
                check(cudaGraphLaunch(exec, phb::S()), "graph launch");
                hs = get1(st.p);
            }
        }
    } catch (...) {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (hs.not_spd) throw SolverError("pcg: operator is not positive definite");
    CgResult res;
    res.iterations = hs.it;
    res.rel_residual = hs.rel_residual;
    res.converged = hs.converged != 0;
    return res;
}

std::string tri_str(const Tri3& f) {
    return "[" + std::to_string(f[0] + 1) + " " + std::to_string(f[1] + 1) + " " + std::to_string(f[2] + 1) + "]";
}

}  // namespace

// =================================================================== mesh

Mesh initial_cube_mesh() {  // mesh.cpp:12-32
    Mesh m;
    for (int i = 0; i < 8; ++i) m.coords.emplace_back(double(i & 1), double((i >> 1) & 1), double((i >> 2) & 1));
    const int t[5][4] = {{1, 2, 3, 5}, {5, 8, 6, 2}, {7, 3, 8, 5}, {4, 8, 3, 2}, {8, 3, 2, 5}};
    const int d[2][3] = {{7, 8, 5}, {5, 8, 6}};
    const int nb[10][3] = {{1, 5, 2}, {5, 6, 2}, {1, 3, 5}, {7, 5, 3}, {7, 3, 8},
                           {4, 8, 3}, {2, 6, 8}, {4, 2, 8}, {4, 3, 2}, {1, 2, 3}};
    for (const auto& e : t) m.tetra.push_back({e[0] - 1, e[1] - 1, e[2] - 1, e[3] - 1});
    for (const auto& f : d) m.dirichlet_faces.push_back({f[0] - 1, f[1] - 1, f[2] - 1});
    for (const auto& f : nb) m.neumann_faces.push_back({f[0] - 1, f[1] - 1, f[2] - 1});
    return m;
}

std::array<Tri3, 4> elem_oriented_faces(const Tet4& t) {
    std::array<Tri3, 4> f;
    for (int k = 0; k < 4; ++k) f[k] = {t[kFaceVerts[k][0]], t[kFaceVerts[k][1]], t[kFaceVerts[k][2]]};
    return f;
}

double signed_volume6(const Mesh& mesh, ElemId t) {
    const Tet4& e = mesh.tetra[t];
    const Vec3& a = mesh.coords[e[0]];
    return dot(cross(mesh.coords[e[1]] - a, mesh.coords[e[2]] - a), mesh.coords[e[3]] - a);
}

double elem_volume(const Mesh& mesh, ElemId t) { return std::fabs(signed_volume6(mesh, t)) / 6.0; }

bool elem_is_oriented(const Mesh& mesh, ElemId t) {  // mesh.cpp:51-66
    const Tet4& e = mesh.tetra[t];
    for (int k = 0; k < 4; ++k) {
        const Vec3& a = mesh.coords[e[kFaceVerts[k][0]]];
        const Vec3& b = mesh.coords[e[kFaceVerts[k][1]]];
        const Vec3& c = mesh.coords[e[kFaceVerts[k][2]]];
        // the vertex off face k: 3 for faces 0-2, 0 for face 3 (by node id,
        // as the reference picks it)
        NodeId off = -1;
        for (NodeId n : e)
            if (n != e[kFaceVerts[k][0]] && n != e[kFaceVerts[k][1]] && n != e[kFaceVerts[k][2]]) off = n;
        if (off < 0) return false;
        if (dot(cross(c - a, b - a), mesh.coords[off] - a) >= 0.0) return false;
    }
    return true;
}

void validate_orientation(const Mesh& mesh) {  // mesh.cpp:68-74
    for (ElemId t = 0; t < mesh.num_elems(); ++t) {
        if (signed_volume6(mesh, t) <= 0.0)
            throw MeshError("element " + std::to_string(t + 1) +
                            " violates the orientation convention (signed 6-volume <= 0)");
        if (!elem_is_oriented(mesh, t))
            throw MeshError("element " + std::to_string(t + 1) + " has a non-outward oriented face");
    }
}

FaceGeometry face_area_and_normal(const Mesh& mesh, const Tri3& f) {  // mesh.cpp:76-84
    const Vec3& a = mesh.coords[f[0]];
    const Vec3 n = cross(mesh.coords[f[2]] - a, mesh.coords[f[1]] - a);
    const double len = norm(n);
    if (len == 0.0) throw MeshError("degenerate face with collinear nodes " + tri_str(f));
    return {0.5 * len, n / len};
}

Vec3 face_centroid(const Mesh& mesh, const Tri3& f) {
    return (mesh.coords[f[0]] + mesh.coords[f[1]] + mesh.coords[f[2]]) / 3.0;
}

double elem_diameter(const Mesh& mesh, ElemId t) {
    const Tet4& e = mesh.tetra[t];
    double m2 = 0.0;
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j) {
            const Vec3 d = mesh.coords[e[i]] - mesh.coords[e[j]];
            m2 = std::max(m2, dot(d, d));
        }
    return std::sqrt(m2);
}

double mesh_diameter(const Mesh& mesh) {
    if (mesh.tetra.empty()) throw MeshError("mesh_diameter on empty mesh");
    return phb::mesh_diameter(*upload(mesh));
}

std::string format_double(double v) { return phb::format_double(v); }

void write_mesh(std::ostream& os, const Mesh& mesh) {  // mesh.cpp:117-130
    os << "COORD " << mesh.coords.size() << "\n";
    for (const Vec3& p : mesh.coords)
        os << format_double(p.x) << ' ' << format_double(p.y) << ' ' << format_double(p.z) << "\n";
    os << "TETRA " << mesh.tetra.size() << "\n";
    for (const Tet4& t : mesh.tetra) os << t[0] + 1 << ' ' << t[1] + 1 << ' ' << t[2] + 1 << ' ' << t[3] + 1 << "\n";
    for (const auto* list : {&mesh.dirichlet_faces, &mesh.neumann_faces}) {
        os << (list == &mesh.dirichlet_faces ? "DB " : "NB ") << list->size() << "\n";
        for (const Tri3& f : *list) os << f[0] + 1 << ' ' << f[1] + 1 << ' ' << f[2] + 1 << "\n";
    }
}

void write_mesh_file(const std::string& path, const Mesh& mesh) {
    std::ofstream os(path);
    if (!os) throw IoError("cannot open '" + path + "' for writing");
    write_mesh(os, mesh);
    if (!os) throw IoError("write failure on '" + path + "'");
}

Mesh read_mesh(std::istream& is) {  // mesh.cpp:139-182
    auto section = [&](const char* name) -> size_t {
        std::string tok;
        if (!(is >> tok) || tok != name)
            throw IoError(std::string("mesh format: expected section '") + name + "', got '" + tok + "'");
        long long n = -1;
        if (!(is >> n) || n < 0) throw IoError(std::string("mesh format: bad row count for section '") + name + "'");
        return (size_t)n;
    };
    Mesh m;
    m.coords.resize(section("COORD"));
    for (Vec3& p : m.coords)
        if (!(is >> p.x >> p.y >> p.z)) throw IoError("mesh format: bad coordinate row");
    auto index = [&](NodeId& out) {
        long long v;
        if (!(is >> v)) throw IoError("mesh format: expected a node index");
        if (v < 1 || v > m.num_nodes())
            throw IoError("mesh format: node index " + std::to_string(v) + " out of range 1.." +
                          std::to_string(m.num_nodes()));
        out = (NodeId)(v - 1);
    };
    m.tetra.resize(section("TETRA"));
    for (Tet4& t : m.tetra)
        for (NodeId& v : t) index(v);
    m.dirichlet_faces.resize(section("DB"));
    for (Tri3& f : m.dirichlet_faces)
        for (NodeId& v : f) index(v);
    m.neumann_faces.resize(section("NB"));
    for (Tri3& f : m.neumann_faces)
        for (NodeId& v : f) index(v);
    return m;
}

Mesh read_mesh_file(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw IoError("cannot open '" + path + "' for reading");
    return read_mesh(is);
}

// ============================================================= quadrature

QuadRule1d gauss_legendre(int n) {
    if (n < 1) throw InvalidArgument("gauss_legendre: n must be positive");
    QuadRule1d r;
    phb::gauss_legendre(n, r.x, r.w);
    return r;
}

TetRule tet_rule(int degree) {
    if (degree < 1) throw InvalidArgument("tet_rule: degree must be positive");
    std::vector<double> lam, w;
    phb::tet_rule(degree, lam, w);
    TetRule r;
    r.exact_degree = 2 * ((degree + 4) / 2) - 3;
    r.points.resize(w.size());
    for (size_t q = 0; q < w.size(); ++q) {
        for (int i = 0; i < 4; ++i) r.points[q].lambda[i] = lam[4 * q + i];
        r.points[q].w = w[q];
    }
    return r;
}

TriRule tri_midpoint_rule() {
    TriRule r;
    r.points[0] = {{0.5, 0.5, 0.0}, 1.0 / 3.0};
    r.points[1] = {{0.0, 0.5, 0.5}, 1.0 / 3.0};
    r.points[2] = {{0.5, 0.0, 0.5}, 1.0 / 3.0};
    return r;
}

// =========================================================== connectivity

EdgeTable num_edges(const Mesh& mesh) {
    auto m = upload(mesh);
    phb::Connectivity c;
    phb::build_connectivity(*m, c, false);
    EdgeTable tab;
    tab.n_nodes = mesh.num_nodes();
    tab.edge_nodes.resize(c.ned);
    if (c.ned) c.edge_nodes.download_to(tab.edge_nodes[0].data(), 2 * c.ned);
    phb::sync();
    tab.pair_map.reserve((size_t)c.ned);
    for (EdgeId e = 0; e < (EdgeId)c.ned; ++e)
        tab.pair_map.emplace(uint64_t(tab.edge_nodes[e][0]) * uint64_t(tab.n_nodes) + uint64_t(tab.edge_nodes[e][1]), e);
    return tab;
}

ElemId EdgePairToElem::lookup(EdgeId from, EdgeId to) const {
    const uint64_t key = uint64_t(from) * uint64_t(n_edges) + uint64_t(to);
    const auto it = std::lower_bound(entries.begin(), entries.end(), key,
                                     [](const std::pair<uint64_t, ElemId>& e, uint64_t k) { return e.first < k; });
    return it != entries.end() && it->first == key ? it->second : -1;
}

namespace {
void check_edges(const Mesh& mesh, const EdgeTable& edges, int64_t ned, const char* who) {
    if (edges.n_edges() != ned || edges.n_nodes != mesh.num_nodes())
        throw InvalidArgument(std::string(who) + ": the edge table does not belong to this mesh");
}
}  // namespace

// The E2T map on demand (connectivity.cpp:46-70): entries from the device
// edge ids, grouped by the first edge, each group sorted by (second edge,
// entry index) = the reference's sorted (key, element) order
EdgePairToElem edge_pairs_to_elems(const Mesh& mesh, const EdgeTable& edges) {
    auto m = upload(mesh);
    phb::Connectivity c;
    phb::build_connectivity(*m, c, false);
    check_edges(mesh, edges, c.ned, "edge_pairs_to_elems");
    const int64_t ne = mesh.num_elems(), n = 12 * ne, ned = c.ned;
    EdgePairToElem map;
    map.n_edges = ned;
    // ned + 1 segments: the last holds the keys that wrap (phfem_gpu_e2t_entries)
    DBuf<int64_t> from(n > 0 ? n : 1), to(n > 0 ? n : 1), seg_ptr(ned + 2), perm(n > 0 ? n : 1), tmp(n > 0 ? n : 1);
    DBuf<int32_t> cnt(ned + 1), elem(n > 0 ? n : 1);
    DBuf<unsigned long long> key(n > 0 ? n : 1), dup(1);
    DBuf<unsigned char> ss;
    dup.fill_bytes(0xff);
    check(phfem_gpu_e2t_entries(ne, ned, c.edge_of_slot.p, c.edge_nodes.p, from.p, to.p, phb::SV()), "e2t entries");
    check(phfem_gpu_seg_sort(n, ned + 1, from.p, to.p, seg_ptr.p, perm.p, cnt.p, tmp.p, scan_scratch(ss, ned + 1),
                             phb::SV()),
          "e2t sort");
    check(phfem_gpu_e2t_finish(n, ned, perm.p, from.p, to.p, key.p, elem.p, dup.p, phb::SV()), "e2t finish");
    const unsigned long long j = get1(dup.p);
    if (j != kNone) {
        int32_t pair[2];
        check(cudaMemcpyAsync(pair, elem.p + j - 1, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, phb::S()), "D2H");
        phb::sync();
        throw MeshError("inconsistent mesh: elements " + std::to_string(pair[0] + 1) + " and " +
                        std::to_string(pair[1] + 1) + " claim the same oriented face");
    }
    std::vector<unsigned long long> hk((size_t)n);
    std::vector<int32_t> he((size_t)n);
    get(key, hk.data(), n);
    get(elem, he.data(), n);
    phb::sync();
    map.entries.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) map.entries[i] = {hk[i], he[i]};
    return map;
}

namespace {

// device face table -> host FaceTable (connectivity.hpp:57-77)
FaceTable face_table_of(const phb::Connectivity& c, int64_t ne) {
    FaceTable ft;
    const int64_t nf = c.nf;
    ft.faces.resize(nf);
    ft.face_area.resize(nf);
    ft.face_class.resize(nf);
    ft.multiplier_index.resize(nf);
    ft.face_slots.resize(nf);
    ft.slot_to_face.resize(4 * ne);
    ft.sigma.resize(4 * ne);
    std::vector<int32_t> fs(2 * nf);
    std::vector<int8_t> sg(4 * ne);
    std::vector<uint8_t> cls(nf);
    if (nf) {
        c.faces.download_to(ft.faces[0].data(), 3 * nf);
        c.face_area.download_to(ft.face_area.data(), nf);
        c.face_mrow.download_to(ft.multiplier_index.data(), nf);
        c.face_slots.download_to(fs.data(), 2 * nf);
        c.face_class.download_to(cls.data(), nf);
    }
    if (ne) {
        c.face_of_slot.download_to(ft.slot_to_face.data(), 4 * ne);
        c.sigma.download_to(sg.data(), 4 * ne);
    }
    phb::sync();
    for (int64_t f = 0; f < nf; ++f) {
        ft.face_slots[f] = {fs[2 * f], fs[2 * f + 1]};
        ft.face_class[f] = static_cast<FaceClass>(cls[f]);
    }
    for (int64_t s = 0; s < 4 * ne; ++s) ft.sigma[s] = sg[s];
    ft.n_interior = c.n_int;
    ft.n_dirichlet = c.n_dir;
    ft.n_neumann = c.n_neu;
    return ft;
}

}  // namespace

std::vector<Tri3> faces_up(const Mesh& mesh, const EdgePairToElem& e2t, const EdgeTable& edges) {
    auto m = upload(mesh);
    phb::Connectivity c;
    // the device numbering emits exactly the faces_up list: each face at the
    // rank of its owner (lower-element) slot, in the owner's orientation
    phb::build_connectivity(*m, c, true, nullptr, false);
    check_edges(mesh, edges, c.ned, "faces_up");
    if (e2t.n_edges != c.ned || (int64_t)e2t.entries.size() != 12 * mesh.num_elems())
        throw InvalidArgument("faces_up: the edge-pair map does not belong to this mesh");
    std::vector<Tri3> faces(c.nf);
    if (c.nf) c.faces.download_to(faces[0].data(), 3 * c.nf);
    phb::sync();
    return faces;
}

FaceTable full_face_table(const Mesh& mesh, const std::vector<Tri3>& faces) {
    auto m = upload(mesh);
    phb::Connectivity c;
    phb::build_connectivity(*m, c, true);
    FaceTable ft = face_table_of(c, mesh.num_elems());
    if (ft.faces != faces)
        throw InvalidArgument("full_face_table: `faces` must be faces_up() of this mesh");
    return ft;
}

FaceTable build_face_table(const Mesh& mesh) {
    auto m = upload(mesh);
    phb::Connectivity c;
    phb::build_connectivity(*m, c, true);
    return face_table_of(c, mesh.num_elems());
}

void dump_edges_csv(std::ostream& os, const EdgeTable& edges) {  // connectivity.cpp:211-215
    os << "edge_id,node1,node2\n";
    for (EdgeId e = 0; e < edges.n_edges(); ++e)
        os << e + 1 << ',' << edges.edge_nodes[e][0] + 1 << ',' << edges.edge_nodes[e][1] + 1 << "\n";
}

void dump_faces_csv(std::ostream& os, const FaceTable& ft) {  // connectivity.cpp:217-225
    static const char* const kName[3] = {"interior", "dirichlet", "neumann"};
    os << "face_id,n1,n2,n3,class\n";
    for (FaceId f = 0; f < ft.n_faces(); ++f)
        os << f + 1 << ',' << ft.faces[f][0] + 1 << ',' << ft.faces[f][1] + 1 << ',' << ft.faces[f][2] + 1 << ','
           << kName[static_cast<int>(ft.face_class[f])] << "\n";
}

// ============================================================= refinement

namespace {

Mesh mesh_of(const phb::MeshData& d) {
    Mesh m;
    m.level = d.level;
    m.coords.resize(d.nc);
    m.tetra.resize(d.ne);
    m.dirichlet_faces.resize(d.nd);
    m.neumann_faces.resize(d.nn);
    if (d.nc) d.coords.download_to(&m.coords[0].x, 3 * d.nc);
    if (d.ne) d.tets.download_to(m.tetra[0].data(), 4 * d.ne);
    if (d.nd) d.db.download_to(m.dirichlet_faces[0].data(), 3 * d.nd);
    if (d.nn) d.nb.download_to(m.neumann_faces[0].data(), 3 * d.nn);
    phb::sync();
    return m;
}

}  // namespace

std::pair<Mesh, RefinementMap> red_refine(const Mesh& mesh, const EdgeTable& edges) {
    auto m = upload(mesh);
    phb::Connectivity c;
    phb::build_connectivity(*m, c, false);
    check_edges(mesh, edges, c.ned, "red_refine");
    phb::RefineMap rm;
    auto child = phb::refine_mesh(*m, c, &rm);
    const int64_t ne = mesh.num_elems();
    RefinementMap map;
    map.midpoint_node.resize(c.ned);
    map.centroid_node.resize(ne);
    map.parent_elem.resize(12 * ne);
    DBuf<int32_t> parent(12 * ne > 0 ? 12 * ne : 1);
    check(phfem_gpu_refine_parents(ne, parent.p, phb::SV()), "parents");
    get(rm.midpoint, map.midpoint_node.data(), c.ned);
    get(rm.centroid, map.centroid_node.data(), ne);
    get(parent, map.parent_elem.data(), 12 * ne);
    Mesh out = mesh_of(*child);
    out.level = mesh.level + 1;
    return {std::move(out), std::move(map)};
}

// refine.cpp:76-96 through the device kernel of the pipeline: the boundary
// list's edge ids come from the host EdgeTable (the caller's), the midpoint
// ids from the caller's map
std::vector<Tri3> refine_boundary_faces(const std::vector<Tri3>& faces, const EdgeTable& edges,
                                        const RefinementMap& map) {
    const int64_t nf = (int64_t)faces.size();
    std::vector<int32_t> mids((size_t)(3 * nf));
    for (int64_t f = 0; f < nf; ++f) {
        const Tri3& t = faces[f];
        const NodeId pr[3][2] = {{t[0], t[1]}, {t[1], t[2]}, {t[0], t[2]}};
        for (int j = 0; j < 3; ++j) {
            const EdgeId e = edges.pair_to_edge(pr[j][0], pr[j][1]);
            if (e < 0 || e >= (EdgeId)map.midpoint_node.size() || map.midpoint_node[e] < 0)
                throw MeshError("inconsistent mesh: boundary face edge (" + std::to_string(pr[j][0] + 1) + "," +
                                std::to_string(pr[j][1] + 1) + ") is not an element edge");
            mids[3 * f + j] = map.midpoint_node[e];
        }
    }
    DBuf<int32_t> din(3 * nf > 0 ? 3 * nf : 1), dmid(3 * nf > 0 ? 3 * nf : 1), dout(12 * nf > 0 ? 12 * nf : 1);
    put(din, flat(faces), 3 * nf);
    put(dmid, mids.data(), 3 * nf);
    check(phfem_gpu_split_boundary(nf, din.p, dmid.p, dout.p, phb::SV()), "boundary split");
    std::vector<Tri3> out((size_t)(4 * nf));
    if (nf) dout.download_to(out[0].data(), 12 * nf);
    phb::sync();
    return out;
}

Mesh refine_to_level(int level, std::vector<LevelInfo>* log) {  // refine.cpp:98-132
    if (level < 0) throw InvalidArgument("refinement level must be non-negative");
    auto since = [](std::chrono::steady_clock::time_point t0) {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    auto m = upload(initial_cube_mesh());
    double t_refine = 0.0;
    for (int lv = 0;; ++lv) {
        phb::Connectivity c;
        auto t0 = std::chrono::steady_clock::now();
        phb::build_connectivity(*m, c, log != nullptr, nullptr, false);
        phb::sync();
        if (log) {
            LevelInfo info;
            info.level = lv;
            info.n_elems = m->ne;
            info.n_nodes = m->nc;
            info.n_edges = c.ned;
            info.n_faces = c.nf;
            // the device pass numbers edges and faces together; the E2T map
            // is never built
            info.timings.t_numedges = since(t0);
            info.timings.t_redrefine = t_refine;
            log->push_back(info);
        }
        if (lv == level) break;
        t0 = std::chrono::steady_clock::now();
        m = phb::refine_mesh(*m, c, nullptr);
        phb::sync();
        t_refine = since(t0);
    }
    return mesh_of(*m);
}

// ================================================================= sparse

CsrMatrix CsrMatrix::from_triplets(std::int64_t rows, std::int64_t cols, const Triplets& t) {
    const int64_t n = (int64_t)t.val.size();
    if ((int64_t)t.row.size() != n || (int64_t)t.col.size() != n)
        throw InvalidArgument("from_triplets: row/col/val sizes differ");
    for (int64_t i = 0; i < n; ++i)
        if (t.row[i] < 0 || t.row[i] >= rows || t.col[i] < 0 || t.col[i] >= cols)
            throw InvalidArgument("from_triplets: entry " + std::to_string(i) + " outside the matrix");
    DBuf<int64_t> tr, tc32w;
    DBuf<int32_t> tc;
    DBuf<double> tv;
    put(tr, t.row.data(), n);
    put(tc, t.col.data(), n);
    put(tv, t.val.data(), n);
    tc32w.alloc(n > 0 ? n : 1);
    check(phfem_gpu_widen(n, tc.p, tc32w.p, phb::SV()), "widen");
    DCsr out;
    triplets_to_csr(rows, cols, n, tr, tc32w, tv, out);
    return down(out);
}

void CsrMatrix::multiply(std::span<const double> x, std::span<double> y) const {
    DCsr a;
    up(*this, a);
    DBuf<double> dx, dy(n_rows > 0 ? n_rows : 1);
    put(dx, x.data(), (int64_t)x.size());
    check(phfem_gpu_csr_spmv(n_rows, a.ptr.p, a.col.p, a.val.p, dx.p, dy.p, phb::SV()), "spmv");
    get(dy, y.data(), n_rows);
    phb::sync();
}

void CsrMatrix::multiply_transpose(std::span<const double> x, std::span<double> y) const {
    // y[col] += val x[row] in row order == the transposed rows summed from
    // zero in storage order (sparse.cpp:54-58)
    DCsr a, t;
    up(*this, a);
    transpose_dev(a, t);
    DBuf<double> dx, dy(n_cols > 0 ? n_cols : 1);
    put(dx, x.data(), (int64_t)x.size());
    check(phfem_gpu_csr_spmv(t.rows, t.ptr.p, t.col.p, t.val.p, dx.p, dy.p, phb::SV()), "spmv");
    get(dy, y.data(), n_cols);
    phb::sync();
}

std::vector<double> CsrMatrix::diagonal() const {
    DCsr a;
    up(*this, a);
    DBuf<double> d(n_rows > 0 ? n_rows : 1);
    check(phfem_gpu_csr_diag(n_rows, a.ptr.p, a.col.p, a.val.p, d.p, phb::SV()), "diagonal");
    std::vector<double> h((size_t)n_rows);
    get(d, h.data(), n_rows);
    phb::sync();
    return h;
}

CsrMatrix CsrMatrix::transpose() const {
    DCsr a, t;
    up(*this, a);
    transpose_dev(a, t);
    return down(t);
}

double CsrMatrix::max_abs() const {
    double m = 0.0;
    for (double v : val) m = std::max(m, std::fabs(v));
    return m;
}

double CsrMatrix::symmetry_gap() const {  // sparse.cpp:96-120
    if (n_rows != n_cols) throw InvalidArgument("symmetry_gap requires a square matrix");
    const CsrMatrix t = transpose();
    double gap = 0.0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t i = row_ptr[r], j = t.row_ptr[r];
        const int64_t ie = row_ptr[r + 1], je = t.row_ptr[r + 1];
        while (i < ie || j < je) {
            const int32_t ci = i < ie ? col[i] : (int32_t)n_cols, cj = j < je ? t.col[j] : (int32_t)n_cols;
            if (ci == cj) gap = std::max(gap, std::fabs(val[i++] - t.val[j++]));
            else if (ci < cj) gap = std::max(gap, std::fabs(val[i++]));
            else gap = std::max(gap, std::fabs(t.val[j++]));
        }
    }
    return gap;
}

CsrMatrix spgemm(const CsrMatrix& a, const CsrMatrix& b) {
    if (a.n_cols != b.n_rows) throw InvalidArgument("spgemm: dimension mismatch");
    DCsr da, db, dc;
    up(a, da);
    up(b, db);
    spgemm_dev(da, db, dc);
    return down(dc);
}

void dump_matrix_coo(std::ostream& os, const CsrMatrix& a) {
    for (int64_t r = 0; r < a.n_rows; ++r)
        for (int64_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
            os << r + 1 << ' ' << a.col[k] + 1 << ' ' << a.val[k] << "\n";
}

double norm2(std::span<const double> v) {
    DBuf<double> d;
    put(d, v.data(), (int64_t)v.size());
    return std::sqrt(sumsq_max(d.p, (int64_t)v.size()).first);
}

CgResult pcg_jacobi(const CsrMatrix& a, std::span<const double> b, std::span<double> x, const CgOptions& opt) {
    DCsr da;
    up(a, da);
    DBuf<double> db, dx(a.n_rows > 0 ? a.n_rows : 1);
    put(db, b.data(), (int64_t)b.size());
    const CgResult r = pcg_dev(da, db.p, dx.p, opt);
    get(dx, x.data(), a.n_rows);
    phb::sync();
    return r;
}

// =============================================================== assembly

LocalStiffnessMass local_stiffness_mass(const Mesh& mesh, ElemId t) {  // assembly.cpp:7-33
    const Tet4& e = mesh.tetra[t];
    const Vec3 p0 = mesh.coords[e[0]];
    const Vec3 d1 = mesh.coords[e[1]] - p0, d2 = mesh.coords[e[2]] - p0, d3 = mesh.coords[e[3]] - p0;
    const double det = dot(cross(d1, d2), d3);
    if (det == 0.0) throw MeshError("degenerate element " + std::to_string(t + 1) + " (zero volume)");
    LocalStiffnessMass L;
    L.volume = std::fabs(det) / 6.0;
    L.grads[1] = cross(d2, d3) / det;
    L.grads[2] = cross(d3, d1) / det;
    L.grads[3] = cross(d1, d2) / det;
    L.grads[0] = (L.grads[1] + L.grads[2] + L.grads[3]) * -1.0;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            L.k[i][j] = L.volume * dot(L.grads[i], L.grads[j]);
            L.m[i][j] = L.volume / 20.0 * (i == j ? 2.0 : 1.0);
        }
    return L;
}

Mat4 local_multiplier(const FaceTable& ft, ElemId t) {  // assembly.cpp:35-44
    Mat4 c = mat4_zero();
    for (int k = 0; k < 4; ++k) {
        const int64_t s = 4 * int64_t(t) + k;
        const double v = ft.sigma[s] * ft.face_area[ft.slot_to_face[s]] / 3.0;
        for (int j = 0; j < 3; ++j) c[k][kFaceVerts[k][j]] = v;
    }
    return c;
}

namespace {

// device rule tables for the tabulated kernels
struct DevRule {
    int nq = 0;
    DBuf<double> lam, w;
    explicit DevRule(int degree) {
        std::vector<double> l, ww;
        phb::tet_rule(degree, l, ww);
        nq = (int)ww.size();
        put(lam, l.data(), (int64_t)l.size());
        put(w, ww.data(), (int64_t)ww.size());
    }
};

// The caller's FaceTable on the device (the fields the kernels read)
struct DevFaces {
    int64_t nf = 0, ne = 0;
    DBuf<int32_t> faces, slot_to_face, mult;
    DBuf<double> sigma, area;
    DBuf<uint8_t> cls;
    DBuf<int64_t> slots;
    DevFaces(const FaceTable& ft, int64_t ne_) : nf(ft.n_faces()), ne(ne_) {
        if ((int64_t)ft.slot_to_face.size() != 4 * ne || (int64_t)ft.sigma.size() != 4 * ne)
            throw InvalidArgument("face table does not match the mesh (4 slots per element)");
        put(faces, flat(ft.faces), 3 * nf);
        put(slot_to_face, ft.slot_to_face.data(), 4 * ne);
        put(mult, ft.multiplier_index.data(), nf);
        put(sigma, ft.sigma.data(), 4 * ne);
        put(area, ft.face_area.data(), nf);
        std::vector<uint8_t> c((size_t)nf);
        for (int64_t f = 0; f < nf; ++f) c[f] = static_cast<uint8_t>(ft.face_class[f]);
        put(cls, c.data(), nf);
        put(slots, nf ? ft.face_slots[0].data() : nullptr, 2 * nf);
    }
};

std::vector<double> download_vec(const DBuf<double>& d, int64_t n) {
    std::vector<double> h((size_t)n);
    get(d, h.data(), n);
    phb::sync();
    return h;
}

// load_vector on an uploaded mesh into db [4 nE] (device)
void load_vector_dev(const phb::MeshData& m, const std::function<double(const Vec3&)>& f, LoadRule rule,
                     DBuf<double>& db) {
    const int64_t ne = m.ne;
    const int r = rule == LoadRule::Gauss ? 0 : 1;
    DevRule q(5);
    const int nq = r == 0 ? q.nq : 4;
    DBuf<double> vol(ne > 0 ? ne : 1), pts(3 * nq * ne > 0 ? 3 * nq * ne : 1), fv;
    check(phfem_gpu_load_points(ne, m.coords.p, m.tets.p, r, nq, q.lam.p, vol.p, pts.p, phb::SV()), "load points");
    const std::vector<double> hp = download_vec(pts, 3 * nq * ne);
    std::vector<double> hf((size_t)(nq * ne));
    for (int64_t i = 0; i < nq * ne; ++i) hf[i] = f(Vec3(hp[3 * i], hp[3 * i + 1], hp[3 * i + 2]));
    put(fv, hf.data(), nq * ne);
    db.alloc(4 * ne > 0 ? 4 * ne : 1);
    check(phfem_gpu_load_tab(ne, r, nq, q.lam.p, q.w.p, vol.p, fv.p, db.p, phb::SV()), "load vector");
}

// geometry (area, unit normal, centroid) of the faces of class `cls`
struct BoundaryGeo {
    std::vector<int32_t> ids;      // face ids of the class
    std::vector<int32_t> of_face;  // face -> geometry row (-1)
    std::vector<double> geo;       // 7 per row
    DBuf<double> dgeo;
    DBuf<int32_t> dof;
};

void boundary_geometry(const phb::MeshData& m, const FaceTable& ft, const DevFaces& df, FaceClass cls,
                       BoundaryGeo& g) {
    const int64_t nf = ft.n_faces();
    g.of_face.assign((size_t)nf, -1);
    for (int64_t f = 0; f < nf; ++f)
        if (ft.face_class[f] == cls) {
            g.of_face[f] = (int32_t)g.ids.size();
            g.ids.push_back((int32_t)f);
        }
    const int64_t n = (int64_t)g.ids.size();
    DBuf<int32_t> dids;
    DBuf<unsigned long long> bad(1);
    bad.fill_bytes(0xff);
    put(dids, g.ids.data(), n);
    g.dgeo.alloc(7 * n > 0 ? 7 * n : 1);
    check(phfem_gpu_face_geom(n, dids.p, df.faces.p, m.coords.p, g.dgeo.p, bad.p, phb::SV()), "face geometry");
    const unsigned long long b = get1(bad.p);
    if (b != kNone) throw MeshError("degenerate face with collinear nodes " + tri_str(ft.faces[g.ids[b]]));
    g.geo = download_vec(g.dgeo, 7 * n);
    put(g.dof, g.of_face.data(), nf);
}

void neumann_dev(const phb::MeshData& m, const FaceTable& ft, const DevFaces& df,
                 const std::function<double(const Vec3&, const Vec3&)>& gfun, DBuf<double>& dln) {
    BoundaryGeo g;
    boundary_geometry(m, ft, df, FaceClass::Neumann, g);
    const int64_t n = (int64_t)g.ids.size();
    std::vector<double> gv((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        const double* r = &g.geo[7 * i];
        gv[i] = gfun(Vec3(r[4], r[5], r[6]), Vec3(r[1], r[2], r[3]));
    }
    DBuf<double> dgv;
    put(dgv, gv.data(), n);
    dln.alloc(4 * m.ne > 0 ? 4 * m.ne : 1);
    check(phfem_gpu_neumann_tab(m.ne, df.slot_to_face.p, df.cls.p, df.slots.p, g.dof.p, g.dgeo.p, dgv.p, dln.p,
                                phb::SV()),
          "neumann");
}

// b_D = |F| u_D(centroid) per Dirichlet face (assembly.cpp:96-104); the
// centroid from the device face geometry, the product on the host as the
// single multiplication it is
std::vector<double> dirichlet_host(const phb::MeshData& m, const FaceTable& ft, const DevFaces& df,
                                   const std::function<double(const Vec3&)>& u_d) {
    BoundaryGeo g;
    boundary_geometry(m, ft, df, FaceClass::Dirichlet, g);
    std::vector<double> bd((size_t)ft.n_multipliers(), 0.0);
    for (size_t i = 0; i < g.ids.size(); ++i) {
        const double* r = &g.geo[7 * i];
        bd[ft.multiplier_index[g.ids[i]]] = ft.face_area[g.ids[i]] * u_d(Vec3(r[4], r[5], r[6]));
    }
    return bd;
}

}  // namespace

std::vector<double> load_vector(const Mesh& mesh, const std::function<double(const Vec3&)>& f, LoadRule rule) {
    auto m = upload(mesh);
    DBuf<double> db;
    load_vector_dev(*m, f, rule, db);
    return download_vec(db, 4 * mesh.num_elems());
}

std::vector<double> neumann_vector(const Mesh& mesh, const FaceTable& ft,
                                   const std::function<double(const Vec3&, const Vec3&)>& g) {
    auto m = upload(mesh);
    DevFaces df(ft, mesh.num_elems());
    DBuf<double> dln;
    neumann_dev(*m, ft, df, g, dln);
    return download_vec(dln, 4 * mesh.num_elems());
}

std::vector<double> dirichlet_vector(const Mesh& mesh, const FaceTable& ft,
                                     const std::function<double(const Vec3&)>& u_d) {
    auto m = upload(mesh);
    DevFaces df(ft, mesh.num_elems());
    return dirichlet_host(*m, ft, df, u_d);
}

// assemble_system (assembly.cpp:106-138): element blocks and C rows from the
// device kernel of the pipeline (debug views of phb::assemble_system are not
// used: the caller's FaceTable is what the blocks are formed from here), C
// from the device from_triplets, load data tabulated
LinearSystem assemble_system(const Mesh& mesh, const FaceTable& ft, const ProblemData& problem, LoadRule rule) {
    auto m = upload(mesh);
    const int64_t ne = mesh.num_elems();
    DevFaces df(ft, ne);
    LinearSystem sys;
    sys.n = 4 * ne;
    sys.l = ft.n_multipliers();
    // blocks, slot rows / coefficients, C triplets
    DBuf<double> a(16 * ne > 0 ? 16 * ne : 1), coef(4 * ne > 0 ? 4 * ne : 1);
    DBuf<int32_t> mrow(4 * ne > 0 ? 4 * ne : 1);
    DBuf<unsigned long long> bad(1);
    bad.fill_bytes(0xff);
    check(phfem_gpu_element_blocks(ne, m->coords.p, m->tets.p, df.slot_to_face.p, df.sigma.p, df.area.p, df.mult.p,
                                   a.p, coef.p, mrow.p, bad.p, phb::SV()),
          "element blocks");
    const unsigned long long b0 = get1(bad.p);
    if (b0 != kNone) throw MeshError("degenerate element " + std::to_string(b0 + 1) + " (zero volume)");
    sys.a_blocks.resize(ne);
    sys.slot_coef.resize(ne);
    sys.slot_mrow.resize(ne);
    if (ne) {
        a.download_to(&sys.a_blocks[0][0][0], 16 * ne);
        coef.download_to(sys.slot_coef[0].data(), 4 * ne);
        mrow.download_to(sys.slot_mrow[0].data(), 4 * ne);
    }
    phb::sync();
    {
        // C triplets in the reference's order (element, slot, face vertex),
        // then the device from_triplets
        DBuf<int32_t> cs(ne > 0 ? ne : 1), cr(ne > 0 ? ne : 1);
        DBuf<int64_t> orr(ne + 1);
        DBuf<unsigned char> ss;
        check(phfem_gpu_schur_counts(ne, mrow.p, cs.p, cr.p, phb::SV()), "c counts");
        check(phfem_gpu_scan_i32(cr.p, orr.p, ne, scan_scratch(ss, ne), phb::SV()), "c scan");
        const int64_t nt = 3 * get1(orr.p + ne);
        DBuf<int64_t> trow(nt > 0 ? nt : 1), tcol(nt > 0 ? nt : 1);
        DBuf<double> tval(nt > 0 ? nt : 1);
        check(phfem_gpu_c_triplets(ne, mrow.p, coef.p, orr.p, trow.p, tcol.p, tval.p, phb::SV()), "c triplets");
        DCsr dc;
        triplets_to_csr(sys.l, sys.n, nt, trow, tcol, tval, dc);
        sys.c = down(dc);
    }
    DBuf<double> db, dln;
    load_vector_dev(*m, problem.f, rule, db);
    neumann_dev(*m, ft, df, problem.neumann_flux, dln);
    check(phfem_gpu_add_inplace(4 * ne, db.p, dln.p, phb::SV()), "rhs");
    sys.rhs = download_vec(db, 4 * ne);
    sys.dirichlet_rhs = dirichlet_host(*m, ft, df, problem.u_dirichlet);
    return sys;
}

CsrMatrix system_a_csr(const LinearSystem& sys) {
    Triplets t;
    t.reserve(sys.a_blocks.size() * 16);
    for (size_t e = 0; e < sys.a_blocks.size(); ++e)
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) t.add(int64_t(4 * e + i), int32_t(4 * e + j), sys.a_blocks[e][i][j]);
    return CsrMatrix::from_triplets(sys.n, sys.n, t);
}

// ================================================================= solver

namespace {

struct DevSystem {
    int64_t ne = 0, n = 0, l = 0;
    DBuf<double> a, coef, rhs, bd;
    DBuf<int32_t> mrow;
    explicit DevSystem(const LinearSystem& sys) : ne((int64_t)sys.a_blocks.size()), n(sys.n), l(sys.l) {
        if (n != 4 * ne || (int64_t)sys.rhs.size() != n || (int64_t)sys.dirichlet_rhs.size() != l ||
            (int64_t)sys.slot_mrow.size() != ne || (int64_t)sys.slot_coef.size() != ne)
            throw InvalidArgument("LinearSystem: inconsistent sizes");
        put(a, ne ? &sys.a_blocks[0][0][0] : nullptr, 16 * ne);
        put(coef, ne ? sys.slot_coef[0].data() : nullptr, 4 * ne);
        put(mrow, ne ? sys.slot_mrow[0].data() : nullptr, 4 * ne);
        put(rhs, sys.rhs.data(), n);
        put(bd, sys.dirichlet_rhs.data(), l);
    }
};

// build_schur on the device (solver.cpp:90-147): S and rhs_neg stay on the
// device (ds, drhs); the LU factors optionally come back
void build_schur_dev(const DevSystem& d, DCsr& ds, DBuf<double>& drhs, std::vector<Mat4Lu>* factors) {
    const int64_t ne = d.ne, l = d.l;
    DBuf<double> lu(16 * ne > 0 ? 16 * ne : 1), s_loc(16 * ne > 0 ? 16 * ne : 1), r_loc(4 * ne > 0 ? 4 * ne : 1);
    DBuf<int32_t> perm(4 * ne > 0 ? 4 * ne : 1);
    DBuf<uint8_t> sing(ne > 0 ? ne : 1);
    DBuf<unsigned long long> first(1);
    first.fill_bytes(0xff);
    check(phfem_gpu_condense_blocks(ne, d.a.p, d.coef.p, d.mrow.p, d.rhs.p, lu.p, perm.p, sing.p, s_loc.p, r_loc.p,
                                    first.p, phb::SV()),
          "condense");
    const unsigned long long fs = get1(first.p);
    if (fs != kNone) throw MeshError("degenerate element block " + std::to_string(fs + 1));
    DBuf<int32_t> cs(ne > 0 ? ne : 1), cr(ne > 0 ? ne : 1);
    DBuf<int64_t> os(ne + 1), orr(ne + 1);
    DBuf<unsigned char> ss;
    check(phfem_gpu_schur_counts(ne, d.mrow.p, cs.p, cr.p, phb::SV()), "schur counts");
    check(phfem_gpu_scan_i32(cs.p, os.p, ne, scan_scratch(ss, ne), phb::SV()), "schur scan");
    check(phfem_gpu_scan_i32(cr.p, orr.p, ne, scan_scratch(ss, ne), phb::SV()), "schur scan");
    const int64_t nt = get1(os.p + ne), nr = get1(orr.p + ne);
    DBuf<int64_t> trow(nt > 0 ? nt : 1), tcol(nt > 0 ? nt : 1), rrow(nr > 0 ? nr : 1);
    DBuf<double> tval(nt > 0 ? nt : 1), rval(nr > 0 ? nr : 1);
    check(phfem_gpu_schur_triplets(ne, d.mrow.p, s_loc.p, r_loc.p, os.p, orr.p, trow.p, tcol.p, tval.p, rrow.p, rval.p,
                                   phb::SV()),
          "schur triplets");
    triplets_to_csr(l, l, nt, trow, tcol, tval, ds);
    // rhs_neg: terms of each row in stream order, subtracted from b_D
    DBuf<int64_t> idx(nr > 0 ? nr : 1), rptr(l + 1), rperm(nr > 0 ? nr : 1), tmp(nr > 0 ? nr : 1);
    DBuf<int32_t> cnt(l > 0 ? l : 1);
    {
        std::vector<int64_t> io((size_t)nr);
        std::iota(io.begin(), io.end(), 0);
        put(idx, io.data(), nr);
    }
    check(phfem_gpu_seg_sort(nr, l, rrow.p, idx.p, rptr.p, rperm.p, cnt.p, tmp.p, scan_scratch(ss, l), phb::SV()),
          "rhs sort");
    drhs.alloc(l > 0 ? l : 1);
    check(phfem_gpu_rhs_neg(l, rptr.p, rperm.p, rval.p, d.bd.p, drhs.p, phb::SV()), "rhs_neg");
    if (factors) {
        std::vector<double> hl((size_t)(16 * ne));
        std::vector<int32_t> hp((size_t)(4 * ne));
        std::vector<uint8_t> hs((size_t)ne);
        get(lu, hl.data(), 16 * ne);
        get(perm, hp.data(), 4 * ne);
        get(sing, hs.data(), ne);
        phb::sync();
        factors->resize(ne);
        for (int64_t t = 0; t < ne; ++t) {
            Mat4Lu& f = (*factors)[t];
            for (int i = 0; i < 4; ++i) {
                f.perm[i] = hp[4 * t + i];
                for (int j = 0; j < 4; ++j) f.lu[i][j] = hl[16 * t + 4 * i + j];
            }
            f.singular = hs[t] != 0;
        }
    }
}

CgOptions inner_cg(const LinearSystem& sys, const SolverOptions& opt, double nrm_rhs, double nrm_bd) {
    CgOptions cg;  // inner_cg_options, solver.cpp:78-86
    cg.tol = opt.tol;
    cg.abs_tol = 0.2 * opt.tol * std::hypot(nrm_rhs, nrm_bd);
    cg.max_iter = opt.max_iter > 0 ? opt.max_iter : 10 * std::max<int64_t>(sys.l, 1);
    return cg;
}

// verify_solution (solver.cpp:44-76) on device vectors: r1 = A U - B - C' L
// (r1 holds A U - B on entry), r2 = C U - b_D
void verify_dev(const LinearSystem& sys, const DevSystem& d, const DCsr& dc, const DBuf<double>& du,
                const DBuf<double>& dl, DBuf<double>& r1, Solution& sol, double tol) {
    DCsr ct;
    transpose_dev(dc, ct);
    DBuf<double> ctl(d.n > 0 ? d.n : 1), r2(d.l > 0 ? d.l : 1);
    check(phfem_gpu_csr_spmv(ct.rows, ct.ptr.p, ct.col.p, ct.val.p, dl.p, ctl.p, phb::SV()), "C' lambda");
    check(phfem_gpu_sub_inplace(d.n, r1.p, ctl.p, phb::SV()), "r1");
    check(phfem_gpu_csr_spmv(dc.rows, dc.ptr.p, dc.col.p, dc.val.p, du.p, r2.p, phb::SV()), "C u");
    check(phfem_gpu_sub_inplace(d.l, r2.p, d.bd.p, phb::SV()), "r2");
    const auto n1 = sumsq_max(r1.p, d.n), n2 = sumsq_max(r2.p, d.l), nb = sumsq_max(d.rhs.p, d.n),
               nd = sumsq_max(d.bd.p, d.l);
    const double r1n = std::sqrt(n1.first), r2n = std::sqrt(n2.first), bn = std::sqrt(nb.first),
                 dn = std::sqrt(nd.first);
    const double rhs_norm = std::hypot(bn, dn), res_norm = std::hypot(r1n, r2n);
    sol.stats.residual = rhs_norm > 0.0 ? res_norm / rhs_norm : res_norm;
    sol.stats.constraint_residual = n2.second / (1.0 + nd.second);
    const bool ok = sol.stats.residual <= tol && r1n <= tol * std::max(bn, 1e-300) && r2n <= tol * (1.0 + dn);
    (void)sys;
    if (!ok) {
        std::ostringstream os;
        os << "solver '" << sol.stats.method << "' missed the residual target: " << sol.stats.residual << " > " << tol;
        throw SolverError(os.str());
    }
}

}  // namespace

SchurSystem build_schur(const LinearSystem& sys, int workers) {
    (void)workers;  // the device path is one deterministic pass for any worker count
    DevSystem d(sys);
    DCsr ds;
    DBuf<double> drhs;
    SchurSystem out;
    build_schur_dev(d, ds, drhs, &out.a_factor);
    out.s_neg = down(ds);
    out.rhs_neg = download_vec(drhs, sys.l);
    return out;
}

Solution solve_schur_parallel(const LinearSystem& sys, int workers, const SolverOptions& opt) {
    if (workers < 1) throw InvalidArgument("workers must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    Solution sol;
    sol.stats.method = workers > 1 ? "schur-parallel" : "schur";
    sol.stats.n = sys.n;
    sol.stats.l = sys.l;
    sol.stats.workers = workers;
    sol.stats.peak_dim = sys.l;
    DevSystem d(sys);
    DCsr ds, dc;
    DBuf<double> drhs, dl(sys.l > 0 ? sys.l : 1), du(sys.n > 0 ? sys.n : 1), r1(sys.n > 0 ? sys.n : 1);
    build_schur_dev(d, ds, drhs, nullptr);
    const double nrm_rhs = std::sqrt(sumsq_max(d.rhs.p, d.n).first), nrm_bd = std::sqrt(sumsq_max(d.bd.p, d.l).first);
    const CgResult cg = pcg_dev(ds, drhs.p, dl.p, inner_cg(sys, opt, nrm_rhs, nrm_bd));
    sol.stats.iterations = cg.iterations;
    if (!cg.converged) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%f", cg.rel_residual);
        throw SolverError("schur: conjugate gradients stalled at relative residual " + std::string(buf) + " after " +
                          std::to_string(cg.iterations) + " iterations");
    }
    check(phfem_gpu_recover_blocks(d.ne, d.a.p, d.coef.p, d.mrow.p, d.rhs.p, dl.p, du.p, r1.p, phb::SV()), "recover");
    sol.lambda = download_vec(dl, sys.l);
    sol.u = download_vec(du, sys.n);
    up(sys.c, dc);
    verify_dev(sys, d, dc, du, dl, r1, sol, opt.tol);
    sol.stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

Solution solve_schur(const LinearSystem& sys, const SolverOptions& opt) { return solve_schur_parallel(sys, 1, opt); }

// solve_direct (solver.cpp:192-244): A^-1 as a block CSR, S = C (A^-1 C')
// by two device spgemms, rhs_neg = b_D - C A^-1 B, PCG, U = A^-1 (B + C' L)
Solution solve_direct(const LinearSystem& sys, const SolverOptions& opt) {
    const auto t0 = std::chrono::steady_clock::now();
    Solution sol;
    sol.stats.method = "direct";
    sol.stats.n = sys.n;
    sol.stats.l = sys.l;
    sol.stats.workers = 1;
    sol.stats.peak_dim = sys.n + sys.l;
    DevSystem d(sys);
    const int64_t ne = d.ne, n = d.n, l = d.l;
    // element inverses as triplets (4e+i, 4e+j) in the reference's order
    DBuf<double> inv(16 * ne > 0 ? 16 * ne : 1);
    DBuf<unsigned long long> first(1);
    first.fill_bytes(0xff);
    check(phfem_gpu_block_inverses(ne, d.a.p, inv.p, first.p, phb::SV()), "block inverses");
    const unsigned long long fs = get1(first.p);
    if (fs != kNone) throw MeshError("degenerate element block " + std::to_string(fs + 1));
    DCsr ainv, dc, ct, w, s;
    {
        DBuf<int64_t> trow(16 * ne > 0 ? 16 * ne : 1), tcol(16 * ne > 0 ? 16 * ne : 1);
        check(phfem_gpu_block_pattern(ne, trow.p, tcol.p, phb::SV()), "block pattern");
        triplets_to_csr(n, n, 16 * ne, trow, tcol, inv, ainv);
    }
    up(sys.c, dc);
    transpose_dev(dc, ct);
    spgemm_dev(ainv, ct, w);
    spgemm_dev(dc, w, s);
    DBuf<double> ab(n > 0 ? n : 1), rhs_neg(l > 0 ? l : 1), dl(l > 0 ? l : 1), tmp(n > 0 ? n : 1),
        du(n > 0 ? n : 1), r1(n > 0 ? n : 1);
    check(phfem_gpu_csr_spmv(n, ainv.ptr.p, ainv.col.p, ainv.val.p, d.rhs.p, ab.p, phb::SV()), "A^-1 B");
    check(phfem_gpu_csr_spmv(l, dc.ptr.p, dc.col.p, dc.val.p, ab.p, rhs_neg.p, phb::SV()), "C A^-1 B");
    check(phfem_gpu_rsub_inplace(l, rhs_neg.p, d.bd.p, phb::SV()), "rhs_neg");
    const double nrm_rhs = std::sqrt(sumsq_max(d.rhs.p, n).first), nrm_bd = std::sqrt(sumsq_max(d.bd.p, l).first);
    const CgResult cg = pcg_dev(s, rhs_neg.p, dl.p, inner_cg(sys, opt, nrm_rhs, nrm_bd));
    sol.stats.iterations = cg.iterations;
    if (!cg.converged) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%f", cg.rel_residual);
        throw SolverError("direct: inner solve stalled at relative residual " + std::string(buf));
    }
    // U = A^-1 (B + C' L): tmp = C' L + B, then the element solves (the
    // recovery kernel with the C' L already added: zero coefficients)
    check(phfem_gpu_csr_spmv(ct.rows, ct.ptr.p, ct.col.p, ct.val.p, dl.p, tmp.p, phb::SV()), "C' L");
    check(phfem_gpu_add_inplace(n, tmp.p, d.rhs.p, phb::SV()), "B + C' L");
    check(phfem_gpu_block_solve(ne, d.a.p, tmp.p, du.p, phb::SV()), "element solves");
    // r1 = A U - B for verify
    check(phfem_gpu_block_residual(ne, d.a.p, du.p, d.rhs.p, r1.p, phb::SV()), "A U - B");
    sol.lambda = download_vec(dl, l);
    sol.u = download_vec(du, n);
    verify_dev(sys, d, dc, du, dl, r1, sol, opt.tol);
    sol.stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

Solution solve(const LinearSystem& sys, const std::string& method, const SolverOptions& opt) {
    if (method == "direct") return solve_direct(sys, opt);
    if (method == "schur") return solve_schur_parallel(sys, 1, opt);
    if (method == "schur-parallel") return solve_schur_parallel(sys, std::max(opt.workers, 1), opt);
    throw InvalidArgument("unknown solver '" + method + "' (expected direct|schur|schur-parallel)");
}

std::string stats_json(const SolverStats& s) {  // solver.cpp:253-261
    std::ostringstream os;
    os.precision(17);
    os << "{\"solver\":\"" << s.method << "\",\"n\":" << s.n << ",\"l\":" << s.l << ",\"iterations\":" << s.iterations
       << ",\"residual\":" << s.residual << ",\"constraint_residual\":" << s.constraint_residual
       << ",\"seconds\":" << s.seconds << ",\"workers\":" << s.workers << ",\"peak_dim\":" << s.peak_dim << "}";
    return os.str();
}

// =============================================================== analysis

ManufacturedProblem manufactured_problem() {  // analysis.cpp:9-25
    ManufacturedProblem p;
    p.name = "manufactured";
    auto u = [](const Vec3& x) { return x.x * x.x * x.y * x.y * x.z * x.z; };
    auto grad = [](const Vec3& x) {
        return Vec3(2.0 * x.x * x.y * x.y * x.z * x.z, 2.0 * x.x * x.x * x.y * x.z * x.z,
                    2.0 * x.x * x.x * x.y * x.y * x.z);
    };
    p.data.f = [u](const Vec3& x) {
        return -2.0 * (x.y * x.y * x.z * x.z + x.x * x.x * x.z * x.z + x.x * x.x * x.y * x.y) + u(x);
    };
    p.data.u_dirichlet = u;
    p.data.neumann_flux = [grad](const Vec3& x, const Vec3& n) { return dot(grad(x), n); };
    p.data.exact_u = u;
    p.data.exact_grad_u = grad;
    return p;
}

ManufacturedProblem linear_patch_problem() {  // analysis.cpp:27-38
    ManufacturedProblem p;
    p.name = "linear-patch";
    auto u = [](const Vec3& x) { return x.x + 2.0 * x.y + 3.0 * x.z + 4.0; };
    const Vec3 g(1.0, 2.0, 3.0);
    p.data.f = u;  // -laplace u = 0, so f = u
    p.data.u_dirichlet = u;
    p.data.neumann_flux = [g](const Vec3&, const Vec3& n) { return dot(g, n); };
    p.data.exact_u = u;
    p.data.exact_grad_u = [g](const Vec3&) { return g; };
    return p;
}

ManufacturedProblem zero_problem() {
    ManufacturedProblem p;
    p.name = "zero";
    p.data.f = [](const Vec3&) { return 0.0; };
    p.data.u_dirichlet = [](const Vec3&) { return 0.0; };
    p.data.neumann_flux = [](const Vec3&, const Vec3&) { return 0.0; };
    p.data.exact_u = [](const Vec3&) { return 0.0; };
    p.data.exact_grad_u = [](const Vec3&) { return Vec3(); };
    return p;
}

namespace {
double device_total(const DBuf<double>& acc, int64_t n) { return sumsq_sum(acc.p, n); }
}  // namespace

double y_norm_error(const Mesh& mesh, const Solution& sol, const ProblemData& prob) {
    if (!prob.exact_u || !prob.exact_grad_u) throw InvalidArgument("y_norm_error requires the exact solution fields");
    const int64_t ne = mesh.num_elems();
    if ((int64_t)sol.u.size() != 4 * ne) throw InvalidArgument("y_norm_error: solution does not match the mesh");
    auto m = upload(mesh);
    const double h = phb::mesh_diameter(*m);
    DevRule q(9);
    const int64_t np = (int64_t)q.nq * ne;
    DBuf<double> pts(3 * np > 0 ? 3 * np : 1), ex, du, acc(ne > 0 ? ne : 1);
    check(phfem_gpu_ynorm_points(ne, m->coords.p, m->tets.p, q.nq, q.lam.p, pts.p, phb::SV()), "y points");
    const std::vector<double> hp = download_vec(pts, 3 * np);
    std::vector<double> he((size_t)(4 * np));
    for (int64_t i = 0; i < np; ++i) {
        const Vec3 x(hp[3 * i], hp[3 * i + 1], hp[3 * i + 2]);
        const Vec3 g = prob.exact_grad_u(x);
        he[4 * i] = prob.exact_u(x);
        he[4 * i + 1] = g.x;
        he[4 * i + 2] = g.y;
        he[4 * i + 3] = g.z;
    }
    put(ex, he.data(), 4 * np);
    put(du, sol.u.data(), 4 * ne);
    check(phfem_gpu_ynorm_elem(ne, m->coords.p, m->tets.p, du.p, q.nq, q.lam.p, q.w.p, ex.p, 1.0 / (h * h), acc.p,
                               phb::SV()),
          "y norm");
    return std::sqrt(device_total(acc, ne));
}

double multiplier_norm_error(const Mesh& mesh, const FaceTable& ft, const Solution& sol, const ProblemData& prob) {
    if (!prob.exact_grad_u) throw InvalidArgument("multiplier_norm_error requires the exact gradient");
    const int64_t ne = mesh.num_elems();
    auto m = upload(mesh);
    const double h = phb::mesh_diameter(*m);
    DevFaces df(ft, ne);
    DBuf<double> pts(36 * ne > 0 ? 36 * ne : 1), gr, dl, acc(ne > 0 ? ne : 1);
    check(phfem_gpu_kappa_points(ne, m->coords.p, m->tets.p, pts.p, phb::SV()), "kappa points");
    const std::vector<double> hp = download_vec(pts, 36 * ne);
    std::vector<double> hg((size_t)(36 * ne), 0.0);
    for (int64_t t = 0; t < ne; ++t)
        for (int k = 0; k < 4; ++k) {
            if (ft.face_class[ft.slot_to_face[4 * t + k]] == FaceClass::Neumann) continue;
            for (int j = 0; j < 3; ++j) {
                const int64_t i = 12 * t + 3 * k + j;
                const Vec3 g = prob.exact_grad_u(Vec3(hp[3 * i], hp[3 * i + 1], hp[3 * i + 2]));
                hg[3 * i] = g.x;
                hg[3 * i + 1] = g.y;
                hg[3 * i + 2] = g.z;
            }
        }
    put(gr, hg.data(), 36 * ne);
    put(dl, sol.lambda.data(), (int64_t)sol.lambda.size());
    check(phfem_gpu_kappa_elem(ne, m->coords.p, m->tets.p, df.slot_to_face.p, df.sigma.p, df.cls.p, df.mult.p, dl.p,
                               gr.p, h, acc.p, phb::SV()),
          "kappa norm");
    return std::sqrt(device_total(acc, ne));
}

double evaluate_uh(const Solution& sol, const Mesh& mesh, ElemId t, const Vec3& p) {  // analysis.cpp:107-121
    const LocalStiffnessMass L = local_stiffness_mass(mesh, t);
    const Vec3 p0 = mesh.coords[mesh.tetra[t][0]];
    double uh = 0.0;
    for (int v = 0; v < 4; ++v) {
        const double lv = (v == 0 ? 1.0 : 0.0) + dot(L.grads[v], p - p0);
        if (lv < -1e-10 || lv > 1.0 + 1e-10)
            throw InvalidArgument("evaluate_uh: point outside element " + std::to_string(t + 1));
        uh += lv * sol.u[4 * t + v];
    }
    return uh;
}

std::vector<ErrorReport> convergence_study(int max_level, const std::string& solver_name, const SolverOptions& opt,
                                           const ManufacturedProblem& prob, LoadRule rule) {
    if (max_level < 1) throw InvalidArgument("convergence_study: max_level must be >= 1");
    std::vector<ErrorReport> out;
    Mesh mesh = initial_cube_mesh();
    for (int level = 1; level <= max_level; ++level) {
        try {
            mesh = red_refine(mesh, num_edges(mesh)).first;
            const EdgeTable edges = num_edges(mesh);
            const FaceTable ft = build_face_table(mesh);
            const LinearSystem sys = assemble_system(mesh, ft, prob.data, rule);
            const Solution sol = solve(sys, solver_name, opt);
            ErrorReport rep;
            rep.level = level;
            rep.n_elems = mesh.num_elems();
            rep.n_nodes = mesh.num_nodes();
            rep.n_edges = edges.n_edges();
            rep.n_faces = ft.n_faces();
            rep.n = sys.n;
            rep.l = sys.l;
            rep.h = mesh_diameter(mesh);
            rep.err_u = y_norm_error(mesh, sol, prob.data);
            rep.err_kappa = multiplier_norm_error(mesh, ft, sol, prob.data);
            rep.stats = sol.stats;
            if (!out.empty()) {
                if (rep.err_u > 0.0 && out.back().err_u > 0.0) rep.order_u = std::log2(out.back().err_u / rep.err_u);
                if (rep.err_kappa > 0.0 && out.back().err_kappa > 0.0)
                    rep.order_kappa = std::log2(out.back().err_kappa / rep.err_kappa);
            }
            out.push_back(rep);
        } catch (const SolverError& e) {
            throw SolverError("level " + std::to_string(level) + ": " + e.what());
        }
    }
    return out;
}

// ==================================================================== vtk

namespace {
std::ofstream vtk_open(const std::string& path) {
    std::ofstream os(path);
    if (!os) throw IoError("cannot open '" + path + "' for writing");
    return os;
}
void vtk_points(std::ostream& os, const Mesh& mesh) {  // vtk.cpp:15-24
    os << "# vtk DataFile Version 3.0\nphfem level " << mesh.level << "\nASCII\nDATASET UNSTRUCTURED_GRID\nPOINTS "
       << mesh.coords.size() << " double\n";
    for (const Vec3& p : mesh.coords)
        os << format_double(p.x) << ' ' << format_double(p.y) << ' ' << format_double(p.z) << "\n";
}
}  // namespace

void export_vtk(const std::string& path, const Mesh& mesh, const Solution* sol, bool point_data) {  // vtk.cpp:27-58
    std::ofstream os = vtk_open(path);
    vtk_points(os, mesh);
    const size_t ne = mesh.tetra.size();
    os << "CELLS " << ne << ' ' << 5 * ne << "\n";
    for (const Tet4& t : mesh.tetra) os << "4 " << t[0] << ' ' << t[1] << ' ' << t[2] << ' ' << t[3] << "\n";
    os << "CELL_TYPES " << ne << "\n";
    for (size_t i = 0; i < ne; ++i) os << "10\n";
    if (!sol) return;
    os << "CELL_DATA " << ne << "\nSCALARS u_mean double 1\nLOOKUP_TABLE default\n";
    for (size_t t = 0; t < ne; ++t)
        os << format_double((sol->u[4 * t] + sol->u[4 * t + 1] + sol->u[4 * t + 2] + sol->u[4 * t + 3]) / 4.0) << "\n";
    if (point_data) {
        std::vector<double> sum(mesh.coords.size(), 0.0);
        std::vector<int> cnt(mesh.coords.size(), 0);
        for (size_t t = 0; t < ne; ++t)
            for (int v = 0; v < 4; ++v) {
                sum[mesh.tetra[t][v]] += sol->u[4 * t + v];
                ++cnt[mesh.tetra[t][v]];
            }
        os << "POINT_DATA " << mesh.coords.size() << "\nSCALARS u_nodal_average double 1\nLOOKUP_TABLE default\n";
        for (size_t i = 0; i < sum.size(); ++i) os << format_double(cnt[i] ? sum[i] / cnt[i] : 0.0) << "\n";
    }
    if (!os) throw IoError("write failure on '" + path + "'");
}

void export_multiplier_vtk(const std::string& path, const Mesh& mesh, const FaceTable& ft,
                           const Solution& sol) {  // vtk.cpp:60-80
    std::ofstream os = vtk_open(path);
    vtk_points(os, mesh);
    const int64_t nl = ft.n_multipliers();
    os << "CELLS " << nl << ' ' << 4 * nl << "\n";
    for (FaceId f = 0; f < ft.n_faces(); ++f)
        if (ft.multiplier_index[f] >= 0)
            os << "3 " << ft.faces[f][0] << ' ' << ft.faces[f][1] << ' ' << ft.faces[f][2] << "\n";
    os << "CELL_TYPES " << nl << "\n";
    for (int64_t i = 0; i < nl; ++i) os << "5\n";
    os << "CELL_DATA " << nl << "\nSCALARS lambda double 1\nLOOKUP_TABLE default\n";
    for (FaceId f = 0; f < ft.n_faces(); ++f)
        if (ft.multiplier_index[f] >= 0) os << format_double(sol.lambda[ft.multiplier_index[f]]) << "\n";
    if (!os) throw IoError("write failure on '" + path + "'");
}

}  // namespace phfem

namespace phb {

// The pair edge_pairs_to_elems names when two elements claim the same
// oriented face (connectivity.cpp:62-68): the first repeated key of the
// sorted E2T entries.  The pipeline never builds the E2T; on that error path
// it is built once on the device to report the reference's exact pair.
bool e2t_first_duplicate(const MeshData& m, const Connectivity& c, int32_t& a, int32_t& b) {
    const int64_t ne = m.ne, n = 12 * ne, ned = c.ned;
    if (!c.has_edges || n == 0) return false;
    // ned + 1 segments: the last holds the keys that wrap (phfem_gpu_e2t_entries)
    DBuf<int64_t> from(n), to(n), seg_ptr(ned + 2), perm(n), tmp(n);
    DBuf<int32_t> cnt(ned + 1), elem(n);
    DBuf<unsigned long long> key(n), dup(1);
    DBuf<unsigned char> ss(phfem_gpu_scan_scratch(ned + 1));
    dup.fill_bytes(0xff);
    check(phfem_gpu_e2t_entries(ne, ned, c.edge_of_slot.p, c.edge_nodes.p, from.p, to.p, SV()), "e2t entries");
    check(phfem_gpu_seg_sort(n, ned + 1, from.p, to.p, seg_ptr.p, perm.p, cnt.p, tmp.p, ss.p, SV()), "e2t sort");
    check(phfem_gpu_e2t_finish(n, ned, perm.p, from.p, to.p, key.p, elem.p, dup.p, SV()), "e2t finish");
    unsigned long long j;
    check(cudaMemcpyAsync(&j, dup.p, sizeof j, cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
    if (j == ~0ull) return false;
    int32_t pair[2];
    check(cudaMemcpyAsync(pair, elem.p + j - 1, sizeof pair, cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
    a = pair[0];
    b = pair[1];
    return true;
}

}  // namespace phb
