// C ABI of libphfem.so: the reference's phfem.h (capi.cpp:95-310 of the
// reference) plus phfem_ext.h, implemented over the device runtime.
//
// Semantics kept from the reference: opaque handles; thread-local last error
// cleared on success; exceptions mapped to status codes by `guarded`
// (capi.cpp:27-46); lazily built connectivity invalidated by refinement
// (capi.cpp:63-85); solutions hold a snapshot of the mesh and its
// connectivity so they survive later refinement (capi.cpp:87-93, 202).  Here
// the snapshot shares the immutable device buffers by reference count.
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "phfem.h"
#include "phfem_ext.h"
#include "phfem_cxx/analysis.hpp"
#include "phfem_cxx/solver.hpp"
#include "runtime.hpp"

using namespace phb;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_last_error.clear();
        return PHFEM_OK;
    } catch (const InvalidArgument& e) {
        return set_error(PHFEM_ERR_ARGUMENT, e.what());
    } catch (const MeshError& e) {
        return set_error(PHFEM_ERR_MESH, e.what());
    } catch (const SolverError& e) {
        return set_error(PHFEM_ERR_SOLVER, e.what());
    } catch (const IoError& e) {
        return set_error(PHFEM_ERR_IO, e.what());
    } catch (const std::bad_alloc&) {
        return set_error(PHFEM_ERR_MESH, "out of memory");
    } catch (const std::exception& e) {
        return set_error(PHFEM_ERR_ARGUMENT, e.what());
    }
}

// host copy of a mesh for the text formats
struct HostMesh {
    std::vector<double> coords;
    std::vector<int32_t> tets, db, nb;
    int level = 0;
};

HostMesh to_host(const MeshData& m) {
    HostMesh h;
    h.coords = m.coords.download();
    h.tets = m.tets.download();
    h.db = m.db.download();
    h.nb = m.nb.download();
    h.level = m.level;
    return h;
}

// The 8-node, 5-tetrahedron unit cube (mesh.cpp:12-32).
std::shared_ptr<MeshData> cube_mesh() {
    const double coords[24] = {0, 0, 0, 1, 0, 0, 0, 1, 0, 1, 1, 0, 0, 0, 1, 1, 0, 1, 0, 1, 1, 1, 1, 1};
    const int32_t tets[20] = {0, 1, 2, 4, 4, 7, 5, 1, 6, 2, 7, 4, 3, 7, 2, 1, 7, 2, 1, 4};
    const int32_t db[6] = {6, 7, 4, 4, 7, 5};
    const int32_t nb[30] = {0, 4, 1, 4, 5, 1, 0, 2, 4, 6, 4, 2, 6, 2, 7, 3, 7, 2, 1, 5, 7, 3, 1, 7, 3, 2, 1, 0, 1, 2};
    return upload_mesh(coords, 8, tets, 5, db, 2, nb, 10, 0);
}

// read_mesh (mesh.cpp:139-182): sections COORD/TETRA/DB/NB, 1-based
std::shared_ptr<MeshData> read_mesh(std::istream& is) {
    auto section = [&](const char* name) -> int64_t {
        std::string tok;
        if (!(is >> tok) || tok != name)
            throw IoError(std::string("mesh format: expected section '") + name + "', got '" + tok + "'");
        long long n = -1;
        if (!(is >> n) || n < 0) throw IoError(std::string("mesh format: bad row count for section '") + name + "'");
        return n;
    };
    HostMesh h;
    const int64_t nc = section("COORD");
    h.coords.resize(3 * nc);
    for (int64_t i = 0; i < 3 * nc; i += 3)
        if (!(is >> h.coords[i] >> h.coords[i + 1] >> h.coords[i + 2]))
            throw IoError("mesh format: bad coordinate row");
    auto read_index = [&](int32_t& out) {
        long long v;
        if (!(is >> v)) throw IoError("mesh format: expected a node index");
        if (v < 1 || v > nc)
            throw IoError("mesh format: node index " + std::to_string(v) + " out of range 1.." + std::to_string(nc));
        out = (int32_t)(v - 1);
    };
    const int64_t ne = section("TETRA");
    h.tets.resize(4 * ne);
    for (auto& v : h.tets) read_index(v);
    const int64_t nd = section("DB");
    h.db.resize(3 * nd);
    for (auto& v : h.db) read_index(v);
    const int64_t nn = section("NB");
    h.nb.resize(3 * nn);
    for (auto& v : h.nb) read_index(v);
    return upload_mesh(h.coords.data(), nc, h.tets.data(), ne, h.db.data(), nd, h.nb.data(), nn, 0);
}

void write_mesh(std::ostream& os, const HostMesh& h) {  // mesh.cpp:117-130
    const size_t nc = h.coords.size() / 3;
    os << "COORD " << nc << "\n";
    for (size_t i = 0; i < nc; ++i)
        os << format_double(h.coords[3 * i]) << ' ' << format_double(h.coords[3 * i + 1]) << ' '
           << format_double(h.coords[3 * i + 2]) << "\n";
    os << "TETRA " << h.tets.size() / 4 << "\n";
    for (size_t t = 0; t < h.tets.size(); t += 4)
        os << h.tets[t] + 1 << ' ' << h.tets[t + 1] + 1 << ' ' << h.tets[t + 2] + 1 << ' ' << h.tets[t + 3] + 1 << "\n";
    os << "DB " << h.db.size() / 3 << "\n";
    for (size_t f = 0; f < h.db.size(); f += 3) os << h.db[f] + 1 << ' ' << h.db[f + 1] + 1 << ' ' << h.db[f + 2] + 1 << "\n";
    os << "NB " << h.nb.size() / 3 << "\n";
    for (size_t f = 0; f < h.nb.size(); f += 3) os << h.nb[f] + 1 << ' ' << h.nb[f + 1] + 1 << ' ' << h.nb[f + 2] + 1 << "\n";
}

std::string stats_json(const std::string& method, int64_t n, int64_t l, int64_t iterations, double residual,
                       double constraint, double seconds, int workers, int64_t peak_dim) {  // solver.cpp:253-261
    std::ostringstream os;
    os.precision(17);
    os << "{\"solver\":\"" << method << "\",\"n\":" << n << ",\"l\":" << l << ",\"iterations\":" << iterations
       << ",\"residual\":" << residual << ",\"constraint_residual\":" << constraint << ",\"seconds\":" << seconds
       << ",\"workers\":" << workers << ",\"peak_dim\":" << peak_dim << "}";
    return os.str();
}

}  // namespace

// Workspaces (connectivity, system, refinement target) of destroyed mesh
// handles, handed to the next handle's pipeline pass: a stream of meshes (the
// end-to-end path, one handle per mesh) then allocates nothing per mesh in
// the middle of a pass, like repeated passes on one handle.  All their device
// work is ordered on the library stream, so reuse is safe.
template <class T>
struct Recycle {
    std::mutex mu;
    std::vector<std::shared_ptr<T>> spare;
    std::shared_ptr<T> take() {
        std::lock_guard<std::mutex> lk(mu);
        if (spare.empty()) return std::make_shared<T>();
        auto p = std::move(spare.back());
        spare.pop_back();
        return p;
    }
    void give(std::shared_ptr<T>& p) {
        if (p && p.use_count() == 1) {
            std::lock_guard<std::mutex> lk(mu);
            if (spare.empty()) spare.push_back(std::move(p));
        }
        p.reset();
    }
};
Recycle<Connectivity>& conn_pool() {
    static Recycle<Connectivity> r;
    return r;
}
Recycle<System>& sys_pool() {
    static Recycle<System> r;
    return r;
}
Recycle<MeshData>& child_pool() {
    static Recycle<MeshData> r;
    return r;
}

// Mesh handle: device mesh + lazily built connectivity and system caches.
struct phfem_mesh {
    ~phfem_mesh() {
        try {
            if (conn) conn->has_edges = conn->has_faces = false;
            if (sys) sys->problem = -1;
            conn_pool().give(conn);
            sys_pool().give(sys);
            child_pool().give(scratch_child);
        } catch (...) {
        }
    }
    // the mesh; an asynchronous upload completes on first access
    mutable std::shared_ptr<MeshData> data_;
    std::shared_ptr<MeshData>& data() const {
        if (data_ && data_->pending) finish_upload(*data_);
        return data_;
    }
    std::shared_ptr<Coefs> coef = std::make_shared<Coefs>();
    std::shared_ptr<Connectivity> conn;
    std::shared_ptr<System> sys;
    RefineMap last_map;
    int64_t map_ned = -1, map_ne = -1;
    std::shared_ptr<MeshData> scratch_child;  // phfem_pipeline's refinement target

    const Connectivity& table() {
        if (!conn || !conn->has_faces) {
            auto c = std::make_shared<Connectivity>();
            build_connectivity(*data(), *c, true);
            conn = c;
        }
        return *conn;
    }
    const Connectivity& edges() {
        if (!conn || !conn->has_edges) {
            auto c = std::make_shared<Connectivity>();
            build_connectivity(*data(), *c, false);
            conn = c;
        }
        return *conn;
    }
    const System& system(int problem, bool debug) {
        table();
        if (!sys || sys->problem != problem || sys->coef_version != coef->version || (debug && !sys->a_blocks.p)) {
            auto s = std::make_shared<System>();
            assemble_system(*data(), *coef, *conn, problem, *s, debug);
            sys = s;
        }
        return *sys;
    }
    void invalidate() {
        conn.reset();
        sys.reset();
    }
};

struct phfem_solution {
    std::shared_ptr<MeshData> mesh;
    std::shared_ptr<Coefs> coef;
    std::shared_ptr<Connectivity> conn;
    int problem = 0;
    SolveResult res;
    std::string method, stats;
    int workers = 1;
    int64_t n = 0, l = 0, peak_dim = 0;
    mutable std::vector<double> u_host, lambda_host;
    mutable bool host_ready = false;
    std::optional<std::array<double, 3>> errors;

    void materialise() const {
        if (host_ready) return;
        u_host = res.u.download();
        lambda_host = res.lambda.download();
        host_ready = true;
    }
};

namespace {

phfem_solution* do_solve(phfem_mesh* m, int problem, const std::string& method, int workers, double tol,
                         int64_t max_iter, int64_t peak_dim_override) {
    auto snapshot_conn = (m->table(), m->conn);
    const System& sys = m->system(problem, false);
    auto sol = std::make_unique<phfem_solution>();
    sol->mesh = m->data();
    sol->coef = m->coef;
    sol->conn = snapshot_conn;
    sol->problem = problem;
    sol->method = method;
    sol->workers = workers;
    sol->n = sys.n;
    sol->l = sys.l;
    sol->peak_dim = peak_dim_override > 0 ? peak_dim_override : sys.l;
    if (method == "direct") {
        // the reference's global route (solver.cpp:192-244) through the C++
        // API: the builtin problem's host data, assemble_system, solve_direct
        // (block inverses, device transpose and spgemms, CSR PCG)
        const HostMesh h = to_host(*m->data());
        phfem::Mesh hm;
        hm.level = h.level;
        for (size_t i = 0; i < h.coords.size(); i += 3)
            hm.coords.emplace_back(h.coords[i], h.coords[i + 1], h.coords[i + 2]);
        for (size_t i = 0; i < h.tets.size(); i += 4)
            hm.tetra.push_back({h.tets[i], h.tets[i + 1], h.tets[i + 2], h.tets[i + 3]});
        for (size_t i = 0; i < h.db.size(); i += 3) hm.dirichlet_faces.push_back({h.db[i], h.db[i + 1], h.db[i + 2]});
        for (size_t i = 0; i < h.nb.size(); i += 3) hm.neumann_faces.push_back({h.nb[i], h.nb[i + 1], h.nb[i + 2]});
        const phfem::ManufacturedProblem prob = problem == 0   ? phfem::manufactured_problem()
                                                : problem == 1 ? phfem::linear_patch_problem()
                                                               : phfem::zero_problem();
        const phfem::FaceTable ft = phfem::build_face_table(hm);
        const phfem::LinearSystem ls = phfem::assemble_system(hm, ft, prob.data);
        phfem::SolverOptions opt;
        opt.tol = tol;
        opt.max_iter = max_iter;
        const phfem::Solution hs = phfem::solve_direct(ls, opt);
        sol->res.u.upload(hs.u.data(), (int64_t)hs.u.size());
        sol->res.lambda.upload(hs.lambda.data(), (int64_t)hs.lambda.size());
        sol->res.iterations = hs.stats.iterations;
        sol->res.residual = hs.stats.residual;
        sol->res.constraint_residual = hs.stats.constraint_residual;
        sol->res.seconds = hs.stats.seconds;
        sol->res.converged = sol->res.accepted = true;
    } else {
        solve_schur(*m->data(), *m->coef, *snapshot_conn, sys, problem, tol, max_iter, method, sol->res);
    }
    sol->stats = stats_json(method, sol->n, sol->l, sol->res.iterations, sol->res.residual,
                            sol->res.constraint_residual, sol->res.seconds, workers, sol->peak_dim);
    return sol.release();
}

}  // namespace

extern "C" {

const char* phfem_last_error(void) { return g_last_error.c_str(); }

int phfem_mesh_create_cube(phfem_mesh** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("null output handle");
        auto m = std::make_unique<phfem_mesh>();
        m->data() = cube_mesh();
        *out = m.release();
    });
}

int phfem_mesh_read(const char* path, phfem_mesh** out) {
    return guarded([&] {
        if (!path || !out) throw InvalidArgument("null argument");
        std::ifstream is(path);
        if (!is) throw IoError(std::string("cannot open '") + path + "' for reading");
        auto m = std::make_unique<phfem_mesh>();
        m->data() = read_mesh(is);
        *out = m.release();
    });
}

int phfem_mesh_write(const phfem_mesh* mesh, const char* path) {
    return guarded([&] {
        if (!mesh || !path) throw InvalidArgument("null argument");
        std::ofstream os(path);
        if (!os) throw IoError(std::string("cannot open '") + path + "' for writing");
        HostMesh h = to_host(*mesh->data());
        write_mesh(os, h);
        if (!os) throw IoError(std::string("write failure on '") + path + "'");
    });
}

void phfem_mesh_destroy(phfem_mesh* mesh) { delete mesh; }

int phfem_mesh_refine(phfem_mesh* mesh, phfem_refine_times* times) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        const auto t0 = std::chrono::steady_clock::now();
        Connectivity& c = const_cast<Connectivity&>(mesh->edges());
        const int64_t ned = c.ned, ne = mesh->data()->ne;
        auto child = refine_mesh(*mesh->data(), c, &mesh->last_map);
        if (c.has_faces && !std::getenv("PHG_NO_REFINED_CONN")) {
            // keep the parent's tables for the child's closed-form grouping
            // (its own parent link is no longer needed)
            child->parent_mesh = mesh->data();
            child->parent_conn = mesh->conn;
            mesh->data()->parent_mesh.reset();
            mesh->data()->parent_conn.reset();
        }
        mesh->map_ned = ned;
        mesh->map_ne = ne;
        mesh->data() = child;
        mesh->coef = std::make_shared<Coefs>();
        mesh->invalidate();
        if (times) {
            *times = {};
            times->t_redrefine = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

// the level is known when the handle is made: no upload wait, no throw
int phfem_mesh_level(const phfem_mesh* mesh) { return mesh && mesh->data_ ? mesh->data_->level : -1; }

int phfem_mesh_counts(const phfem_mesh* mesh, int64_t* n_elems, int64_t* n_nodes, int64_t* n_edges,
                      int64_t* n_faces, phfem_refine_times* times) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        auto* m = const_cast<phfem_mesh*>(mesh);
        if (n_elems) *n_elems = m->data()->ne;
        if (n_nodes) *n_nodes = m->data()->nc;
        if (n_edges || n_faces || times) {
            const Connectivity& c = m->table();
            if (n_edges) *n_edges = c.ned;
            if (n_faces) *n_faces = c.nf;
            if (times) {
                *times = {};
                times->t_numedges = c.t_edges;
                times->t_edge2tetra = 0.0;
                times->t_faceup = c.t_faces;
            }
        }
    });
}

int phfem_mesh_system_dims(const phfem_mesh* mesh, int64_t* n, int64_t* l) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        auto* m = const_cast<phfem_mesh*>(mesh);
        if (n) *n = 4 * m->data()->ne;
        if (l) *l = m->table().l;
    });
}

int phfem_mesh_diameter(const phfem_mesh* mesh, double* h) {
    return guarded([&] {
        if (!mesh || !h) throw InvalidArgument("null argument");
        *h = mesh_diameter(*mesh->data());
    });
}

int phfem_mesh_dump_connectivity(const phfem_mesh* mesh, const char* edges_csv_path, const char* faces_csv_path) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        auto* m = const_cast<phfem_mesh*>(mesh);
        if (edges_csv_path) {  // dump_edges_csv, connectivity.cpp:211-216
            std::ofstream os(edges_csv_path);
            if (!os) throw IoError(std::string("cannot open '") + edges_csv_path + "'");
            const std::vector<int32_t> en = m->edges().edge_nodes.download();
            os << "edge_id,node1,node2\n";
            for (size_t e = 0; e < en.size() / 2; ++e)
                os << e + 1 << ',' << en[2 * e] + 1 << ',' << en[2 * e + 1] + 1 << "\n";
        }
        if (faces_csv_path) {  // dump_faces_csv, connectivity.cpp:218-225
            std::ofstream os(faces_csv_path);
            if (!os) throw IoError(std::string("cannot open '") + faces_csv_path + "'");
            const Connectivity& c = m->table();
            const std::vector<int32_t> f = c.faces.download();
            const std::vector<uint8_t> cls = c.face_class.download();
            static const char* names[] = {"interior", "dirichlet", "neumann"};
            os << "face_id,n1,n2,n3,class\n";
            for (int64_t i = 0; i < c.nf; ++i)
                os << i + 1 << ',' << f[3 * i] + 1 << ',' << f[3 * i + 1] + 1 << ',' << f[3 * i + 2] + 1 << ','
                   << names[cls[i]] << "\n";
        }
    });
}

int phfem_solve(const phfem_mesh* mesh, int problem, const char* solver, int workers, double tol,
                phfem_solution** out) {
    return guarded([&] {
        if (!mesh || !solver || !out) throw InvalidArgument("null argument");
        if (problem < 0 || problem > 2) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        const std::string name(solver);
        if (name != "direct" && name != "schur" && name != "schur-parallel")
            throw InvalidArgument("unknown solver '" + name + "' (expected direct|schur|schur-parallel)");
        auto* m = const_cast<phfem_mesh*>(mesh);
        const double t = tol > 0.0 ? tol : 1e-10;
        const int w = workers > 0 ? workers : 1;
        // solve() dispatch, solver.cpp:246-251
        std::string method = "schur";
        int wk = 1;
        int64_t peak = 0;
        if (name == "direct") {
            method = "direct";
            peak = 4 * m->data()->ne + m->table().l;
        } else if (name == "schur-parallel") {
            wk = w;
            method = w > 1 ? "schur-parallel" : "schur";
        }
        *out = do_solve(m, problem, method, wk, t, -1, peak);
    });
}

void phfem_solution_destroy(phfem_solution* sol) { delete sol; }

int phfem_solution_values(const phfem_solution* sol, const double** u, int64_t* n, const double** lambda,
                          int64_t* l) {
    return guarded([&] {
        if (!sol) throw InvalidArgument("null solution");
        sol->materialise();
        if (u) *u = sol->u_host.data();
        if (n) *n = (int64_t)sol->u_host.size();
        if (lambda) *lambda = sol->lambda_host.data();
        if (l) *l = (int64_t)sol->lambda_host.size();
    });
}

int phfem_solution_stats_json(const phfem_solution* sol, const char** json) {
    return guarded([&] {
        if (!sol || !json) throw InvalidArgument("null argument");
        *json = sol->stats.c_str();
    });
}

static const std::array<double, 3>& solution_errors(const phfem_solution* sol) {
    auto* s = const_cast<phfem_solution*>(sol);
    if (!s->errors) {
        std::array<double, 3> e{};
        error_norms(*s->mesh, *s->coef, *s->conn, s->problem, s->res.u.p, s->res.lambda.p, e.data());
        s->errors = e;
    }
    return *s->errors;
}

int phfem_solution_errors(const phfem_solution* sol, double* err_u, double* err_kappa) {
    return guarded([&] {
        if (!sol) throw InvalidArgument("null solution");
        const auto& e = solution_errors(sol);
        if (err_u) *err_u = e[0];
        if (err_kappa) *err_kappa = e[1];
    });
}

int phfem_solution_write(const phfem_solution* sol, const char* u_path, const char* lambda_path) {
    return guarded([&] {
        if (!sol) throw InvalidArgument("null solution");
        sol->materialise();
        auto write_vec = [](const char* path, const std::vector<double>& v) {
            if (!path) return;
            std::ofstream os(path);
            if (!os) throw IoError(std::string("cannot open '") + path + "'");
            for (double x : v) os << format_double(x) << "\n";
            if (!os) throw IoError(std::string("write failure on '") + path + "'");
        };
        write_vec(u_path, sol->u_host);
        write_vec(lambda_path, sol->lambda_host);
    });
}

namespace {
void write_vtk_points(std::ostream& os, const HostMesh& h) {  // vtk.cpp:15-23
    os << "# vtk DataFile Version 3.0\n"
       << "phfem level " << h.level << "\n"
       << "ASCII\n"
       << "DATASET UNSTRUCTURED_GRID\n"
       << "POINTS " << h.coords.size() / 3 << " double\n";
    for (size_t i = 0; i < h.coords.size(); i += 3)
        os << format_double(h.coords[i]) << ' ' << format_double(h.coords[i + 1]) << ' '
           << format_double(h.coords[i + 2]) << "\n";
}
}  // namespace

int phfem_export_vtk(const phfem_mesh* mesh, const phfem_solution* sol, const char* path, int with_point_data) {
    return guarded([&] {
        if (!mesh || !path) throw InvalidArgument("null argument");
        std::ofstream os(path);
        if (!os) throw IoError(std::string("cannot open '") + path + "' for writing");
        const HostMesh h = to_host(*mesh->data());
        const size_t ne = h.tets.size() / 4;
        write_vtk_points(os, h);  // export_vtk, vtk.cpp:27-58
        os << "CELLS " << ne << ' ' << 5 * ne << "\n";
        for (size_t t = 0; t < ne; ++t)
            os << "4 " << h.tets[4 * t] << ' ' << h.tets[4 * t + 1] << ' ' << h.tets[4 * t + 2] << ' '
               << h.tets[4 * t + 3] << "\n";
        os << "CELL_TYPES " << ne << "\n";
        for (size_t t = 0; t < ne; ++t) os << "10\n";
        if (!sol) return;
        sol->materialise();
        const std::vector<double>& u = sol->u_host;
        os << "CELL_DATA " << ne << "\n"
           << "SCALARS u_mean double 1\nLOOKUP_TABLE default\n";
        for (size_t t = 0; t < ne; ++t)
            os << format_double((u[4 * t] + u[4 * t + 1] + u[4 * t + 2] + u[4 * t + 3]) / 4.0) << "\n";
        if (with_point_data) {
            const size_t nc = h.coords.size() / 3;
            std::vector<double> sum(nc, 0.0);
            std::vector<int> count(nc, 0);
            for (size_t t = 0; t < ne; ++t)
                for (int v = 0; v < 4; ++v) {
                    sum[h.tets[4 * t + v]] += u[4 * t + v];
                    count[h.tets[4 * t + v]]++;
                }
            os << "POINT_DATA " << nc << "\n"
               << "SCALARS u_nodal_average double 1\nLOOKUP_TABLE default\n";
            for (size_t n = 0; n < nc; ++n) os << format_double(count[n] ? sum[n] / count[n] : 0.0) << "\n";
        }
        if (!os) throw IoError(std::string("write failure on '") + path + "'");
    });
}

int phfem_export_multiplier_vtk(const phfem_solution* sol, const char* path) {
    return guarded([&] {
        if (!sol || !path) throw InvalidArgument("null argument");
        std::ofstream os(path);
        if (!os) throw IoError(std::string("cannot open '") + path + "' for writing");
        const HostMesh h = to_host(*sol->mesh);  // export_multiplier_vtk, vtk.cpp:60-80
        write_vtk_points(os, h);
        const Connectivity& c = *sol->conn;
        const std::vector<int32_t> f = c.faces.download();
        const std::vector<int32_t> mrow = c.face_mrow.download();
        sol->materialise();
        os << "CELLS " << c.l << ' ' << 4 * c.l << "\n";
        for (int64_t i = 0; i < c.nf; ++i)
            if (mrow[i] >= 0) os << "3 " << f[3 * i] << ' ' << f[3 * i + 1] << ' ' << f[3 * i + 2] << "\n";
        os << "CELL_TYPES " << c.l << "\n";
        for (int64_t i = 0; i < c.l; ++i) os << "5\n";
        os << "CELL_DATA " << c.l << "\n"
           << "SCALARS lambda double 1\nLOOKUP_TABLE default\n";
        for (int64_t i = 0; i < c.nf; ++i)
            if (mrow[i] >= 0) os << format_double(sol->lambda_host[mrow[i]]) << "\n";
        if (!os) throw IoError(std::string("write failure on '") + path + "'");
    });
}

int phfem_dump_system(const phfem_mesh* mesh, int problem, const char* directory) {
    return guarded([&] {
        if (!mesh || !directory) throw InvalidArgument("null argument");
        if (problem < 0 || problem > 2) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        auto* m = const_cast<phfem_mesh*>(mesh);
        const System& sys = m->system(problem, true);
        const std::string dir(directory);
        auto open = [](const std::string& p) {
            std::ofstream os(p);
            if (!os) throw IoError("cannot open '" + p + "'");
            return os;
        };
        const std::vector<double> a = sys.a_blocks.download();
        const std::vector<double> coef = sys.slot_coef.download();
        const std::vector<int32_t> mrow = sys.slot_mrow.download();
        const std::vector<double> rhs = sys.rhs.download();
        const std::vector<double> bd = sys.bd.download();
        const int64_t ne = m->data()->ne;
        {  // system_a_csr dumped row-major (assembly.cpp:140-148, sparse.cpp:224-228)
            auto os = open(dir + "/a.txt");
            for (int64_t t = 0; t < ne; ++t)
                for (int i = 0; i < 4; ++i)
                    for (int j = 0; j < 4; ++j)
                        os << 4 * t + i + 1 << ' ' << 4 * t + j + 1 << ' ' << a[16 * t + 4 * i + j] << "\n";
        }
        {  // C from the slot rows, sorted by (row, col)
            static const int kFV[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {3, 2, 1}};
            std::vector<std::vector<std::pair<int64_t, double>>> rows((size_t)sys.l);
            for (int64_t t = 0; t < ne; ++t)
                for (int k = 0; k < 4; ++k) {
                    const int32_t r = mrow[4 * t + k];
                    if (r < 0) continue;
                    for (int v : kFV[k]) rows[r].push_back({4 * t + v, coef[4 * t + k]});
                }
            auto os = open(dir + "/c.txt");
            for (int64_t r = 0; r < sys.l; ++r) {
                std::sort(rows[r].begin(), rows[r].end(),
                          [](const auto& x, const auto& y) { return x.first < y.first; });
                for (const auto& e : rows[r]) os << r + 1 << ' ' << e.first + 1 << ' ' << e.second << "\n";
            }
        }
        {
            auto os = open(dir + "/rhs.txt");
            for (double v : rhs) os << format_double(v) << "\n";
        }
        {
            auto os = open(dir + "/bd.txt");
            for (double v : bd) os << format_double(v) << "\n";
        }
    });
}

// ---------------------------------------------------------------- phfem_ext

int phfem_mesh_create_from_arrays(const double* coords, int64_t n_nodes, const int32_t* tetra, int64_t n_elems,
                                  const int32_t* dirichlet, int64_t n_dir, const int32_t* neumann, int64_t n_neu,
                                  int level, phfem_mesh** out) {
    return guarded([&] {
        if (!out || (n_nodes && !coords) || (n_elems && !tetra) || (n_dir && !dirichlet) || (n_neu && !neumann))
            throw InvalidArgument("null argument");
        auto m = std::make_unique<phfem_mesh>();
        m->data() = upload_mesh(coords, n_nodes, tetra, n_elems, dirichlet, n_dir, neumann, n_neu, level);
        // index range check on the device (the host copy stays untouched)
        const MeshData& d = *m->data();
        DBuf<unsigned long long> bad(3);
        bad.fill_bytes(0xff);
        check(phfem_gpu_check_indices(d.tets.p, 4 * d.ne, d.nc, bad.p, SV()), "check indices");
        check(phfem_gpu_check_indices(d.db.p, 3 * d.nd, d.nc, bad.p + 1, SV()), "check indices");
        check(phfem_gpu_check_indices(d.nb.p, 3 * d.nn, d.nc, bad.p + 2, SV()), "check indices");
        const std::vector<unsigned long long> b = bad.download();
        const int32_t* src[3] = {tetra, dirichlet, neumann};
        for (int i = 0; i < 3; ++i)
            if (b[i] != ~0ull)
                throw InvalidArgument("node index " + std::to_string((long long)src[i][b[i]] + 1) +
                                      " out of range 1.." + std::to_string(n_nodes));
        *out = m.release();
    });
}

int phfem_mesh_create_from_arrays_async(const double* coords, int64_t n_nodes, const int32_t* tetra, int64_t n_elems,
                                        const int32_t* dirichlet, int64_t n_dir, const int32_t* neumann,
                                        int64_t n_neu, int level, phfem_mesh** out) {
    return guarded([&] {
        if (!out || (n_nodes && !coords) || (n_elems && !tetra) || (n_dir && !dirichlet) || (n_neu && !neumann))
            throw InvalidArgument("null argument");
        auto m = std::make_unique<phfem_mesh>();
        m->data_ = upload_mesh_async(coords, n_nodes, tetra, n_elems, dirichlet, n_dir, neumann, n_neu, level);
        *out = m.release();
    });
}

int phfem_mesh_create_kuhn(int nx, int ny, int nz, double lx, double ly, double lz, double jitter, uint64_t seed,
                           uint32_t dirichlet_mask, phfem_mesh** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("null output handle");
        auto m = std::make_unique<phfem_mesh>();
        m->data() = kuhn_mesh(nx, ny, nz, lx, ly, lz, jitter, seed, dirichlet_mask);
        *out = m.release();
    });
}

int phfem_mesh_sizes(const phfem_mesh* mesh, int64_t out[4]) {
    return guarded([&] {
        if (!mesh || !out) throw InvalidArgument("null argument");
        out[0] = mesh->data()->nc;
        out[1] = mesh->data()->ne;
        out[2] = mesh->data()->nd;
        out[3] = mesh->data()->nn;
    });
}

int phfem_mesh_get_arrays(const phfem_mesh* mesh, double* coords, int32_t* tetra, int32_t* dirichlet,
                          int32_t* neumann) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        const MeshData& d = *mesh->data();
        if (coords) d.coords.download_to(coords, 3 * d.nc);
        if (tetra) d.tets.download_to(tetra, 4 * d.ne);
        if (dirichlet) d.db.download_to(dirichlet, 3 * d.nd);
        if (neumann) d.nb.download_to(neumann, 3 * d.nn);
        phb::sync();
    });
}

int phfem_mesh_set_coefficients(phfem_mesh* mesh, const double* a_elem, const double* a_diag, double c) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        auto k = std::make_shared<Coefs>();
        const int64_t ne = mesh->data()->ne;
        if (a_diag) {
            k->a_diag.upload(a_diag, 3 * ne);
            k->has_diag = true;
        } else if (a_elem) {
            k->a_elem.upload(a_elem, ne);
            k->has_elem = true;
        }
        k->c = c;
        k->version = mesh->coef->version + 1;
        phb::sync();
        mesh->coef = k;
        mesh->sys.reset();
    });
}

int phfem_mesh_connectivity(const phfem_mesh* mesh, int64_t counts[6]) {
    return guarded([&] {
        if (!mesh || !counts) throw InvalidArgument("null argument");
        const Connectivity& c = const_cast<phfem_mesh*>(mesh)->table();
        counts[0] = c.ned;
        counts[1] = c.nf;
        counts[2] = c.n_int;
        counts[3] = c.n_dir;
        counts[4] = c.n_neu;
        counts[5] = c.l;
    });
}

int phfem_mesh_get_edges(const phfem_mesh* mesh, int32_t* edge_nodes, int32_t* edge_of_slot) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        const Connectivity& c = const_cast<phfem_mesh*>(mesh)->edges();
        if (edge_nodes) c.edge_nodes.download_to(edge_nodes, 2 * c.ned);
        if (edge_of_slot) c.edge_of_slot.download_to(edge_of_slot, 6 * mesh->data()->ne);
        phb::sync();
    });
}

int phfem_mesh_get_faces(const phfem_mesh* mesh, int32_t* faces, int32_t* face_of_slot, int8_t* sigma,
                         int64_t* face_slots, uint8_t* face_class, int32_t* multiplier_index, double* face_area) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        const Connectivity& c = const_cast<phfem_mesh*>(mesh)->table();
        const int64_t ne = mesh->data()->ne;
        if (faces) c.faces.download_to(faces, 3 * c.nf);
        if (face_of_slot) c.face_of_slot.download_to(face_of_slot, 4 * ne);
        if (sigma) c.sigma.download_to(sigma, 4 * ne);
        if (face_class) c.face_class.download_to(face_class, c.nf);
        if (multiplier_index) c.face_mrow.download_to(multiplier_index, c.nf);
        if (face_area) c.face_area.download_to(face_area, c.nf);
        phb::sync();
        if (face_slots) {
            const std::vector<int32_t> fs = c.face_slots.download();
            for (size_t i = 0; i < fs.size(); ++i) face_slots[i] = fs[i];
        }
    });
}

int phfem_mesh_refinement_map(const phfem_mesh* mesh, int64_t sizes[2], int32_t* midpoint_node,
                              int32_t* centroid_node) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        if (mesh->map_ned < 0) throw InvalidArgument("the mesh has not been refined");
        if (sizes) {
            sizes[0] = mesh->map_ned;
            sizes[1] = mesh->map_ne;
        }
        if (midpoint_node) mesh->last_map.midpoint.download_to(midpoint_node, mesh->map_ned);
        if (centroid_node) mesh->last_map.centroid.download_to(centroid_node, mesh->map_ne);
        phb::sync();
    });
}

int phfem_mesh_assemble(const phfem_mesh* mesh, int problem, int64_t sizes[3]) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        auto* m = const_cast<phfem_mesh*>(mesh);
        const System& sys = m->system(problem, true);
        if (sizes) {
            sizes[0] = sys.n;
            sizes[1] = sys.l;
            DBuf<int32_t> nnz(sys.l);
            check(phfem_gpu_sell_row_nnz(sys.l, sys.sell_col.p, nnz.p, SV()), "row nnz");
            DBuf<int64_t> ptr(sys.l + 1);
            DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(sys.l));
            check(phfem_gpu_scan_i32(nnz.p, ptr.p, sys.l, scratch.p, SV()), "scan");
            sizes[2] = read_scalar(ptr.p + sys.l);
        }
    });
}

int phfem_mesh_get_system(const phfem_mesh* mesh, double* a_blocks, double* slot_coef, int32_t* slot_mrow,
                          double* rhs, double* bd, int64_t* s_rowptr, int32_t* s_col, double* s_val,
                          double* rhs_neg) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        if (!mesh->sys) throw InvalidArgument("phfem_mesh_assemble has not been called");
        const System& sys = *mesh->sys;
        const int64_t ne = mesh->data()->ne;
        if ((a_blocks || slot_coef || slot_mrow) && !sys.a_blocks.p)
            throw InvalidArgument("element views were not kept");
        if ((s_rowptr || s_col || s_val) && sys.elem)
            throw InvalidArgument("the Schur matrix was not kept in row form (call phfem_mesh_assemble)");
        if (a_blocks) sys.a_blocks.download_to(a_blocks, 16 * ne);
        if (slot_coef) sys.slot_coef.download_to(slot_coef, 4 * ne);
        if (slot_mrow) sys.slot_mrow.download_to(slot_mrow, 4 * ne);
        if (rhs) sys.rhs.download_to(rhs, 4 * ne);
        if (bd) sys.bd.download_to(bd, sys.l);
        if (rhs_neg) {
            sys.finish();  // an element-major system's halves
            sys.rhs_neg.download_to(rhs_neg, sys.l);
        }
        if (s_rowptr || s_col || s_val) {
            DBuf<int32_t> nnz(sys.l);
            check(phfem_gpu_sell_row_nnz(sys.l, sys.sell_col.p, nnz.p, SV()), "row nnz");
            DBuf<int64_t> ptr(sys.l + 1);
            DBuf<unsigned char> scratch((int64_t)phfem_gpu_scan_scratch(sys.l));
            check(phfem_gpu_scan_i32(nnz.p, ptr.p, sys.l, scratch.p, SV()), "scan");
            const int64_t total = read_scalar(ptr.p + sys.l);
            DBuf<int32_t> col(total);
            DBuf<double> val(total);
            check(phfem_gpu_sell_to_csr(sys.l, sys.sell_col.p, sys.sell_val.p, ptr.p, col.p, val.p, SV()), "to csr");
            if (s_rowptr) ptr.download_to(s_rowptr, sys.l + 1);
            if (s_col) col.download_to(s_col, total);
            if (s_val) val.download_to(s_val, total);
            phb::sync();
        }
        phb::sync();
    });
}

int phfem_solve_ex(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter, phfem_solution** out) {
    return guarded([&] {
        if (!mesh || !out) throw InvalidArgument("null argument");
        if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        auto* m = const_cast<phfem_mesh*>(mesh);
        *out = do_solve(m, problem, "schur", 1, tol > 0.0 ? tol : 1e-10, max_iter, 0);
    });
}

int phfem_mesh_solve_faces(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter, double* lambda,
                           double out[3]) {
    return guarded([&] {
        if (!mesh || !out) throw InvalidArgument("null argument");
        if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        auto* m = const_cast<phfem_mesh*>(mesh);
        const System& sys = m->system(problem, false);
        SolveResult r;
        solve_schur(*m->data(), *m->coef, *m->conn, sys, problem, tol > 0.0 ? tol : 1e-10, max_iter, "schur", r, true);
        if (lambda) r.lambda.download_to(lambda, sys.l);
        phb::sync();
        out[0] = (double)r.iterations;
        out[1] = r.rel_residual;
        out[2] = r.converged ? 1.0 : 0.0;
    });
}

int phfem_mesh_solve_unverified(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter, double* u,
                                double* lambda, double out[13]) {
    return guarded([&] {
        if (!mesh || !out) throw InvalidArgument("null argument");
        if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        auto* m = const_cast<phfem_mesh*>(mesh);
        const System& sys = m->system(problem, false);
        SolveResult r;
        solve_schur(*m->data(), *m->coef, *m->conn, sys, problem, tol > 0.0 ? tol : 1e-10, max_iter, "schur", r, false,
                    false);
        double e[3];
        error_norms(*m->data(), *m->coef, *m->conn, problem, r.u.p, r.lambda.p, e);
        if (u) r.u.download_to(u, 4 * m->data()->ne);
        if (lambda) r.lambda.download_to(lambda, sys.l);
        phb::sync();
        const double v[13] = {(double)r.iterations, r.residual, r.constraint_residual, r.converged ? 1.0 : 0.0,
                              r.accepted ? 1.0 : 0.0, r.r1, r.r2, r.nrm_rhs, r.nrm_bd, r.rel_residual, e[0], e[1], e[2]};
        for (int i = 0; i < 13; ++i) out[i] = v[i];
    });
}

int phfem_solution_stats(const phfem_solution* sol, double out[4]) {
    return guarded([&] {
        if (!sol || !out) throw InvalidArgument("null argument");
        out[0] = (double)sol->res.iterations;
        out[1] = sol->res.residual;
        out[2] = sol->res.constraint_residual;
        out[3] = sol->res.seconds;
    });
}

int phfem_solution_errors_ex(const phfem_solution* sol, double out[3]) {
    return guarded([&] {
        if (!sol || !out) throw InvalidArgument("null argument");
        const auto& e = solution_errors(sol);
        for (int i = 0; i < 3; ++i) out[i] = e[i];
    });
}

void* phfem_stream(void) {
    try {
        return SV();
    } catch (...) {
        return nullptr;
    }
}

// PHFEM_FUSED_REFINE=0 keeps the separate refinement kernel in the pipeline
// pass (A/B measurements)
static bool fused_refine_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PHFEM_FUSED_REFINE");
        return !(v && v[0] == '0');
    }();
    return on;
}

int phfem_pipeline(phfem_mesh* mesh, int problem, int flags, phfem_stage_ms* ms, int64_t counts[5]) {
    return guarded([&] {
        if (!mesh) throw InvalidArgument("null mesh");
        if (problem < 0 || problem > 5) throw InvalidArgument("unknown problem id " + std::to_string(problem));
        const bool do_refine = flags & PHFEM_PIPE_REFINE;
        const bool do_assemble = !(flags & PHFEM_PIPE_NO_ASSEMBLY);
        Stages st;
        st.defer = true;  // error checks at the end of the pass (one synchronisation)
        Timer total;
        total.start();
        // rebuild everything; reuse the previous pass's device memory when no
        // solution snapshot shares it
        auto c = (mesh->conn && mesh->conn.use_count() == 1) ? mesh->conn : conn_pool().take();
        auto s = (mesh->sys && mesh->sys.use_count() == 1) ? mesh->sys : sys_pool().take();
        mesh->invalidate();
        build_connectivity(*mesh->data(), *c, true, &st);
        mesh->conn = c;
        // with both stages asked for, the assembly kernel writes the child's
        // elements and coordinates itself (assemble.cu: refine_elem); the
        // refinement stage is then the boundary lists alone
        const bool fused = do_refine && do_assemble && fused_refine_enabled();
        if (do_refine && !mesh->scratch_child) mesh->scratch_child = child_pool().take();
        if (do_assemble) {
            const MeshData& m = *mesh->data();
            phg_refine_out ro{};
            if (fused) {
                prepare_child(m, *c, mesh->scratch_child);
                ro = {m.nc, c->edge_first.p, c->edge_of_slot.p, c->edge_off.p, mesh->scratch_child->coords.p,
                      mesh->scratch_child->tets.p};
            }
            assemble_system(m, *mesh->coef, *c, problem, *s, false, &st, fused ? &ro : nullptr);
            mesh->sys = s;
        }
        int64_t ne_child = 0;
        if (do_refine) {
            auto child = refine_mesh(*mesh->data(), *c, nullptr, &st, mesh->scratch_child, fused);
            ne_child = child->ne;
        }
        const double tot = total.stop_ms();
        try {
            st.resolve();  // deferred assembly / refinement error checks
        } catch (...) {
            mesh->invalidate();  // the cached system is not valid
            throw;
        }
        if (ms) {
            ms->star = st.star;
            ms->groups = st.groups;
            ms->number = st.number;
            ms->classify = st.classify;
            ms->assemble = st.assemble;
            ms->refine = st.refine;
            ms->total = tot;
            ms->assemble_kernel = st.assemble_kernel;
        }
        if (counts) {
            counts[0] = c->ned;
            counts[1] = c->nf;
            counts[2] = c->l;
            // stored S values: element-major 10 per element, or SELL slots
            counts[3] = !do_assemble ? 0 : (s->elem ? 10 * mesh->data()->ne : s->nchunks * PHG_SELL_C * PHG_SELL_W);
            counts[4] = ne_child;
        }
    });
}

int phfem_pipeline_child(const phfem_mesh* mesh, int64_t sizes[4], double* coords, int32_t* tets, int32_t* db,
                         int32_t* nb) {
    return guarded([&] {
        if (!mesh || !sizes) throw InvalidArgument("null argument");
        const auto& ch = mesh->scratch_child;
        if (!ch || !ch->tets.p) throw InvalidArgument("no pipeline pass has refined this mesh");
        sizes[0] = ch->nc;
        sizes[1] = ch->ne;
        sizes[2] = ch->nd;
        sizes[3] = ch->nn;
        if (coords) ch->coords.download_to(coords, 3 * ch->nc);
        if (tets) ch->tets.download_to(tets, 4 * ch->ne);
        if (db) ch->db.download_to(db, 3 * ch->nd);
        if (nb) ch->nb.download_to(nb, 3 * ch->nn);
    });
}

int phfem_solve_timed(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter, double out[8],
                      double* out8) {
    return guarded([&] {
        if (!mesh || !out) throw InvalidArgument("null argument");
        auto* m = const_cast<phfem_mesh*>(mesh);
        const System& sys = m->system(problem, false);
        SolveResult r;
        bool accepted = true;
        try {
            solve_schur(*m->data(), *m->coef, *m->conn, sys, problem, tol > 0.0 ? tol : 1e-10, max_iter, "schur", r,
                        false);
        } catch (const SolverError& e) {
            // verify_solution's refusal of a converged solve (finding 8)
            if (!r.converged || std::string(e.what()).find("missed the residual target") == std::string::npos) throw;
            accepted = false;
        }
        out[0] = (double)r.iterations;
        out[1] = r.cg_ms;
        out[2] = r.iterations ? r.cg_ms / (double)r.iterations : 0.0;
        out[3] = r.converged ? 1.0 : 0.0;
        out[4] = r.seconds;
        out[5] = accepted ? 1.0 : 0.0;
        out[6] = r.residual;
        out[7] = r.constraint_residual;
        if (out8) {
            const double v[4] = {r.r1, r.r2, r.nrm_rhs, r.nrm_bd};
            for (int i = 0; i < 4; ++i) out8[i] = v[i];
        }
    });
}

}  // extern "C"
