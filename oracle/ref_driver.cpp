// Reference driver: a thin extern "C" shim over the UNMODIFIED reference
// library, compiled from the sources where they lie under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
//
// TEST INFRASTRUCTURE ONLY (see oracle/README.md): it exists to (1) pin the
// CPU restatement in phfem_oracle.c against the reference itself and
// (2) time the reference's own CPU path for bench.py's reference arm.  It
// never runs on the product path.
//
// Everything here calls the reference's public C++ entry points:
//   num_edges / edge_pairs_to_elems / faces_up / full_face_table
//     (connectivity.hpp:35, 51, 57, 79), red_refine (refine.hpp:40),
//   assemble_system (assembly.hpp:85), build_schur (solver.hpp:41),
//   pcg_jacobi (sparse.hpp:68), solve (solver.hpp:56),
//   y_norm_error / multiplier_norm_error (analysis.hpp:29-37).
// The only addition is the coefficient extension of SURVEY.md 7.1 item 1,
// applied by patching the assembled element blocks and feeding per-element
// data to the reference's load/flux callbacks (see oracle/problems.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "analysis.hpp"
#include "assembly.hpp"
#include "connectivity.hpp"
#include "mesh.hpp"
#include "refine.hpp"
#include "solver.hpp"
#include "sparse.hpp"

extern "C" {
#include "problems.h"
}

using namespace phfem;

namespace {

thread_local std::string g_err;

double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return 0;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return 1;
    } catch (const MeshError& e) {
        g_err = e.what();
        return 2;
    } catch (const SolverError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::bad_alloc&) {
        g_err = "out of memory";
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

struct Ctx {
    Mesh mesh;
    std::unique_ptr<EdgeTable> edges;
    std::unique_ptr<EdgePairToElem> e2t;
    std::unique_ptr<FaceTable> ft;
    std::unique_ptr<RefinementMap> rmap;
    // coefficient extension (empty = reference operator A = I, c = 1)
    std::vector<double> a_elem, a_diag;
    double c = 1.0;
    int problem = 0;
    std::unique_ptr<LinearSystem> sys;
    std::unique_ptr<SchurSystem> schur;
    std::unique_ptr<Solution> sol;
    double bnorm_rhs = 0.0, bnorm_bd = 0.0;

    bool default_coef() const { return a_elem.empty() && a_diag.empty() && c == 1.0; }
    void coef(std::int64_t t, double A[3]) const {
        if (!a_diag.empty()) {
            A[0] = a_diag[3 * t]; A[1] = a_diag[3 * t + 1]; A[2] = a_diag[3 * t + 2];
        } else if (!a_elem.empty()) {
            A[0] = A[1] = A[2] = a_elem[t];
        } else {
            A[0] = A[1] = A[2] = 1.0;
        }
    }
    void drop_connectivity() { edges.reset(); e2t.reset(); ft.reset(); }
    void drop_system() { sys.reset(); schur.reset(); sol.reset(); }
};

Ctx* C(void* p) { return static_cast<Ctx*>(p); }

// ProblemData with per-element coefficients.  The reference's load_vector
// calls f exactly 64 times per element in element order (assembly.cpp:65-78,
// tet_rule(5)), and neumann_vector calls g once per Neumann face in face
// order (assembly.cpp:84-92): the callbacks count calls to know the element.
struct CoefProblem {
    const Ctx* ctx;
    std::vector<std::int64_t> neumann_owner; // element of each Neumann face, face order
    std::int64_t f_calls = 0, g_calls = 0;
};

ProblemData make_data(const std::shared_ptr<CoefProblem>& cp) {
    const int kind = cp->ctx->problem;
    ProblemData d;
    d.f = [cp, kind](const Vec3& x) {
        const std::int64_t t = cp->f_calls++ / 64;
        double A[3];
        cp->ctx->coef(t, A);
        return orp_f(kind, x.x, x.y, x.z, A, cp->ctx->c);
    };
    d.u_dirichlet = [kind](const Vec3& x) { return orp_u(kind, x.x, x.y, x.z); };
    d.neumann_flux = [cp, kind](const Vec3& x, const Vec3& n) {
        const std::int64_t t = cp->neumann_owner[cp->g_calls++];
        double A[3];
        cp->ctx->coef(t, A);
        const double nn[3] = {n.x, n.y, n.z};
        return orp_g(kind, x.x, x.y, x.z, nn, A);
    };
    d.exact_u = [kind](const Vec3& x) { return orp_u(kind, x.x, x.y, x.z); };
    d.exact_grad_u = [kind](const Vec3& x) {
        double g[3];
        orp_grad(kind, x.x, x.y, x.z, g);
        return Vec3{g[0], g[1], g[2]};
    };
    return d;
}

void require_table(Ctx* c) {
    if (!c->ft) {
        c->edges = std::make_unique<EdgeTable>(num_edges(c->mesh));
        c->e2t = std::make_unique<EdgePairToElem>(edge_pairs_to_elems(c->mesh, *c->edges));
        c->ft = std::make_unique<FaceTable>(
            full_face_table(c->mesh, faces_up(c->mesh, *c->e2t, *c->edges)));
    }
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_ctx_new(const double* coords, std::int64_t nc, const std::int32_t* tets, std::int64_t ne,
                  const std::int32_t* db, std::int64_t nd, const std::int32_t* nb, std::int64_t nn,
                  int level) {
    auto* c = new Ctx;
    c->mesh.coords.resize(nc);
    for (std::int64_t i = 0; i < nc; ++i)
        c->mesh.coords[i] = Vec3{coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
    c->mesh.tetra.resize(ne);
    for (std::int64_t i = 0; i < ne; ++i)
        for (int v = 0; v < 4; ++v) c->mesh.tetra[i][v] = tets[4 * i + v];
    c->mesh.dirichlet_faces.resize(nd);
    for (std::int64_t i = 0; i < nd; ++i)
        for (int v = 0; v < 3; ++v) c->mesh.dirichlet_faces[i][v] = db[3 * i + v];
    c->mesh.neumann_faces.resize(nn);
    for (std::int64_t i = 0; i < nn; ++i)
        for (int v = 0; v < 3; ++v) c->mesh.neumann_faces[i][v] = nb[3 * i + v];
    c->mesh.level = level;
    return c;
}

void* ref_ctx_new_cube(void) {
    auto* c = new Ctx;
    c->mesh = initial_cube_mesh();
    return c;
}

void ref_ctx_free(void* p) { delete C(p); }

// sizes: [nC, nE, nD, nN, level]
void ref_mesh_sizes(void* p, std::int64_t out[5]) {
    const Mesh& m = C(p)->mesh;
    out[0] = m.num_nodes();
    out[1] = m.num_elems();
    out[2] = static_cast<std::int64_t>(m.dirichlet_faces.size());
    out[3] = static_cast<std::int64_t>(m.neumann_faces.size());
    out[4] = m.level;
}

void ref_mesh_get(void* p, double* coords, std::int32_t* tets, std::int32_t* db, std::int32_t* nb) {
    const Mesh& m = C(p)->mesh;
    if (coords)
        for (std::size_t i = 0; i < m.coords.size(); ++i) {
            coords[3 * i] = m.coords[i].x;
            coords[3 * i + 1] = m.coords[i].y;
            coords[3 * i + 2] = m.coords[i].z;
        }
    if (tets)
        for (std::size_t i = 0; i < m.tetra.size(); ++i)
            for (int v = 0; v < 4; ++v) tets[4 * i + v] = m.tetra[i][v];
    if (db)
        for (std::size_t i = 0; i < m.dirichlet_faces.size(); ++i)
            for (int v = 0; v < 3; ++v) db[3 * i + v] = m.dirichlet_faces[i][v];
    if (nb)
        for (std::size_t i = 0; i < m.neumann_faces.size(); ++i)
            for (int v = 0; v < 3; ++v) nb[3 * i + v] = m.neumann_faces[i][v];
}

// Connectivity through the reference, with the stage timings of
// refine.cpp:104-126.  times: [t_numedges, t_edge2tetra, t_faceup, t_fulltable]
int ref_connectivity(void* p, double times[4]) {
    return guard([&] {
        Ctx* c = C(p);
        c->drop_connectivity();
        auto t0 = std::chrono::steady_clock::now();
        c->edges = std::make_unique<EdgeTable>(num_edges(c->mesh));
        times[0] = secs(t0);
        t0 = std::chrono::steady_clock::now();
        c->e2t = std::make_unique<EdgePairToElem>(edge_pairs_to_elems(c->mesh, *c->edges));
        times[1] = secs(t0);
        t0 = std::chrono::steady_clock::now();
        std::vector<Tri3> faces = faces_up(c->mesh, *c->e2t, *c->edges);
        times[2] = secs(t0);
        t0 = std::chrono::steady_clock::now();
        c->ft = std::make_unique<FaceTable>(full_face_table(c->mesh, faces));
        times[3] = secs(t0);
    });
}

// Only num_edges (for the refine-only path).
int ref_num_edges(void* p, double* t) {
    return guard([&] {
        Ctx* c = C(p);
        auto t0 = std::chrono::steady_clock::now();
        c->edges = std::make_unique<EdgeTable>(num_edges(c->mesh));
        if (t) *t = secs(t0);
    });
}

// counts: [nEd, nF, n_interior, n_dirichlet, n_neumann, L]
void ref_conn_counts(void* p, std::int64_t out[6]) {
    Ctx* c = C(p);
    out[0] = c->edges ? c->edges->n_edges() : -1;
    if (c->ft) {
        out[1] = c->ft->n_faces();
        out[2] = c->ft->n_interior;
        out[3] = c->ft->n_dirichlet;
        out[4] = c->ft->n_neumann;
        out[5] = c->ft->n_multipliers();
    } else {
        out[1] = out[2] = out[3] = out[4] = out[5] = -1;
    }
}

// edge_nodes [2 nEd]; edge_of_slot [6 nE] via pair_to_edge over the local
// pair order (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) (connectivity.cpp:15-18).
void ref_get_edges(void* p, std::int32_t* edge_nodes, std::int32_t* edge_of_slot) {
    Ctx* c = C(p);
    const EdgeTable& e = *c->edges;
    if (edge_nodes)
        for (std::int64_t i = 0; i < e.n_edges(); ++i) {
            edge_nodes[2 * i] = e.edge_nodes[i][0];
            edge_nodes[2 * i + 1] = e.edge_nodes[i][1];
        }
    if (edge_of_slot) {
        static const int P[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
        for (std::int64_t t = 0; t < c->mesh.num_elems(); ++t)
            for (int k = 0; k < 6; ++k)
                edge_of_slot[6 * t + k] =
                    e.pair_to_edge(c->mesh.tetra[t][P[k][0]], c->mesh.tetra[t][P[k][1]]);
    }
}

std::int64_t ref_e2t_size(void* p) { return static_cast<std::int64_t>(C(p)->e2t->entries.size()); }

void ref_get_e2t(void* p, std::uint64_t* keys, std::int32_t* elems) {
    const auto& en = C(p)->e2t->entries;
    for (std::size_t i = 0; i < en.size(); ++i) {
        keys[i] = en[i].first;
        elems[i] = en[i].second;
    }
}

// faces [3 nF], face_of_slot [4 nE], sigma [4 nE] (+1/-1 as int8),
// face_slots [2 nF] int64, face_class [nF] (0 int, 1 dir, 2 neu),
// mrow [nF], area [nF]
void ref_get_faces(void* p, std::int32_t* faces, std::int32_t* face_of_slot, std::int8_t* sigma,
                   std::int64_t* face_slots, std::uint8_t* face_class, std::int32_t* mrow,
                   double* area) {
    const FaceTable& ft = *C(p)->ft;
    for (std::int64_t f = 0; f < ft.n_faces(); ++f) {
        if (faces)
            for (int v = 0; v < 3; ++v) faces[3 * f + v] = ft.faces[f][v];
        if (face_slots) {
            face_slots[2 * f] = ft.face_slots[f][0];
            face_slots[2 * f + 1] = ft.face_slots[f][1];
        }
        if (face_class) face_class[f] = static_cast<std::uint8_t>(ft.face_class[f]);
        if (mrow) mrow[f] = ft.multiplier_index[f];
        if (area) area[f] = ft.face_area[f];
    }
    for (std::size_t s = 0; s < ft.slot_to_face.size(); ++s) {
        if (face_of_slot) face_of_slot[s] = ft.slot_to_face[s];
        if (sigma) sigma[s] = ft.sigma[s] > 0 ? 1 : -1;
    }
}

// One red refinement through the reference (refine.cpp:16-96), replacing the
// context's mesh; reuses the edge table when present.
int ref_refine(void* p, double* t_refine) {
    return guard([&] {
        Ctx* c = C(p);
        if (!c->edges) c->edges = std::make_unique<EdgeTable>(num_edges(c->mesh));
        auto t0 = std::chrono::steady_clock::now();
        auto res = red_refine(c->mesh, *c->edges);
        if (t_refine) *t_refine = secs(t0);
        c->mesh = std::move(res.first);
        c->rmap = std::make_unique<RefinementMap>(std::move(res.second));
        c->drop_connectivity();
        c->drop_system();
        c->a_elem.clear();
        c->a_diag.clear();
    });
}

// midpoint_node [nEd of the parent], centroid_node [nE parent]
void ref_get_refinement_map(void* p, std::int32_t* midpoint, std::int32_t* centroid) {
    const RefinementMap& m = *C(p)->rmap;
    if (midpoint) std::copy(m.midpoint_node.begin(), m.midpoint_node.end(), midpoint);
    if (centroid) std::copy(m.centroid_node.begin(), m.centroid_node.end(), centroid);
}

void ref_set_coefficients(void* p, const double* a_elem, const double* a_diag, double cc) {
    Ctx* c = C(p);
    const std::int64_t ne = c->mesh.num_elems();
    c->a_elem.clear();
    c->a_diag.clear();
    if (a_elem) c->a_elem.assign(a_elem, a_elem + ne);
    if (a_diag) c->a_diag.assign(a_diag, a_diag + 3 * ne);
    c->c = cc;
    c->drop_system();
}

// assemble_system (assembly.cpp:106-138) with the coefficient extension:
// A_T = K_T(A) + c M_T with K_ij = V * ((A0 gx gx' + A1 gy gy') + A2 gz gz'),
// which is bit-identical to mat4_add(k, m) at A = I, c = 1.
// times: [assemble]
int ref_assemble(void* p, int problem, double* t_asm) {
    return guard([&] {
        Ctx* c = C(p);
        c->problem = problem;
        require_table(c);
        auto cp = std::make_shared<CoefProblem>();
        cp->ctx = c;
        for (std::int64_t f = 0; f < c->ft->n_faces(); ++f)
            if (c->ft->face_class[f] == FaceClass::Neumann)
                cp->neumann_owner.push_back(c->ft->face_slots[f][0] / 4);
        const ProblemData data = make_data(cp);
        auto t0 = std::chrono::steady_clock::now();
        c->sys = std::make_unique<LinearSystem>(assemble_system(c->mesh, *c->ft, data));
        if (!c->default_coef()) {
            for (std::int64_t t = 0; t < c->mesh.num_elems(); ++t) {
                const LocalStiffnessMass loc = local_stiffness_mass(c->mesh, ElemId(t));
                double A[3];
                c->coef(t, A);
                for (int i = 0; i < 4; ++i)
                    for (int j = 0; j < 4; ++j) {
                        const Vec3& gi = loc.grads[i];
                        const Vec3& gj = loc.grads[j];
                        const double d =
                            A[0] * (gi.x * gj.x) + A[1] * (gi.y * gj.y) + A[2] * (gi.z * gj.z);
                        c->sys->a_blocks[t][i][j] = loc.volume * d + c->c * loc.m[i][j];
                    }
            }
        }
        if (t_asm) *t_asm = secs(t0);
        c->bnorm_rhs = norm2(c->sys->rhs);
        c->bnorm_bd = norm2(c->sys->dirichlet_rhs);
    });
}

// sizes: [n, l, nnz(C)]
void ref_system_sizes(void* p, std::int64_t out[3]) {
    const LinearSystem& s = *C(p)->sys;
    out[0] = s.n;
    out[1] = s.l;
    out[2] = s.c.nnz();
}

void ref_get_system(void* p, double* a_blocks, double* slot_coef, std::int32_t* slot_mrow,
                    double* rhs, double* bd, std::int64_t* c_rowptr, std::int32_t* c_col,
                    double* c_val) {
    const LinearSystem& s = *C(p)->sys;
    const std::size_t ne = s.a_blocks.size();
    for (std::size_t t = 0; t < ne; ++t) {
        if (a_blocks)
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) a_blocks[16 * t + 4 * i + j] = s.a_blocks[t][i][j];
        for (int k = 0; k < 4; ++k) {
            if (slot_coef) slot_coef[4 * t + k] = s.slot_coef[t][k];
            if (slot_mrow) slot_mrow[4 * t + k] = s.slot_mrow[t][k];
        }
    }
    if (rhs) std::copy(s.rhs.begin(), s.rhs.end(), rhs);
    if (bd) std::copy(s.dirichlet_rhs.begin(), s.dirichlet_rhs.end(), bd);
    if (c_rowptr) std::copy(s.c.row_ptr.begin(), s.c.row_ptr.end(), c_rowptr);
    if (c_col) std::copy(s.c.col.begin(), s.c.col.end(), c_col);
    if (c_val) std::copy(s.c.val.begin(), s.c.val.end(), c_val);
}

// build_schur (solver.cpp:90-147).  times: [build_schur]
int ref_build_schur(void* p, int workers, double* t_schur) {
    return guard([&] {
        Ctx* c = C(p);
        auto t0 = std::chrono::steady_clock::now();
        c->schur = std::make_unique<SchurSystem>(build_schur(*c->sys, workers));
        if (t_schur) *t_schur = secs(t0);
    });
}

std::int64_t ref_schur_nnz(void* p) { return C(p)->schur->s_neg.nnz(); }

void ref_get_schur(void* p, std::int64_t* rowptr, std::int32_t* col, double* val, double* rhs_neg) {
    const SchurSystem& s = *C(p)->schur;
    if (rowptr) std::copy(s.s_neg.row_ptr.begin(), s.s_neg.row_ptr.end(), rowptr);
    if (col) std::copy(s.s_neg.col.begin(), s.s_neg.col.end(), col);
    if (val) std::copy(s.s_neg.val.begin(), s.s_neg.val.end(), val);
    if (rhs_neg) std::copy(s.rhs_neg.begin(), s.rhs_neg.end(), rhs_neg);
}

// A bounded CG prefix on the built Schur system with the reference's
// inner_cg_options (solver.cpp:78-86), for per-iteration timing.
int ref_cg_prefix(void* p, std::int64_t iters, double tol, double* seconds, std::int64_t* done) {
    return guard([&] {
        Ctx* c = C(p);
        CgOptions o;
        o.tol = tol;
        o.abs_tol = 0.2 * tol * std::hypot(c->bnorm_rhs, c->bnorm_bd);
        o.max_iter = iters;
        std::vector<double> x(c->sys->l, 0.0);
        auto t0 = std::chrono::steady_clock::now();
        const CgResult r = pcg_jacobi(c->schur->s_neg, c->schur->rhs_neg, x, o);
        if (seconds) *seconds = secs(t0);
        if (done) *done = r.iterations;
    });
}

// Full solve through solve() (solver.cpp:246-251): "schur" / "schur-parallel" /
// "direct".  stats: [iterations, residual, constraint_residual, seconds]
int ref_solve(void* p, const char* method, int workers, double tol, std::int64_t max_iter,
              double stats[4]) {
    return guard([&] {
        Ctx* c = C(p);
        SolverOptions opt;
        if (tol > 0.0) opt.tol = tol;
        opt.workers = workers > 0 ? workers : 1;
        if (max_iter > 0) opt.max_iter = max_iter;
        c->sol = std::make_unique<Solution>(solve(*c->sys, method, opt));
        stats[0] = double(c->sol->stats.iterations);
        stats[1] = c->sol->stats.residual;
        stats[2] = c->sol->stats.constraint_residual;
        stats[3] = c->sol->stats.seconds;
    });
}

void ref_get_solution(void* p, double* u, double* lambda) {
    const Solution& s = *C(p)->sol;
    if (u) std::copy(s.u.begin(), s.u.end(), u);
    if (lambda) std::copy(s.lambda.begin(), s.lambda.end(), lambda);
}

// Errors of the current solution.  At the reference operator these are the
// reference's y_norm_error / multiplier_norm_error (analysis.cpp:51-105); the
// L2 error (the north-star check) mirrors y_norm_error's quadrature without
// the gradient term and the h weight.  out: [err_y, err_kappa, err_l2]
int ref_errors(void* p, double out[3]) {
    return guard([&] {
        Ctx* c = C(p);
        const int kind = c->problem;
        auto cp = std::make_shared<CoefProblem>();
        cp->ctx = c;
        const ProblemData data = make_data(cp);
        const Mesh& mesh = c->mesh;
        const Solution& sol = *c->sol;
        if (c->default_coef()) {
            out[0] = y_norm_error(mesh, sol, data);
            out[1] = multiplier_norm_error(mesh, *c->ft, sol, data);
        } else {
            out[0] = -1.0;
            out[1] = -1.0;
        }
        static const TetRule quad = tet_rule(9);
        double acc = 0.0;
        for (ElemId t = 0; t < mesh.num_elems(); ++t) {
            const Tet4& e = mesh.tetra[t];
            const Vec3 pt[4] = {mesh.coords[e[0]], mesh.coords[e[1]], mesh.coords[e[2]],
                                mesh.coords[e[3]]};
            const double vol = elem_volume(mesh, t);
            for (const auto& q : quad.points) {
                const Vec3 x = pt[0] * q.lambda[0] + pt[1] * q.lambda[1] + pt[2] * q.lambda[2] +
                               pt[3] * q.lambda[3];
                double uh = 0.0;
                for (int v = 0; v < 4; ++v) uh += q.lambda[v] * sol.u[4 * t + v];
                const double dv = orp_u(kind, x.x, x.y, x.z) - uh;
                acc += vol * q.w * (dv * dv);
            }
        }
        out[2] = std::sqrt(acc);
    });
}

} // extern "C"
