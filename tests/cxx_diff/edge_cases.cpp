// Differential test of the C++ API on edge cases: the same program is built
// against the reference (/root/reference/proj/src headers, oracle/_ref's
// libphfem_ref.so: the reference's own code) and against this repository's
// drop-in (include/phfem_cxx, libphfem.so), and the two reports must agree
// (tests/test_cxx_edge_cases.py; the reference's report is committed as
// tests/golden/cxx_edge_cases.txt by tests/cxx_diff/Makefile).
//
// Each line is "key value..." and exact (integers, tables, and the element /
// Schur data, which the device path reproduces bit for bit), except lines
// starting with '~' whose numbers are compared to 1e-9 relative (solutions:
// the CG's dot products are summed in another order).  Exceptions print
// their class and message.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "analysis.hpp"
#include "connectivity.hpp"
#include "errors.hpp"
#include "mesh.hpp"
#include "refine.hpp"
#include "solver.hpp"

using namespace phfem;

namespace {

void put_ints(const char* key, const std::vector<long long>& v) {
    std::printf("%s %zu", key, v.size());
    for (long long x : v) std::printf(" %lld", x);
    std::printf("\n");
}

void put_exact(const char* key, const std::vector<double>& v) {
    std::printf("%s %zu", key, v.size());
    for (double x : v) std::printf(" %a", x);
    std::printf("\n");
}

double norm(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

template <class F>
void run(const char* name, F f) {
    std::printf("== %s\n", name);
    try {
        f();
    } catch (const MeshError& e) {
        std::printf("MeshError %s\n", e.what());
    } catch (const SolverError& e) {
        std::printf("SolverError %s\n", e.what());
    } catch (const InvalidArgument& e) {
        std::printf("InvalidArgument %s\n", e.what());
    }
}

Mesh single_tet(const std::vector<int>& dirichlet_faces) {
    Mesh m;
    m.coords = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    m.tetra = {{0, 1, 2, 3}};
    const int fv[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {3, 2, 1}};
    for (int k = 0; k < 4; ++k) {
        const Tri3 f = {m.tetra[0][fv[k][0]], m.tetra[0][fv[k][1]], m.tetra[0][fv[k][2]]};
        bool dir = false;
        for (int d : dirichlet_faces) dir = dir || d == k;
        (dir ? m.dirichlet_faces : m.neumann_faces).push_back(f);
    }
    return m;
}

void report_tables(const Mesh& m) {
    const EdgeTable e = num_edges(m);
    std::vector<long long> en;
    for (const auto& p : e.edge_nodes) {
        en.push_back(p[0]);
        en.push_back(p[1]);
    }
    put_ints("edge_nodes", en);
    const FaceTable ft = build_face_table(m);
    std::vector<long long> fs, fc, mi;
    for (const auto& f : ft.faces)
        for (int j = 0; j < 3; ++j) fs.push_back(f[j]);
    for (auto c : ft.face_class) fc.push_back((long long)c);
    for (auto r : ft.multiplier_index) mi.push_back(r);
    put_ints("faces", fs);
    put_ints("face_class", fc);
    put_ints("multiplier_index", mi);
    put_exact("face_area", ft.face_area);
    std::printf("counts %lld %lld %lld\n", (long long)ft.n_interior, (long long)ft.n_dirichlet,
                (long long)ft.n_neumann);
}

void report_solve(const Mesh& m, const char* method) {
    const FaceTable ft = build_face_table(m);
    const ManufacturedProblem p = manufactured_problem();
    const LinearSystem sys = assemble_system(m, ft, p.data);
    put_exact("rhs", sys.rhs);
    put_exact("dirichlet_rhs", sys.dirichlet_rhs);
    const SchurSystem s = build_schur(sys);
    put_exact("s_val", s.s_neg.val);
    put_exact("rhs_neg", s.rhs_neg);
    SolverOptions opt;
    const Solution sol = solve(sys, method, opt);
    std::printf("l %lld n %lld\n", (long long)sol.stats.l, (long long)sol.stats.n);
    std::printf("~norms %.17g %.17g\n", norm(sol.u), norm(sol.lambda));
    std::printf("~errors %.17g %.17g\n", y_norm_error(m, sol, p.data), multiplier_norm_error(m, ft, sol, p.data));
}

}  // namespace

int main() {
    run("empty mesh tables", [] {
        Mesh m;
        m.coords = {{0, 0, 0}};
        report_tables(m);
        const EdgeTable e = num_edges(m);
        const auto [child, map] = red_refine(m, e);
        std::printf("child %zu %zu\n", child.coords.size(), child.tetra.size());
    });
    run("single element all Dirichlet", [] {
        const Mesh m = single_tet({0, 1, 2, 3});
        report_tables(m);
        report_solve(m, "schur");
    });
    run("single element all Neumann", [] {
        const Mesh m = single_tet({});
        report_tables(m);
        report_solve(m, "schur");
    });
    run("single element mixed, direct", [] {
        const Mesh m = single_tet({0, 3});
        report_solve(m, "direct");
    });
    run("repeated node id", [] {
        Mesh m;
        m.coords = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 1}};
        m.tetra = {{0, 1, 2, 3}, {1, 1, 2, 4}};
        const EdgeTable e = num_edges(m);
        std::vector<long long> en;
        for (const auto& p : e.edge_nodes) {
            en.push_back(p[0]);
            en.push_back(p[1]);
        }
        put_ints("edge_nodes", en);
        const EdgePairToElem e2t = edge_pairs_to_elems(m, e);
        std::vector<long long> keys, elems;
        for (const auto& kv : e2t.entries) {
            keys.push_back((long long)kv.first);
            elems.push_back(kv.second);
        }
        put_ints("e2t_keys", keys);
        put_ints("e2t_elems", elems);
        report_tables(m);
    });
    run("cube level 1 schur", [] {
        const Mesh m0 = initial_cube_mesh();
        const auto [m, map] = red_refine(m0, num_edges(m0));
        report_solve(m, "schur");
    });
    run("refine_to_level 2 log", [] {
        std::vector<LevelInfo> log;
        const Mesh m = refine_to_level(2, &log);
        std::printf("mesh %zu %zu %zu %zu\n", m.coords.size(), m.tetra.size(), m.dirichlet_faces.size(),
                    m.neumann_faces.size());
        for (const auto& li : log)
            std::printf("level %d %lld %lld %lld %lld\n", li.level, (long long)li.n_elems, (long long)li.n_nodes,
                        (long long)li.n_edges, (long long)li.n_faces);
    });
    run("linear patch, schur and parallel schur", [] {
        const Mesh m0 = initial_cube_mesh();
        const auto [m, map] = red_refine(m0, num_edges(m0));
        const FaceTable ft = build_face_table(m);
        const ManufacturedProblem p = linear_patch_problem();
        const LinearSystem sys = assemble_system(m, ft, p.data);
        SolverOptions opt;
        const Solution a = solve(sys, "schur", opt);
        opt.workers = 4;
        const Solution b = solve_schur_parallel(sys, 4, opt);
        std::printf("~patch %.17g %.17g %.17g %.17g\n", norm(a.u), norm(a.lambda), norm(b.u), norm(b.lambda));
        std::printf("~patch_errors %.17g %.17g\n", y_norm_error(m, a, p.data) + 1.0,
                    multiplier_norm_error(m, ft, a, p.data) + 1.0);
    });
    run("pcg on an empty and a 1x1 matrix", [] {
        CsrMatrix a;
        a.row_ptr = {0};
        std::vector<double> b, x;
        const CgResult r0 = pcg_jacobi(a, b, x);
        std::printf("empty %lld %d %a\n", (long long)r0.iterations, (int)r0.converged, r0.rel_residual);
        CsrMatrix one;
        one.n_rows = one.n_cols = 1;
        one.row_ptr = {0, 1};
        one.col = {0};
        one.val = {4.0};
        std::vector<double> b1 = {2.0}, x1 = {0.0};
        const CgResult r1 = pcg_jacobi(one, b1, x1);
        std::printf("one %lld %d %a %a\n", (long long)r1.iterations, (int)r1.converged, r1.rel_residual, x1[0]);
    });
    return 0;
}
