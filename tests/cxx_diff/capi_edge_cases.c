/* Differential test of the C ABI (include/phfem.h) on edge-case meshes read
 * from the reference's text format: built against the reference's C ABI
 * (oracle/_ref/libphfem_ref.so) for the golden report and against this
 * library (tests/test_cxx_edge_cases.py).  Per mesh: refinement, counts,
 * system sizes, diameter, the Schur and direct solves (iterations; solution
 * norms and error norms on '~' lines, compared to 1e-9), and every output
 * file the ABI writes, as a byte checksum (exact) or, for files carrying
 * solution values, as a value norm ('~').  Errors print their status and
 * message.  usage: capi_edge_cases WORKDIR */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "phfem.h"

static char dir[4096];

static void path(char* out, const char* name) { snprintf(out, 4096, "%s/%s", dir, name); }

/* FNV-1a of a file's bytes, or -1 when it cannot be read */
static long long file_hash(const char* p) {
    FILE* f = fopen(p, "rb");
    if (!f) return -1;
    unsigned long long h = 1469598103934665603ull;
    int c;
    while ((c = fgetc(f)) != EOF) h = (h ^ (unsigned char)c) * 1099511628211ull;
    fclose(f);
    return (long long)(h >> 1);
}

/* l2 norm of every number in a text file (whitespace / comma separated
 * tokens that parse fully as doubles) */
static double file_norm(const char* p) {
    FILE* f = fopen(p, "r");
    if (!f) return -1.0;
    char tok[256];
    double s = 0.0;
    int c, n = 0;
    while ((c = fgetc(f)) != EOF) {
        if (c == ' ' || c == '\n' || c == ',' || c == '\t' || c == '\r') {
            if (n) {
                tok[n] = 0;
                char* end;
                double v = strtod(tok, &end);
                if (*end == 0) s += v * v;
                n = 0;
            }
        } else if (n < 255) {
            tok[n++] = (char)c;
        }
    }
    fclose(f);
    return sqrt(s);
}

static int report_rc(const char* what, int rc) {
    if (rc != PHFEM_OK) printf("%s status %d: %s\n", what, rc, phfem_last_error());
    return rc;
}

static double vnorm(const double* v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* refine = 0 where the reference's red_refine is undefined (an element
 * repeating a node id: its pair_to_edge(a, a) = -1 indexes the midpoint
 * table at -1, refine.cpp:40-41) */
static void run_mesh(const char* name, const char* text, int refine) {
    printf("== %s\n", name);
    char p[4096], q[4096], r[4096];
    path(p, "in.mesh");
    FILE* f = fopen(p, "w");
    fputs(text, f);
    fclose(f);
    phfem_mesh* m = NULL;
    if (report_rc("read", phfem_mesh_read(p, &m))) return;
    int64_t ne = 0, nc = 0, ned = 0, nf = 0, n = 0, l = 0;
    if (!report_rc("counts", phfem_mesh_counts(m, &ne, &nc, &ned, &nf, NULL)))
        printf("counts %lld %lld %lld %lld\n", (long long)ne, (long long)nc, (long long)ned, (long long)nf);
    if (!report_rc("dims", phfem_mesh_system_dims(m, &n, &l))) printf("dims %lld %lld\n", (long long)n, (long long)l);
    double h = 0.0;
    if (!report_rc("diameter", phfem_mesh_diameter(m, &h))) printf("diameter %a\n", h);
    path(p, "edges.csv");
    path(q, "faces.csv");
    if (!report_rc("dump", phfem_mesh_dump_connectivity(m, p, q)))
        printf("dump %lld %lld\n", file_hash(p), file_hash(q));
    if (!report_rc("dump_system", phfem_dump_system(m, PHFEM_PROBLEM_MANUFACTURED, dir))) {
        const char* files[4] = {"a.txt", "c.txt", "rhs.txt", "bd.txt"};
        printf("system");
        for (int i = 0; i < 4; ++i) {
            path(p, files[i]);
            printf(" %lld", file_hash(p));
        }
        printf("\n");
    }
    const char* solvers[2] = {"schur", "direct"};
    for (int k = 0; k < 2; ++k) {
        phfem_solution* s = NULL;
        char what[64];
        snprintf(what, sizeof what, "solve %s", solvers[k]);
        if (report_rc(what, phfem_solve(m, PHFEM_PROBLEM_MANUFACTURED, solvers[k], 1, 0.0, &s))) continue;
        const double *u, *lam;
        int64_t nu, nl;
        phfem_solution_values(s, &u, &nu, &lam, &nl);
        printf("%s sizes %lld %lld\n", solvers[k], (long long)nu, (long long)nl);
        printf("~%s norms %.17g %.17g\n", solvers[k], vnorm(u, nu) + 1.0, vnorm(lam, nl) + 1.0);
        double eu = 0, ek = 0;
        if (!report_rc("errors", phfem_solution_errors(s, &eu, &ek))) printf("~%s errors %.17g %.17g\n", solvers[k], eu + 1.0, ek + 1.0);
        path(p, "u.txt");
        path(q, "lambda.txt");
        if (!report_rc("solution_write", phfem_solution_write(s, p, q)))
            printf("~%s files %.17g %.17g\n", solvers[k], file_norm(p) + 1.0, file_norm(q) + 1.0);
        path(r, "sol.vtk");
        if (!report_rc("export_vtk", phfem_export_vtk(m, s, r, 1))) printf("~%s vtk %.17g\n", solvers[k], file_norm(r) + 1.0);
        path(r, "mult.vtk");
        if (!report_rc("export_multiplier_vtk", phfem_export_multiplier_vtk(s, r)))
            printf("~%s mvtk %.17g\n", solvers[k], file_norm(r) + 1.0);
        phfem_solution_destroy(s);
    }
    path(p, "mesh.vtk");
    if (!report_rc("export_vtk mesh", phfem_export_vtk(m, NULL, p, 0))) printf("mesh_vtk %lld\n", file_hash(p));
    if (refine && !report_rc("refine", phfem_mesh_refine(m, NULL))) {
        printf("level %d\n", phfem_mesh_level(m));
        if (!report_rc("counts", phfem_mesh_counts(m, &ne, &nc, &ned, &nf, NULL)))
            printf("counts %lld %lld %lld %lld\n", (long long)ne, (long long)nc, (long long)ned, (long long)nf);
        path(p, "out.mesh");
        if (!report_rc("write", phfem_mesh_write(m, p))) printf("refined_mesh %lld\n", file_hash(p));
    }
    phfem_mesh_destroy(m);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    snprintf(dir, sizeof dir, "%s", argv[1]);
    const char* tet = "COORD 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nTETRA 1\n1 2 3 4\n";
    char buf[1024];
    snprintf(buf, sizeof buf, "%sDB 4\n1 2 3\n1 3 4\n1 4 2\n4 3 2\nNB 0\n", tet);
    run_mesh("single element all Dirichlet", buf, 1);
    snprintf(buf, sizeof buf, "%sDB 0\nNB 4\n1 2 3\n1 3 4\n1 4 2\n4 3 2\n", tet);
    run_mesh("single element all Neumann", buf, 1);
    snprintf(buf, sizeof buf, "%sDB 2\n1 2 3\n4 3 2\nNB 2\n1 3 4\n1 4 2\n", tet);
    run_mesh("single element mixed", buf, 1);
    run_mesh("no elements", "COORD 2\n0 0 0\n1 1 1\nTETRA 0\nDB 0\nNB 0\n", 1);
    run_mesh("repeated node id",
             "COORD 5\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n1 1 1\nTETRA 2\n1 2 3 4\n2 2 3 5\nDB 0\nNB 0\n", 0);
    run_mesh("bad index", "COORD 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nTETRA 1\n1 2 3 9\nDB 0\nNB 0\n", 1);
    run_mesh("face not on the boundary list",
             "COORD 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nTETRA 1\n1 2 3 4\nDB 1\n1 2 3\nNB 0\n", 1);
    /* the reference cube: refined twice, the three problems, a parallel
     * Schur solve, and the dispatch's argument errors */
    printf("== cube\n");
    phfem_mesh* m = NULL;
    phfem_mesh_create_cube(&m);
    phfem_mesh_refine(m, NULL);
    phfem_mesh_refine(m, NULL);
    for (int problem = 0; problem < 3; ++problem) {
        phfem_solution* s = NULL;
        if (report_rc("solve", phfem_solve(m, problem, problem == 1 ? "schur-parallel" : "schur", 4, 0.0, &s)))
            continue;
        const double *u, *lam;
        int64_t nu, nl;
        phfem_solution_values(s, &u, &nu, &lam, &nl);
        double eu = 0, ek = 0;
        phfem_solution_errors(s, &eu, &ek);
        printf("~problem %d %.17g %.17g %.17g %.17g\n", problem, vnorm(u, nu) + 1.0, vnorm(lam, nl) + 1.0, eu + 1.0,
               ek + 1.0);
        phfem_solution_destroy(s);
    }
    phfem_solution* s = NULL;
    report_rc("unknown solver", phfem_solve(m, 0, "cholesky", 1, 0.0, &s));
    report_rc("unknown problem", phfem_solve(m, 7, "schur", 1, 0.0, &s));
    report_rc("null out", phfem_solve(m, 0, "schur", 1, 0.0, NULL));
    report_rc("null mesh", phfem_mesh_refine(NULL, NULL));
    phfem_mesh_destroy(m);
    return 0;
}
