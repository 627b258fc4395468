/* phfem_ext.h — extensions of the reference C ABI (phfem.h) needed by the
 * BASELINE.json configs and by parity/benchmark harnesses.  The reference has
 * only the 5-tet cube, a text reader and three built-in problems
 * (phfem.h:31-47); configs 2-5 need Kuhn meshes, per-element coefficients and
 * the config problems.  All entry points follow the
 * reference's conventions: status codes of phfem_status, message in
 * phfem_last_error(), 0-based indices, host pointers.
 */
#ifndef PHFEM_EXT_H
#define PHFEM_EXT_H

#include "phfem.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Problem kinds beyond phfem_problem (0..2). */
enum phfem_problem_ext {
    PHFEM_PROBLEM_SIN3 = 3,    /* u = sin(pi x) sin(pi y) sin(pi z)  (configs 1, 4) */
    PHFEM_PROBLEM_EXPCOS = 4,  /* u = exp(x) cos(pi y) z^2           (config 3) */
    PHFEM_PROBLEM_POLYSIN = 5  /* u = x (8-x) sin(pi y) sin(pi z)    (config 5) */
};

/* Mesh from host arrays: coords [3 nC], tetra [4 nE], dirichlet [3 nD],
 * neumann [3 nN], 0-based.  Replaces phfem_mesh_read for in-memory data
 * (mesh.cpp:162-182 validates the same index ranges). */
int phfem_mesh_create_from_arrays(const double* coords, int64_t n_nodes, const int32_t* tetra,
                                  int64_t n_elems, const int32_t* dirichlet, int64_t n_dir,
                                  const int32_t* neumann, int64_t n_neu, int level,
                                  phfem_mesh** out);

/* The same, returning before the upload completes: the copies (and the
 * index check) run on a separate stream and copy engine, so a caller can
 * stage the next mesh while the device still works on the previous one.
 * The host arrays (page-locked for overlap) must stay valid and unchanged
 * until the mesh's first use, which waits for the upload and reports an
 * out-of-range index as PHFEM_ERR_INVALID_ARGUMENT. */
int phfem_mesh_create_from_arrays_async(const double* coords, int64_t n_nodes, const int32_t* tetra,
                                        int64_t n_elems, const int32_t* dirichlet, int64_t n_dir,
                                        const int32_t* neumann, int64_t n_neu, int level,
                                        phfem_mesh** out);

/* n_x*n_y*n_z cells x 6 Kuhn tetrahedra on [0,lx]x[0,ly]x[0,lz], generated
 * on the device.  Interior nodes move by (2u-1)*jitter*h per axis with
 * u = (splitmix64(seed ^ (3n+axis)) >> 11) * 2^-53.  dirichlet_mask bit p
 * makes plane p Dirichlet (0:x=0 1:x=lx 2:y=0 3:y=ly 4:z=0 5:z=lz), the other
 * boundary planes are Neumann. */
int phfem_mesh_create_kuhn(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                           uint64_t seed, uint32_t dirichlet_mask, phfem_mesh** out);

/* sizes out: [nC, nE, nD, nN] */
int phfem_mesh_sizes(const phfem_mesh* mesh, int64_t out[4]);
/* device -> host copies; any pointer may be NULL */
int phfem_mesh_get_arrays(const phfem_mesh* mesh, double* coords, int32_t* tetra,
                          int32_t* dirichlet, int32_t* neumann);

/* Coefficient extension -div(A grad u) + c u = f with A = a_elem[t] I or
 * diag(a_diag[3t..3t+2]) per element (a_diag wins; both NULL: A = I).
 * Reduces bit-exactly to the reference operator at A = I, c = 1. */
int phfem_mesh_set_coefficients(phfem_mesh* mesh, const double* a_elem, const double* a_diag,
                                double c);

/* Connectivity (built lazily like phfem_mesh_counts).
 * counts out: [nEd, nF, n_interior, n_dirichlet, n_neumann, L] */
int phfem_mesh_connectivity(const phfem_mesh* mesh, int64_t counts[6]);
/* EdgeTable: edge_nodes [2 nEd] (sorted pairs, first-occurrence order),
 * edge_of_slot [6 nE] (pair_to_edge of the local pairs) */
int phfem_mesh_get_edges(const phfem_mesh* mesh, int32_t* edge_nodes, int32_t* edge_of_slot);
/* FaceTable (connectivity.hpp:57-77): faces [3 nF], face_of_slot [4 nE],
 * sigma [4 nE] (+1/-1), face_slots [2 nF], face_class [nF] (0 interior,
 * 1 Dirichlet, 2 Neumann), multiplier_index [nF], face_area [nF] */
int phfem_mesh_get_faces(const phfem_mesh* mesh, int32_t* faces, int32_t* face_of_slot,
                         int8_t* sigma, int64_t* face_slots, uint8_t* face_class,
                         int32_t* multiplier_index, double* face_area);
/* RefinementMap of the last phfem_mesh_refine on this handle
 * (refine.hpp:13-17): midpoint_node [nEd parent], centroid_node [nE parent] */
int phfem_mesh_refinement_map(const phfem_mesh* mesh, int64_t sizes[2], int32_t* midpoint_node,
                              int32_t* centroid_node);

/* Assembly + condensation of `problem` on the mesh (cached on the handle).
 * sizes out: [N, L, nnz(S)] */
int phfem_mesh_assemble(const phfem_mesh* mesh, int problem, int64_t sizes[3]);
/* LinearSystem / SchurSystem views (assembly.hpp:69-84, solver.hpp:36-40):
 * a_blocks [16 nE], slot_coef [4 nE], slot_mrow [4 nE], rhs [N], bd [L],
 * S as CSR (rows sorted by column) s_rowptr [L+1], s_col, s_val [nnz],
 * rhs_neg [L].  Any pointer may be NULL. */
int phfem_mesh_get_system(const phfem_mesh* mesh, double* a_blocks, double* slot_coef,
                          int32_t* slot_mrow, double* rhs, double* bd, int64_t* s_rowptr,
                          int32_t* s_col, double* s_val, double* rhs_neg);

/* phfem_solve for any problem kind and the handle's coefficients; the
 * solver is always the element-local Schur path. max_iter <= 0: 10 L. */
int phfem_solve_ex(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter,
                   phfem_solution** out);
/* The face solve alone: pcg_jacobi on s_neg with inner_cg_options
 * (sparse.cpp:163-212, solver.cpp:78-86), no recovery and no
 * verify_solution (which can reject a converged solve, SURVEY finding 8).
 * lambda [L] host output; out: [iterations, rel_residual, converged]. */
int phfem_mesh_solve_faces(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter,
                           double* lambda, double out[3]);
/* The whole Schur path (face solve, recovery, verify_solution's residuals,
 * error norms) without raising on verify_solution's refusal of a converged
 * solve (SURVEY finding 8), for parity checks of U and Lambda where the
 * reference itself refuses.  u [4 nE], lambda [L] host outputs (may be
 * NULL).  out: [iterations, residual, constraint_residual, converged,
 * accepted, ||AU - C'L - B||, ||CU - b_D||, ||B||, ||b_D||, CG rel_residual,
 * y-norm error, multiplier h-norm error, L2 error] */
int phfem_mesh_solve_unverified(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter,
                                double* u, double* lambda, double out[13]);
/* out: [iterations, residual, constraint_residual, seconds] */
int phfem_solution_stats(const phfem_solution* sol, double out[4]);
/* out: [broken Y-norm error, multiplier h-norm error, L2 error] */
int phfem_solution_errors_ex(const phfem_solution* sol, double out[3]);

/* --- device-resident pipeline (benchmarking) ---------------------------- */

/* The library's CUDA stream (cudaStream_t) so callers can time on it. */
void* phfem_stream(void);

/* Stage times of one pass of the hot path, milliseconds from CUDA events on
 * phfem_stream(). */
typedef struct phfem_stage_ms {
    double star;      /* vertex -> element incidence */
    double groups;    /* edge/face grouping per vertex */
    double number;    /* scans + id assignment + slot fill */
    double classify;  /* boundary classification + multiplier rows */
    double assemble;  /* fused assembly + condensation */
    double refine;    /* red refinement (children + nodes + boundary) */
    double total;
    double assemble_kernel; /* the fused assembly kernel alone (roofline) */
} phfem_stage_ms;

/* One full pass on a device-resident mesh: connectivity (edges + faces),
 * assembly + condensation of `problem` and one red refinement into a scratch
 * mesh that is discarded.  flags: PHFEM_PIPE_REFINE (1) includes the
 * refinement, PHFEM_PIPE_NO_ASSEMBLY (2) skips assembly + condensation.
 * Caches on the handle are rebuilt (not reused).  counts out (may be NULL):
 * [nEd, nF, L, nnz(S) padded, nE children] */
#define PHFEM_PIPE_REFINE 1
#define PHFEM_PIPE_NO_ASSEMBLY 2
int phfem_pipeline(phfem_mesh* mesh, int problem, int flags, phfem_stage_ms* ms,
                   int64_t counts[5]);
/* The last phfem_pipeline refinement's child: sizes out [nC, nE, nD, nN];
 * arrays (each may be NULL) sized from them.  PHFEM_ERR_ARGUMENT when no
 * pass refined. */
int phfem_pipeline_child(const phfem_mesh* mesh, int64_t sizes[4], double* coords, int32_t* tets,
                         int32_t* db, int32_t* nb);

/* Schur solve (assembly cached): Jacobi-PCG timed on the device, then
 * recovery and verify_solution; a verify refusal (SURVEY finding 8) is
 * reported, not raised.  out: [iterations, cg_ms, ms_per_iteration,
 * converged, total_s (CG + recovery + verify wall time), accepted,
 * residual, constraint_residual]; verify_terms (may be NULL): [||AU - C'L - B||,
 * ||CU - b_D||, ||B||, ||b_D||] (verify_solution, solver.cpp:44-76) */
int phfem_solve_timed(const phfem_mesh* mesh, int problem, double tol, int64_t max_iter,
                      double out[8], double* verify_terms);

#ifdef __cplusplus
}
#endif

#endif
