/* CPU oracle for the phfem hot path — TEST INFRASTRUCTURE.
 *
 * A plain-C restatement of the reference algorithm (proj/src of
 * arXiv 2509.11133's phfem library), used only by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg, always as the
 * checker and never as the thing measured or shipped.  Every function cites
 * the reference file:line it restates (paths relative to proj/src).
 *
 * Parity pinning: tests/test_oracle_pins.py checks this restatement against
 * (a) the golden vectors in the reference's own unit tests
 *     (test_connectivity.cpp, test_refine.cpp, test_assembly.cpp,
 *      test_solver.cpp, test_analysis.cpp) and
 * (b) the reference library itself, compiled from its sources into
 *     oracle/_ref by oracle/Makefile, bit for bit on connectivity, refinement
 *     and element/Schur entries, on the 5-tet cube family and Kuhn meshes.
 * The coefficient extension (A != I or c != 1) is pinned against the
 * reference with its element blocks patched the same way (ref_driver.cpp).
 *
 * Conventions: coords double[3 nC] (x,y,z per node), tets int32[4 nE],
 * boundary faces int32[3 n], all 0-based; slot s = 4t+k (faces) or 6t+k
 * (edges).  Functions return 0 on success or the reference's status code
 * (1 argument, 2 mesh, 3 solver) with or_last_error() set to the reference's
 * message.
 */
#ifndef PHFEM_ORACLE_H
#define PHFEM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* --- seeded inputs ------------------------------- */
uint64_t or_splitmix64(uint64_t x);
double or_uniform(uint64_t seed, uint64_t idx); /* (splitmix64(seed^idx) >> 11) * 2^-53 */

/* n_x*n_y*n_z cells x 6 Kuhn tetrahedra on [0,lx]x[0,ly]x[0,lz].
 * sizes out: [nC, nE, nD, nN].  dirichlet_mask bit p marks plane p Dirichlet:
 * 0:x=0 1:x=lx 2:y=0 3:y=ly 4:z=0 5:z=lz (the rest are Neumann). */
void or_kuhn_sizes(int nx, int ny, int nz, uint32_t dirichlet_mask, int64_t out[4]);
void or_kuhn_mesh(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                  uint64_t seed, uint32_t dirichlet_mask, double* coords, int32_t* tets,
                  int32_t* db, int32_t* nb);

/* --- connectivity ------------------------------------------------------- */
/* num_edges (connectivity.cpp:22-37). edge_of_slot [6 nE]; edge_nodes [2 nEd]
 * (capacity 12 nE).  Returns nEd. */
int64_t or_num_edges(int64_t nc, int64_t ne, const int32_t* tets, int32_t* edge_of_slot,
                     int32_t* edge_nodes);

/* edge_pairs_to_elems (connectivity.cpp:46-70): sorted keys/elems [12 nE]. */
int or_edge_pairs_to_elems(int64_t nc, int64_t ne, const int32_t* tets, uint64_t* keys,
                           int32_t* elems);

/* faces_up + full_face_table (connectivity.cpp:72-203).  Capacities 4 nE
 * faces.  counts out: [nF, n_interior, n_dirichlet, n_neumann, L]. */
int or_face_table(int64_t nc, int64_t ne, const int32_t* tets, const double* coords, int64_t nd,
                  const int32_t* db, int64_t nn, const int32_t* nb, int32_t* faces,
                  int32_t* face_of_slot, int8_t* sigma, int64_t* face_slots, uint8_t* face_class,
                  int32_t* mrow, double* area, int64_t counts[5]);

/* red_refine + refine_boundary_faces (refine.cpp:16-96).  Outputs sized
 * coords_out [3 (nC+nEd+nE)], tets_out [48 nE], db_out [12 nD], nb_out
 * [12 nN]; midpoint_node [nEd] and centroid_node [nE] may be NULL. */
int or_refine(int64_t nc, int64_t ne, const double* coords, const int32_t* tets, int64_t nd,
              const int32_t* db, int64_t nn, const int32_t* nb, double* coords_out,
              int32_t* tets_out, int32_t* db_out, int32_t* nb_out, int32_t* midpoint_node,
              int32_t* centroid_node);

/* --- assembly + condensation -------------------------------------------- */
typedef struct or_problem {
    int kind;            /* oracle/problems.h */
    double c;            /* reaction (reference operator: 1) */
    const double* a_elem; /* [nE] scalar diffusion or NULL */
    const double* a_diag; /* [3 nE] diagonal tensor or NULL (wins over a_elem) */
} or_problem;

/* assemble_system (assembly.cpp:106-138) + build_schur (solver.cpp:90-147)
 * over the face table of or_face_table.  Any output may be NULL except
 * s_rowptr/s_col/s_val/rhs_neg when the Schur system is wanted; s_col/s_val
 * need capacity 16 nE.  s_nnz receives nnz(S).  c_* is the constraint matrix
 * C (capacity 12 nE). */
int or_assemble_condense(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                         int64_t nf, const int32_t* faces, const int32_t* face_of_slot,
                         const int8_t* sigma, const int64_t* face_slots,
                         const uint8_t* face_class, const int32_t* mrow, const double* area,
                         int64_t l, const or_problem* prob, double* a_blocks, double* slot_coef,
                         int32_t* slot_mrow, double* rhs, double* bd, int64_t* c_rowptr,
                         int32_t* c_col, double* c_val, int64_t* s_rowptr, int32_t* s_col,
                         double* s_val, double* rhs_neg, int64_t* s_nnz);

/* Componentwise magnitudes for per-entry parity of B_T (rhs_scale [4 nE])
 * and rhs_neg (rhsneg_scale [L]): the summed magnitudes of their summands
 * (test infrastructure, see phfem_oracle.c). */
int or_entry_scales(int64_t nc, int64_t ne, const double* coords, const int32_t* tets, int64_t nf,
                    const int32_t* faces, const int32_t* face_of_slot, const int8_t* sigma,
                    const int64_t* face_slots, const uint8_t* face_class, const int32_t* mrow,
                    const double* area, int64_t l, const or_problem* prob, double* rhs_scale,
                    double* rhsneg_scale);

/* pcg_jacobi (sparse.cpp:163-212).  res out: [iterations, rel_residual,
 * converged]. */
int or_pcg(int64_t n, const int64_t* rowptr, const int32_t* col, const double* val,
           const double* b, double* x, double tol, double abs_tol, int64_t max_iter,
           double res[3]);

/* Full Schur-path solve (solver.cpp:149-186 with inner_cg_options 78-86 and
 * verify_solution 44-76) on an assembled system.  stats out:
 * [iterations, residual, constraint_residual]. */
int or_solve_schur(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                   const or_problem* prob, int64_t l, const double* slot_coef,
                   const int32_t* slot_mrow, const double* rhs, const double* bd,
                   const int64_t* c_rowptr, const int32_t* c_col, const double* c_val,
                   const int64_t* s_rowptr, const int32_t* s_col, const double* s_val,
                   const double* rhs_neg, double tol, int64_t max_iter, double* u,
                   double* lambda, double stats[3]);

/* Errors (analysis.cpp:51-105 + the L2 extension).  out: [y_norm,
 * kappa_norm, l2]. */
int or_errors(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
              const int32_t* face_of_slot, const int8_t* sigma, const int32_t* mrow,
              const or_problem* prob, const double* u, const double* lambda, double out[3]);

/* SHA-256 (FIPS 180-4) of n bytes */
void or_sha256(const void* data, int64_t n, uint8_t out[32]);
/* Streaming connectivity digests for meshes whose full oracle tables do not
 * fit host memory (config 2 level 7): digests [9 x 32] of edge_nodes int32
 * [nEd][2], edge_of_slot int32 [nE][6], faces int32 [nF][3], face_of_slot
 * int32 [4 nE], sigma int8 [4 nE], face_slots int64 [nF][2], face_area f64
 * [nF], face_class u8 [nF], multiplier_index int32 [nF] of an all-Dirichlet
 * mesh; counts [nEd, nF]. */
int or_conn_digests(int64_t nc, int64_t ne, const int32_t* tets, const double* coords, uint8_t* digests,
                    int64_t counts[2]);

/* max element diameter (mesh.cpp:90-106) */
double or_mesh_diameter(int64_t nc, int64_t ne, const double* coords, const int32_t* tets);

/* Quadrature tables (quadrature.cpp:9-62): n^3 points, lambda [4 n^3], w [n^3]. */
int or_tet_rule(int degree, double* lambda, double* w);

#ifdef __cplusplus
}
#endif

#endif
