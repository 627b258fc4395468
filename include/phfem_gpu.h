/* phfem_gpu.h — the thin C ABI between the host runtime (capi.cpp) and the
 * sm_100a kernels of the phfem hot path.
 *
 * Every entry point takes device pointers, sizes and a cudaStream_t (passed
 * as void*), launches kernels on that stream and returns without
 * synchronising.  None allocates memory: the host runtime sizes every buffer
 * (reading back the few device counts it needs) and owns it.
 *
 * Each launcher names the reference function whose semantics it implements
 * (paths relative to /root/reference/proj/src).  Layout conventions (device):
 *   coords  double[3 nC]  (x,y,z per node, AoS: one 24-byte gather per vertex)
 *   tets    int32[4 nE]   (16-byte aligned, loaded as int4)
 *   db, nb  int32[3 n]    boundary triangles, outward oriented
 *   slot    s = 4t+k for faces, 6t+k for edges (element-major)
 *   S       SELL-32, width 7, column-major within each 32-row chunk:
 *           entry (row, pos) at (row/32)*224 + pos*32 + row%32; pos 0 is the
 *           diagonal, 1-3 the other faces of the owner element, 4-6 those of
 *           the second element; padding has col == row and value 0.
 */
#ifndef PHFEM_GPU_H
#define PHFEM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error slots of the device error vector (unsigned long long[PHG_ERR_COUNT],
 * initialised to all ones); each keeps the minimum offending key. */
enum phg_err_slot {
    PHG_ERR_DUP_ORIENT = 0,  /* key = t1<<32 | t2: two elements claim one oriented face (connectivity.cpp:62-68) */
    PHG_ERR_CLASSIFY = 1,    /* key = entry<<2 | kind (0 no match, 1 listed twice, 2 interior) (connectivity.cpp:156-175) */
    PHG_ERR_FACE = 2,        /* key = face<<2 | kind (0 degenerate, 1 unclassified boundary) (connectivity.cpp:177-194, mesh.cpp:80-82) */
    PHG_ERR_ZERO_VOLUME = 3, /* key = element (assembly.cpp:13-14) */
    PHG_ERR_SINGULAR = 4,    /* key = element (solver.cpp:103-109, 128-129) */
    PHG_ERR_BOUNDARY_EDGE = 5, /* key = (list index)<<2 | pair (refine.cpp:80-85) */
    PHG_ERR_VALENCE = 6,     /* key = vertex: star larger than the supported maximum */
    PHG_ERR_DEGEN_FACE = 7,  /* key = slot 4t+k: a face with a repeated node id, which faces_up never lists
                                (connectivity.cpp:81-84) and full_face_table cannot match (:140-143) */
    PHG_ERR_COUNT = 8
};

#define PHG_SELL_C 32
#define PHG_SELL_W 7

/* Problem data (oracle/problems.h restates the same formulas on the CPU). */
typedef struct phg_problem {
    int kind;              /* 0 manufactured, 1 linear, 2 zero, 3 sin3, 4 expcos, 5 polysin */
    double c;              /* reaction coefficient */
    const double* a_elem;  /* device [nE] scalar diffusion, or NULL */
    const double* a_diag;  /* device [3 nE] diagonal diffusion, or NULL (wins) */
} phg_problem;

/* ---------------------------------------------------------------- scans */
/* Exclusive scan of n int32 counts into int64 offsets (out[n] = total).
 * scratch needs phfem_gpu_scan_scratch(n) bytes. */
size_t phfem_gpu_scan_scratch(int64_t n);
int phfem_gpu_scan_i32(const int32_t* in, int64_t* out, int64_t n, void* scratch, void* stream);

/* ------------------------------------------------------------ mesh input */
/* Kuhn mesh generator (oracle: or_kuhn_mesh). */
int phfem_gpu_kuhn_nodes(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                         uint64_t seed, double* coords, void* stream);
/* tets + per-element boundary-face counts packed (nDir | nNeu<<8) */
int phfem_gpu_kuhn_tets(int nx, int ny, int nz, uint32_t dirichlet_mask, int32_t* tets,
                        int32_t* bcount, void* stream);
/* boundary lists in element/slot order from the exclusive scans of the
 * Dirichlet and Neumann counts */
int phfem_gpu_kuhn_boundary(int nx, int ny, int nz, uint32_t dirichlet_mask, const int32_t* tets,
                            const int64_t* dir_off, const int64_t* neu_off, int32_t* db,
                            int32_t* nb, void* stream);
int phfem_gpu_split_counts(const int32_t* packed, int32_t* dir, int32_t* neu, int64_t n, void* stream);

/* range check of uploaded node indices (mesh.cpp:151-158): atomicMin of the
 * first position holding an index outside [0, nc) into *first_bad */
int phfem_gpu_check_indices(const int32_t* a, int64_t n, int64_t nc, unsigned long long* first_bad,
                            void* stream);

/* small device-to-host reads without the copy engine: word i of dst (host
 * memory mapped into the device address space) = *src[i], i < n <= 16.  A
 * cudaMemcpyAsync D2H queues behind a running H2D upload on the copy
 * engine; this kernel does not. */
int phfem_gpu_gather_words(const unsigned long long* const* src, int n, unsigned long long* dst, void* stream);

/* max element diameter (mesh.cpp:90-106); out: one double (device) */
int phfem_gpu_diameter(const double* coords, const int32_t* tets, int64_t ne, double* out,
                       double* partials, void* stream);

/* -------------------------------------------------------- connectivity */
/* vertex -> (element, local vertex) incidence ("star"), CSR by vertex,
 * without the incidence of each element's largest vertex (3 nE entries:
 * every edge and face is grouped at its smallest vertex, and an element's
 * largest vertex has no candidate above it):
 * count[v] (zeroed) += incidences; star_ptr = exclusive scan of count;
 * star_fill places each incidence at star_ptr[v] + --count[v] (the order
 * inside a vertex's segment is unspecified; every consumer is order free)
 * and leaves count zeroed. */
/* repeated (may be NULL, zeroed by the caller) is set to 1 if an element
 * repeats a node id; star_groups then checks its stars for such elements */
int phfem_gpu_star_count(const int32_t* tets, int64_t ne, int32_t* count, int32_t* repeated, void* stream);
int phfem_gpu_star_fill(const int32_t* tets, int64_t ne, const int64_t* star_ptr, int32_t* count, int32_t* star,
                        void* stream);

/* Per vertex v, group the edges (v,b), b>v and the faces whose smallest
 * vertex is v among the incident element slots: edge_first[6t+k] = smallest
 * slot of the edge (first occurrence, connectivity.cpp:22-37); slot_mate[4t+k]
 * = the other slot of the face or -1 (faces_up/full_face_table,
 * connectivity.cpp:72-153).  slot_mate may be NULL (edges only).  Three
 * passes without host round trips: warps over stars <= 32, warps over the
 * deferred stars <= 64, blocks over anything larger (stars above 2730
 * incidences are listed for phfem_gpu_star_groups_global and set
 * PHG_ERR_VALENCE, their slots hold in-bounds placeholders).  defer_list
 * needs 3 nC entries, defer_count 3. */
int phfem_gpu_star_groups(int64_t nc, const int64_t* star_ptr, const int32_t* star,
                          const int32_t* tets, int32_t* edge_first, int32_t* slot_mate,
                          int32_t* defer_list, int32_t* defer_count, unsigned long long* err,
                          const int32_t* repeated, void* stream);
/* The child of a red refinement (refine_conn.cu): edge_first [6 x 12 n] and
 * slot_mate [4 x 12 n] (may be NULL) of the child mesh in closed form from
 * the parent's tets [4 n], edge_of_slot, edge_first, slot_mate and nEd;
 * a0 is scratch [2 nEd].  Also the child's slot masks [12 n] and the tile
 * sums of phfem_gpu_element_offsets in scratch (its layout), so that
 * phfem_gpu_element_offsets_scan finishes the offsets. */
int phfem_gpu_refined_groups(int64_t n, const int32_t* tets, const int32_t* edge_of_slot,
                             const int32_t* edge_first, const int32_t* slot_mate, int64_t ned,
                             int32_t* a0, int32_t* ef_out, int32_t* sm_out, uint16_t* masks, void* scratch,
                             void* stream);
/* classification (connectivity.cpp:120-160) of a refined mesh's lists: the
 * child entries' faces from the parent's classification (nd, nn, db, nb,
 * entry_face, face_slots, tets of the PARENT, n = parent nE), the child's
 * face_of_slot / face_slots; claims and errors as phfem_gpu_classify;
 * face_class (may be NULL, else zeroed) gets 1 / 2 on the listed faces */
int phfem_gpu_refined_classify(int64_t nd, int64_t nn, const int32_t* db, const int32_t* nb,
                               const int32_t* p_entry_face, const int32_t* p_face_slots, const int32_t* p_tets,
                               int64_t n, const int32_t* face_of_slot, const int32_t* face_slots,
                               uint32_t* claim, int32_t* entry_face, uint8_t* face_class,
                               unsigned long long* err, void* stream);
/* a star listed by star_groups as too large for shared memory (defer_list
 * + 2 nC, count defer_count[2], PHG_ERR_VALENCE set): tables of capacity
 * cap (power of two > 3 m) in global scratch [20 cap bytes] */
int phfem_gpu_star_groups_global(int32_t v, const int64_t* star_ptr, const int32_t* star,
                                 const int32_t* tets, int32_t* edge_first, int32_t* slot_mate,
                                 void* scratch, unsigned cap, unsigned long long* err, void* stream);

/* Per-element slot masks [ne] (bit k < 6: edge slot 6t+k is its edge's
 * first occurrence; bit 6+k: face slot 4t+k owns its face) and the exclusive
 * offsets [ne + 1] of their popcounts: edge_off, face_off (skipped when
 * slot_mate is NULL).  Entry t < ne packs the offset (low 32 bits; totals
 * stay below 2^31) with element t's edge / face mask above it; entry ne is
 * the plain total.  scratch needs phfem_gpu_element_offsets_scratch(ne)
 * bytes. */
size_t phfem_gpu_element_offsets_scratch(int64_t ne);
int phfem_gpu_element_offsets(int64_t ne, const int32_t* edge_first, const int32_t* slot_mate, uint16_t* masks,
                              int64_t* edge_off, int64_t* face_off, void* scratch, void* stream);
/* the same from masks and tile sums already in scratch (refined_groups) */
int phfem_gpu_element_offsets_scan(int64_t ne, const uint16_t* masks, bool faces, int64_t* edge_off,
                                   int64_t* face_off, void* scratch, void* stream);

/* Numbering from the exclusive offsets: edge ids = rank of the first slot,
 * face ids = rank of the owner slot (the faces_up order).  One thread per
 * element writes the ids of all its slots (the others rank in their group's
 * first element), the edge/face tables, sigma and the face areas.  Either
 * output group may be NULL (edge_first / slot_mate NULL). */
int phfem_gpu_number(int64_t ne, const int32_t* tets, const double* coords,
                     const int32_t* edge_first, const int64_t* edge_off, int32_t* edge_of_slot,
                     int32_t* edge_nodes, const int32_t* slot_mate, const int64_t* face_off,
                     int32_t* face_of_slot, int8_t* sigma, int32_t* faces, int32_t* face_slots,
                     double* face_area, unsigned long long* err, void* stream);

/* Boundary classification (connectivity.cpp:156-175): entries of db then nb
 * are matched through the star of their smallest vertex; entry_face [nd +
 * nn] receives each entry's face id (-1: none), which the check pass and the
 * assembly's boundary terms reuse. */
int phfem_gpu_classify(int64_t nd, const int32_t* db, int64_t nn, const int32_t* nb,
                       const int64_t* star_ptr, const int32_t* star, const int32_t* tets,
                       const int32_t* face_of_slot, const int32_t* face_slots, uint32_t* claim,
                       int32_t* entry_face, unsigned long long* err, void* stream);
int phfem_gpu_classify_check(int64_t nd, int64_t nn, const int32_t* entry_face, const uint32_t* claim,
                             unsigned long long* err, void* stream);
/* face classes (connectivity.cpp:177-201); claim[f] is the first list entry
 * naming face f (all ones: none); counts[3] += interior, dirichlet, neumann
 * (device int64, zeroed by the caller); *n_rows (device) = number of row
 * (non-Neumann) faces.  scratch (phfem_gpu_face_rows_scratch(nf) bytes)
 * carries the per-tile row offsets to phfem_gpu_face_rows. */
size_t phfem_gpu_face_rows_scratch(int64_t nf);
int phfem_gpu_face_class(int64_t nf, int64_t nd, const uint32_t* claim, const int32_t* face_slots,
                         uint8_t* face_class, unsigned long long* counts, void* scratch, int64_t* n_rows,
                         unsigned long long* err, void* stream);
/* multiplier rows = rank among the row faces (face_mrow, -1 for Neumann
 * faces) and the inverse map row -> face, from face_class and the scratch of
 * phfem_gpu_face_class */
int phfem_gpu_face_rows(int64_t nf, const uint8_t* face_class, const void* scratch, int32_t* face_mrow,
                        int32_t* row_face, void* stream);
/* phfem_gpu_face_class's tile row counts (scratch) from classes already in
 * face_class (a refined child's, refined_classify) */
int phfem_gpu_face_tile_rows(int64_t nf, const uint8_t* face_class, void* scratch, int64_t* n_rows,
                             void* stream);
/* rows when every face is a row (no Neumann faces): face_mrow = row_face =
 * 0..nf-1 */
int phfem_gpu_face_rows_identity(int64_t nf, int32_t* face_mrow, int32_t* row_face, void* stream);

/* ----------------------------------------------------------- refinement */
/* red_refine (refine.cpp:16-74): one thread per parent; child 0 at row t,
 * children 1..11 at rows nE + 11t + q-1; new nodes by the closed form
 * centroid(t) = nC + t + E_t, midpoint(e) = nC + firstElem(e) + 1 + e.
 * coords_out must hold nC + nEd + nE nodes; the first nC are copied. */
int phfem_gpu_refine(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                     const int32_t* edge_first, const int32_t* edge_of_slot,
                     const int64_t* edge_off, double* coords_out, int32_t* tets_out,
                     int32_t* midpoint_node, int32_t* centroid_node, void* stream);
/* refine_boundary_faces (refine.cpp:76-96) over one list; list_base offsets
 * the error key (0 for db, nd for nb). */
int phfem_gpu_refine_boundary(int64_t nf, const int32_t* faces, int64_t list_base, int64_t nc,
                              const int64_t* star_ptr, const int32_t* star, const int32_t* tets,
                              const int32_t* edge_first, const int32_t* edge_of_slot,
                              int32_t* out, unsigned long long* err, void* stream);
/* the same split for a classified mesh: midpoints through the owner slot of
 * each entry's face (entry_face + list_base, face_slots), no star */
int phfem_gpu_refine_boundary_owned(int64_t nf, const int32_t* faces, int64_t list_base, int64_t nc,
                                    const int32_t* entry_face, const int32_t* face_slots, const int32_t* tets,
                                    const int32_t* edge_first, const int32_t* edge_of_slot, int32_t* out,
                                    void* stream);

/* ------------------------------------------------- assembly + condensation */
/* Upload tet_rule(5) and tet_rule(9) (quadrature.cpp:36-62), built on the
 * host exactly like the reference, into constant memory. */
int phfem_gpu_set_rules(const double* lam5, const double* w5, int n5, const double* lam9,
                        const double* w9, int n9);

/* Fused assemble_system + build_schur local part (assembly.cpp:7-138,
 * solver.cpp:90-127) with the direct scatter into SELL S and rhs_neg.
 * Rows 0..l-1 of the SELL arrays, rhs_neg and bd are fully written (the
 * row owners clear the accumulated entries first); padding rows of the
 * last slice are left untouched.  Optional
 * debug outputs (may be NULL): a_blocks [16 nE], slot_coef [4 nE],
 * slot_mrow [4 nE].  rhs [4 nE] (= b + LN) is always written (recovery).
 * norms [2] (device) receive sum(rhs^2), sum(bd^2) over the l face rows,
 * reduced deterministically through partials[2 * grid].  redo [ne + 1] is
 * scratch: the count and list of elements whose operands leave the
 * reciprocal-division window and are recomputed with IEEE division.
 * face_bval [nf] is scratch: the boundary faces' Dirichlet traces / Neumann
 * terms, formed first by a pass over the nd + nn boundary entries
 * (entry_face of the classification, face_slots).  ev_begin / ev_end (cudaEvent_t, may be NULL) bracket the
 * main kernel.  S goes to SELL-32 (sell_col, sell_val: the reference's rows,
 * both triangles) or, when st_val is not NULL, element-major: st_val [10 ne]
 * (S_T[r][q], r <= q, in 32-element chunks: (t/32)*320 + pair*32 + t%32),
 * the rows slot_mrow [4 ne] (required) and the assembled diagonal diag [l].
 * refine (may be NULL): the same kernel also writes one red refinement of the
 * mesh (phfem_gpu_refine's coords_out / tets_out, without the node maps) from
 * the connectivity's edge tables. */
typedef struct phg_refine_out {
    int64_t nc;
    const int32_t* edge_first;
    const int32_t* edge_of_slot;
    const int64_t* edge_off;
    double* coords_out;
    int32_t* tets_out;
} phg_refine_out;
int phfem_gpu_assemble_condense(int64_t ne, int64_t l, const double* coords, const int32_t* tets,
                                const phg_problem* prob, const int32_t* face_of_slot,
                                const int32_t* slot_mate, const int32_t* face_mrow,
                                const double* face_area, int64_t nd, int64_t nn,
                                const int32_t* entry_face, const int32_t* face_slots, double* face_bval,
                                int32_t* sell_col, double* sell_val, double* st_val, double* diag,
                                double* rhs_neg, double* bd, double* rhs, double* a_blocks,
                                double* slot_coef, int32_t* slot_mrow, int32_t* redo, double* halves,
                                unsigned long long* err, const phg_refine_out* refine, void* ev_begin,
                                void* ev_end, void* stream);
/* halves (element-major only, may be NULL) [2 l]: the second element's S
 * diagonal and rhs_neg terms of each row (zero on boundary rows), the
 * owner's going to diag / rhs_neg, all by plain stores; sum_halves then
 * gives the assembled diag / rhs_neg (what the atomics on cleared rows that
 * a NULL halves selects give, bit for bit). */
int phfem_gpu_sum_halves(int64_t l, double* diag, double* rhs_neg, const double* halves, void* stream);
int phfem_gpu_assemble_grid(int64_t ne);
/* norms [2] (device) = ||rhs||^2 [n], ||bd||^2 [l], deterministic; partials
 * [2 phfem_gpu_assemble_grid(n)] */
int phfem_gpu_sumsq2(const double* rhs, int64_t n, const double* bd, int64_t l, double* partials,
                     double* norms, void* stream);

/* --------------------------------------------------------------- solver */
typedef struct phg_cg_state {
    double rz, pq, alpha, beta, rnorm, bnorm, stop, rel_residual;
    long long it, max_iter;
    int done, converged, not_spd;
    int x_pending; /* set with done by the stop test: cg_pdir still adds alpha p to x */
    unsigned int counter[4];
} phg_cg_state;

/* Jacobi-PCG on S (pcg_jacobi, sparse.cpp:163-212; stopping rule of
 * inner_cg_options, solver.cpp:78-86).  cg_init sets x=0, r=b, z=d r, p=z,
 * d = 1/diag (1 where the diagonal is 0), computes ||b|| and the stop
 * level from tol, abs_tol (<= 0 means none) and max_iter.  cg_iterations
 * enqueues n iterations (kernels turn into no-ops once done). */
int phfem_gpu_cg_init(int64_t l, const int32_t* sell_col, const double* sell_val, const double* b,
                      double* x, double* r, double* p, double* d, double tol, double abs_tol,
                      long long max_iter, phg_cg_state* st, double* partials, void* stream);
int phfem_gpu_cg_iterations(int n, int64_t l, const int32_t* sell_col, const double* sell_val,
                            double* x, double* r, double* p, double* q, const double* d,
                            phg_cg_state* st, double* partials, void* stream);
/* SELL-32 rows of an element-major S (phfem_gpu_assemble_condense with
 * sell_col NULL): the layout the SELL assembly writes, S[r][q] = S[q][r] =
 * the stored upper-triangle value, diagonal = diag; needs slot_mate for the
 * owner / second-slot positions.  Once per solve (the CG streams rows). */
int phfem_gpu_elem_to_sell(int64_t ne, int64_t l, const double* st_val, const int32_t* slot_mrow,
                           const int32_t* slot_mate, const double* diag, int32_t* sell_col, double* sell_val,
                           void* stream);
/* The same CG on the element-major S itself (no SELL copy): row_slots
 * [2 L] = (owner slot, second slot or -1) of each row, built once per solve
 * by cg_em_rows; cg_em_iterations sums each row in the SELL order of
 * elem_to_sell, so the iterates equal cg_iterations' on that SELL copy. */
int phfem_gpu_cg_em_rows(int64_t ne, const int32_t* slot_mrow, const int32_t* slot_mate, int32_t* row_slots,
                         void* stream);
int phfem_gpu_cg_em_init(int64_t l, const double* diag, const double* b, double* x, double* r, double* p,
                         double* d, double tol, double abs_tol, long long max_iter, phg_cg_state* st,
                         double* partials, void* stream);
int phfem_gpu_cg_em_iterations(int n, int64_t l, const int32_t* row_slots, const double* st_val,
                               const int32_t* slot_mrow, const double* diag, double* x, double* r, double* p,
                               double* q, const double* d, phg_cg_state* st, double* partials, void* stream);

/* Element-local recovery U_T = A_T^-1 (B_T + C_T' Lambda_T) (solver.cpp:168-181)
 * fused with the primal block residual of verify_solution (solver.cpp:44-53):
 * sums [0] += ||A U - rhs - C' Lambda||^2. */
int phfem_gpu_recover(int64_t ne, const double* coords, const int32_t* tets,
                      const phg_problem* prob, const int32_t* face_of_slot,
                      const int32_t* slot_mate, const int32_t* face_mrow,
                      const double* face_area, const double* rhs, const double* lambda,
                      double* u, double* sums, double* partials, unsigned long long* err,
                      void* stream);
/* Constraint residual r2 = C U - b_D per multiplier row (solver.cpp:54-62):
 * out[0] = ||r2||^2, out[1] = max|r2|, out[2] = max|b_D| */
int phfem_gpu_constraint_residual(int64_t l, const int32_t* row_face, const int32_t* face_slots,
                                  const int32_t* slot_mate, const int32_t* face_of_slot,
                                  const double* face_area, const int32_t* tets, const double* u,
                                  const double* bd, double* out, double* partials, void* stream);

/* Error norms (analysis.cpp:51-105 + L2 extension): out [y^2, kappa^2, l2^2] */
int phfem_gpu_errors(int64_t ne, const double* coords, const int32_t* tets,
                     const phg_problem* prob, const int32_t* face_of_slot,
                     const int32_t* slot_mate, const int32_t* face_mrow, const double* u,
                     const double* lambda, double h, double* out, double* partials,
                     void* stream);

/* SELL -> CSR export of S for parity checks (host orchestrated; dense rows
 * sorted by column, padding dropped). row_nnz [L] */
int phfem_gpu_sell_row_nnz(int64_t l, const int32_t* sell_col, int32_t* row_nnz, void* stream);
int phfem_gpu_sell_to_csr(int64_t l, const int32_t* sell_col, const double* sell_val,
                          const int64_t* row_ptr, int32_t* col, double* val, void* stream);

/* self-test: n random quotients of the kernels' shared-reciprocal division
 * compared bit for bit with IEEE division; *mismatches (device) += count */
int phfem_gpu_division_selftest(int64_t n, uint64_t seed, unsigned long long* mismatches, void* stream);

/* fp64 FMA throughput probe: *flops = floating-point operations of one
 * launch; time it between ev_begin / ev_end (cudaEvent_t, may be NULL) */
int phfem_gpu_fp64_peak(int iters, double* sink, void* ev_begin, void* ev_end, double* flops, void* stream);

/* ------------------------------------------------- C++ API support (api.cu)
 * Kernels behind the value-returning C++ API (include/phfem_cxx), whose
 * inputs are host structs (LinearSystem, CsrMatrix, Triplets, FaceTable).
 * Every sequential sum the reference defines is owned by one thread and
 * replayed in the reference's order. */

/* group n items by seg[i] in [0, nseg) and sort each group by
 * (minor[i], i): seg_ptr [nseg+1] (exclusive offsets), perm [n] (item ids in
 * sorted order).  Scratch: cnt [nseg], tmp [n], scan_scratch
 * (phfem_gpu_scan_scratch(nseg)). */
int phfem_gpu_seg_sort(int64_t n, int64_t nseg, const int64_t* seg, const int64_t* minor,
                       int64_t* seg_ptr, int64_t* perm, int32_t* cnt, int64_t* tmp, void* scan_scratch,
                       void* stream);
/* items already grouped by seg_ptr: perm = identity, then sorted per group */
int phfem_gpu_sort_within(int64_t n, int64_t nseg, const int64_t* seg_ptr, const int64_t* minor,
                          int64_t* perm, int64_t* tmp, void* stream);

/* edge_pairs_to_elems (connectivity.cpp:46-70): entry 12 m + 3 k + j of
 * element m, the reference's key from * ned + to (uint64, pair_to_edge = -1
 * for an edge of two equal node ids: edge_nodes, may be NULL for meshes
 * without) stored as (segment, minor) in [0, ned] x [0, ned]; after seg_sort
 * by segment (ned + 1 of them) with that minor, e2t_finish writes the sorted
 * keys / elements and atomicMin's the first position j whose key equals key
 * j-1. */
int phfem_gpu_e2t_entries(int64_t ne, int64_t ned, const int32_t* edge_of_slot, const int32_t* edge_nodes,
                          int64_t* from, int64_t* to, void* stream);
int phfem_gpu_e2t_finish(int64_t n, int64_t ned, const int64_t* perm, const int64_t* from,
                         const int64_t* to, unsigned long long* key, int32_t* elem,
                         unsigned long long* first_dup, void* stream);

int phfem_gpu_widen(int64_t n, const int32_t* a, int64_t* b, void* stream);
/* from_triplets (sparse.cpp:12-44) after seg_sort by row with minor col:
 * distinct columns per row, then the CSR with duplicates summed in
 * insertion order */
int phfem_gpu_csr_unique(int64_t rows, const int64_t* ptr, const int64_t* perm, const int64_t* col,
                         int32_t* cnt, void* stream);
int phfem_gpu_csr_write(int64_t rows, const int64_t* ptr, const int64_t* perm, const int64_t* col,
                        const double* val, const int64_t* out_ptr, int32_t* out_col, double* out_val,
                        void* stream);
/* y = A x (sparse.cpp:46-52), diagonal (60-66) */
int phfem_gpu_csr_spmv(int64_t rows, const int64_t* ptr, const int32_t* col, const double* val,
                       const double* x, double* y, void* stream);
int phfem_gpu_csr_diag(int64_t rows, const int64_t* ptr, const int32_t* col, const double* val,
                       double* d, void* stream);
/* transpose (sparse.cpp:68-87): rowof [nnz] = row of each entry; after
 * seg_sort by column with minor = entry index, tcol/tval from perm */
int phfem_gpu_csr_rowof(int64_t rows, const int64_t* ptr, int64_t* rowof, void* stream);
int phfem_gpu_csr_transpose(int64_t nnz, const int64_t* perm, const int64_t* rowof, const double* val,
                            int32_t* tcol, double* tval, void* stream);
/* spgemm (sparse.cpp:122-149): products per row of A (count, fill in the
 * accumulation order), sort_within by column, then per column
 * acc = 0.0; acc += product in that order */
int phfem_gpu_spgemm_count(int64_t rows, const int64_t* aptr, const int32_t* acol, const int64_t* bptr,
                           int32_t* cnt, void* stream);
int phfem_gpu_spgemm_fill(int64_t rows, const int64_t* aptr, const int32_t* acol, const double* aval,
                          const int64_t* bptr, const int32_t* bcol, const double* bval,
                          const int64_t* pptr, int64_t* pcol, double* pval, void* stream);
int phfem_gpu_spgemm_write(int64_t rows, const int64_t* pptr, const int64_t* perm, const int64_t* pcol,
                           const double* pval, const int64_t* out_ptr, int32_t* out_col,
                           double* out_val, void* stream);

/* build_schur's element part (solver.cpp:101-127) from given blocks:
 * lu [16 nE], perm [4 nE], singular [nE], s_loc [16 nE], r_loc [4 nE];
 * *first_singular = min singular element (init ULLONG_MAX) */
int phfem_gpu_condense_blocks(int64_t ne, const double* a_blocks, const double* coef, const int32_t* mrow,
                              const double* rhs, double* lu, int32_t* perm, uint8_t* singular,
                              double* s_loc, double* r_loc, unsigned long long* first_singular,
                              void* stream);
/* per element: S triplets nr^2, rhs_neg terms nr (nr = non-Neumann rows) */
int phfem_gpu_schur_counts(int64_t ne, const int32_t* mrow, int32_t* cs, int32_t* cr, void* stream);
/* the reference's triplet stream (solver.cpp:131-145) at offsets os / orr */
int phfem_gpu_schur_triplets(int64_t ne, const int32_t* mrow, const double* s_loc, const double* r_loc,
                             const int64_t* os, const int64_t* orr, int64_t* trow, int64_t* tcol,
                             double* tval, int64_t* rrow, double* rval, void* stream);
/* rhs_neg[r] = ((b_D[r] - t0) - t1) over row r's terms in stream order */
int phfem_gpu_rhs_neg(int64_t l, const int64_t* ptr, const int64_t* perm, const double* rval,
                      const double* bd, double* out, void* stream);
/* recovery (solver.cpp:168-181) + r1 = A U - B per element (44-50) */
int phfem_gpu_recover_blocks(int64_t ne, const double* a_blocks, const double* coef, const int32_t* mrow,
                             const double* rhs, const double* lambda, double* u, double* r1, void* stream);
int phfem_gpu_sub_inplace(int64_t n, double* a, const double* b, void* stream);
/* out (device) [sum x^2, max |x|], deterministic; partials
 * [2 phfem_gpu_sumsq_max_partials()] */
int phfem_gpu_sumsq_max_partials(void);
int phfem_gpu_sumsq_max(int64_t n, const double* x, double* partials, double* out, void* stream);

/* tabulated problem data (assembly.cpp:46-104): rule 0 = Gauss (nq points
 * lam [4 nq], w [nq]), 1 = face centroids (4 per element).  load_points:
 * vol [nE], pts [3 nq nE]; load_tab: b [4 nE] from f values fv [nq nE]. */
int phfem_gpu_load_points(int64_t ne, const double* coords, const int32_t* tets, int rule, int nq,
                          const double* lam, double* vol, double* pts, void* stream);
int phfem_gpu_load_tab(int64_t ne, int rule, int nq, const double* lam, const double* w,
                       const double* vol, const double* fv, double* b, void* stream);
/* face_area_and_normal + face_centroid (mesh.cpp:76-88) of faces ids[i]
 * (ids NULL: 0..n-1): out [7 n] = area, unit normal, centroid; *bad = first
 * degenerate position (init ULLONG_MAX) */
int phfem_gpu_face_geom(int64_t n, const int32_t* ids, const int32_t* faces, const double* coords,
                        double* out, unsigned long long* bad, void* stream);
/* neumann_vector (assembly.cpp:81-94) from g values gv [per geometry row];
 * geo_of_face maps a face to its face_geom row */
int phfem_gpu_neumann_tab(int64_t ne, const int32_t* slot_to_face, const uint8_t* face_class,
                          const int64_t* face_slots, const int32_t* geo_of_face, const double* geo,
                          const double* gv, double* ln, void* stream);
/* y_norm_error (analysis.cpp:51-76): points [3 nq nE]; per-element sums
 * from ex [4 nq nE] = (u, grad u) at the points */
int phfem_gpu_ynorm_points(int64_t ne, const double* coords, const int32_t* tets, int nq,
                           const double* lam, double* pts, void* stream);
int phfem_gpu_ynorm_elem(int64_t ne, const double* coords, const int32_t* tets, const double* u, int nq,
                         const double* lam, const double* w, const double* ex, double inv_h2,
                         double* acc, void* stream);
/* multiplier_norm_error (analysis.cpp:78-105): points [36 nE] (3 edge
 * midpoints of each oriented face); per-element sums from grad u [36 nE] */
int phfem_gpu_kappa_points(int64_t ne, const double* coords, const int32_t* tets, double* pts,
                           void* stream);
int phfem_gpu_kappa_elem(int64_t ne, const double* coords, const int32_t* tets,
                         const int32_t* slot_to_face, const double* sigma, const uint8_t* face_class,
                         const int32_t* mult, const double* lambda, const double* gr, double h,
                         double* acc, void* stream);
/* assemble_system's element part (assembly.cpp:115-130) from a given face
 * table: a [16 nE] = K + M, coef [4 nE] = (sigma |F|) / 3, mrow [4 nE];
 * *bad = first zero-volume element (init ULLONG_MAX) */
int phfem_gpu_element_blocks(int64_t ne, const double* coords, const int32_t* tets,
                             const int32_t* slot_to_face, const double* sigma, const double* area,
                             const int32_t* mult, double* a, double* coef, int32_t* mrow,
                             unsigned long long* bad, void* stream);
/* C triplets in the reference's order at offsets 3 orr[t] (orr = exclusive
 * scan of the non-Neumann slot counts) */
int phfem_gpu_c_triplets(int64_t ne, const int32_t* mrow, const double* coef, const int64_t* orr,
                         int64_t* trow, int64_t* tcol, double* tval, void* stream);
/* solve_direct (solver.cpp:192-244): block inverses inv [16 nE] with the
 * block pattern (4t+i, 4t+j); block solves; r1 = A U - B */
int phfem_gpu_block_inverses(int64_t ne, const double* a, double* inv, unsigned long long* first_singular,
                             void* stream);
int phfem_gpu_block_pattern(int64_t ne, int64_t* row, int64_t* col, void* stream);
int phfem_gpu_block_solve(int64_t ne, const double* a, const double* b, double* u, void* stream);
int phfem_gpu_block_residual(int64_t ne, const double* a, const double* u, const double* rhs, double* r1,
                             void* stream);
/* a += b; a = b - a; out (device) = sum x (deterministic, partials as
 * phfem_gpu_sumsq_max) */
int phfem_gpu_add_inplace(int64_t n, double* a, const double* b, void* stream);
int phfem_gpu_rsub_inplace(int64_t n, double* a, const double* b, void* stream);
int phfem_gpu_sum(int64_t n, const double* x, double* partials, double* out, void* stream);
/* refine_boundary_faces' split (refine.cpp:88-94): in [3 nf], the
 * midpoint ids mid [3 nf] = (m12, m23, m13) per face, out [12 nf] */
int phfem_gpu_split_boundary(int64_t nf, const int32_t* in, const int32_t* mid, int32_t* out, void* stream);
/* RefinementMap::parent_elem [12 nE] (refine.cpp:58-68) */
int phfem_gpu_refine_parents(int64_t ne, int32_t* parent, void* stream);
/* Jacobi-PCG on a general CSR matrix (the C++ API's pcg_jacobi) */
int phfem_gpu_cgcsr_init(int64_t l, const int64_t* ptr, const int32_t* col, const double* val,
                         const double* b, double* x, double* r, double* p, double* d, double tol,
                         double abs_tol, long long max_iter, phg_cg_state* st, double* partials,
                         void* stream);
int phfem_gpu_cgcsr_iterations(int n, int64_t l, const int64_t* ptr, const int32_t* col,
                               const double* val, double* x, double* r, double* p, double* q,
                               const double* d, phg_cg_state* st, double* partials, void* stream);

/* kernels launched by this library since load (benchmark accounting) */
long long phfem_gpu_launch_count(void);

/* last CUDA error as text (for the host runtime's messages) */
const char* phfem_gpu_error_string(int code);

#ifdef __cplusplus
}
#endif

#endif
