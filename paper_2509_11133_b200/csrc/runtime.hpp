// Host runtime of the B200 phfem library: device buffers, the mesh /
// connectivity / system objects behind the C ABI handles, and the stage
// orchestration that calls the kernels through phfem_gpu.h.
#pragma once

#include <cstring>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "phfem_cxx/errors.hpp"
#include "phfem_gpu.h"

namespace phb {

// Error taxonomy of the reference (errors.hpp:9-27): the C++ API's own
// classes, so errors raised here reach C++ callers with the reference's type;
// the C ABI wrapper maps them 1:1 onto the status codes.
using phfem::InvalidArgument;
using phfem::IoError;
using phfem::MeshError;
using phfem::SolverError;

void check(cudaError_t e, const char* what);
inline void check(int e, const char* what) { check(static_cast<cudaError_t>(e), what); }

// One stream per process; every call synchronises on it before returning.
struct Runtime {
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;  // asynchronous mesh uploads (copy engine)
    int device = 0;
    Runtime();
};
Runtime& rt();
inline cudaStream_t S() { return rt().stream; }
inline cudaStream_t SC() { return rt().copy; }
inline void* SV() { return static_cast<void*>(rt().stream); }
void sync();

// Stream-ordered device buffer (cudaMallocAsync on the library stream,
// served from the device memory pool between pipeline passes).
// alloc() keeps the current block when it is large enough, so objects that
// are rebuilt every pass (connectivity, system, workspaces) stop paying for
// allocation after the first pass.
template <class T>
struct DBuf {
    T* p = nullptr;
    int64_t n = 0;
    int64_t cap = 0;
    DBuf() = default;
    explicit DBuf(int64_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) { o.p = nullptr; o.n = o.cap = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            cap = o.cap;
            o.p = nullptr;
            o.n = o.cap = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(int64_t count) {
        if (p && count <= cap) {
            n = count;
            return;
        }
        release();
        n = cap = count;
        if (count > 0) check(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (size_t)count, S()), "allocate");
    }
    void release() {
        if (p) cudaFreeAsync(p, S());
        p = nullptr;
        n = cap = 0;
    }
    void zero() {
        if (n) check(cudaMemsetAsync(p, 0, sizeof(T) * (size_t)n, S()), "memset");
    }
    void fill_bytes(int byte) {
        if (n) check(cudaMemsetAsync(p, byte, sizeof(T) * (size_t)n, S()), "memset");
    }
    void upload(const T* h, int64_t count) {
        alloc(count);
        if (count) check(cudaMemcpyAsync(p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, S()), "H2D");
    }
    // allocation and copy ordered on another stream (the upload stream);
    // users on the library stream wait for an event recorded after it
    void upload_on(const T* h, int64_t count, cudaStream_t s) {
        release();
        n = cap = count;
        if (count > 0) {
            check(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (size_t)count, s), "allocate");
            check(cudaMemcpyAsync(p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, s), "H2D");
        }
    }
    std::vector<T> download() const {
        std::vector<T> h((size_t)n);
        if (n) check(cudaMemcpyAsync(h.data(), p, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, S()), "D2H");
        sync();
        return h;
    }
    void download_to(T* h, int64_t count) const {
        if (count) check(cudaMemcpyAsync(h, p, sizeof(T) * (size_t)count, cudaMemcpyDeviceToHost, S()), "D2H");
    }
};

// n <= 16 device words to the host in one synchronisation, through host
// memory mapped into the device (phfem_gpu_gather_words): no copy-engine
// transfer, so the read does not wait behind an upload in flight
void read_words(const unsigned long long* const* src, int n, unsigned long long* out);

template <class T>
T read_scalar(const T* dptr) {
    static_assert(sizeof(T) == 8, "read_scalar reads one 8-byte word");
    const unsigned long long* src[1] = {reinterpret_cast<const unsigned long long*>(dptr)};
    unsigned long long w;
    read_words(src, 1, &w);
    T v;
    std::memcpy(&v, &w, sizeof(T));
    return v;
}

// Device events for stage timing on the library stream.
struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    Timer();
    ~Timer();
    void start();
    double stop_ms();  // records b, synchronises, returns ms
};

// ---------------------------------------------------------------- objects

// An upload still in flight on the copy stream (upload_mesh_async): the
// event follows the copies, the index check and its D2H into `flags`.
struct PendingUpload {
    cudaEvent_t ready = nullptr;
    unsigned long long* flags = nullptr;  // pinned [3]: first bad index per array
    DBuf<unsigned long long> dflags;
    const int32_t* src[3] = {nullptr, nullptr, nullptr};  // caller's arrays, read once for the message
    std::string error;  // set by the first failed check; later uses rethrow it
    ~PendingUpload();
};

struct Connectivity;

struct MeshData {
    int64_t nc = 0, ne = 0, nd = 0, nn = 0;
    int level = 0;
    // the mesh this one was red-refined from, with its full connectivity:
    // the child's edge / face grouping then follows in closed form
    // (refine_conn.cu) instead of the vertex-star hashing
    std::shared_ptr<MeshData> parent_mesh;
    std::shared_ptr<Connectivity> parent_conn;
    DBuf<double> coords;  // [3 nC]
    DBuf<int32_t> tets;   // [4 nE]
    DBuf<int32_t> db, nb; // [3 nD], [3 nN]
    std::unique_ptr<PendingUpload> pending;
    MeshData() = default;
    MeshData(const MeshData&) = delete;
    MeshData& operator=(const MeshData&) = delete;
    ~MeshData();  // an unused pending upload is waited for before the free
};

// Completes an asynchronous upload before the mesh's first use: waits for
// its event on the host (instant once the copy engine is done), replays the
// index check, and orders the library stream after the upload.
void finish_upload(MeshData& m);

struct Coefs {
    DBuf<double> a_elem, a_diag;
    bool has_elem = false, has_diag = false;
    double c = 1.0;
    uint64_t version = 0;
};

// transient device buffers of one connectivity / refinement / assembly pass,
// kept with their owner so repeated passes reuse them
struct Work {
    DBuf<int32_t> cnt, big_list, big_count, packed, redo, a0;
    DBuf<double> face_bval;  // boundary faces' b_D / Neumann terms (assembly)
    DBuf<int64_t> face_off;
    DBuf<unsigned char> scratch;
    DBuf<uint32_t> claim;
    DBuf<unsigned long long> counts, err;
    DBuf<uint16_t> masks;
    DBuf<double> partials, norms;
};

struct Connectivity {
    Work w;
    // vertex star
    DBuf<int64_t> star_ptr;
    DBuf<int32_t> star;
    bool has_star = false;  // skipped for a classified refined mesh
    // edges
    bool has_edges = false;
    int64_t ned = 0;
    DBuf<int32_t> edge_first, edge_of_slot, edge_nodes;
    DBuf<int64_t> edge_off;
    // faces
    bool has_faces = false;
    int64_t nf = 0, n_int = 0, n_dir = 0, n_neu = 0, l = 0;
    DBuf<int32_t> slot_mate, face_of_slot, faces, face_slots, face_mrow, row_face;
    DBuf<int8_t> sigma;
    DBuf<uint8_t> face_class;
    DBuf<double> face_area;
    DBuf<int32_t> entry_face;  // boundary list entry (db then nb) -> face id
    // timings (seconds)
    double t_edges = 0.0, t_faces = 0.0;
};

struct System {
    Work w;
    int problem = -1;
    uint64_t coef_version = 0;
    int64_t n = 0, l = 0, nchunks = 0;
    // S: SELL-32 (debug / export systems) or element-major (solve path:
    // st_val + slot_mrow + diag); elem says which
    bool elem = false;
    DBuf<int32_t> sell_col;
    DBuf<double> sell_val, rhs_neg, bd, rhs;
    DBuf<double> st_val, diag;
    // element-major: the rows' second halves of diag / rhs_neg [2 l] until a
    // solve sums them in (split)
    DBuf<double> halves;
    mutable bool split = false;
    // diag / rhs_neg assembled (sums the halves once)
    void finish() const;
    // sum(B_T^2), sum(b_D^2) for inner_cg_options: reduced on the device
    // when a solve asks (the reference computes them at solve time too)
    void norms(double& sum_rhs2, double& sum_bd2) const;
    // debug views (filled only on request)
    DBuf<double> a_blocks, slot_coef;
    DBuf<int32_t> slot_mrow;
};

struct RefineMap {
    DBuf<int32_t> midpoint, centroid;
};

// Stage times from events recorded on the library stream without host
// synchronisation; resolve() (one synchronisation) turns the recorded spans
// into milliseconds after the pass.
struct Stages {
    double star = 0, groups = 0, number = 0, classify = 0, assemble = 0, refine = 0;
    double assemble_kernel = 0;  // assemble_k alone
    Stages() = default;
    Stages(const Stages&) = delete;
    Stages& operator=(const Stages&) = delete;
    ~Stages();
    // records an event now; returns its handle
    cudaEvent_t mark();
    // an event for the caller to record
    cudaEvent_t event();
    // adds the time between `from` and an event recorded now to *field
    void span(double* field, cudaEvent_t from);
    // adds the time between two recorded events to *field
    void span(double* field, cudaEvent_t from, cudaEvent_t to);
    // resolve() also runs the error checks deferred with defer_errors()
    void resolve();
    // Deferred error checks (one synchronisation for the whole pass): the
    // device error slots are copied into page-locked memory now and `check`
    // runs on them in resolve(); only when `defer` is set.
    bool defer = false;
    void defer_errors(const unsigned long long* dev_err, std::function<void(const unsigned long long*)> check);

  private:
    std::vector<cudaEvent_t> events_;
    size_t used_ = 0;
    std::vector<std::tuple<double*, cudaEvent_t, cudaEvent_t>> pending_;
    std::vector<std::pair<unsigned long long*, std::function<void(const unsigned long long*)>>> checks_;
};

// --------------------------------------------------------------- pipeline

std::shared_ptr<MeshData> upload_mesh(const double* coords, int64_t nc, const int32_t* tets, int64_t ne,
                                      const int32_t* db, int64_t nd, const int32_t* nb, int64_t nn, int level);
// Host arrays must stay valid (and unchanged) until the mesh's first use.
std::shared_ptr<MeshData> upload_mesh_async(const double* coords, int64_t nc, const int32_t* tets, int64_t ne,
                                            const int32_t* db, int64_t nd, const int32_t* nb, int64_t nn, int level);
std::shared_ptr<MeshData> kuhn_mesh(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                                    uint64_t seed, uint32_t mask);

// star + edges (+ faces, classification and multiplier rows)
// (classify = false: the face numbering alone, as faces_up gives it, without
// the boundary classification and multiplier rows)
void build_connectivity(const MeshData& m, Connectivity& c, bool faces, Stages* st = nullptr, bool classify = true);
// red refinement; needs edges.  `into` (optional) is reused for the child.
// `elements_written`: the child's elements and coordinates were written by
// the assembly kernel (prepare_child + assemble_system's refine argument);
// only the boundary lists are refined here.
std::shared_ptr<MeshData> refine_mesh(const MeshData& m, Connectivity& c, RefineMap* map, Stages* st = nullptr,
                                      std::shared_ptr<MeshData> into = nullptr, bool elements_written = false);
// the child mesh of one red refinement, sized and allocated (contents unset)
std::shared_ptr<MeshData> prepare_child(const MeshData& m, const Connectivity& c, std::shared_ptr<MeshData> into);
// fused assembly + condensation (+ the child's elements and coordinates
// when `refine` is given)
void assemble_system(const MeshData& m, const Coefs& k, const Connectivity& c, int problem, System& sys,
                     bool debug_views, Stages* st = nullptr, const phg_refine_out* refine = nullptr);
phg_problem device_problem(const Coefs& k, int problem);

struct SolveResult {
    DBuf<double> u, lambda;
    int64_t iterations = 0;
    double residual = 0.0, constraint_residual = 0.0, seconds = 0.0, cg_ms = 0.0, rel_residual = 0.0;
    // verify_solution's terms (solver.cpp:44-76): ||AU - C'L - B||, ||CU - b_D||, ||B||, ||b_D||
    double r1 = 0.0, r2 = 0.0, nrm_rhs = 0.0, nrm_bd = 0.0;
    bool converged = false, accepted = false;
};
// Jacobi-PCG on S, then (unless cg_only) recovery and verify_solution;
// with refuse_throws = false a verify refusal only clears `accepted`.
void solve_schur(const MeshData& m, const Coefs& k, const Connectivity& c, const System& sys, int problem,
                 double tol, int64_t max_iter, const std::string& method, SolveResult& out, bool cg_only = false,
                 bool refuse_throws = true);

double mesh_diameter(const MeshData& m);
// edge_pairs_to_elems' duplicate error pair (cxx_api.cpp), for the error path
bool e2t_first_duplicate(const MeshData& m, const Connectivity& c, int32_t& a, int32_t& b);
// [y-norm, kappa-norm, L2]
void error_norms(const MeshData& m, const Coefs& k, const Connectivity& c, int problem, const double* u,
                 const double* lambda, double out[3]);

// host helpers
std::string format_double(double v);
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w);
void tet_rule(int degree, std::vector<double>& lam, std::vector<double>& w);

}  // namespace phb
