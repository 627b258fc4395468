// Host runtime: stage orchestration of the device pipeline.  Sizes that only
// the device knows (nEd, nF, L) are read back once per stage; everything else
// stays on the stream.  Device error slots are replayed in the reference's
// check order so the same exception (and message shape) surfaces.
#include <mutex>

#include "runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace phb {

// ------------------------------------------------------------------ basics

void check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw MeshError(std::string("out of memory (device, ") + what + ")");
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
    check(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "create stream");
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

Stages::~Stages() {
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
}
cudaEvent_t Stages::event() {
    if (used_ == events_.size()) {
        cudaEvent_t e;
        check(cudaEventCreate(&e), "event");
        events_.push_back(e);
    }
    return events_[used_++];
}
cudaEvent_t Stages::mark() {
    cudaEvent_t e = event();
    check(cudaEventRecord(e, S()), "event record");
    return e;
}
void Stages::span(double* field, cudaEvent_t from) { pending_.emplace_back(field, from, mark()); }
void Stages::span(double* field, cudaEvent_t from, cudaEvent_t to) { pending_.emplace_back(field, from, to); }
namespace {
// host memory mapped into the device address space, written by
// phfem_gpu_gather_words (allocated once per thread: cudaHostAlloc
// synchronises the device): slot 0 for read_words, 1.. for deferred error
// reads
constexpr size_t kWordSlots = 17;
unsigned long long* word_slot(size_t i) {
    static thread_local unsigned long long* base = nullptr;
    if (!base)
        check(cudaHostAlloc(reinterpret_cast<void**>(&base), kWordSlots * 16 * sizeof(unsigned long long),
                            cudaHostAllocMapped | cudaHostAllocPortable),
              "mapped alloc");
    if (i >= kWordSlots) throw MeshError("too many deferred error checks");
    return base + 16 * i;
}
void gather_to(const unsigned long long* const* src, int n, unsigned long long* h) {
    unsigned long long* d = nullptr;
    check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0), "mapped pointer");
    check(phfem_gpu_gather_words(src, n, d, S()), "gather words");
}
}  // namespace

void read_words(const unsigned long long* const* src, int n, unsigned long long* out) {
    if (n > 16) throw MeshError("read_words: at most 16 words");
    volatile unsigned long long* h = word_slot(0);
    gather_to(src, n, const_cast<unsigned long long*>(h));
    sync();
    for (int i = 0; i < n; ++i) out[i] = h[i];
}

void Stages::defer_errors(const unsigned long long* dev_err, std::function<void(const unsigned long long*)> f) {
    unsigned long long* h = word_slot(1 + checks_.size());
    const unsigned long long* src[PHG_ERR_COUNT];
    for (int i = 0; i < PHG_ERR_COUNT; ++i) src[i] = dev_err + i;
    gather_to(src, PHG_ERR_COUNT, h);
    checks_.emplace_back(h, std::move(f));
}

void Stages::resolve() {
    if (pending_.empty() && checks_.empty()) return;
    sync();
    for (auto& [field, a, b] : pending_) {
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, a, b), "event time");
        *field += ms;
    }
    pending_.clear();
    auto checks = std::move(checks_);
    checks_.clear();
    for (auto& [h, f] : checks) f(h);
}
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

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
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

// Page-locked result slots for the asynchronous index checks, allocated once:
// cudaMallocHost / cudaFreeHost synchronise the device, which would serialise
// an upload with the work it is meant to overlap.
namespace {
struct FlagSlots {
    static constexpr int kSlots = 256;
    std::mutex mu;
    unsigned long long* base = nullptr;
    std::vector<int> free_list;
    unsigned long long* take() {
        std::lock_guard<std::mutex> lk(mu);
        if (!base) {
            check(cudaMallocHost(reinterpret_cast<void**>(&base), kSlots * 4 * sizeof(unsigned long long)),
                  "pinned alloc");
            for (int i = kSlots - 1; i >= 0; --i) free_list.push_back(i);
        }
        if (free_list.empty()) throw MeshError("too many mesh uploads in flight");
        const int i = free_list.back();
        free_list.pop_back();
        return base + 4 * i;
    }
    void give(unsigned long long* p) {
        std::lock_guard<std::mutex> lk(mu);
        free_list.push_back((int)((p - base) / 4));
    }
};
FlagSlots& flag_slots() {
    static FlagSlots s;
    return s;
}
}  // namespace

PendingUpload::~PendingUpload() {
    if (ready) cudaEventDestroy(ready);
    if (flags) flag_slots().give(flags);
}

std::shared_ptr<MeshData> upload_mesh_async(const double* coords, int64_t nc, const int32_t* tets, int64_t ne,
                                            const int32_t* db, int64_t nd, const int32_t* nb, int64_t nn, int level) {
    if (nc < 0 || ne < 0 || nd < 0 || nn < 0) throw InvalidArgument("negative mesh size");
    if (6 * ne >= (int64_t)INT32_MAX) throw MeshError("mesh too large: 6 nE must stay below 2^31");
    auto m = std::make_shared<MeshData>();
    m->nc = nc;
    m->ne = ne;
    m->nd = nd;
    m->nn = nn;
    m->level = level;
    auto pu = std::make_unique<PendingUpload>();
    cudaStream_t s = SC();
    m->coords.upload_on(coords, 3 * nc, s);
    m->tets.upload_on(tets, 4 * ne, s);
    m->db.upload_on(db, 3 * nd, s);
    m->nb.upload_on(nb, 3 * nn, s);
    // index range check on the copy stream, result to pinned memory
    pu->flags = flag_slots().take();
    pu->dflags.release();
    pu->dflags.n = pu->dflags.cap = 3;
    check(cudaMallocAsync(reinterpret_cast<void**>(&pu->dflags.p), 3 * sizeof(unsigned long long), s), "allocate");
    check(cudaMemsetAsync(pu->dflags.p, 0xff, 3 * sizeof(unsigned long long), s), "memset");
    check(phfem_gpu_check_indices(m->tets.p, 4 * ne, nc, pu->dflags.p, s), "check indices");
    check(phfem_gpu_check_indices(m->db.p, 3 * nd, nc, pu->dflags.p + 1, s), "check indices");
    check(phfem_gpu_check_indices(m->nb.p, 3 * nn, nc, pu->dflags.p + 2, s), "check indices");
    check(cudaMemcpyAsync(pu->flags, pu->dflags.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaEventCreateWithFlags(&pu->ready, cudaEventDisableTiming), "event");
    check(cudaEventRecord(pu->ready, s), "event record");
    pu->src[0] = tets;
    pu->src[1] = db;
    pu->src[2] = nb;
    m->pending = std::move(pu);
    return m;
}

MeshData::~MeshData() {
    if (pending && pending->ready) {
        cudaEventSynchronize(pending->ready);
        cudaStreamWaitEvent(S(), pending->ready, 0);
    }
}

void finish_upload(MeshData& m) {
    if (!m.pending) return;
    PendingUpload& pu = *m.pending;
    // an invalid mesh stays pending: every later use fails the same way,
    // from the saved message (the caller's arrays need only live until the
    // first use, phfem_ext.h)
    if (!pu.error.empty()) throw InvalidArgument(pu.error);
    check(cudaEventSynchronize(pu.ready), "upload");
    for (int i = 0; i < 3; ++i)
        if (pu.flags[i] != ~0ull) {
            pu.error = "node index " + std::to_string((long long)pu.src[i][pu.flags[i]] + 1) + " out of range 1.." +
                       std::to_string(m.nc);
            pu.src[0] = pu.src[1] = pu.src[2] = nullptr;
            throw InvalidArgument(pu.error);
        }
    check(cudaStreamWaitEvent(S(), pu.ready, 0), "wait upload");
    m.pending.reset();
}

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

// ------------------------------------------------------------------- solve

void System::norms(double& sum_rhs2, double& sum_bd2) const {
    DBuf<double> partials(2 * (int64_t)phfem_gpu_assemble_grid(n / 4)), out(2);
    check(phfem_gpu_sumsq2(rhs.p, n, bd.p, l, partials.p, out.p, SV()), "norms");
    double h[2];
    check(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, S()), "D2H");
    sync();
    sum_rhs2 = h[0];
    sum_bd2 = h[1];
}

void solve_schur(const MeshData& m, const Coefs& k, const Connectivity& c, const System& sys, int problem,
                 double tol, int64_t max_iter, const std::string& method, SolveResult& out, bool cg_only,
                 bool refuse_throws) {
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t l = sys.l;
    sys.finish();  // an element-major system's diag / rhs_neg halves
    double sum_rhs2, sum_bd2;
    sys.norms(sum_rhs2, sum_bd2);
    const double nrm_rhs = std::sqrt(sum_rhs2), nrm_bd = std::sqrt(sum_bd2);
    // inner_cg_options, solver.cpp:78-86
    const double abs_tol = 0.2 * tol * std::hypot(nrm_rhs, nrm_bd);
    const long long mi = max_iter > 0 ? max_iter : 10 * std::max<int64_t>(l, 1);
    out.lambda.alloc(l);
    DBuf<double> r(l), p(l), q(l), d(l);
    DBuf<phg_cg_state> state(1);
    DBuf<double> partials(2 * 148 * 8 + 64);
    Timer tm;
    tm.start();
    // An element-major system is streamed by rows straight from its blocks
    // (cg_spmv_em: per row its two slots, the elements' off-diagonal values
    // and row ids gathered); PHFEM_CG_SELL=1 lays it out as SELL-32 once
    // instead (S_T's upper triangle mirrored; the same iterates bit for bit).
    // A SELL system (exports) is streamed as it is.
    static const bool force_sell = [] {
        const char* e = std::getenv("PHFEM_CG_SELL");
        return e && std::atoi(e) != 0;
    }();
    const bool em = sys.elem && !force_sell;
    DBuf<int32_t> tmp_col, row_slots;
    DBuf<double> tmp_val;
    const int32_t* sell_col = sys.sell_col.p;
    const double* sell_val = sys.sell_val.p;
    if (em) {
        row_slots.alloc(2 * l);
        check(phfem_gpu_cg_em_rows(m.ne, sys.slot_mrow.p, c.slot_mate.p, row_slots.p, SV()), "cg rows");
        check(phfem_gpu_cg_em_init(l, sys.diag.p, sys.rhs_neg.p, out.lambda.p, r.p, p.p, d.p, tol, abs_tol, mi,
                                   state.p, partials.p, SV()),
              "cg init");
    } else {
        if (sys.elem) {
            tmp_col.alloc(sys.nchunks * PHG_SELL_C * PHG_SELL_W);
            tmp_val.alloc(sys.nchunks * PHG_SELL_C * PHG_SELL_W);
            check(phfem_gpu_elem_to_sell(m.ne, l, sys.st_val.p, sys.slot_mrow.p, c.slot_mate.p, sys.diag.p,
                                         tmp_col.p, tmp_val.p, SV()),
                  "elem to sell");
            sell_col = tmp_col.p;
            sell_val = tmp_val.p;
        }
        check(phfem_gpu_cg_init(l, sell_col, sell_val, sys.rhs_neg.p, out.lambda.p, r.p, p.p, d.p, tol, abs_tol,
                                mi, state.p, partials.p, SV()),
              "cg init");
    }
    phg_cg_state hs{};
    phg_cg_state* pinned = nullptr;
    check(cudaMallocHost(reinterpret_cast<void**>(&pinned), sizeof(phg_cg_state)), "pinned alloc");
    // iterations per graph launch / host poll: a poll (D2H + stream sync +
    // relaunch) costs ~20-30 us, so small systems batch more; iterations past
    // convergence are no-op launches (a few us each)
    const int batch = l < 200000 ? 64 : (l < 8000000 ? 32 : 16);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    try {
        check(cudaMemcpyAsync(pinned, state.p, sizeof(phg_cg_state), cudaMemcpyDeviceToHost, S()), "D2H");
        sync();
        hs = *pinned;
        if (!hs.done) {
            check(cudaStreamBeginCapture(S(), cudaStreamCaptureModeThreadLocal), "capture");
            if (em)
                phfem_gpu_cg_em_iterations(batch, l, row_slots.p, sys.st_val.p, sys.slot_mrow.p, sys.diag.p,
                                           out.lambda.p, r.p, p.p, q.p, d.p, state.p, partials.p, SV());
            else
                phfem_gpu_cg_iterations(batch, l, sell_col, sell_val, out.lambda.p, r.p, p.p, q.p, d.p, state.p,
                                        partials.p, SV());
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
    out.rel_residual = hs.rel_residual;
    if (hs.not_spd) throw SolverError("pcg: operator is not positive definite");
    if (!hs.converged) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "%f", hs.rel_residual);
        throw SolverError("schur: conjugate gradients stalled at relative residual " + std::string(buf) + " after " +
                          std::to_string(hs.it) + " iterations");
    }
    if (cg_only) {
        out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return;
    }
    // recovery + verify_solution (solver.cpp:44-76, 168-181)
    out.u.alloc(4 * m.ne);
    const phg_problem pr = device_problem(k, problem);
    DBuf<double> rpart(148 * 16 * 3 + 64), sums(1), cres(3);
    DBuf<unsigned long long> err(PHG_ERR_COUNT);
    err.fill_bytes(0xff);
    check(phfem_gpu_recover(m.ne, m.coords.p, m.tets.p, &pr, c.face_of_slot.p, c.slot_mate.p, c.face_mrow.p,
                            c.face_area.p, sys.rhs.p, out.lambda.p, out.u.p, sums.p, rpart.p, err.p, SV()),
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
    out.r1 = r1;
    out.r2 = r2;
    out.nrm_rhs = nrm_rhs;
    out.nrm_bd = nrm_bd;
    out.accepted = ok;
    if (!ok && refuse_throws) {
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
