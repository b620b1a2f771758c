// capi.cu — the extern "C" boundary of librafem_b200 (include/rafem_b200.h)
// and the native time loop (rafem_simulate).
#include "common.cuh"
#include "internal.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

using namespace rafem;

int rafem_fail(rafem_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int rafem_fail_cuda(rafem_ctx* ctx, cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    if (ctx) ctx->err = buf;
    return RAFEM_ERR_CUDA;
}

namespace rafem {

int ensure(rafem_ctx* ctx, DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes && b.p) return RAFEM_OK;
    if (b.p) {
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
    }
    const size_t want = std::max<size_t>(bytes, 256);
    RF_CUDA_TRY(ctx, cudaMalloc(&b.p, want));
    b.bytes = want;
    return RAFEM_OK;
}

cudaError_t dmalloc(rafem_ctx* ctx, void** p, size_t bytes) {
    bytes = std::max<size_t>((bytes + 255) / 256 * 256, 256);
    auto it = ctx->free_blocks.lower_bound(bytes);
    if (it != ctx->free_blocks.end() && it->first <= 2 * bytes) {  // reuse a block of close size
        *p = it->second;
        ctx->cached_bytes -= it->first;
        ctx->free_set.erase(it->second);
        ctx->free_blocks.erase(it);
        return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {  // give the cache back to the driver and retry once
        cudaGetLastError();
        dcache_release(ctx);
        e = cudaMalloc(p, bytes);
    }
    if (e == cudaSuccess) ctx->block_size[*p] = bytes;
    return e;
}

void dfree(rafem_ctx* ctx, void* p) {
    if (!p) return;
    auto it = ctx->block_size.find(p);
    if (it == ctx->block_size.end()) {
        cudaFree(p);
        return;
    }
    if (!ctx->free_set.insert(p).second) {  // already free: a second release would alias two later blocks
        if (ctx->double_frees++ == 0)
            if (const char* dbg = getenv("RAFEM_DEBUG_ALLOC"))
                if (dbg[0] == '1') std::fprintf(stderr, "rafem: double free of device block %p ignored\n", p);
        return;
    }
    ctx->free_blocks.emplace(it->second, p);
    ctx->cached_bytes += it->second;
    // keep at most 8 GiB cached
    while (ctx->cached_bytes > (8ull << 30) && !ctx->free_blocks.empty()) {
        auto big = std::prev(ctx->free_blocks.end());
        cudaFree(big->second);
        ctx->block_size.erase(big->second);
        ctx->free_set.erase(big->second);
        ctx->cached_bytes -= big->first;
        ctx->free_blocks.erase(big);
    }
}

void dcache_release(rafem_ctx* ctx) {
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->free_blocks) {
        cudaFree(kv.second);
        ctx->block_size.erase(kv.second);
    }
    ctx->free_blocks.clear();
    ctx->free_set.clear();
    ctx->cached_bytes = 0;
}

void* pinned(rafem_ctx* ctx, size_t bytes) {
    if (ctx->pin_bytes >= bytes && ctx->pin) return ctx->pin;
    if (ctx->pin) {
        cudaStreamSynchronize(ctx->stream);
        cudaFreeHost(ctx->pin);
        ctx->pin = nullptr;
        ctx->pin_bytes = 0;
    }
    const size_t want = std::max<size_t>(bytes, 1 << 16);
    if (cudaMallocHost(&ctx->pin, want) != cudaSuccess) {
        ctx->pin = nullptr;
        return nullptr;
    }
    ctx->pin_bytes = want;
    return ctx->pin;
}

}  // namespace rafem

namespace {

// host -> device through the pinned staging buffer (async wrt the host
// only up to the final stream sync the callers do)
int upload(rafem_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return RAFEM_OK;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return RAFEM_OK;
}

void fill_stats(const KResult& r, float ms, rafem_solve_stats* st) {
    st->iterations = r.iterations;
    st->restarts = r.restarts;
    st->final_relative_residual = r.final_rel;
    st->converged = r.converged;
    st->stagnated = r.stagnated;
    st->cycles = r.cycles;
    st->history_len = r.hist_len;
    st->device_ms = ms;
}

int check_params(rafem_ctx* ctx, const rafem_solver_params* p) {
    if (!p) return rafem_fail(ctx, RAFEM_ERR_INVALID, "solver params missing");
    if (p->method != RAFEM_METHOD_GMRES && p->method != RAFEM_METHOD_PCG)
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "unknown Krylov method");
    if (p->restart_m < 1) return rafem_fail(ctx, RAFEM_ERR_INVALID, "restart_m must be at least 1");
    if (!(p->tolerance > 0.0 && p->tolerance < 1.0))
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "tolerance must lie in (0, 1)");
    if (p->precondition < RAFEM_PRECOND_NONE || p->precondition > RAFEM_PRECOND_BLOCK_JACOBI)
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "unknown preconditioner");
    return RAFEM_OK;
}

MatView system_view(rafem_system* s) {
    // stencil classes pay off only when the matrix streams from HBM
    if (!s->mesh->cls_tried && (long long)s->mesh->slots * 20 > (48LL << 20)) mesh_stencil_classes(s->mesh);
    MatView A;
    A.rp = s->mesh->rp;
    A.col = s->mesh->col;
    A.val = s->val2;
    A.ngroups = s->mesh->N;
    A.W = 2;
    A.slots = s->mesh->slots;
    A.pattern_id = s->mesh->id;
    A.maxdeg = s->mesh->maxdeg;
    A.cls = s->mesh->cls;
    A.cls_off = s->mesh->cls_off;
    A.ncls = s->mesh->ncls;
    A.coords = s->mesh->nodes;
    return A;
}

// device layout of sys->status
struct SysStatus {
    PassStatus pass;
    int flag;  // zero-diagonal flag of the Jacobi setup
    int pad;
};

SysStatus* sys_status(rafem_system* s) { return reinterpret_cast<SysStatus*>(s->status); }

// solve on a matrix view with host b/x0/x; shared by system and matrix paths
// RAFEM_HOST_TIMING=1: per-phase host microseconds of each solve to stderr
static double host_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int solve_common(rafem_ctx* ctx, const MatView& A, double* b_dev, bool b_is_host, const double* b,
                 const double* x0, const rafem_solver_params* p, double* x_out, rafem_solve_stats* st,
                 double* hist, int64_t hist_cap, int64_t* cycle_lens, int64_t cycle_cap, double* minv,
                 double* xbuf, SysStatus* dstat) {
    const int n = A.ngroups * A.W;
    static const bool timing = [] { const char* e = getenv("RAFEM_HOST_TIMING"); return e && e[0] == '1'; }();
    const double t0 = timing ? host_us() : 0.0;
    if (int rc = check_params(ctx, p)) return rc;
    // one pinned staging area and one stream synchronisation per solve:
    // [b | x0 | x out | KResult | history head | cycle-length head]
    constexpr long long kHistHead = 4096, kCycHead = 512;
    const size_t nb = sizeof(double) * (size_t)n;
    char* pin = static_cast<char*>(pinned(ctx, 3 * nb + sizeof(KResult) + 8 * (kHistHead + kCycHead)));
    if (!pin) return rafem_fail(ctx, RAFEM_ERR_CUDA, "pinned staging allocation failed");
    double* pb = reinterpret_cast<double*>(pin);
    double* px0 = pb + n;
    double* px = px0 + n;
    KResult* pr = reinterpret_cast<KResult*>(px + n);
    double* ph = reinterpret_cast<double*>(pr + 1);
    long long* pc = reinterpret_cast<long long*>(ph + kHistHead);
    if (b_is_host && b && n > 0) {
        std::memcpy(pb, b, nb);
        if (int rc = upload(ctx, b_dev, pb, nb)) return rc;
    }
    const double* x0_dev = nullptr;
    if (x0) {
        if (n > 0) {
            std::memcpy(px0, x0, nb);
            if (int rc = upload(ctx, xbuf, px0, nb)) return rc;
        }
        x0_dev = xbuf;
    }
    const double t1 = timing ? host_us() : 0.0;
    int* flag = &dstat->flag;
    if (p->precondition != RAFEM_PRECOND_NONE) {
        if (int rc = jacobi_minv(ctx, A, minv, flag)) return rc;
    } else {
        RF_CUDA_TRY(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    }
    const double t2 = timing ? host_us() : 0.0;
    if (int rc = krylov_solve(ctx, A, b_dev, x0_dev, xbuf, minv, *p, &dstat->pass.solve, flag, ctx->ev0, ctx->ev1))
        return rc;
    const double t3 = timing ? host_us() : 0.0;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(pr, &dstat->pass.solve, sizeof(KResult), cudaMemcpyDeviceToHost, ctx->stream));
    if (n > 0) RF_CUDA_TRY(ctx, cudaMemcpyAsync(px, xbuf, nb, cudaMemcpyDeviceToHost, ctx->stream));
    // the heads of the residual history and the cycle lengths ride along
    const long long hh = std::min<long long>(kHistHead, (long long)(ctx->ws_hist.bytes / sizeof(double)));
    const long long ch = std::min<long long>(kCycHead, (long long)(ctx->ws_cyc.bytes / sizeof(long long)));
    if (hist && hist_cap > 0 && hh > 0)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(ph, ctx->ws_hist.p, sizeof(double) * hh, cudaMemcpyDeviceToHost, ctx->stream));
    if (cycle_lens && cycle_cap > 0 && ch > 0)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(pc, ctx->ws_cyc.p, sizeof(long long) * ch, cudaMemcpyDeviceToHost, ctx->stream));
    const double t4 = timing ? host_us() : 0.0;
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const double t5 = timing ? host_us() : 0.0;
    const KResult r = *pr;
    if (n > 0) std::memcpy(x_out, px, nb);
    if (timing)
        std::fprintf(stderr, "solve host us: uploads %.1f, jacobi %.1f, krylov_solve %.1f, d2h enqueue %.1f, sync %.1f\n",
                     t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    if (st) fill_stats(r, ms, st);
    const long long nh = std::min<long long>(r.hist_len, hist ? hist_cap : 0);
    const long long nc = std::min<long long>(r.cycles, cycle_lens ? cycle_cap : 0);
    if (nh <= hh && nc <= ch) {
        if (nh > 0) std::memcpy(hist, ph, sizeof(double) * nh);
        if (nc > 0) std::memcpy(cycle_lens, pc, sizeof(long long) * nc);
    } else if (int rc = krylov_read_history(ctx, r, hist, hist_cap, reinterpret_cast<long long*>(cycle_lens),
                                            cycle_cap)) {
        return rc;
    }
    if (r.status == RAFEM_ERR_INVALID)
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "Jacobi preconditioning requires a zero-free diagonal");
    if (r.status == RAFEM_ERR_BREAKDOWN) {
        char buf[256];
        std::snprintf(buf, sizeof(buf), "Arnoldi breakdown with relative residual %.3e above tolerance %.3e",
                      r.final_rel, p->tolerance);
        if (p->method == RAFEM_METHOD_PCG)
            std::snprintf(buf, sizeof(buf), "CG breakdown (operator not SPD under the preconditioner), "
                          "relative residual %.3e", r.final_rel);
        return rafem_fail(ctx, RAFEM_ERR_BREAKDOWN, buf);
    }
    return RAFEM_OK;
}

}  // namespace

extern "C" {

int rafem_ctx_create(int device, rafem_ctx** out) {
    if (!out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    rafem_ctx* ctx = new rafem_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        int rc = rafem_fail_cuda(ctx, e, "cudaSetDevice", __FILE__, __LINE__);
        *out = ctx;  // keep the message readable
        return rc;
    }
    cudaDeviceProp prop;
    RF_CUDA_TRY(ctx, cudaGetDeviceProperties(&prop, device));
    ctx->sm_count = prop.multiProcessorCount;
    ctx->cc_major = prop.major;
    ctx->cc_minor = prop.minor;
    ctx->total_mem = (long long)prop.totalGlobalMem;
    if (!prop.cooperativeLaunch) {
        *out = ctx;
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "device lacks cooperative launch");
    }
    RF_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    RF_CUDA_TRY(ctx, cudaEventCreate(&ctx->ev0));
    RF_CUDA_TRY(ctx, cudaEventCreate(&ctx->ev1));
    RF_CUDA_TRY(ctx, cudaEventCreate(&ctx->ev2));
    ensure(ctx, ctx->ws_res, 4096);
    *out = ctx;
    return RAFEM_OK;
}

void rafem_ctx_destroy(rafem_ctx* ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->ws_basis, &ctx->ws_vec, &ctx->ws_partial, &ctx->ws_hess, &ctx->ws_hist,
                      &ctx->ws_cyc, &ctx->ws_part, &ctx->ws_res, &ctx->ws_trace, &ctx->ws_flags, &ctx->ws_simout,
                      &ctx->ws_diag, &ctx->ws_gal})
        if (b->p) cudaFree(b->p);
    for (auto& e : ctx->part_cache) dfree(ctx, e.gpart);
    ctx->part_cache.clear();
    cluster_plans_release(ctx);
    dcache_release(ctx);
    if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
    if (ctx->mapped) cudaFreeHost(ctx->mapped);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev2) cudaEventDestroy(ctx->ev2);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* rafem_last_error(const rafem_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int rafem_device_info(rafem_ctx* ctx, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor,
                      int64_t* total_mem) {
    if (!ctx) return RAFEM_ERR_INVALID;
    if (sm_count) *sm_count = ctx->sm_count;
    if (cc_major) *cc_major = ctx->cc_major;
    if (cc_minor) *cc_minor = ctx->cc_minor;
    if (total_mem) *total_mem = ctx->total_mem;
    return RAFEM_OK;
}

int64_t rafem_kernel_launches(const rafem_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* rafem_stream(const rafem_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int rafem_last_solve_mode(const rafem_ctx* ctx, int32_t* mode, int32_t* ctas) {
    if (!ctx) return RAFEM_ERR_INVALID;
    if (mode) *mode = ctx->last_mode;
    if (ctas) *ctas = ctx->last_ctas;
    return RAFEM_OK;
}

int rafem_last_solve_precond(const rafem_ctx* ctx, int32_t* precond) {
    if (!ctx || !precond) return RAFEM_ERR_INVALID;
    *precond = ctx->last_precond;
    return RAFEM_OK;
}

int rafem_set_trace(rafem_ctx* ctx, int32_t on) {
    if (!ctx) return RAFEM_ERR_INVALID;
    ctx->trace_on = on ? 1 : 0;
    return RAFEM_OK;
}

int64_t rafem_get_trace(rafem_ctx* ctx, int64_t* out, int64_t cap) {
    if (!ctx || !ctx->ws_trace.p) return 0;
    const int64_t n = std::min<int64_t>(cap, (int64_t)(ctx->ws_trace.bytes / sizeof(long long)));
    if (cudaMemcpyAsync(out, ctx->ws_trace.p, sizeof(long long) * n, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return 0;
    return n;
}

// ---- sparse ---------------------------------------------------------------

int rafem_spmv(rafem_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr,
               const int64_t* col_idx, const double* vals, const double* x, double* y) {
    if (!ctx) return RAFEM_ERR_INVALID;
    if (nrows < 0 || ncols < 0 || nnz < 0) return rafem_fail(ctx, RAFEM_ERR_INVALID, "negative size");
    if (nrows >= (1LL << 31) || ncols >= (1LL << 31) || nnz >= (1LL << 31))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "spmv: sizes must fit in int32");
    if (nrows == 0) return RAFEM_OK;
    std::vector<int> rp(nrows + 1), ci(nnz);
    for (int64_t i = 0; i <= nrows; ++i) rp[i] = (int)row_ptr[i];
    for (int64_t k = 0; k < nnz; ++k) ci[k] = (int)col_idx[k];
    int *drp = nullptr, *dci = nullptr;
    double *dv = nullptr, *dx = nullptr, *dy = nullptr;
    auto cleanup = [&]() { cudaFree(drp); cudaFree(dci); cudaFree(dv); cudaFree(dx); cudaFree(dy); };
    cudaError_t e;
#define RF_S(x) do { e = (x); if (e != cudaSuccess) { cleanup(); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    RF_S(cudaMalloc(&drp, sizeof(int) * (nrows + 1)));
    RF_S(cudaMalloc(&dci, sizeof(int) * std::max<int64_t>(nnz, 1)));
    RF_S(cudaMalloc(&dv, sizeof(double) * std::max<int64_t>(nnz, 1)));
    RF_S(cudaMalloc(&dx, sizeof(double) * std::max<int64_t>(ncols, 1)));
    RF_S(cudaMalloc(&dy, sizeof(double) * nrows));
    RF_S(cudaMemcpyAsync(drp, rp.data(), sizeof(int) * (nrows + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (nnz) {
        RF_S(cudaMemcpyAsync(dci, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, ctx->stream));
        RF_S(cudaMemcpyAsync(dv, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (ncols) RF_S(cudaMemcpyAsync(dx, x, sizeof(double) * ncols, cudaMemcpyHostToDevice, ctx->stream));
    MatView A{drp, dci, dv, (int)nrows, 1, nnz};
    if (int rc = spmv_launch(ctx, A, dx, dy)) { cleanup(); return rc; }
    RF_S(cudaMemcpyAsync(y, dy, sizeof(double) * nrows, cudaMemcpyDeviceToHost, ctx->stream));
    RF_S(cudaStreamSynchronize(ctx->stream));
#undef RF_S
    cleanup();
    return RAFEM_OK;
}

int rafem_coo_to_csr(rafem_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz_in, const int64_t* rows,
                     const int64_t* cols, const double* vals, int64_t* row_ptr_out, int64_t* col_idx_out,
                     double* vals_out, int64_t* nnz_out) {
    if (!ctx) return RAFEM_ERR_INVALID;
    return coo_to_csr_device(ctx, nrows, ncols, nnz_in, rows, cols, vals, row_ptr_out, col_idx_out, vals_out,
                             nnz_out);
}

// ---- general matrix ---------------------------------------------------------

int rafem_matrix_create(rafem_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, rafem_matrix** out) {
    if (!ctx || !out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    if (nrows < 0 || nnz < 0) return rafem_fail(ctx, RAFEM_ERR_INVALID, "negative size");
    if (nrows >= (1LL << 31) || nnz >= (1LL << 31))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "matrix sizes must fit in int32");
    rafem_matrix* a = new rafem_matrix();
    a->ctx = ctx;
    a->n = (int)nrows;
    a->nnz = nnz;
    std::vector<int> rp(nrows + 1), ci(nnz);
    for (int64_t i = 0; i <= nrows; ++i) rp[i] = (int)row_ptr[i];
    for (int64_t k = 0; k < nnz; ++k) ci[k] = (int)col_idx[k];
    cudaError_t e;
#define RF_M(x) do { e = (x); if (e != cudaSuccess) { rafem_matrix_destroy(a); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    RF_M(cudaMalloc(&a->rp, sizeof(int) * (nrows + 1)));
    RF_M(cudaMalloc(&a->col, sizeof(int) * std::max<int64_t>(nnz, 1)));
    RF_M(cudaMalloc(&a->val, sizeof(double) * std::max<int64_t>(nnz, 1)));
    RF_M(cudaMalloc(&a->minv, sizeof(double) * (3 * (size_t)std::max<int64_t>(nrows, 1) + 64)));
    RF_M(cudaMemcpyAsync(a->rp, rp.data(), sizeof(int) * (nrows + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (nnz) {
        RF_M(cudaMemcpyAsync(a->col, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, ctx->stream));
        RF_M(cudaMemcpyAsync(a->val, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    }
    RF_M(cudaStreamSynchronize(ctx->stream));
#undef RF_M
    *out = a;
    return RAFEM_OK;
}

void rafem_matrix_destroy(rafem_matrix* a) {
    if (!a) return;
    cudaFree(a->rp);
    cudaFree(a->col);
    cudaFree(a->val);
    cudaFree(a->minv);
    delete a;
}

int rafem_matrix_solve(rafem_matrix* a, const double* b, const double* x0, const rafem_solver_params* p,
                       double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap,
                       int64_t* cycle_lens, int64_t cycle_cap) {
    if (!a) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = a->ctx;
    const int n = a->n;
    if (n == 0) {
        if (st) std::memset(st, 0, sizeof(*st)), st->converged = 1;
        return RAFEM_OK;
    }
    // minv buffer doubles as b and x staging: [minv | b | x | status]
    double* minv = a->minv;
    double* bdev = a->minv + n;
    double* xdev = a->minv + 2 * (size_t)n;
    if (int rc = ensure(ctx, ctx->ws_res, sizeof(SysStatus) + 256)) return rc;
    SysStatus* ds = static_cast<SysStatus*>(ctx->ws_res.p);
    MatView A{a->rp, a->col, a->val, n, 1, a->nnz};
    return solve_common(ctx, A, bdev, true, b, x0, p, x_out, st, hist, hist_cap, cycle_lens, cycle_cap, minv, xdev, ds);
}

// ---- mesh / system -----------------------------------------------------------

int rafem_mesh_create(rafem_ctx* ctx, int64_t n_nodes, const double* nodes, int64_t n_tets, const int64_t* tets,
                      const int32_t* region_index, int32_t n_regions, const double* k, const double* rho_c,
                      const double* sigma0, const double* alpha, const double* t_ref, const uint8_t* dof_kind,
                      rafem_mesh** out) {
    if (!ctx || !out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    if (n_nodes < 0 || n_tets < 0 || n_regions < 1) return rafem_fail(ctx, RAFEM_ERR_INVALID, "bad mesh sizes");
    if (n_nodes >= (1LL << 30) || n_tets >= (1LL << 30))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "mesh too large for 30-bit element ids");
    std::vector<int> t32(4 * (size_t)n_tets);
    for (int64_t i = 0; i < 4 * n_tets; ++i) {
        if (tets[i] < 0 || tets[i] >= n_nodes) return rafem_fail(ctx, RAFEM_ERR_INVALID, "tet references a node out of range");
        t32[i] = (int)tets[i];
    }
    std::vector<int> reg(n_tets, 0);
    if (region_index)
        for (int64_t e = 0; e < n_tets; ++e) {
            if (region_index[e] < 0 || region_index[e] >= n_regions) return rafem_fail(ctx, RAFEM_ERR_INVALID, "region index out of range");
            reg[e] = region_index[e];
        }
    std::vector<double> tab(5 * (size_t)n_regions);
    for (int r = 0; r < n_regions; ++r) {
        tab[r] = k[r];
        tab[n_regions + r] = rho_c[r];
        tab[2 * n_regions + r] = sigma0[r];
        tab[3 * n_regions + r] = alpha[r];
        tab[4 * n_regions + r] = t_ref[r];
    }
    rafem_mesh* m = new rafem_mesh();
    static unsigned long long next_id = 1;
    m->ctx = ctx;
    m->id = next_id++;
    m->N = (int)n_nodes;
    m->M = (int)n_tets;
    m->nreg = n_regions;
    cudaError_t e;
#define RF_MS(x) do { e = (x); if (e != cudaSuccess) { rafem_mesh_destroy(m); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    const size_t N = std::max<int64_t>(n_nodes, 1), M = std::max<int64_t>(n_tets, 1);
    RF_MS(dmalloc(ctx, (void**)&m->nodes, sizeof(double) * 3 * N));
    RF_MS(dmalloc(ctx, (void**)&m->tets, sizeof(int) * 4 * M));
    RF_MS(dmalloc(ctx, (void**)&m->region, sizeof(int) * M));
    RF_MS(dmalloc(ctx, (void**)&m->regtab, sizeof(double) * 5 * n_regions));
    RF_MS(dmalloc(ctx, (void**)&m->kind, 2 * N));
    // every copy on the library stream (non-blocking: legacy-stream copies
    // are not ordered with it); the host vectors live until the sync below
    RF_MS(cudaMemcpyAsync(m->nodes, nodes, sizeof(double) * 3 * n_nodes, cudaMemcpyHostToDevice, ctx->stream));
    RF_MS(cudaMemcpyAsync(m->tets, t32.data(), sizeof(int) * 4 * n_tets, cudaMemcpyHostToDevice, ctx->stream));
    RF_MS(cudaMemcpyAsync(m->region, reg.data(), sizeof(int) * n_tets, cudaMemcpyHostToDevice, ctx->stream));
    RF_MS(cudaMemcpyAsync(m->regtab, tab.data(), sizeof(double) * 5 * n_regions, cudaMemcpyHostToDevice, ctx->stream));
    RF_MS(cudaMemcpyAsync(m->kind, dof_kind, 2 * n_nodes, cudaMemcpyHostToDevice, ctx->stream));
    RF_MS(cudaStreamSynchronize(ctx->stream));
#undef RF_MS
    if (int rc = mesh_symbolic(m)) {
        rafem_mesh_destroy(m);
        return rc;
    }
    if (int rc = mesh_geometry(m)) {
        rafem_mesh_destroy(m);
        return rc;
    }
    cudaError_t se = cudaStreamSynchronize(ctx->stream);
    if (se != cudaSuccess) {
        rafem_mesh_destroy(m);
        return rafem_fail_cuda(ctx, se, "mesh setup", __FILE__, __LINE__);
    }
    *out = m;
    return RAFEM_OK;
}

int rafem_mesh_set_geometry(rafem_mesh* m, const double* grad, const double* vol) {
    if (!m || !grad || !vol) return RAFEM_ERR_INVALID;
    return mesh_set_geometry(m, grad, vol);
}

void rafem_mesh_destroy(rafem_mesh* m) {
    if (!m) return;
    auto& pc = m->ctx->part_cache;  // partitions cached for this mesh's pattern
    for (size_t i = 0; i < pc.size();)
        if (pc[i].pattern_id == m->id) {
            dfree(m->ctx, pc[i].gpart);
            pc.erase(pc.begin() + i);
        } else {
            ++i;
        }
    for (void* p : {(void*)m->nodes, (void*)m->tets, (void*)m->region, (void*)m->regtab, (void*)m->kind,
                    (void*)m->rp, (void*)m->col, (void*)m->diag, (void*)m->inc_ptr, (void*)m->inc_ea,
                    (void*)m->inc_slot, (void*)m->base, (void*)m->grad, (void*)m->vol, (void*)m->slot_ptr,
                    (void*)m->slot_src, (void*)m->cls, (void*)m->cls_off, (void*)m->contrib_pos,
                    (void*)m->load_pos})
        if (p) dfree(m->ctx, p);
    delete m;
}

int64_t rafem_mesh_slots(const rafem_mesh* m) { return m ? m->slots : -1; }

int32_t rafem_mesh_stencil_classes(rafem_mesh* m) {
    if (!m) return -1;
    if (!m->cls_tried && mesh_stencil_classes(m) != RAFEM_OK) return -1;
    return m->ncls;
}

int rafem_mesh_set_shard_order(rafem_mesh* m, int64_t n_owned, int64_t n_below) {
    if (!m) return RAFEM_ERR_INVALID;
    if (n_owned < 0 || n_below < 0 || n_owned + n_below > m->N)
        return rafem_fail(m->ctx, RAFEM_ERR_INVALID, "shard order: owned + below-owner ghosts exceed the nodes");
    if (m->maxdeg > 32 && n_below > 0)
        return rafem_fail(m->ctx, RAFEM_ERR_UNSUPPORTED, "shard order: rows longer than 32 slots");
    m->own_end = (int)n_owned;
    m->below_end = (int)(n_owned + n_below);
    return RAFEM_OK;
}

int rafem_mesh_pattern(rafem_mesh* m, int64_t* node_row_ptr, int32_t* node_col) {
    if (!m) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = m->ctx;
    std::vector<int> rp(m->N + 1);
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(rp.data(), m->rp, sizeof(int) * (m->N + 1), cudaMemcpyDeviceToHost, ctx->stream));
    if (m->slots)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(node_col, m->col, sizeof(int) * m->slots, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i <= m->N; ++i) node_row_ptr[i] = rp[i];
    return RAFEM_OK;
}

int rafem_system_create(rafem_mesh* m, rafem_system** out) {
    if (!m || !out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    rafem_ctx* ctx = m->ctx;
    rafem_system* s = new rafem_system();
    s->mesh = m;
    const size_t N = std::max(m->N, 1), M = std::max(m->M, 1), S = std::max<long long>(m->slots, 1);
    cudaError_t e;
#define RF_SS(x) do { e = (x); if (e != cudaSuccess) { rafem_system_destroy(s); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    RF_SS(dmalloc(ctx, (void**)&s->val2, sizeof(double) * 2 * S));
    RF_SS(dmalloc(ctx, (void**)&s->rhs, sizeof(double) * 2 * N));
    // s->contrib / s->load (288 B per tet) only for the paths that stage
    // per-element outputs: system_contrib() allocates them on first use
    RF_SS(dmalloc(ctx, (void**)&s->diagpart, sizeof(double) * 2 * N));
    RF_SS(dmalloc(ctx, (void**)&s->minv, sizeof(double) * 2 * N));
    RF_SS(dmalloc(ctx, (void**)&s->xin, sizeof(double) * (3 * N + 2 * S)));  // host inputs / dof expansion
    RF_SS(dmalloc(ctx, (void**)&s->status, 1024));
    RF_SS(dmalloc(ctx, (void**)&s->xs, sizeof(double) * 6 * 2 * N));
    // on the library stream: ctx->stream is non-blocking, so a legacy-stream
    // cudaMemset could land after the first assembly's reset of the bad-element
    // flag (seen as a spurious PhysicsRangeError with two processes on a GPU)
    RF_SS(cudaMemsetAsync(s->status, 0, 1024, ctx->stream));
#undef RF_SS
    *out = s;
    return RAFEM_OK;
}

void rafem_system_destroy(rafem_system* s) {
    if (!s) return;
    if (s->kp) rafem_kp_destroy(s->kp);
    for (void* p : {(void*)s->val2, (void*)s->rhs, (void*)s->contrib, (void*)s->load, (void*)s->esig,
                    (void*)s->eload, (void*)s->diagpart,
                    (void*)s->minv, (void*)s->xin, (void*)s->status, (void*)s->xs})
        if (p) dfree(s->mesh->ctx, p);
    delete s;
}

int rafem_assemble(rafem_system* s, const double* t_iter, const double* v_iter, const double* t_prev,
                   const rafem_assemble_params* p, double* scale_out, int64_t* bad_element) {
    return rafem_assemble_rhs(s, t_iter, v_iter, t_prev, p, scale_out, bad_element, nullptr);
}

int rafem_assemble_rhs(rafem_system* s, const double* t_iter, const double* v_iter, const double* t_prev,
                       const rafem_assemble_params* p, double* scale_out, int64_t* bad_element, double* rhs_out) {
    if (!s || !p) return RAFEM_ERR_INVALID;
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    if (!(p->dt > 0.0)) return rafem_fail(ctx, RAFEM_ERR_INVALID, "dt must be positive");
    const int N = m->N;
    // pinned staging: [t_iter | v_iter | t_prev] in, [rhs (2N) | PassStatus] out
    const size_t in_b = sizeof(double) * 3 * (size_t)std::max(N, 1);
    const size_t rhs_b = sizeof(double) * 2 * (size_t)N;
    double* pin = static_cast<double*>(pinned(ctx, in_b + rhs_b + sizeof(PassStatus)));
    if (!pin) return rafem_fail(ctx, RAFEM_ERR_CUDA, "pinned staging allocation failed");
    std::memcpy(pin, t_iter, sizeof(double) * N);
    std::memcpy(pin + N, v_iter, sizeof(double) * N);
    std::memcpy(pin + 2 * (size_t)N, t_prev, sizeof(double) * N);
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(s->xin, pin, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
    SysStatus* ds = sys_status(s);
    if (int rc = assemble_launch(s, s->xin, 1, s->xin + N, 1, s->xin + 2 * (size_t)N, 1, *p, &ds->pass.scale,
                                 &ds->pass.bad_element))
        return rc;
    double* prhs = pin + in_b / sizeof(double);
    PassStatus* phs = reinterpret_cast<PassStatus*>(reinterpret_cast<char*>(pin) + in_b + rhs_b);
    if (rhs_out && N > 0) RF_CUDA_TRY(ctx, cudaMemcpyAsync(prhs, s->rhs, rhs_b, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(phs, &ds->pass, sizeof(PassStatus), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const PassStatus hs = *phs;
    if (rhs_out && N > 0) std::memcpy(rhs_out, prhs, rhs_b);
    s->scale = hs.scale;
    if (scale_out) *scale_out = hs.scale;
    if (bad_element) *bad_element = hs.bad_element;
    if (hs.bad_element >= 0) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "sigma(T) <= 0 in element %lld", hs.bad_element);
        return rafem_fail(ctx, RAFEM_ERR_PHYSICS, buf);
    }
    return RAFEM_OK;
}

int rafem_system_download(rafem_system* s, double* vals_out, double* rhs_out) {
    if (!s) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = s->mesh->ctx;
    const int N = s->mesh->N;
    if (vals_out && s->mesh->slots) {
        double* scratch = s->xin;  // 2*slots fits in xin (3N + 2S)
        if (int rc = expand_dof_vals(s, scratch)) return rc;
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(vals_out, scratch, sizeof(double) * 2 * s->mesh->slots, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (rhs_out) RF_CUDA_TRY(ctx, cudaMemcpyAsync(rhs_out, s->rhs, sizeof(double) * 2 * N, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

int rafem_system_solve(rafem_system* s, const double* b, const double* x0, const rafem_solver_params* p,
                       double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap, int64_t* cycle_lens,
                       int64_t cycle_cap) {
    if (!s) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = s->mesh->ctx;
    if (int rc = kp_system_solve(s, b, x0, p, x_out, st, hist, hist_cap, cycle_lens, cycle_cap);
        rc != RAFEM_ERR_UNSUPPORTED)
        return rc;
    const size_t n2 = 2 * (size_t)s->mesh->N;
    double* bdev = b ? s->xs + 4 * n2 : s->rhs;
    double* xdev = s->xs + 5 * n2;
    return solve_common(ctx, system_view(s), bdev, b != nullptr, b, x0, p, x_out, st, hist, hist_cap, cycle_lens,
                        cycle_cap, s->minv, xdev, sys_status(s));
}

int rafem_system_spmv(rafem_system* s, const double* x, double* y) {
    if (!s) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = s->mesh->ctx;
    const size_t n2 = 2 * (size_t)s->mesh->N;
    double* dx = s->xs + 4 * n2;
    double* dy = s->xs + 5 * n2;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(dx, x, sizeof(double) * n2, cudaMemcpyHostToDevice, ctx->stream));
    if (int rc = spmv_launch(ctx, system_view(s), dx, dy)) return rc;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(y, dy, sizeof(double) * n2, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

int rafem_system_spmv_bench(rafem_system* s, int32_t reps, int32_t flush_l2, double* ms_per_launch) {
    if (!s || reps < 1) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = s->mesh->ctx;
    const size_t n2 = 2 * (size_t)s->mesh->N;
    double* dx = s->xs + 4 * n2;
    double* dy = s->xs + 5 * n2;
    if (int rc = fill_initial(ctx, dx, s->mesh->N, 1.25)) return rc;
    const MatView A = system_view(s);
    if (int rc = spmv_launch(ctx, A, dx, dy)) return rc;  // warm-up
    if (!flush_l2) {
        // back to back: each launch may stream its first matrix tiles while
        // the previous one drains (programmatic dependent launch; the matrix
        // is constant here, x and y are touched only after the dependency
        // wait).  RAFEM_NO_PDL=1: plain stream order.
        const char* np = getenv("RAFEM_NO_PDL");
        ctx->spmv_pdl = !(np && np[0] == '1');
        RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
        for (int r = 0; r < reps; ++r)
            if (int rc = spmv_launch(ctx, A, dx, dy)) {
                ctx->spmv_pdl = false;
                return rc;
            }
        ctx->spmv_pdl = false;
        RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
        RF_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        RF_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *ms_per_launch = ms / reps;
        return RAFEM_OK;
    }
    // cold L2: a 256 MB write between launches, each launch timed alone
    void* flush = nullptr;
    const size_t fb = 256u << 20;
    RF_CUDA_TRY(ctx, cudaMalloc(&flush, fb));
    double total = 0.0;
    for (int r = 0; r < reps; ++r) {
        RF_CUDA_TRY(ctx, cudaMemsetAsync(flush, r & 0xff, fb, ctx->stream));
        RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
        if (int rc = spmv_launch(ctx, A, dx, dy)) {
            cudaFree(flush);
            return rc;
        }
        RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
        RF_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        RF_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        total += ms;
    }
    cudaFree(flush);
    *ms_per_launch = total / reps;
    return RAFEM_OK;
}

// ---- native time loop -------------------------------------------------------
// run_simulation (fem.py:554-644) + corrector_step (fem.py:463-540) with all
// vectors resident in HBM; the host only reads a 96-byte PassStatus per
// corrector pass to take the same control decisions the reference takes.

namespace {

// SimulationSummary from the fused kernel's device summary; maps the run's
// status onto the error taxonomy
int fused_summary(rafem_ctx* ctx, const SimDevOut& so, std::chrono::steady_clock::time_point t_wall,
                  rafem_sim_summary* out) {
    out->accepted_steps = so.accepted;
    out->total_corrector_iters = so.corr;
    out->total_solver_iterations = so.inner;
    out->dt_halvings = so.halvings;
    out->passes = so.passes;
    out->final_time = so.t;
    out->status = so.status;
    out->failed_step = so.failed_step;
    out->failed_dt = so.failed_dt;
    out->bad_element = so.bad;
    out->assemble_ms = so.asm_ns * 1e-6;
    out->solve_ms = so.solve_ns * 1e-6;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall).count();
    if (so.status == RAFEM_ERR_PHYSICS) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "sigma(T) <= 0 in element %lld", (long long)so.bad);
        return rafem_fail(ctx, so.status, buf);
    }
    if (so.status == RAFEM_ERR_STEP_FAILURE) {
        char buf[160];
        std::snprintf(buf, sizeof(buf), "step %d failed to converge with dt already at the floor (%g s)",
                      so.failed_step, so.failed_dt);
        return rafem_fail(ctx, so.status, buf);
    }
    if (so.status == RAFEM_ERR_INVALID)
        return rafem_fail(ctx, so.status, "Jacobi preconditioning requires a zero-free diagonal");
    return so.status;
}

int check_sim(rafem_ctx* ctx, const rafem_sim_params* p) {
    if (int rc = check_params(ctx, &p->solver)) return rc;
    if (!(p->total_time > 0.0) || !(p->dt_min > 0.0 && p->dt_min <= p->dt_init && p->dt_init <= p->dt_max) ||
        !(p->corrector_tol > 0.0) || p->max_corrector_iters < 1)
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "invalid SimConfig");
    return RAFEM_OK;
}

// host side of the record stream: copy each published record out of the
// device ring on a side stream while the simulation kernel keeps running
struct StreamPump {
    rafem_ctx* ctx;
    cudaStream_t copy;
    const double* ring;  // device
    int slots;
    size_t rec_doubles;  // 2N + 4
    volatile long long* prog;  // host view
    volatile long long* cons;
    double* hbuf;        // pinned, one record
    rafem_record_fn fn;
    void* user;
    int cb_status;
    long long consumed;
};

int pump_records(void* u) {
    StreamPump& P = *static_cast<StreamPump*>(u);
    const long long n2 = (long long)P.rec_doubles - 4;
    while (true) {
        const bool kernel_done = cudaStreamQuery(P.ctx->stream) != cudaErrorNotReady;
        const long long produced = *P.prog;
        if (P.consumed >= produced) {
            if (kernel_done) break;
            std::this_thread::sleep_for(std::chrono::microseconds(20));
            continue;
        }
        while (P.consumed < produced) {
            const double* slot = P.ring + (P.consumed % P.slots) * P.rec_doubles;
            RF_CUDA_TRY(P.ctx, cudaMemcpyAsync(P.hbuf, slot, sizeof(double) * P.rec_doubles, cudaMemcpyDeviceToHost,
                                               P.copy));
            RF_CUDA_TRY(P.ctx, cudaStreamSynchronize(P.copy));
            if (P.cb_status == 0 && P.fn)
                P.cb_status = P.fn(P.user, P.consumed, P.hbuf[0], P.hbuf[1], (int32_t)P.hbuf[2], P.hbuf + 4);
            ++P.consumed;
            *P.cons = P.cb_status ? (1LL << 60) : P.consumed;  // a failed sink releases the kernel
        }
        (void)n2;
    }
    return RAFEM_OK;
}


// rafem_simulate's record sink: the first rec_cap steps into the caller's arrays
struct RecordArrays {
    long long cap;
    int64_t* step;
    double* time;
    double* dt;
    int32_t* iters;
    double* x;
    size_t n2;
    cudaStream_t st;
};

int record_to_arrays(void* u, long long step, double t, double dt, int iters, const double* xacc) {
    auto& R = *static_cast<RecordArrays*>(u);
    if (step >= R.cap) return 0;
    if (R.step) R.step[step] = step;
    if (R.time) R.time[step] = t;
    if (R.dt) R.dt[step] = dt;
    if (R.iters) R.iters[step] = iters;
    if (R.x) {
        const cudaError_t e = cudaMemcpyAsync(R.x + (size_t)step * R.n2, xacc, sizeof(double) * R.n2,
                                              cudaMemcpyDeviceToHost, R.st);
        if (e != cudaSuccess) return RAFEM_ERR_CUDA;
    }
    return 0;
}

// rafem_simulate_stream's sink on the per-pass loop: each accepted state
// through one pinned record buffer straight to the caller's fn
struct RecordStream {
    rafem_ctx* ctx;
    double* hbuf;  // pinned, 2N
    size_t n2;
    rafem_record_fn fn;
    void* user;
};

int record_to_stream(void* u, long long step, double t, double dt, int iters, const double* xacc) {
    auto& R = *static_cast<RecordStream*>(u);
    if (cudaMemcpyAsync(R.hbuf, xacc, sizeof(double) * R.n2, cudaMemcpyDeviceToHost, R.ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(R.ctx->stream) != cudaSuccess)
        return RAFEM_ERR_CUDA;
    return R.fn ? (R.fn(R.user, step, t, dt, (int32_t)iters, R.hbuf) ? 1 : 0) : 0;
}

// Per-pass native loop (the fallback when the fused kernel does not apply,
// e.g. GMRES): every accepted step's device state xacc (2N dofs) is handed
// to fn as it is accepted — a record costs 2N doubles of host memory only
// for as long as fn holds it.  fn returns 0, a CUDA status (< 0, aborts)
// or > 0 (the sink refused: delivery stops, the run completes, the call
// returns RAFEM_ERR_INVALID).
using AcceptFn = int (*)(void* u, long long step, double t, double dt, int iters, const double* xacc_dev);

int simulate_host_loop(rafem_system* s, const rafem_sim_params* p, rafem_sim_summary* out,
                       std::chrono::steady_clock::time_point t_wall, AcceptFn fn, void* u) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    const int N = m->N;
    const size_t n2 = 2 * (size_t)N;
    cudaStream_t st = ctx->stream;
    double* xacc = s->xs;            // accepted (V, T)
    double* xprev = s->xs + n2;      // accepted one step earlier
    double* xit = s->xs + 2 * n2;    // current iterate (x_old)
    double* xnew = s->xs + 3 * n2;   // solve output
    if (int rc = fill_initial(ctx, xacc, N, p->initial_temp)) return rc;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(xprev, xacc, sizeof(double) * n2, cudaMemcpyDeviceToDevice, st));
    SysStatus* ds = sys_status(s);
    const MatView A = system_view(s);
    const bool pre = p->solver.precondition != RAFEM_PRECOND_NONE;
    rafem_assemble_params ap{};
    ap.applied_voltage = p->applied_voltage;
    ap.boundary_temp = p->boundary_temp;
    ap.apply_constraints = 1;
    ap.equilibrate = 1;

    bool rec_failed = false;
    double t = 0.0, dt_state = p->dt_init, dt_prev = p->dt_init;
    long long step = 0, passes = 0, total_corr = 0, total_inner = 0, halvings = 0;
    double asm_ms = 0.0, sol_ms = 0.0;
    int status = RAFEM_OK;
    while (t < p->total_time) {
        if (p->max_steps > 0 && step >= p->max_steps) break;
        const double remaining = p->total_time - t;
        const bool final_step = dt_state >= remaining;
        const double dt = final_step ? remaining : dt_state;
        // PCG: the first pass's solver starts from V extrapolated in time as
        // well (same system and delta reference; simulate_dev.cuh)
        const char* nv = getenv("RAFEM_NO_VX0");
        const bool vx0 = p->solver.method == RAFEM_METHOD_PCG && !(nv && nv[0] == '1');
        if (int rc = predictor_launch(ctx, xit, xacc, xprev, N, (int)step, dt / dt_prev, vx0 ? xnew : nullptr))
            return rc;
        bool converged = false;
        int iters = 0;
        for (int it = 1; it <= p->max_corrector_iters; ++it) {
            iters = it;
            ++passes;
            ap.dt = dt;
            RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
            if (int rc = assemble_launch(s, xit + 1, 2, xit, 2, xacc + 1, 2, ap, &ds->pass.scale, &ds->pass.bad_element))
                return rc;
            if (pre) {
                if (int rc = jacobi_minv(ctx, A, s->minv, &ds->flag)) return rc;
            } else {
                RF_CUDA_TRY(ctx, cudaMemsetAsync(&ds->flag, 0, sizeof(int), st));
            }
            if (int rc = krylov_solve(ctx, A, s->rhs, (vx0 && it == 1) ? xnew : xit, xnew, s->minv, p->solver,
                                      &ds->pass.solve, &ds->flag, ctx->ev1, ctx->ev2))
                return rc;
            if (int rc = vec_delta_launch(ctx, xnew, xit, (int)n2, &ds->pass.delta)) return rc;
            PassStatus hs;
            RF_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, &ds->pass, sizeof(hs), cudaMemcpyDeviceToHost, st));
            RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
            float a_ms = 0.f, s_ms = 0.f;
            cudaEventElapsedTime(&a_ms, ctx->ev0, ctx->ev1);
            cudaEventElapsedTime(&s_ms, ctx->ev1, ctx->ev2);
            asm_ms += a_ms;
            sol_ms += s_ms;
            if (hs.bad_element >= 0) {  // PhysicsRangeError aborts the run (fem.py:274)
                out->bad_element = hs.bad_element;
                status = RAFEM_ERR_PHYSICS;
                break;
            }
            if (hs.solve.status == RAFEM_ERR_INVALID) {  // ValueError aborts the run
                status = RAFEM_ERR_INVALID;
                ctx->err = "Jacobi preconditioning requires a zero-free diagonal";
                break;
            }
            if (hs.solve.status == RAFEM_ERR_BREAKDOWN) break;  // SolverError -> step failure (fem.py:511-515)
            total_inner += hs.solve.iterations;
            if (!hs.solve.converged) break;                   // fem.py:517-524
            std::swap(xit, xnew);                              // x_old = x_new (fem.py:529-530)
            if (hs.delta < p->corrector_tol) {
                converged = true;
                break;
            }
        }
        if (status != RAFEM_OK) break;
        total_corr += iters;
        if (converged) {
            // rotate: prev <- acc <- iterate   (fem.py:604-607)
            double* old_prev = xprev;
            xprev = xacc;
            xacc = xit;
            xit = old_prev;
            dt_prev = dt;
            t = final_step ? p->total_time : t + dt;
            if (fn && !rec_failed)
                if (int rc = fn(u, step, t, dt, iters, xacc)) {
                    if (rc < 0) return rc;  // CUDA error while handing the record over
                    rec_failed = true;      // the sink refused: stop delivering, finish the run
                }
            ++step;
            if (iters <= 5)
                dt_state = std::min(dt * 1.5, p->dt_max);
            else if (iters >= 20)
                dt_state = std::max(dt * 0.75, p->dt_min);
            else
                dt_state = dt;
        } else {
            if (dt <= p->dt_min) {  // StepFailureError (fem.py:629-631)
                status = RAFEM_ERR_STEP_FAILURE;
                out->failed_step = (int)step;
                out->failed_dt = dt;
                break;
            }
            dt_state = std::max(dt * 0.5, p->dt_min);
            ++halvings;
        }
    }
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    // keep the final accepted state at the front of xs for callers
    if (xacc != s->xs) {
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(s->xs, xacc, sizeof(double) * n2, cudaMemcpyDeviceToDevice, st));
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    }
    out->accepted_steps = step;
    out->total_corrector_iters = total_corr;
    out->total_solver_iterations = total_inner;
    out->dt_halvings = halvings;
    out->passes = passes;
    out->final_time = t;
    out->status = status;
    out->assemble_ms = asm_ms;
    out->solve_ms = sol_ms;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall).count();
    if (status == RAFEM_ERR_PHYSICS) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "sigma(T) <= 0 in element %lld", (long long)out->bad_element);
        return rafem_fail(ctx, status, buf);
    }
    if (status == RAFEM_ERR_STEP_FAILURE) {
        char buf[160];
        std::snprintf(buf, sizeof(buf), "step %d failed to converge with dt already at the floor (%g s)",
                      out->failed_step, out->failed_dt);
        return rafem_fail(ctx, status, buf);
    }
    if (status == RAFEM_OK && rec_failed) return rafem_fail(ctx, RAFEM_ERR_INVALID, "record sink failed");
    return status;
}

}  // namespace

int rafem_simulate_stream(rafem_system* s, const rafem_sim_params* p, rafem_sim_summary* out, int32_t ring_slots,
                          rafem_record_fn fn, void* user) {
    if (!s || !p || !out || ring_slots < 1) return RAFEM_ERR_INVALID;
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    std::memset(out, 0, sizeof(*out));
    out->failed_step = -1;
    out->bad_element = -1;
    if (int rc = check_sim(ctx, p)) return rc;
    const auto t_wall = std::chrono::steady_clock::now();
    const size_t n2 = 2 * (size_t)m->N;
    const char* nofused = getenv("RAFEM_NO_FUSED");
    if (p->solver.method == RAFEM_METHOD_PCG && !(nofused && nofused[0] == '1')) {
        StreamPump P{};
        P.ctx = ctx;
        P.slots = ring_slots;
        P.rec_doubles = n2 + 4;
        P.fn = fn;
        P.user = user;
        double* ring = nullptr;
        long long* dcounters = nullptr;
        auto cleanup = [&]() {
            if (ring) dfree(ctx, ring);
        };
        // ring from the context cache; side stream, mapped counters and the
        // pinned record buffer are created once per context
        cudaError_t e = dmalloc(ctx, reinterpret_cast<void**>(&ring), sizeof(double) * P.rec_doubles * ring_slots);
        if (e == cudaSuccess && !ctx->mapped)
            e = cudaHostAlloc(reinterpret_cast<void**>(&ctx->mapped), 2 * sizeof(long long), cudaHostAllocMapped);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dcounters), ctx->mapped, 0);
        if (e == cudaSuccess && !ctx->side_stream) e = cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking);
        P.hbuf = e == cudaSuccess ? static_cast<double*>(pinned(ctx, sizeof(double) * P.rec_doubles)) : nullptr;
        if (e == cudaSuccess && !P.hbuf) e = cudaErrorMemoryAllocation;
        if (e != cudaSuccess) {
            cleanup();
            return rafem_fail_cuda(ctx, e, "record stream setup", __FILE__, __LINE__);
        }
        long long* counters = ctx->mapped;
        P.copy = ctx->side_stream;
        counters[0] = 0;
        counters[1] = 0;
        P.ring = ring;
        P.prog = counters;
        P.cons = counters + 1;
        SimStream ss{ring, ring_slots, dcounters, dcounters + 1, pump_records, &P};
        SimDevOut so{};
        float kms = 0.f;
        const int frc = simulate_fused(s, p, &so, nullptr, nullptr, nullptr, nullptr, 0, s->xs + 5 * n2, &kms, &ss);
        if (frc == RAFEM_OK && P.consumed < so.accepted) pump_records(&P);  // drain (kernel is done)
        const int cb = P.cb_status;
        cleanup();
        if (frc == RAFEM_OK) {
            const int rc = fused_summary(ctx, so, t_wall, out);
            if (cb) return rafem_fail(ctx, RAFEM_ERR_INVALID, "record sink failed");
            return rc;
        }
        if (frc != RAFEM_ERR_UNSUPPORTED) return frc;
    }
    // not eligible for the fused kernel: the per-pass loop hands each
    // accepted step to fn as it is accepted (bounded memory at any size)
    RecordStream rs{ctx, static_cast<double*>(pinned(ctx, sizeof(double) * n2)), n2, fn, user};
    if (!rs.hbuf) return rafem_fail(ctx, RAFEM_ERR_CUDA, "pinned record buffer");
    return simulate_host_loop(s, p, out, t_wall, record_to_stream, &rs);
}

int rafem_simulate(rafem_system* s, const rafem_sim_params* p, rafem_sim_summary* out, int64_t rec_cap,
                   int64_t* rec_step, double* rec_time, double* rec_dt, int32_t* rec_iters, double* rec_x) {
    if (!s || !p || !out) return RAFEM_ERR_INVALID;
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    std::memset(out, 0, sizeof(*out));
    out->failed_step = -1;
    out->bad_element = -1;
    if (int rc = check_sim(ctx, p)) return rc;
    const auto t_wall = std::chrono::steady_clock::now();
    const int N = m->N;
    const size_t n2 = 2 * (size_t)N;
    cudaStream_t st = ctx->stream;

    // Preferred path: the whole simulation in one persistent kernel (PCG).
    const char* nofused = getenv("RAFEM_NO_FUSED");
    if (p->solver.method == RAFEM_METHOD_PCG && !(nofused && nofused[0] == '1')) {
        const long long cap = std::max<long long>(rec_cap, 0);
        double* d_rx = nullptr;
        double* d_rt = nullptr;
        double* d_rd = nullptr;
        int* d_ri = nullptr;
        // record buffers from the context's allocation cache: the field buffer
        // is sized for the caller's capacity (hundreds of MB for a 900 s run),
        // and a cudaMalloc / cudaFree pair of that size per call cost more
        // than the simulation itself (45 vs 26 ms per mesh-B run)
        auto release = [&]() {
            for (void* q : {(void*)d_rx, (void*)d_rt, (void*)d_rd, (void*)d_ri})
                if (q) dfree(ctx, q);
        };
        if (cap > 0) {
            RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&d_rt), sizeof(double) * cap));
            RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&d_rd), sizeof(double) * cap));
            RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&d_ri), sizeof(int) * cap));
            if (p->record_fields && rec_x)
                RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&d_rx), sizeof(double) * n2 * cap));
        }
        SimDevOut so{};
        float kms = 0.f;
        const int frc = simulate_fused(s, p, &so, d_rx, d_rt, d_rd, d_ri, cap, s->xs + 5 * n2, &kms);
        if (frc == RAFEM_OK) {
            const long long nrec = std::min<long long>(so.accepted, cap);
            if (nrec > 0) {
                std::vector<double> ht(nrec), hd(nrec);
                std::vector<int> hi(nrec);
                RF_CUDA_TRY(ctx, cudaMemcpyAsync(ht.data(), d_rt, sizeof(double) * nrec, cudaMemcpyDeviceToHost, ctx->stream));
                RF_CUDA_TRY(ctx, cudaMemcpyAsync(hd.data(), d_rd, sizeof(double) * nrec, cudaMemcpyDeviceToHost, ctx->stream));
                RF_CUDA_TRY(ctx, cudaMemcpyAsync(hi.data(), d_ri, sizeof(int) * nrec, cudaMemcpyDeviceToHost, ctx->stream));
                RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
                for (long long k = 0; k < nrec; ++k) {
                    if (rec_step) rec_step[k] = k;
                    if (rec_time) rec_time[k] = ht[k];
                    if (rec_dt) rec_dt[k] = hd[k];
                    if (rec_iters) rec_iters[k] = hi[k];
                }
                if (d_rx) {
                    RF_CUDA_TRY(ctx, cudaMemcpyAsync(rec_x, d_rx, sizeof(double) * n2 * nrec, cudaMemcpyDeviceToHost,
                                                     ctx->stream));
                    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
                }
            }
            release();
            return fused_summary(ctx, so, t_wall, out);
        }
        release();
        if (frc != RAFEM_ERR_UNSUPPORTED) return frc;
    }
    RecordArrays ra{rec_cap, rec_step, rec_time, rec_dt, rec_iters, p->record_fields ? rec_x : nullptr, n2, st};
    return simulate_host_loop(s, p, out, t_wall, record_to_arrays, &ra);
}

}  // extern "C"
