// internal.hpp — host-side structures shared by the librafem_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/rafem_b200.h"

namespace rafem {

// Result block a Krylov kernel leaves in device memory (read back by the
// host API, or inspected on device by the native time loop).
struct KResult {
    long long iterations;
    long long restarts;
    long long cycles;
    long long hist_len;
    double final_rel;
    int converged;
    int stagnated;
    int status;  // RAFEM_OK / RAFEM_ERR_BREAKDOWN / RAFEM_ERR_INVALID
    int pad;
};

// Per-pass status the native loop reads back (one small D2H per pass).
struct PassStatus {
    KResult solve;
    double delta;          // corrector delta max|dx|/max(1,|x_old|)
    long long bad_element; // PhysicsRangeError element or -1
    double scale;          // voltage_row_scale of the pass
};

// Summary the fused simulation kernel leaves in device memory.
struct SimDevOut {
    long long accepted, corr, inner, halvings, passes;
    double t;
    int status, failed_step;
    double failed_dt;
    long long bad;
    long long asm_ns, solve_ns;
};

// Matrix view consumed by the Krylov and SpMV kernels.  W = dofs per row
// group: 1 for a general CSR (one row per group), 2 for the FEM node
// pattern (rows 2i and 2i+1 share node i's columns; one double2 per slot).
struct MatView {
    const int* rp;      // ngroups + 1
    const int* col;     // slots, GROUP (node) indices
    const double* val;  // W doubles per slot
    int ngroups;
    int W;
    long long slots;
    unsigned long long pattern_id = 0;  // nonzero: partitions may be cached
    int maxdeg = 0;                     // max slots per row group (0: unknown)
    // stencil classes (structured meshes): column k of row g is
    // g + cls_off[cls[g] * kClsWidth + k]; null = explicit columns only
    const uint8_t* cls = nullptr;
    const int* cls_off = nullptr;
    int ncls = 0;
    const double* coords = nullptr;  // N x 3 node coordinates (device) when the pattern is a mesh's
};
constexpr int kClsWidth = 16;   // max row length of a stencil class
constexpr int kMaxClasses = 255;

struct PartCacheEntry {
    unsigned long long pattern_id;
    const int* rp;
    int G;
    int* gpart;
    size_t max_slice;
    int max_groups;
    bool by_rows;
};

// Growable device scratch owned by a context.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace rafem

struct rafem_ctx {
    int device = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
    long long total_mem = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    std::string err;
    long long launches = 0;
    // solver workspace (grown on demand)
    rafem::DevBuf ws_basis, ws_vec, ws_partial, ws_hess, ws_hist, ws_cyc, ws_part, ws_res;
    // host pinned staging
    void* pin = nullptr;
    size_t pin_bytes = 0;
    std::vector<rafem::PartCacheEntry> part_cache;
    int trace_on = 0;
    rafem::DevBuf ws_trace;
    rafem::DevBuf ws_flags;     // grid barrier / all-reduce slots
    rafem::DevBuf ws_simout;    // fused simulation summary
    rafem::DevBuf ws_diag;      // diagonal-sum partials of the assembly
    rafem::DevBuf ws_gal;       // fused simulation: Galerkin-start ring of solution increments
    unsigned epoch = 0;         // per-launch flag epoch
    // device blocks of destroyed meshes / systems kept for reuse (a new mesh
    // of the same size then costs no cudaMalloc / cudaFree, which synchronise)
    std::multimap<size_t, void*> free_blocks;
    std::unordered_set<void*> free_set;  // blocks in free_blocks (a second dfree of one is ignored)
    long long double_frees = 0;
    std::unordered_map<void*, size_t> block_size;
    size_t cached_bytes = 0;
    cudaStream_t side_stream = nullptr;  // record copies of rafem_simulate_stream
    long long* mapped = nullptr;         // 2 mapped host counters (record stream)
    int last_mode = -1;  // 1: cluster-resident solve, 0: grid-wide cooperative solve
    int last_ctas = 0;
    int last_precond = -1;  // preconditioner the last solve applied (RAFEM_PRECOND_*)
    int last_team = 0;
    bool spmv_pdl = false;
    std::vector<void*> cluster_plans;  // cluster.cu plans (ClusterPlan*), released with the context  // streaming SpMV launched with programmatic dependent launch (back-to-back bench)
};

struct rafem_matrix {
    rafem_ctx* ctx = nullptr;
    int n = 0;
    long long nnz = 0;
    int* rp = nullptr;
    int* col = nullptr;
    double* val = nullptr;
    double* minv = nullptr;
};

struct rafem_mesh {
    rafem_ctx* ctx = nullptr;
    int N = 0, M = 0;
    long long slots = 0;
    int maxdeg = 0;     // max slots per node row
    int maxinc = 0;     // max incident tets per node
    unsigned long long id = 0;  // unique per mesh (partition cache key)
    // inputs
    double* nodes = nullptr;  // N x 3
    int* tets = nullptr;      // M x 4
    int* region = nullptr;    // M
    int nreg = 0;
    double* regtab = nullptr; // 5 x nreg: k, rho_c, sigma0, alpha, t_ref
    uint8_t* kind = nullptr;  // 2N dof kinds
    // symbolic pattern
    int* rp = nullptr;        // N + 1
    int* col = nullptr;       // slots
    int* diag = nullptr;      // N: slot offset of the diagonal within its row
    // shard meshes: local ids [own_end, below_end) are ghosts whose global
    // ids precede the owned block; the constraint sums walk each row in
    // global column order (below ghosts, owned, the rest).  -1: natural order
    int own_end = -1, below_end = -1;
    int* inc_ptr = nullptr;   // N + 1
    unsigned* inc_ea = nullptr;   // 4M: tet | (local index << 30)
    unsigned* inc_slot = nullptr; // 4M: 4 x uint8 row offsets of the tet's nodes
    int* slot_ptr = nullptr;  // slots + 1: per-slot contributor lists
    int* slot_src = nullptr;  // 16M: contribution index 16 e + 4 a + b (ascending e per slot)
    bool slot_lists_tried = false;
    int* contrib_pos = nullptr;  // 16M: list position (slot_src order) of contribution 16 e + 4 a + b
    int* load_pos = nullptr;     // 4M: list position (inc_ea order) of load 4 e + a
    uint8_t* cls = nullptr;   // N stencil class per node row (null: none)
    int* cls_off = nullptr;   // ncls x kClsWidth column offsets
    int ncls = 0;
    bool cls_tried = false;
    // geometry (constant per mesh)
    double* base = nullptr;   // M x 10: vol * grad_a . grad_b, symmetric packed
    double* grad = nullptr;   // M x 12
    double* vol = nullptr;    // M
};

struct rafem_system {
    rafem_mesh* mesh = nullptr;
    double* val2 = nullptr;   // slots x 2 (V, T)
    double* rhs = nullptr;    // 2N
    double* contrib = nullptr; // M x 16 x (V, T) element block contributions
    double* load = nullptr;   // M x 4 T-rhs element contributions
    double* esig = nullptr;   // M: sigma(Tbar) per element (fused fill)
    double* eload = nullptr;  // M x 4: T-rhs loads per element (fused fill)
    double* diagpart = nullptr; // 2 x G partial diag sums
    double* minv = nullptr;   // 2N
    double* xin = nullptr;    // 3N staging for host inputs / 2N iterate buffers
    double* status = nullptr; // device PassStatus + scratch
    double scale = 1.0;
    // native-loop state
    double* xs = nullptr;     // 5 x 2N dof vectors
    rafem_kp* kp = nullptr;   // kernel-per-phase PCG for very large systems (shard.cu)
};

// error helpers (capi.cu)
int rafem_fail(rafem_ctx* ctx, int code, const std::string& msg);
int rafem_fail_cuda(rafem_ctx* ctx, cudaError_t e, const char* what, const char* file, int line);

namespace rafem {

// krylov.cu
int krylov_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, const double* x0_dev,
                 double* x_dev, const double* minv_dev, const rafem_solver_params& p,
                 KResult* res_dev, int* flag_dev, cudaEvent_t ev_start = nullptr,
                 cudaEvent_t ev_stop = nullptr);
int jacobi_minv(rafem_ctx* ctx, const MatView& A, double* minv_dev, int* flag_dev);
// Record streaming of the fused simulation: the kernel fills a device ring
// and publishes progress in mapped host memory; `pump` (host) runs right
// after the launch, consuming records until the kernel is done.
struct SimStream {
    double* ring;
    int slots;
    volatile long long* prog;  // device view of the mapped counters
    volatile long long* cons;
    int (*pump)(void* user);
    void* user;
};
// fused device-resident simulation (krylov.cu + simulate_dev.cuh); returns
// RAFEM_ERR_UNSUPPORTED when the system is not eligible (caller falls back)
int simulate_fused(rafem_system* s, const rafem_sim_params* p, SimDevOut* out, double* rec_x_dev,
                   double* rec_time_dev, double* rec_dt_dev, int* rec_iters_dev, long long rec_cap,
                   double* final_x_dev, float* ms, const SimStream* stream = nullptr);
// cluster.cu: cluster-resident PCG for paper-scale node-paired systems;
// RAFEM_ERR_UNSUPPORTED when the system is not eligible
int cluster_pcg_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, double* x_dev, const double* minv_dev,
                      const rafem_solver_params& p, KResult* res_dev, int* flag_dev, cudaEvent_t ev_start,
                      cudaEvent_t ev_stop);
void cluster_plans_release(rafem_ctx* ctx);
// cluster.cu: the whole simulation on one thread-block cluster (same contract
// as simulate_fused); RAFEM_ERR_UNSUPPORTED when not eligible
struct SimStream;
int simulate_cluster(rafem_system* s, const rafem_sim_params* p, SimDevOut* out, double* rec_x_dev,
                     double* rec_time_dev, double* rec_dt_dev, int* rec_iters_dev, long long rec_cap,
                     double* final_x_dev, float* ms, const SimStream* stream);
int krylov_read_history(rafem_ctx* ctx, const KResult& r, double* hist, long long hist_cap,
                        long long* cyc, long long cyc_cap);
int spmv_launch(rafem_ctx* ctx, const MatView& A, const double* x_dev, double* y_dev);
int vec_delta_launch(rafem_ctx* ctx, const double* xn, const double* xo, int n, double* out_dev);

// assembly.cu
int mesh_symbolic(rafem_mesh* m);
int mesh_geometry(rafem_mesh* m);
int mesh_set_geometry(rafem_mesh* m, const double* grad, const double* vol);  // host geometry (exact mode)
int mesh_slot_lists(rafem_mesh* m);  // per-slot contributor lists (built on first use)
int mesh_slot_positions(rafem_mesh* m);  // their inverse maps (fused simulation, built on first use)
// stencil classes of the node pattern (built on first use; none when the
// rows have more than kMaxClasses distinct offset signatures)
int mesh_stencil_classes(rafem_mesh* m);
int assemble_launch(rafem_system* s, const double* t_it, int ts, const double* v_it, int vs,
                    const double* t_prev, int ps, const rafem_assemble_params& p,
                    double* scale_dev, long long* bad_dev);
// shard.cu: single-shard kernel-per-phase PCG on an assembled system;
// RAFEM_ERR_UNSUPPORTED when the system is not eligible
int kp_system_solve(rafem_system* s, const double* b, const double* x0, const rafem_solver_params* p,
                    double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap, int64_t* cycle_lens,
                    int64_t cycle_cap);
int assemble_fill_launch(rafem_system* s, const double* t_it, int ts, const double* v_it, int vs,
                         const double* t_prev, int ps, double dt, long long* bad_dev);
int assemble_constrain_launch(rafem_system* s, const rafem_assemble_params& p, double scale);
// (sum of V, sum of T) raw diagonal entries of the first n node rows, two
// deterministic stages; sums_dev (2 doubles) and/or the equilibration scale
int diag_sums_launch(rafem_ctx* ctx, const double* diag_raw, int n, int equilibrate, double* sums_dev,
                     double* scale_dev);
int expand_dof_vals(rafem_system* s, double* out_dev);
// per-element contribution / load buffers of a system, allocated on first use
int system_contrib(rafem_system* s);
// per-element scalars of the fused fill (sigma, 4 loads), allocated on first use
int system_escal(rafem_system* s);
int predictor_launch(rafem_ctx* ctx, double* x_it, const double* x_acc, const double* x_prev,
                     int N, int step, double ratio,
                     double* x_start = nullptr);
int fill_initial(rafem_ctx* ctx, double* x, int N, double t0);
struct AsmMesh;
AsmMesh asm_mesh(const rafem_mesh* m);

// sparse.cu
int scan_ints(rafem_ctx* ctx, const int* in, int* out, int n);
int coo_to_csr_device(rafem_ctx* ctx, long long nrows, long long ncols, long long nnz,
                      const int64_t* rows, const int64_t* cols, const double* vals,
                      int64_t* row_ptr_out, int64_t* col_idx_out, double* vals_out,
                      int64_t* nnz_out);

// grow a device buffer to at least `bytes`
int ensure(rafem_ctx* ctx, DevBuf& b, size_t bytes);
// context-cached device allocation for mesh / system arrays (stream-ordered
// reuse on the context stream); dfree returns the block to the cache
cudaError_t dmalloc(rafem_ctx* ctx, void** p, size_t bytes);
void dfree(rafem_ctx* ctx, void* p);
void dcache_release(rafem_ctx* ctx);
void* pinned(rafem_ctx* ctx, size_t bytes);

}  // namespace rafem
