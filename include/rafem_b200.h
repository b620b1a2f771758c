/*
 * rafem_b200.h — C ABI of the B200-native RAFEM hot path (librafem_b200.so).
 *
 * The reference (rafem 0.1.0, /root/reference/pkg/src/rafem) is pure
 * Python; its plugin seam is two module globals that corrector_step
 * calls (fem.py:47-48, 492, 501):
 *
 *     assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt,
 *                     apply_constraints=True, equilibrate=True, threads=None)
 *                                                       (fem.py:325-336)
 *     solve(a, b, x0=None, config=None, session=None, tracer=None,
 *           trace_step=-1, trace_corrector_iter=-1)     (solver.py:580-589)
 *
 * plus the sparse kernels they rest on, spmv (sparse.py:205-219) and
 * coo_to_csr (sparse.py:164-197).  These entry points are what a ctypes
 * binding of that seam needs (see INTEGRATION.md for the binding).
 * All pointers are HOST pointers unless a name ends in _dev.  Every call
 * is synchronous with respect to the host unless stated otherwise.
 *
 * Status codes map onto the reference's exception taxonomy:
 *   RAFEM_OK              0
 *   RAFEM_ERR_BREAKDOWN   1  -> rafem.solver.GmresBreakdownError (solver.py:73, 522)
 *   RAFEM_ERR_INVALID     2  -> ValueError (solver.py:173-181, 399-417; fem.py:354-358)
 *   RAFEM_ERR_PHYSICS     3  -> rafem.fem.PhysicsRangeError (fem.py:272-278)
 *   RAFEM_ERR_UNSUPPORTED 4  -> NotImplementedError (e.g. pattern too dense)
 *   RAFEM_ERR_STEP_FAILURE 5 -> rafem.fem.StepFailureError (fem.py:76-82, 629-631)
 *   RAFEM_ERR_CUDA       -1  -> RuntimeError(rafem_last_error(ctx))
 */
#ifndef RAFEM_B200_H
#define RAFEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAFEM_OK 0
#define RAFEM_ERR_BREAKDOWN 1
#define RAFEM_ERR_INVALID 2
#define RAFEM_ERR_PHYSICS 3
#define RAFEM_ERR_UNSUPPORTED 4
#define RAFEM_ERR_STEP_FAILURE 5
#define RAFEM_ERR_CUDA (-1)

/* Krylov method (solver.py:50 lists the reference backends; only its
 * iterative one is on the device path, plus PCG for SPD FEM systems). */
#define RAFEM_METHOD_GMRES 0
#define RAFEM_METHOD_PCG 1

#define RAFEM_PRECOND_NONE 0
#define RAFEM_PRECOND_JACOBI 1
/* block-Jacobi over the persistent solver's row blocks (one per CTA), each
 * block solved by one Neumann step on the Jacobi-scaled block:
 * M^-1 = D^-1 + omega D^-1 (D - A_bb) D^-1.  Used by the paper-scale
 * pipelined PCG (north_star's "Jacobi or block-Jacobi"); the other engines
 * and GMRES treat it as point Jacobi. */
#define RAFEM_PRECOND_BLOCK_JACOBI 2

/* Dirichlet kind per interleaved dof (fem.py:403-413). */
#define RAFEM_DOF_FREE 0
#define RAFEM_DOF_APPLIED_VOLTAGE 1 /* 2*electrode_pos      -> config.applied_voltage */
#define RAFEM_DOF_ZERO 2            /* 2*electrode_neg      -> 0.0                    */
#define RAFEM_DOF_BOUNDARY_TEMP 3   /* 2*outer_boundary + 1 -> config.boundary_temp   */

typedef struct rafem_ctx rafem_ctx;
typedef struct rafem_mesh rafem_mesh;     /* mesh + symbolic pattern + geometry, on device  */
typedef struct rafem_system rafem_system; /* one assembled corrector-pass system, on device */
typedef struct rafem_matrix rafem_matrix; /* a general CSR uploaded from the host            */

/* SolverConfig (solver.py:81-110) restricted to the iterative path. */
typedef struct {
    int32_t method;          /* RAFEM_METHOD_*                                   */
    int32_t restart_m;       /* GMRES(m) restart length, >= 1                    */
    double tolerance;        /* relative residual target, in (0, 1)              */
    int64_t max_total_iters; /* <= 0 means 10 * n (solver.py:411)                */
    int32_t precondition;    /* RAFEM_PRECOND_*                                  */
    int32_t grid_ctas;       /* 0 = auto; otherwise persistent-kernel CTA count  */
} rafem_solver_params;

/* SolveStats (solver.py:113-130). */
typedef struct {
    int64_t iterations;          /* inner steps (Arnoldi / CG iterations)          */
    int64_t restarts;            /* cycles - 1                                     */
    double final_relative_residual; /* last TRUE residual ||b-Ax||/||b||           */
    int32_t converged;
    int32_t stagnated;
    int64_t cycles;              /* entries of cycle_lens                          */
    int64_t history_len;         /* total history entries (may exceed hist_cap)    */
    double device_ms;            /* CUDA-event time of the solve kernel            */
} rafem_solve_stats;

typedef struct {
    double dt;                 /* > 0 (fem.py:354-355)                          */
    double applied_voltage;    /* SimConfig.applied_voltage (fem.py:131)        */
    double boundary_temp;      /* SimConfig.boundary_temp (fem.py:132)          */
    int32_t apply_constraints; /* fem.py:333                                    */
    int32_t equilibrate;       /* fem.py:334                                    */
} rafem_assemble_params;

/* SimConfig (fem.py:121-147) for the native time loop. */
typedef struct {
    double total_time, dt_init, dt_min, dt_max, corrector_tol;
    int32_t max_corrector_iters;
    int32_t record_fields;     /* 1: copy every accepted (V,T) dof vector out    */
    double applied_voltage, boundary_temp, initial_temp;
    int64_t max_steps;         /* <= 0: run to total_time; else stop after n     */
    rafem_solver_params solver;
} rafem_sim_params;

/* SimulationSummary (fem.py:543-551). */
typedef struct {
    int64_t accepted_steps, total_corrector_iters, total_solver_iterations, dt_halvings;
    int64_t passes;            /* corrector passes (assembly + solve pairs)      */
    double final_time;
    int32_t status;            /* RAFEM_OK, or the error that aborted the run    */
    int32_t failed_step;       /* step index of a StepFailureError, else -1      */
    double failed_dt;
    double wall_ms;            /* host wall clock of the whole loop              */
    double assemble_ms, solve_ms; /* CUDA-event sums per region                  */
    int64_t bad_element;       /* PhysicsRangeError element, else -1             */
} rafem_sim_summary;

/* ---- context ----------------------------------------------------------- */
int rafem_ctx_create(int device, rafem_ctx** out);
void rafem_ctx_destroy(rafem_ctx* ctx);
const char* rafem_last_error(const rafem_ctx* ctx);
int rafem_device_info(rafem_ctx* ctx, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor,
                      int64_t* total_mem);
/* launches of the library's own kernels since ctx creation */
int64_t rafem_kernel_launches(const rafem_ctx* ctx);
/* the cudaStream_t every library call runs on (for external CUDA events) */
void* rafem_stream(const rafem_ctx* ctx);
/* diagnostics: last solve's execution mode (1 cluster-resident, 0 grid-wide,
 * 2 fused simulation, 3 grid-wide streaming PCG, 4 kernel-per-phase PCG,
 * 5 cluster-resident pipelined PCG (DSMEM halos), 6 cluster-resident simulation)
 * and CTA count; per-iteration phase timestamps (SM clock64) of CTA 0 when
 * tracing is on: 8 slots per iteration, returns entries copied */
int rafem_last_solve_mode(const rafem_ctx* ctx, int32_t* mode, int32_t* ctas);
/* preconditioner the last solve (or fused simulation) actually applied,
 * RAFEM_PRECOND_*: block-Jacobi exists only in the paper-scale pipelined
 * PCG; the other engines and GMRES apply point Jacobi when it is requested */
int rafem_last_solve_precond(const rafem_ctx* ctx, int32_t* precond);
int rafem_set_trace(rafem_ctx* ctx, int32_t on);
int64_t rafem_get_trace(rafem_ctx* ctx, int64_t* out, int64_t cap);

/* ---- sparse.py ----------------------------------------------------------- */
/* spmv (sparse.py:205-219): y = A x, each row summed left to right over its
 * stored entries with separately rounded products — bit-identical to the
 * reference's bincount route. */
int rafem_spmv(rafem_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr,
               const int64_t* col_idx, const double* vals, const double* x, double* y);

/* coo_to_csr (sparse.py:164-197): stable device sort by (row, col), runs
 * summed first-to-last from 0.0.  Outputs must hold nnz_in entries;
 * *nnz_out receives the compressed count. */
int rafem_coo_to_csr(rafem_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz_in,
                     const int64_t* rows, const int64_t* cols, const double* vals,
                     int64_t* row_ptr_out, int64_t* col_idx_out, double* vals_out,
                     int64_t* nnz_out);

/* ---- general CSR solve (solver.py:580-636 with a host CsrMatrix) --------- */
int rafem_matrix_create(rafem_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* vals, rafem_matrix** out);
void rafem_matrix_destroy(rafem_matrix* a);
int rafem_matrix_solve(rafem_matrix* a, const double* b, const double* x0 /* nullable */,
                       const rafem_solver_params* p, double* x_out, rafem_solve_stats* st,
                       double* hist, int64_t hist_cap, int64_t* cycle_lens, int64_t cycle_cap);

/* ---- mesh, assembly (fem.py:212-430) -------------------------------------- */
/* Symbolic phase, once per mesh: node pattern, incidence lists, slot map and
 * element geometry, all on device.  tets are 0-based node ids; region_index
 * maps each tet to a row of the per-region tables (k, rho_c, sigma0, alpha,
 * t_ref; fem.py:85-118).  dof_kind: 2N RAFEM_DOF_* codes. */
int rafem_mesh_create(rafem_ctx* ctx, int64_t n_nodes, const double* nodes, int64_t n_tets,
                      const int64_t* tets, const int32_t* region_index, int32_t n_regions,
                      const double* k, const double* rho_c, const double* sigma0,
                      const double* alpha, const double* t_ref, const uint8_t* dof_kind,
                      rafem_mesh** out);
void rafem_mesh_destroy(rafem_mesh* mesh);
/* Bit-exact assembly mode: replace the device-computed element geometry with
 * the reference's own (_basis_gradients, fem.py:229-240: np.linalg.det /
 * np.linalg.inv of the edge matrix — LAPACK LU, which a device kernel does
 * not reproduce to the last bit).  grad: n_tets x 4 x 3 basis gradients,
 * vol: n_tets volumes, computed once per mesh on the host; the packed
 * vol * grad_a . grad_b table (fem.py:280-282) is rebuilt on the device in
 * np.einsum's summation order.  Every later assembly of this mesh is then
 * bit-identical to assemble_global (fem.py:325-430). */
int rafem_mesh_set_geometry(rafem_mesh* mesh, const double* grad, const double* vol);
/* node-pattern size (slots); the dof CSR has 2*slots entries */
int64_t rafem_mesh_slots(const rafem_mesh* mesh);
/* stencil classes of the node pattern (built on first call): rows whose
 * column offsets (col - row) coincide share a class, and the streaming
 * SpMV kernels compute their columns instead of reading them (16 instead
 * of 20 bytes per slot).  Returns the class count, 0 when the pattern has
 * more than 255 distinct rows (unstructured meshes keep explicit columns),
 * -1 on error. */
int32_t rafem_mesh_stencil_classes(rafem_mesh* mesh);
/* node-level pattern: row_ptr (N+1), col (slots) */
int rafem_mesh_pattern(rafem_mesh* mesh, int64_t* node_row_ptr, int32_t* node_col);
/* shard sub-mesh (local ids [owned | ghosts by (owner, id)]): the ghosts
 * [n_owned, n_owned + n_below) have global ids below the owned block, so
 * the Dirichlet elimination's moved-column sums (fem.py:419-424) walk each
 * row in GLOBAL column order and the owned rows' rhs is bitwise the
 * unsharded one.  Rows must have <= 32 slots when n_below > 0. */
int rafem_mesh_set_shard_order(rafem_mesh* mesh, int64_t n_owned, int64_t n_below);

int rafem_system_create(rafem_mesh* mesh, rafem_system** out);
void rafem_system_destroy(rafem_system* sys);
/* assemble_global (fem.py:325-430) into sys; fields are host arrays of N.
 * On RAFEM_ERR_PHYSICS, *bad_element holds the lowest offending element. */
int rafem_assemble(rafem_system* sys, const double* t_iter, const double* v_iter,
                   const double* t_prev, const rafem_assemble_params* p, double* scale_out,
                   int64_t* bad_element);
/* rafem_assemble that also returns the rhs (2N, host) from the same
 * stream synchronisation (the plug-in seam reads it on every pass,
 * fem.py:495); rhs_out may be NULL. */
int rafem_assemble_rhs(rafem_system* sys, const double* t_iter, const double* v_iter,
                       const double* t_prev, const rafem_assemble_params* p, double* scale_out,
                       int64_t* bad_element, double* rhs_out);
/* dof-order values (2*slots, CsrMatrix.vals order) and rhs (2N) to host */
int rafem_system_download(rafem_system* sys, double* vals_out, double* rhs_out);
/* solve the device-resident system; b == NULL uses the assembled rhs */
int rafem_system_solve(rafem_system* sys, const double* b, const double* x0,
                       const rafem_solver_params* p, double* x_out, rafem_solve_stats* st,
                       double* hist, int64_t hist_cap, int64_t* cycle_lens, int64_t cycle_cap);
/* y = A x on the device-resident system (dof vectors, host) */
int rafem_system_spmv(rafem_system* sys, const double* x, double* y);
/* device-only SpMV timing on a device-resident x, mean CUDA-event ms per
 * launch: `reps` back-to-back launches, or (flush_l2) each launch timed
 * alone after a 256 MB write that evicts L2 */
int rafem_system_spmv_bench(rafem_system* sys, int32_t reps, int32_t flush_l2, double* ms_per_launch);

/* ---- native time loop (fem.py:554-644 around the device path) ------------ */
/* Runs run_simulation's adaptive predictor-corrector loop with mesh, system,
 * iterates and solver state resident in HBM; one 32-byte status read per
 * corrector pass.  If p->record_fields, rec_x must hold rec_cap * 2N doubles
 * (interleaved V/T per accepted step).  rec_* arrays may be NULL if rec_cap
 * is 0. */
int rafem_simulate(rafem_system* sys, const rafem_sim_params* p, rafem_sim_summary* out,
                   int64_t rec_cap, int64_t* rec_step, double* rec_time, double* rec_dt,
                   int32_t* rec_iters, double* rec_x);

/* ---- row-block shards and the kernel-per-phase PCG ------
 *
 * A shard is a rafem_system assembled on the sub-mesh of the tets touching
 * its owned nodes, with local node ids [owned (n_owned) | ghosts]; its
 * first n_owned node rows are complete rows of the global system.  The
 * reference has no distributed path: these entry points split
 * assemble_global (fem.py:325-430) at its one global reduction (the
 * equilibration sums, fem.py:390-400) and solve (solver.py:580-636) at its
 * dot products, so the caller can put collectives in between. */
typedef struct rafem_kp rafem_kp;

/* element kernel + slot fill (fem.py:247-388) for the whole sub-mesh;
 * diag_sums[0..1] = (sum of V, sum of T) diagonal entries of the first
 * n_owned node rows, the shard's share of fem.py:392-393. */
int rafem_assemble_partial(rafem_system* sys, const double* t_iter, const double* v_iter,
                           const double* t_prev, const rafem_assemble_params* p, int64_t n_owned,
                           double* diag_sums, int64_t* bad_element);
/* V-row scaling by the all-shard scale (fem.py:394-400) and Dirichlet
 * elimination (fem.py:402-428). */
int rafem_assemble_finish(rafem_system* sys, const rafem_assemble_params* p, double scale);

/* PCG over the first n_owned node rows of sys; columns address an
 * extended vector of n_ext nodes whose ghost tail [n_owned, n_ext) the
 * caller refreshes (halo exchange) before each SpMV phase. */
int rafem_kp_create(rafem_system* sys, int64_t n_owned, int64_t n_ext, int32_t nranks, int32_t rank,
                    rafem_kp** out);
void rafem_kp_destroy(rafem_kp* kp);
/* owned node ids whose (V,T) values the neighbours need, in send order */
int rafem_kp_set_halo(rafem_kp* kp, const int32_t* send_idx, int64_t n_send);
/* device buffers for the caller's collectives: x and u extended vectors
 * (double2 per node), packed send buffer, per-shard scalar slots
 * (nranks x 4 doubles; slot `rank` is written by the library) */
int rafem_kp_buffers(rafem_kp* kp, void** x_ext, void** u_ext, void** send_buf, void** rank_part);
/* b (host, 2*n_owned; NULL = the assembled rhs), x0 (host or NULL = 0);
 * Jacobi setup and the shard's ||b||^2 into its scalar slot */
int rafem_kp_begin(rafem_kp* kp, const double* b, const double* x0, const rafem_solver_params* p);
/* asynchronous phase launch (RAFEM_KP_*) */
#define RAFEM_KP_BNORM_FINISH 0
#define RAFEM_KP_HEAD 1
#define RAFEM_KP_SPMV_AFTER_HEAD 2
#define RAFEM_KP_SPMV 3
#define RAFEM_KP_UPDATE_FIRST 4
#define RAFEM_KP_UPDATE 5
#define RAFEM_KP_PACK_X 6
#define RAFEM_KP_PACK_U_AFTER_HEAD 7
#define RAFEM_KP_PACK_U 8
int rafem_kp_launch(rafem_kp* kp, int32_t phase);
/* nranks == 1 (or connected with rafem_kp_ipc_connect): `iters` iterations
 * back to back ([PACK_U +] SPMV + UPDATE each), no host round trip */
int rafem_kp_iterate(rafem_kp* kp, int32_t iters);
/* state (synchronises): flags bit0 done, bit1 need true residual, bit2 converged */
int rafem_kp_state(rafem_kp* kp, int32_t* flags, int64_t* iterations, double* rel);
/* Device-initiated data plane (one process per GPU of a node; also two
 * processes sharing one GPU): instead of the caller's collectives between
 * the phases, the phase kernels write the halo straight into the
 * neighbours' ghost ranges and the 4 scalars into every peer's slot array
 * through CUDA IPC mappings of the peers' kp blocks (NVLink peer memory),
 * each exchange announced by a system-scope release of a sequence word that
 * the consuming kernel acquires.  After connect, RAFEM_KP_PACK_* push,
 * every phase waits for its inputs itself and rafem_kp_iterate runs any
 * number of iterations without the host.
 * export: this shard's 64-byte cudaIpcMemHandle_t and 4 byte offsets
 * (x_ext, u_ext, slot array, flag block).  connect: every shard's handle and
 * offsets (rank order; own entry ignored), the send segments (neighbour,
 * [start, end) in send order, the neighbour's ghost node index of the
 * segment's first entry) and the ranks this shard receives from. */
int rafem_kp_ipc_export(rafem_kp* kp, void* handle, int64_t* offsets);
int rafem_kp_ipc_connect(rafem_kp* kp, const void* handles, const int64_t* offsets, int32_t nseg,
                         const int32_t* seg_peer, const int64_t* seg_start, const int64_t* seg_dst_node,
                         int32_t n_recv_peers, const int32_t* recv_peers);
/* owned x (host, 2*n_owned), SolveStats, history; returns the solve status */
int rafem_kp_finish(rafem_kp* kp, double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap,
                    int64_t* cycle_lens, int64_t cycle_cap);

/* ---- device-resident shard time loop (run_simulation / corrector_step,
 * fem.py:463-644, over one row block) ------------------------------------
 * The shard's accepted, previous and iterate (V, T) states over its
 * extended node set stay in HBM.  Per corrector pass the caller only moves
 * the halo (rafem_sl_pack -> exchange send4 into ghost4 -> rafem_sl_unpack;
 * 4 doubles per node: iterate V, T, accepted V, T), the equilibration sums
 * (rafem_sl_assemble_partial -> reduce -> rafem_assemble_finish), the
 * kp phases' collectives, and the corrector delta (a max over shards). */
typedef struct rafem_shard_loop rafem_shard_loop;
int rafem_sl_create(rafem_kp* kp, rafem_shard_loop** out);
void rafem_sl_destroy(rafem_shard_loop* sl);
/* device buffers: send4 (4 x n_send doubles, kp send order), ghost4 (4 x
 * n_ghost doubles, ghost order) */
int rafem_sl_buffers(rafem_shard_loop* sl, void** send4, void** ghost4);
/* T = initial_temp, V = 0 (fem.py:573-576) */
int rafem_sl_init(rafem_shard_loop* sl, double initial_temp);
/* predictor (fem.py:437-449), ratio = dt / dt_prev; vx0: the solver start
 * extrapolates V as well (the first pass of a step) */
int rafem_sl_predict(rafem_shard_loop* sl, int32_t step, double ratio, int32_t vx0);
int rafem_sl_pack(rafem_shard_loop* sl);
int rafem_sl_unpack(rafem_shard_loop* sl);
/* rafem_assemble_partial on the device iterate */
int rafem_sl_assemble_partial(rafem_shard_loop* sl, double dt, double* diag_sums, int64_t* bad_element);
/* kp solve of the assembled system from the predictor's start (from_start)
 * or the iterate; then rafem_kp_launch phases as for rafem_kp_begin */
int rafem_sl_solve_begin(rafem_shard_loop* sl, const rafem_solver_params* p, int32_t from_start);
/* solve status (return) and stats; the shard's corrector delta
 * (fem.py:526-528) to *delta; the iterate becomes the solution */
int rafem_sl_solve_end(rafem_shard_loop* sl, rafem_solve_stats* st, double* delta);
/* accept the step (fem.py:604-607) */
int rafem_sl_accept(rafem_shard_loop* sl);
/* owned accepted (V, T) dofs, interleaved, 2 x n_owned doubles (host) */
int rafem_sl_download(rafem_shard_loop* sl, double* x_out);

/* ---- device box mesh (mesh.py:306-375) and field comparison -------------
 * generate_box_mesh on the device, bit-identical to the host generator:
 * nodes (numpy.linspace coordinates), Kuhn tets, region 0, Dirichlet kinds
 * (outer surface T dofs; the electrode columns' V dofs, whose node ids the
 * caller computes with the same nearest-column rule); then the symbolic
 * phase.  extent = {x0, x1, y0, y1, z0, z1}.  One material region. */
int rafem_mesh_create_box(rafem_ctx* ctx, int32_t nx, int32_t ny, int32_t nz, const double* extent,
                          const int64_t* electrode_pos, int64_t n_pos, const int64_t* electrode_neg,
                          int64_t n_neg, double k, double rho_c, double sigma0, double alpha, double t_ref,
                          rafem_mesh** out);
/* node count (return) and tet count of a device mesh */
int64_t rafem_mesh_counts(const rafem_mesh* mesh, int64_t* n_tets);
/* host copies of the device mesh: nodes (3N), tets (4M, int32), dof kinds (2N); any may be NULL */
int rafem_mesh_download(rafem_mesh* mesh, double* nodes, int32_t* tets, uint8_t* dof_kind);
/* psnr_series kernels (metrics.py:47-64, 98-166): for each of `steps`
 * field pairs of n values (ref/test, step-major, host or device memory),
 * the sum of squared differences and max |ref|, fixed-order reductions */
int rafem_field_compare(rafem_ctx* ctx, int64_t n, int64_t steps, const double* ref, const double* test,
                        int32_t on_device, double* sq_err, double* max_abs_ref);

/* ---- streamed records (results.py:59-94 ResultWriter.append per step) ----
 * rafem_simulate with every accepted step's fields streamed to `fn` WHILE
 * the simulation runs: the device kernel writes each accepted (V, T) dof
 * vector into a ring of `ring_slots` device slots and publishes progress
 * in mapped host memory; a host loop copies published slots out on a side
 * stream and calls fn(user, step, time, dt, corrector_iters, x) with x the
 * interleaved 2N dof vector in pinned host memory (valid during the call).
 * The kernel waits for a free slot, so memory stays bounded at any record
 * size.  A nonzero return from fn stops the delivery (the run completes)
 * and the call returns RAFEM_ERR_INVALID.  fn must not call back into the
 * library (the record buffer is the context's pinned staging area). */
typedef int32_t (*rafem_record_fn)(void* user, int64_t step, double time, double dt, int32_t corrector_iters,
                                   const double* x);
int rafem_simulate_stream(rafem_system* sys, const rafem_sim_params* p, rafem_sim_summary* out,
                          int32_t ring_slots, rafem_record_fn fn, void* user);

#ifdef __cplusplus
}
#endif
#endif /* RAFEM_B200_H */
