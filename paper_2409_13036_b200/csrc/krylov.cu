// krylov.cu — persistent-kernel Krylov solvers and SpMV for sm_100a.
//
// Reference semantics: solver.py:381-531 (restarted GMRES(m), Givens LSQ,
// right Jacobi, true-residual restarts, stagnation latch, breakdown rules)
// and sparse.py:205-219 (SpMV, per-row left-to-right sums).
//
// One launch runs a whole solve.  Every CTA owns a contiguous block of row
// groups (balanced by slots + rows), keeps its share of every vector, and
// meets the others only at barriers around the scalar reductions.  Engines
// (chosen in krylov_solve):
//
//   * grid mode, smem slices (paper scale, the default there): a
//     cooperative launch of one CTA per SM, each CTA's matrix slice staged
//     in shared memory once; PCG runs the pipelined recurrence
//     (pcg_pipe_core: one barrier per iteration, the dot-product gather
//     overlapped with the SpMV, owner vectors in shared memory, optional
//     block-Jacobi), GMRES keeps its own basis rows in shared memory.
//   * grid mode, global rows: the same bodies reading the matrix from HBM.
//   * streaming PCG (pcg_stream_kernel, matrices >= 48 MB without stencil
//     classes): rows staged by TMA bulk copies, materialised preconditioned
//     residual.  Patterns with stencil classes (and any matrix >= 1 GB) go
//     to the kernel-per-phase engine in shard.cu instead (kp_system_solve).
//   * cluster mode (RAFEM_SOLVER_MODE=cluster): one thread-block cluster
//     with DSMEM barriers; measured slower, kept for experiments.
//   The kernel-per-phase PCG for the largest and sharded systems lives in
//   shard.cu; the whole-simulation kernel in simulate_dev.cuh.
//
// Reductions are deterministic in every mode: per-thread partial sums in
// a fixed order, a fixed xor-butterfly per warp, per-CTA partials in global
// memory, and every CTA re-reduces the G partials in the same fixed order,
// so all CTAs take identical control decisions and results are bitwise
// reproducible run to run.
#include "assembly_dev.cuh"
#include "common.cuh"
#include "internal.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <vector>

namespace rafem {

constexpr int KT = 512;        // threads per CTA of the persistent kernels
constexpr int KTC = 512;      // cluster-mode PCG: one thread per row group at paper scale
constexpr int kMaxCluster = 16;
constexpr size_t kSmemBudget = 220 * 1024;

struct KArgs {
    MatView A;
    const int* gpart;  // G + 1 group partition
    long long ldv;     // basis row stride
    const double* b;
    double* x;
    const double* minv;
    double* V;  // GMRES basis, (m + 1) x ldv
    double* w0;
    double* w1;
    double* r;
    double* z;
    double* p0;
    double* p1;
    double* q;
    double* e0;       // pipelined PCG: s, and the second m buffer
    double* e1;
    double* e2;
    double* partial;  // 2 x (m + 2) x G
    double* hess;     // per-CTA Hessenberg scratch when it does not fit in smem
    long long hess_stride;
    long long hess_smem;  // doubles of Hessenberg scratch at the head of dynamic smem
    int m;
    double tol;
    long long cap;
    double* hist;
    long long hist_cap;
    long long* cyc;
    long long cyc_cap;
    KResult* res;
    const int* flag;  // nonzero: zero diagonal under Jacobi -> ValueError
    long long* trace; // optional per-phase clock64 stamps (CTA 0, thread 0)
    int trace_cap;
    int team;         // lanes per row group in the solver SpMV (power of two)
    unsigned long long* flags;  // 2 x G x 8 words of barrier/all-reduce slots
    unsigned epoch;             // per-launch flag epoch (never 0)
    int pipe;                   // PCG: pipelined recurrence (pcg_pipe_core), W == 2 only
    int block;                  // pipelined PCG: block-Jacobi (Neumann step) on the CTA's diagonal block
    unsigned long long* gbar;   // grid-barrier arrival counter (zeroed before each launch); null: cg grid sync
    long long vs_off;           // GMRES: own rows of the basis in dynamic smem at this double offset (0: global)
    int vs_ld;                  // its row stride (own dofs of the widest CTA)
    int gm1r;                   // GMRES with the basis in smem: one-reduce Arnoldi (gmres_1r_body)
};

// Phase timestamps for diagnosis: slot k of iteration i at trace[i*8 + k].
RF_DEV void stamp(const KArgs& a, long long it, int k) {
    // (thread and block first: every other thread leaves without loading a.trace)
    if (threadIdx.x == 0 && blockIdx.x == 0 && a.trace && it * 8 + k < a.trace_cap)
        a.trace[it * 8 + k] = clock64();
}

// ---------------------------------------------------------------------------
// execution modes

struct GridMode {
    static constexpr bool kCluster = false;
    static constexpr bool kFlags = false;  // LL flag all-reduce (measured slower: L2 hot spot)
    RF_DEV static void sync() { cg::this_grid().sync(); }
};
struct ClusterMode {
    static constexpr bool kCluster = true;
    static constexpr bool kFlags = false;
    RF_DEV static void sync() { cg::this_cluster().sync(); }
};

// Row access: global (read-only / streaming loads) or this CTA's slice in
// shared memory (rp rebased to the CTA's first group).
template <int W, bool SMEM, bool STREAM>
struct Rows {
    const int* rp;
    const int* col;
    const double* val;
    int gbase;
    RF_DEV int start(int g) const { return SMEM ? rp[g - gbase] : __ldg(rp + g); }
    RF_DEV int column(int s) const { return SMEM ? col[s] : (STREAM ? __ldcs(col + s) : __ldg(col + s)); }
    RF_DEV double value1(int s) const { return SMEM ? val[s] : (STREAM ? __ldcs(val + s) : __ldg(val + s)); }
    RF_DEV double2 value2(int s) const {
        const double2* p = reinterpret_cast<const double2*>(val) + s;
        return SMEM ? *p : (STREAM ? __ldcs(p) : __ldg(p));
    }
};

// ---------------------------------------------------------------------------
// SpMV over this CTA's row groups.  Each group's rows are summed left to
// right over the stored slots with separately rounded products: exactly
// the reference's bincount order (sparse.py:217-218), so y is bit-identical.
// Slots are processed in chunks of 8 whose column/value loads and operand
// gathers are all issued before the (sequential) accumulation, so a row
// costs one gather latency per chunk instead of one per slot.

constexpr int kChunk = 8;   // scalar rows
constexpr int kChunk2 = 4;  // paired rows (two double2 per slot in flight)

// Solver SpMV: a team of `team` lanes (power of two <= 32, runtime) per row
// group; lane l takes slots l, l + team, ... (two in flight), and the team
// combines its partial sums with a fixed xor-butterfly.  The summation
// order differs from the reference's left-to-right one but is fixed for a
// given launch shape, so solves stay bit-reproducible.  A team puts every
// gather of a row in flight at once, which matters when rows are few per
// CTA (paper-scale meshes spread over all SMs).  team == 1 is one thread
// per row.  The loop trip count is uniform over the CTA, so every lane
// reaches the shuffles; lane 0 of each team runs the row epilogue.
// `pre(g)` runs on lane 0 before the slot loop (owner-row loads that do not
// depend on the product, so their latency overlaps the gathers) and its
// result is handed to `fin(g, y, pf)` after the team reduction.
struct NoPre {
    RF_DEV int operator()(int) const { return 0; }
};

template <int W, class R, class Src, class Pre, class Fin>
RF_DEV void spmv_team2(const R& rows, int g0, int g1, int team, const Src& src, const Pre& pre, Fin&& fin) {
    const int lane = threadIdx.x & (team - 1);
    const int nteams = blockDim.x / team;
    const int tt = threadIdx.x / team;
    for (int gb = g0; gb < g1; gb += nteams) {
        const int g = gb + tt;
        const bool active = g < g1;
        double av = 0.0, at = 0.0;
        decltype(pre(0)) pf{};
        if (active && lane == 0) pf = pre(g);
        if (active) {
            const int s0 = rows.start(g), s1 = rows.start(g + 1);
            for (int s = s0 + lane; s < s1; s += 2 * team) {
                const int sb = s + team;
                const bool two = sb < s1;
                if constexpr (W == 1) {
                    const int c0 = rows.column(s);
                    const int c1 = two ? rows.column(sb) : c0;
                    const double a0 = rows.value1(s);
                    const double a1 = two ? rows.value1(sb) : 0.0;
                    const double x0 = src.at(c0);
                    const double x1 = two ? src.at(c1) : 0.0;
                    av = add(av, mul(a0, x0));
                    if (two) av = add(av, mul(a1, x1));
                } else {
                    const int c0 = rows.column(s);
                    const int c1 = two ? rows.column(sb) : c0;
                    const double2 a0 = rows.value2(s);
                    const double2 a1 = two ? rows.value2(sb) : make_double2(0.0, 0.0);
                    const double2 x0 = src.at2(c0);
                    const double2 x1 = two ? src.at2(c1) : make_double2(0.0, 0.0);
                    av = add(av, mul(a0.x, x0.x));
                    at = add(at, mul(a0.y, x0.y));
                    if (two) {
                        av = add(av, mul(a1.x, x1.x));
                        at = add(at, mul(a1.y, x1.y));
                    }
                }
            }
        }
        for (int o = team >> 1; o > 0; o >>= 1) {
            av = add(av, __shfl_xor_sync(0xffffffffu, av, o));
            if (W == 2) at = add(at, __shfl_xor_sync(0xffffffffu, at, o));
        }
        if (active && lane == 0) {
            double y[2] = {av, at};
            fin(g, y, pf);
        }
    }
}

template <int W, class R, class Src, class Epi>
RF_DEV void spmv_team(const R& rows, int g0, int g1, int team, const Src& src, Epi&& epi) {
    spmv_team2<W>(rows, g0, g1, team, src, NoPre{}, [&](int g, const double* y, int) { epi(g, y); });
}

template <int W, class R, class Src, class Epi, int CH1 = kChunk, int CH2 = Src::kChunk2>
RF_DEV void spmv_groups(const R& rows, int g0, int g1, const Src& src, Epi&& epi) {
    constexpr int kChunk = CH1;
    constexpr int kChunk2 = CH2;
    for (int g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
        const int s0 = rows.start(g), s1 = rows.start(g + 1);
        if constexpr (W == 1) {
            double acc = 0.0;
            for (int s = s0; s < s1; s += kChunk) {
                int c[kChunk];
                double a[kChunk], xv[kChunk];
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (s + j < s1) {
                        c[j] = rows.column(s + j);
                        a[j] = rows.value1(s + j);
                    }
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (s + j < s1) xv[j] = src.at(c[j]);
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (s + j < s1) acc = add(acc, mul(a[j], xv[j]));
            }
            double y[1] = {acc};
            epi(g, y);
        } else {
            double av = 0.0, at = 0.0;
            for (int s = s0; s < s1; s += kChunk2) {
                int c[kChunk2];
                double2 a[kChunk2], xv[kChunk2];
#pragma unroll
                for (int j = 0; j < kChunk2; ++j)
                    if (s + j < s1) {
                        c[j] = rows.column(s + j);
                        a[j] = rows.value2(s + j);
                    }
#pragma unroll
                for (int j = 0; j < kChunk2; ++j)
                    if (s + j < s1) xv[j] = src.at2(c[j]);
#pragma unroll
                for (int j = 0; j < kChunk2; ++j)
                    if (s + j < s1) {
                        av = add(av, mul(a[j].x, xv[j].x));
                        at = add(at, mul(a[j].y, xv[j].y));
                    }
            }
            double y[2] = {av, at};
            epi(g, y);
        }
    }
}

// Operand sources: the SpMV input is formed on the fly from vectors that
// are final after the previous barrier, which saves a barrier per step.
struct SrcPlain {
    static constexpr int kChunk2 = 4;
    const double* x;
    RF_DEV double at(int j) const { return __ldca(x + j); }
    RF_DEV double2 at2(int c) const { return __ldca(reinterpret_cast<const double2*>(x) + c); }
};

// GMRES: z_j = minv_j * (s_j * c), where v_k = s * c is the next basis
// vector (c = 1/beta or 1/h_{k,k-1}); owners store the same bits in V[k].
template <bool PRE>
struct SrcBasis {
    static constexpr int kChunk2 = 4;
    const double* s;
    double c;
    const double* minv;
    RF_DEV double at(int j) const {
        double v = mul(__ldca(s + j), c);
        return PRE ? mul(v, __ldg(minv + j)) : v;
    }
    RF_DEV double2 at2(int cc) const {
        double2 sv = __ldca(reinterpret_cast<const double2*>(s) + cc);
        double2 v = make_double2(mul(sv.x, c), mul(sv.y, c));
        if (PRE) {
            double2 mv = __ldg(reinterpret_cast<const double2*>(minv) + cc);
            v.x = mul(v.x, mv.x);
            v.y = mul(v.y, mv.y);
        }
        return v;
    }
};

// PCG: p_j = z_j + beta * pold_j (first step: p = z).
struct SrcCg {
    static constexpr int kChunk2 = 4;
    const double* z;
    const double* po;
    double beta;
    int first;
    RF_DEV double at(int j) const {
        double zj = __ldca(z + j);
        return first ? zj : add(zj, mul(beta, __ldca(po + j)));
    }
    RF_DEV double2 at2(int c) const {
        double2 zz = __ldca(reinterpret_cast<const double2*>(z) + c);
        if (first) return zz;
        double2 pp = __ldca(reinterpret_cast<const double2*>(po) + c);
        return make_double2(add(zz.x, mul(beta, pp.x)), add(zz.y, mul(beta, pp.y)));
    }
};

// ---------------------------------------------------------------------------
// reduction plumbing

template <int NV>
RF_DEV void publish(double (&v)[NV], int nv, double* P, int base, int G, double* red) {
    block_sum<NV>(v, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (j < nv) P[(long long)(base + j) * G + blockIdx.x] = v[j];
    }
}

// After a barrier: reduce nv coefficient rows of P into co[] (all CTAs).
RF_DEV void gather(const double* P, int nv, int G, double* co) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = wid; i < nv; i += nw) {
        double s = reduce_partials_warp(P + (long long)i * G, G);
        if (lane == 0) co[i] = s;
    }
    __syncthreads();
}

// Per-CTA dots v_i . w for i < nv over dofs [lo, hi), published into P.
RF_DEV void multidot(const double* V, long long ldv, int nv, const double* w, int lo, int hi,
                     double* P, int G, double* red) {
    for (int i0 = 0; i0 < nv; i0 += 8) {
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        const int cnt = min(8, nv - i0);
        for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) {
            const double we = w[e];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < cnt) acc[j] = add(acc[j], mul(__ldca(V + (long long)(i0 + j) * ldv + e), we));
        }
        publish<8>(acc, cnt, P, i0, G, red);
    }
}

// Per-CTA dots v_i . w over this CTA's own dofs with the basis rows in
// shared memory (Vs[i * ld + (e - lo)]): one warp per coefficient, lanes
// striding the dofs, a fixed xor-butterfly — no block-level reduction.
RF_DEV void multidot_smem(const double* Vs, int ld, int nv, const double* w, int lo, int hi, double* P, int G,
                          bool self = false) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = wid; i < nv + (self ? 1 : 0); i += nw) {
        const double* vi = i < nv ? Vs + (long long)i * ld - lo : w;  // coefficient nv: w . w
        double acc = 0.0;
        for (int e = lo + lane; e < hi; e += 32) acc = add(acc, mul(vi[e], w[e]));
        acc = warp_sum(acc);
        if (lane == 0) P[(long long)i * G + blockIdx.x] = acc;
    }
}

// One-reduce Arnoldi partials (gmres_1r_body): for j < k, v_j . u -> row j
// and v_j . w -> row k + 1 + j; u . u -> row k and u . w -> row 2k + 1.
// w == nullptr: the u rows only.  One warp per j, as multidot_smem.
RF_DEV void multidot_pair_smem(const double* Vs, int ld, int k, const double* u, const double* w, int lo, int hi,
                               double* P, int ldp) {
    // one half-warp per j (all k + 1 in one round for k < 32 at 512 threads),
    // lanes striding the dofs, a fixed xor-butterfly over the 16 lanes
    const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, nh = blockDim.x >> 4;
    const int jend = ((k + 1 + nh - 1) / nh) * nh;  // whole rounds: every lane shuffles
    for (int j = hw; j < jend; j += nh) {
        const bool on = j <= k;
        const double* vj = j < k ? Vs + (long long)j * ld - lo : u;
        double sa = 0.0, sb = 0.0;
        if (on) {
            if (w) {
                for (int e = lo + hl; e < hi; e += 16) {
                    const double v = vj[e];
                    sa = add(sa, mul(v, u[e]));
                    sb = add(sb, mul(v, w[e]));
                }
            } else {
                for (int e = lo + hl; e < hi; e += 16) sa = add(sa, mul(vj[e], u[e]));
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            sa = add(sa, __shfl_xor_sync(0xffffffffu, sa, o));
            sb = add(sb, __shfl_xor_sync(0xffffffffu, sb, o));
        }
        if (on && hl == 0) {
            double* pc = P + (long long)blockIdx.x * ldp;
            pc[j] = sa;
            if (w) pc[k + 1 + j] = sb;
        }
    }
}

// After a barrier: nv coefficients from CTA-major partials P[c * ldp + i]
// into co[] on every CTA.  512 threads load at once (8 groups of
// consecutive CTAs x 64 coefficients, a warp reading 32 adjacent
// coefficients of one CTA), then each coefficient adds its 8 group sums
// left to right: one L2 round trip for G <= 152, the same fixed order on
// every CTA.  gs: 512 doubles of shared scratch.
RF_DEV void gather_wide(const double* P, int ldp, int nv, int G, double* co, double* gs) {
    constexpr int NG = 8, U = 19;
    const int t = threadIdx.x, i0 = t & 63, grp = t >> 6;
    const int per = (G + NG - 1) / NG;
    for (int base = 0; base < nv; base += 64) {
        const int i = base + i0;
        double s = 0.0;
        if (grp < NG && i < nv) {
            const int c0 = grp * per, c1 = min(G, c0 + per);
            for (int c = c0; c < c1; c += U) {
                double v[U];
#pragma unroll
                for (int q = 0; q < U; ++q) v[q] = c + q < c1 ? __ldcg(P + (long long)(c + q) * ldp + i) : 0.0;
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (c + q < c1) s = add(s, v[q]);
            }
        }
        if (grp < NG) gs[t] = s;
        __syncthreads();
        if (t < 64 && base + t < nv) {
            double acc = gs[t];
#pragma unroll
            for (int g = 1; g < NG; ++g) acc = add(acc, gs[g * 64 + t]);
            co[base + t] = acc;
        }
        __syncthreads();
    }
}

// Cluster mode: copy this CTA's slice of the matrix into shared memory
// (16-byte vector loads; the slice is constant for the whole solve).
template <int W>
RF_DEV void stage_slice(const MatView& A, int g0, int g1, double* sval, int* scol, int* srp) {
    const int s0 = __ldg(A.rp + g0), s1 = __ldg(A.rp + g1);
    const int ns = s1 - s0;
    for (int g = g0 + threadIdx.x; g <= g1; g += blockDim.x) srp[g - g0] = __ldg(A.rp + g) - s0;
    if (W == 2) {
        const double2* src = reinterpret_cast<const double2*>(A.val) + s0;
        double2* dst = reinterpret_cast<double2*>(sval);
        for (int s = threadIdx.x; s < ns; s += blockDim.x) dst[s] = __ldg(src + s);
    } else {
        for (int s = threadIdx.x; s < ns; s += blockDim.x) sval[s] = __ldg(A.val + s0 + s);
    }
    for (int s = threadIdx.x; s < ns; s += blockDim.x) scol[s] = __ldg(A.col + s0 + s);
    __syncthreads();
}

RF_DEV void write_result(KResult* res, long long total, long long cycles, long long hlen, double rel,
                         bool converged, bool stagnated, int status) {
    res->iterations = total;
    res->restarts = cycles > 0 ? cycles - 1 : 0;
    res->cycles = cycles;
    res->hist_len = hlen;
    res->final_rel = rel;
    res->converged = converged ? 1 : 0;
    res->stagnated = stagnated ? 1 : 0;
    res->status = status;
}

// ---------------------------------------------------------------------------
// Grid-wide barrier + all-reduce without cooperative_groups.
//
// Each CTA owns a 64-byte slot per round parity.  For up to 3 values the
// slot carries the CTA's block-reduced partials LL-style: every 8-byte
// word holds half of a double in its low 32 bits and the round flag in the
// high 32 bits, and 8-byte stores are single-copy atomic, so a reader that
// sees the current flag in a word also sees its data.  One polling pass of
// warp 0 over the G slots is therefore barrier and gather at once (one L2
// round trip after the last CTA arrives, instead of barrier + gather).
// Publication is release-ordered after the CTA's vector writes
// (bar.sync then __threadfence by the publishing thread) and the poll is
// followed by an acquire fence, so the next phase's gathers see every
// CTA's vectors.  Flags are (launch epoch << 16 | round); slots alternate
// parity, which suffices because a CTA can run at most one round ahead of
// the slowest poller.  A spin cap traps instead of hanging the GPU.

RF_DEV void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
RF_DEV unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
constexpr long long kSpinCap = 1LL << 31;

// Grid barrier on a monotonically increasing arrival counter: after the
// CTA's bar.sync one thread adds 1 with release semantics and spins with
// acquire loads until all G CTAs of this round have arrived (target =
// rounds * G).  Release after bar.sync is cumulative over the CTA's
// writes, and the acquire (which invalidates the SM's L1) before the
// closing bar.sync orders every thread's later loads after them.  Measured
// on B200 with 128 doubles written per CTA before each barrier
// (scripts/microbench_bar.cu): 1.70 us per round vs 2.54 us for
// cooperative_groups' grid sync (see grid_counter for the in-kernel result).
RF_DEV void grid_barrier(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        long long spins = 0;
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (++spins > kSpinCap) asm volatile("trap;");
        } while (v < target);
    }
    __syncthreads();
}

template <class Mode>
struct Sync {
    const KArgs& a;
    unsigned round = 0;
    unsigned long long nbar = 0;  // grid barriers passed (counter-barrier target)

    RF_DEV void grid_sync() {
        if constexpr (Mode::kCluster) {
            Mode::sync();
        } else {
            if (a.gbar) {
                ++nbar;
                grid_barrier(a.gbar, nbar * gridDim.x);
            } else {
                Mode::sync();
            }
        }
    }

    RF_DEV unsigned flag() const { return (a.epoch << 16) | (round & 0xffffu); }
    RF_DEV unsigned long long* slot(int cta) const {
        return a.flags + ((size_t)(round & 1u) * gridDim.x + cta) * 8;
    }

    // Block-reduce v, combine over all CTAs in a fixed order into co[0..nv).
    template <int NV>
    RF_DEV void reduce(double (&v)[NV], int nv, double* P, double* co, double* red) {
        const int G = gridDim.x;
        if constexpr (Mode::kCluster || !Mode::kFlags) {
            publish<NV>(v, nv, P, 0, G, red);
            grid_sync();
            gather(P, nv, G, co);
            return;
        } else {
            static_assert(NV <= 3, "LL slots carry at most three values");
            block_sum<NV>(v, red);
            const unsigned f = flag();
            if (threadIdx.x == 0) {
                __threadfence();
                unsigned long long* s = slot(blockIdx.x);
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    if (j < nv) {
                        const unsigned long long bits = (unsigned long long)__double_as_longlong(v[j]);
                        st_relaxed(s + 2 * j, ((unsigned long long)f << 32) | (bits & 0xffffffffULL));
                        st_relaxed(s + 2 * j + 1, ((unsigned long long)f << 32) | (bits >> 32));
                    }
                }
            }
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                double acc[NV];
#pragma unroll
                for (int j = 0; j < NV; ++j) acc[j] = 0.0;
                for (int c = lane; c < G; c += 32) {
                    const unsigned long long* s = slot(c);
                    unsigned long long w[2 * NV];
                    long long spins = 0;
                    bool ok;
                    do {
                        ok = true;
#pragma unroll
                        for (int k = 0; k < 2 * NV; ++k) {
                            if (k < 2 * nv) {
                                w[k] = ld_relaxed(s + k);
                                ok = ok && (unsigned)(w[k] >> 32) == f;
                            }
                        }
                        if (++spins > kSpinCap) asm volatile("trap;");
                    } while (!ok);
#pragma unroll
                    for (int j = 0; j < NV; ++j)
                        if (j < nv)
                            acc[j] = add(acc[j], __longlong_as_double((long long)((w[2 * j] & 0xffffffffULL) |
                                                                                  (w[2 * j + 1] << 32))));
                }
#pragma unroll
                for (int j = 0; j < NV; ++j) acc[j] = warp_sum(acc[j]);
                if (lane == 0)
                    for (int j = 0; j < nv; ++j) co[j] = acc[j];
                __threadfence();
            }
            __syncthreads();
            ++round;
        }
    }

    // Barrier only (vector visibility).
    RF_DEV void barrier() {
        if constexpr (Mode::kCluster || !Mode::kFlags) {
            grid_sync();
        } else {
            __syncthreads();
            const unsigned f = flag();
            if (threadIdx.x == 0) {
                __threadfence();
                st_relaxed(slot(blockIdx.x) + 7, f);
            }
            if (threadIdx.x < 32) {
                for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) {
                    long long spins = 0;
                    while ((unsigned)ld_relaxed(slot(c) + 7) != f)
                        if (++spins > kSpinCap) asm volatile("trap;");
                }
                __threadfence();
            }
            __syncthreads();
            ++round;
        }
    }

    // Partials already stored in P by publish(); barrier then fixed-order gather.
    RF_DEV void sync_gather(const double* P, int nv, double* co) {
        barrier();
        gather(P, nv, gridDim.x, co);
    }
};

// Shared prologue: invalid flag check and ||b|| (solver.py:413-425).
// Returns bnorm, or a negative value when the kernel must stop.
template <class Mode>
RF_DEV double prologue(const KArgs& a, Sync<Mode>& sy, int lo, int hi, double* co, double* red, int& par,
                       long long pstride) {
    if (*a.flag) {
        if (blockIdx.x == 0 && threadIdx.x == 0) write_result(a.res, 0, 0, 0, INFINITY, false, false, RAFEM_ERR_INVALID);
        return -1.0;
    }
    double v[1] = {0.0};
    for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const double be = a.b[e];
        v[0] = add(v[0], mul(be, be));
    }
    sy.template reduce<1>(v, 1, a.partial + par * pstride, co, red);
    par ^= 1;
    const double bnorm = sqrt(co[0]);
    if (bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
        for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) a.x[e] = 0.0;
        if (blockIdx.x == 0 && threadIdx.x == 0) write_result(a.res, 0, 0, 0, 0.0, true, false, RAFEM_OK);
        return -1.0;
    }
    return bnorm;
}

// ---------------------------------------------------------------------------
// GMRES(m) — solver.py:381-531, with classical Gram-Schmidt applied twice
// (CGS2) in place of the reference's modified Gram-Schmidt: the same
// Arnoldi basis to working precision, but 3 barriers per step instead of
// k + 2 dependent reductions.

template <int W, bool PRE, class R>
RF_DEV void gmres_1r_body(const KArgs& a, const R& rows, double* dyn);

template <int W, bool PRE, class Mode, class R>
RF_DEV void gmres_body(const KArgs& a, const R& rows, double* dyn) {
    if constexpr (!Mode::kCluster) {
        if (a.gm1r) {
            gmres_1r_body<W, PRE>(a, rows, dyn);
            return;
        }
    }
    __shared__ double red[32 * 8];
    __shared__ double sc[4];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const int lo = W * g0, hi = W * g1;
    const int m = a.m;
    const long long ldv = a.ldv;
    double* H = a.hess ? a.hess + (long long)cta * a.hess_stride : dyn;  // col-major (m+1) x m
    double* cs = H + (long long)(m + 1) * m;
    double* sn = cs + m;
    double* gg = sn + m;      // m + 1
    double* yy = gg + m + 1;  // m
    double* co = yy + m;      // m + 2
    const long long pstride = (long long)(m + 2) * G;
    int par = 0;
    Sync<Mode> sy{a};
    // basis row i, own dof e: in shared memory when the host reserved room
    double* const Vs = a.vs_off ? dyn + a.vs_off : nullptr;
    auto vrow = [&](int i) -> double* { return Vs ? Vs + (long long)i * a.vs_ld - lo : a.V + (long long)i * ldv; };

    const double bnorm = prologue<Mode>(a, sy, lo, hi, co, red, par, pstride);
    if (bnorm < 0.0) return;

    // r = b - A x, returns ||r|| / ||b||   (solver.py:438-439, 517-518)
    auto true_residual = [&]() -> double {
        double v[1] = {0.0};
        spmv_team<W>(rows, g0, g1, a.team, SrcPlain{a.x}, [&](int g, const double* y) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int e = W * g + w;
                const double re = sub(a.b[e], y[w]);
                a.r[e] = re;
                v[0] = add(v[0], mul(re, re));
            }
        });
        sy.template reduce<1>(v, 1, a.partial + par * pstride, co, red);
        par ^= 1;
        return sqrt(co[0]) / bnorm;
    };

    long long total = 0, cycles = 0, hlen = 0;
    int weak = 0;
    bool latched = false, have_prev = false, converged = false;
    double prev_start = 0.0, rel = INFINITY;
    int status = RAFEM_OK;
    const double tiny = 2.2250738585072014e-308;  // np.finfo(float64).tiny

    while (true) {
        rel = true_residual();
        if (have_prev) {  // stagnation bookkeeping (solver.py:440-447)
            if (rel > (1.0 - 1e-3) * prev_start) {
                if (++weak >= 3) latched = true;
            } else {
                weak = 0;
            }
            have_prev = false;
        }
        if (rel <= a.tol) {
            converged = true;
            break;
        }
        if (total >= a.cap) break;

        const double cycle_start = rel;
        const double beta = rel * bnorm;
        if (tid == 0) {
            for (int i = 0; i <= m; ++i) gg[i] = 0.0;
            gg[0] = beta;
        }
        const double* src = a.r;
        double src_scale = 1.0 / beta;
        int used = 0;
        bool broke = false, dead = false;
        const long long hstart = hlen;

        for (int k = 0; k < m; ++k) {
            double* wk = (k & 1) ? a.w1 : a.w0;
            double* Vk = vrow(k);
            stamp(a, total, 0);
            // v_k (own rows) and w = A (M^-1 v_k)       (solver.py:469-470)
            for (int e = lo + tid; e < hi; e += bd) Vk[e] = mul(src[e], src_scale);
            spmv_team<W>(rows, g0, g1, a.team, SrcBasis<PRE>{src, src_scale, a.minv}, [&](int g, const double* y) {
#pragma unroll
                for (int w = 0; w < W; ++w) wk[W * g + w] = y[w];
            });
            __syncthreads();
            stamp(a, total, 1);
            // CGS pass 1: h_i = v_i . w
            double* P = a.partial + par * pstride;
            if (Vs)
                multidot_smem(Vs, a.vs_ld, k + 1, wk, lo, hi, P, G);
            else
                multidot(a.V, ldv, k + 1, wk, lo, hi, P, G, red);
            stamp(a, total, 2);
            sy.sync_gather(P, k + 1, co);
            stamp(a, total, 3);
            par ^= 1;
            if (tid == 0)
                for (int i = 0; i <= k; ++i) H[(long long)k * (m + 1) + i] = co[i];
            // w -= sum h_i v_i ; CGS pass 2: c_i = v_i . w
            for (int e = lo + tid; e < hi; e += bd) {
                double acc = wk[e];
                for (int i = 0; i <= k; ++i) acc = sub(acc, mul(co[i], Vs ? vrow(i)[e] : __ldca(vrow(i) + e)));
                wk[e] = acc;
            }
            P = a.partial + par * pstride;
            if (Vs) {
                __syncthreads();  // the warps read other threads' w entries
                multidot_smem(Vs, a.vs_ld, k + 1, wk, lo, hi, P, G, true);
            } else {
                multidot(a.V, ldv, k + 1, wk, lo, hi, P, G, red);
            }
            stamp(a, total, 4);
            sy.sync_gather(P, Vs ? k + 2 : k + 1, co);
            stamp(a, total, 5);
            par ^= 1;
            if (tid == 0)
                for (int i = 0; i <= k; ++i) H[(long long)k * (m + 1) + i] = add(H[(long long)k * (m + 1) + i], co[i]);
            double hk1;
            if (Vs) {
                // ||w - V c||^2 = ||w||^2 - ||c||^2 (V orthonormal, c = V^T w, tiny
                // after the first pass): no third reduction, only the barrier
                // that makes the new w visible to the next SpMV's gathers
                // Near an invariant subspace ||c||^2 approaches ||w||^2 and the
                // difference cancels: then (same decision on every CTA, the
                // scalars are identical) the norm is reduced explicitly.
                double cc = 0.0;
                for (int i = 0; i <= k; ++i) cc = add(cc, mul(co[i], co[i]));
                const bool explicit_norm = cc > 1e-8 * co[k + 1];
                double v[1] = {0.0};
                for (int e = lo + tid; e < hi; e += bd) {
                    double acc = wk[e];
                    for (int i = 0; i <= k; ++i) acc = sub(acc, mul(co[i], vrow(i)[e]));
                    wk[e] = acc;
                    v[0] = add(v[0], mul(acc, acc));
                }
                if (explicit_norm) {
                    P = a.partial + par * pstride;
                    sy.template reduce<1>(v, 1, P, co, red);
                    par ^= 1;
                    hk1 = sqrt(co[0]);
                } else {
                    hk1 = sqrt(sub(co[k + 1], cc));
                    sy.barrier();
                }
            }
            // w -= sum c_i v_i ; ||w||
            else {
                double v[1] = {0.0};
                for (int e = lo + tid; e < hi; e += bd) {
                    double acc = wk[e];
                    for (int i = 0; i <= k; ++i)
                        acc = sub(acc, mul(co[i], Vs ? vrow(i)[e] : __ldca(vrow(i) + e)));
                    wk[e] = acc;
                    v[0] = add(v[0], mul(acc, acc));
                }
                P = a.partial + par * pstride;
                sy.template reduce<1>(v, 1, P, co, red);
                par ^= 1;
                hk1 = sqrt(co[0]);
            }
            stamp(a, total, 6);
            total += 1;
            // Givens update of column k (solver.py:478-496), one thread per CTA
            if (tid == 0) {
                double* hc = H + (long long)k * (m + 1);
                hc[k + 1] = hk1;
                for (int i = 0; i < k; ++i) {
                    const double t = add(mul(cs[i], hc[i]), mul(sn[i], hc[i + 1]));
                    hc[i + 1] = add(mul(-sn[i], hc[i]), mul(cs[i], hc[i + 1]));
                    hc[i] = t;
                }
                const double rad = hypot(hc[k], hc[k + 1]);
                double est = 0.0;
                int isdead = 0;
                if (rad == 0.0) {
                    isdead = 1;
                } else {
                    cs[k] = hc[k] / rad;
                    sn[k] = hc[k + 1] / rad;
                    hc[k] = rad;
                    hc[k + 1] = 0.0;
                    gg[k + 1] = mul(-sn[k], gg[k]);
                    gg[k] = mul(cs[k], gg[k]);
                    est = fabs(gg[k + 1]) / bnorm;
                    if (cta == 0 && hlen < a.hist_cap) a.hist[hlen] = est;
                }
                sc[0] = isdead;
                sc[1] = est;
            }
            __syncthreads();
            if (sc[0] != 0.0) {  // column added nothing (solver.py:483-487)
                dead = true;
                used = k;
                break;
            }
            used = k + 1;
            const double est = sc[1];
            ++hlen;
            if (hk1 < tiny) {  // breakdown (solver.py:497-499)
                broke = true;
                break;
            }
            src = wk;
            src_scale = 1.0 / hk1;
            if (est <= a.tol || total >= a.cap) break;
        }

        if (used > 0) {  // y = R^-1 g ; x += M^-1 (V y)   (solver.py:504-511)
            if (tid == 0) {
                for (int i = used - 1; i >= 0; --i) {
                    double d = 0.0;
                    for (int j = i + 1; j < used; ++j) d = add(d, mul(H[(long long)j * (m + 1) + i], yy[j]));
                    yy[i] = sub(gg[i], d) / H[(long long)i * (m + 1) + i];
                }
            }
            __syncthreads();
            for (int e = lo + tid; e < hi; e += bd) {
                double u = 0.0;
                for (int i = 0; i < used; ++i) u = add(u, mul(Vs ? vrow(i)[e] : __ldca(vrow(i) + e), yy[i]));
                if (PRE) u = mul(a.minv[e], u);
                a.x[e] = add(a.x[e], u);
            }
        }
        if (cta == 0 && tid == 0 && cycles < a.cyc_cap) a.cyc[cycles] = hlen - hstart;
        ++cycles;
        have_prev = true;
        prev_start = cycle_start;
        sy.barrier();  // x final everywhere before the next SpMV

        if (broke || dead) {  // solver.py:516-524
            rel = true_residual();
            if (rel <= a.tol) {
                converged = true;
            } else {
                status = RAFEM_ERR_BREAKDOWN;
            }
            break;
        }
    }
    if (cta == 0 && tid == 0) write_result(a.res, total, cycles, hlen, rel, converged, latched && !converged, status);
}

// ---------------------------------------------------------------------------
// GMRES(m) with a one-reduce Arnoldi step: classical Gram-Schmidt whose
// second (reorthogonalising) pass over each basis vector is delayed into the
// next step, so one fixed-order reduction serves both passes (the
// low-synchronisation "DCGS2" Arnoldi).  Step k holds u_k, the candidate
// for v_k after one projection against V_{k-1}, forms w_k = A M^-1 u_k and
// reduces in ONE round
//     a = V_{k-1}^T u_k,   u_k . u_k,   b = V_{k-1}^T w_k,   u_k . w_k.
// With alpha = ||u_k - V_{k-1} a|| = sqrt(u.u - a.a) (an explicit norm
// reduction when that difference cancels):
//     v_k       = (u_k - V_{k-1} a) / alpha                (second pass)
//     H[:, k-1] = first-pass coefficients + a,  H[k][k-1] = alpha
//     u_{k+1}   = (w_k - V_{k-1} b - v_k g) / alpha,   g = (u.w - a.b) / alpha
//     first pass of column k = ([b; g] - H[0:k+1, 0:k] a) / alpha
// since A M^-1 v_k = (w_k - A M^-1 V_{k-1} a) / alpha and A M^-1 V_{k-1} =
// V_k H.  Column k-1 becomes final — Givens rotation, residual estimate and
// the reference's stop tests (solver.py:478-502) — one step after its SpMV,
// so m columns cost m SpMVs, m + 1 reductions and m barriers (3m
// synchronisations in gmres_body); on convergence one SpMV goes unused.
// Grid mode with the basis rows in shared memory only.
template <int W, bool PRE, class R>
RF_DEV void gmres_1r_body(const KArgs& a, const R& rows, double* dyn) {
    __shared__ double red[32 * 8];
    __shared__ double sc[8];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const int lo = W * g0, hi = W * g1;
    const int m = a.m;
    const long long ld = m + 1;
    double* H = dyn;  // rotated columns (back substitution), col-major ld x m
    double* cs = H + ld * m;
    double* sn = cs + m;
    double* gg = sn + m;          // m + 1
    double* yy = gg + m + 1;      // m
    double* co = yy + m;          // 2m + 4
    double* Hr = co + 2 * m + 4;  // raw Hessenberg columns, col-major ld x m
    double* Hf = Hr + ld * m;     // first-pass coefficients of the open column (2 x ld, alternating)
    double* gs = Hf + 2 * ld;     // 512: gather_wide scratch
    const long long pstride = (long long)(2 * m + 4) * G;
    int par = 0;
    Sync<GridMode> sy{a};
    double* const Vs = dyn + a.vs_off;
    auto vrow = [&](int i) -> double* { return Vs + (long long)i * a.vs_ld - lo; };

    const double bnorm = prologue<GridMode>(a, sy, lo, hi, co, red, par, pstride);
    if (bnorm < 0.0) return;

    auto true_residual = [&]() -> double {  // solver.py:438-439, 517-518
        double v[1] = {0.0};
        spmv_team<W>(rows, g0, g1, a.team, SrcPlain{a.x}, [&](int g, const double* y) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int e = W * g + w;
                const double re = sub(a.b[e], y[w]);
                a.r[e] = re;
                v[0] = add(v[0], mul(re, re));
            }
        });
        sy.template reduce<1>(v, 1, a.partial + par * pstride, co, red);
        par ^= 1;
        return sqrt(co[0]) / bnorm;
    };

    long long total = 0, cycles = 0, hlen = 0, nstep = 0;  // nstep: trace stamps
    int weak = 0;
    bool latched = false, have_prev = false, converged = false;
    double prev_start = 0.0, rel = INFINITY;
    int status = RAFEM_OK;
    const double tiny = 2.2250738585072014e-308;  // np.finfo(float64).tiny

    while (true) {
        rel = true_residual();
        if (have_prev) {  // stagnation bookkeeping (solver.py:440-447)
            if (rel > (1.0 - 1e-3) * prev_start) {
                if (++weak >= 3) latched = true;
            } else {
                weak = 0;
            }
            have_prev = false;
        }
        if (rel <= a.tol) {
            converged = true;
            break;
        }
        if (total >= a.cap) break;

        const double cycle_start = rel;
        const double beta = rel * bnorm;
        if (tid == 0) {
            for (int i = 0; i <= m; ++i) gg[i] = 0.0;
            gg[0] = beta;
        }
        int used = 0;
        bool broke = false, dead = false;
        const long long hstart = hlen;
        double alpha = beta;  // u_0 = r, v_0 = r / beta

        for (int k = 0; k <= m; ++k) {
            const double* u = k == 0 ? a.r : ((k & 1) ? a.w1 : a.w0);
            double* wv = a.z;
            const bool more = k < m;
            stamp(a, nstep, 0);
            if (more) {  // w_k = A (M^-1 u_k)   (solver.py:469-470)
                spmv_team<W>(rows, g0, g1, a.team, SrcBasis<PRE>{u, 1.0, a.minv}, [&](int g, const double* y) {
#pragma unroll
                    for (int w = 0; w < W; ++w) wv[W * g + w] = y[w];
                });
            }
            __syncthreads();
            stamp(a, nstep, 1);
            double* P = a.partial + par * pstride;
            multidot_pair_smem(Vs, a.vs_ld, k, u, more ? wv : nullptr, lo, hi, P, 2 * m + 4);
            stamp(a, nstep, 2);
            sy.barrier();
            stamp(a, nstep, 3);
            gather_wide(P, 2 * m + 4, more ? 2 * k + 2 : k + 1, G, co, gs);
            __syncthreads();
            par ^= 1;
            if (k > 0) {  // alpha = ||u_k - V_{k-1} a||; identical decision on every CTA
                double aa = 0.0;
                for (int i = 0; i < k; ++i) aa = add(aa, mul(co[i], co[i]));
                if (aa > 1e-8 * co[k]) {
                    stamp(a, nstep, 7);
                    double v[1] = {0.0};
                    for (int e = lo + tid; e < hi; e += bd) {
                        double s = 0.0;
                        for (int i = 0; i < k; ++i) s = add(s, mul(co[i], vrow(i)[e]));
                        const double d = sub(u[e], s);
                        v[0] = add(v[0], mul(d, d));
                    }
                    sy.template reduce<1>(v, 1, a.partial + par * pstride, sc + 4, red);
                    par ^= 1;
                    alpha = sqrt(sc[4]);
                } else {
                    alpha = sqrt(fmax(sub(co[k], aa), 0.0));
                }
            }
            stamp(a, nstep, 4);
            // v_k (second pass) and u_{k+1} (first pass of the next vector)
            // over the own rows; then, while the grid barrier that publishes
            // u_{k+1} is in flight (split arrive / wait on the counter),
            // warp 0 rotates column k-1 (Givens, solver.py:478-496) and warp 1
            // stores column k-1's raw values and column k's first-pass
            // coefficients.  The stop tests read warp 0's results after the
            // wait (on convergence v_k / u_{k+1} go unused).
            const int j = k - 1;
            const double ialpha = 1.0 / alpha;
            const int wid = tid >> 5, lane = tid & 31;
            if (more) {
                // four lanes per row, lane q taking basis rows i = q mod 4, and
                // a quad butterfly ((q0 + q1) + (q2 + q3)); a . b rides along
                double* un = ((k + 1) & 1) ? a.w1 : a.w0;
                double* Vk = vrow(k);
                const int q = tid & 3;
                const int nrow = hi - lo;
                for (int r0 = 0; r0 < nrow; r0 += bd >> 2) {
                    const int r = r0 + (tid >> 2);
                    const int e = lo + (r < nrow ? r : nrow - 1);
                    double sa = 0.0, sb = 0.0, ab = 0.0;
                    for (int i = q; i < k; i += 4) {
                        const double vi = vrow(i)[e];
                        const double ci = co[i], bi = co[k + 1 + i];
                        sa = add(sa, mul(ci, vi));
                        sb = add(sb, mul(bi, vi));
                        ab = add(ab, mul(ci, bi));
                    }
                    sa = add(sa, __shfl_xor_sync(0xffffffffu, sa, 1));
                    sb = add(sb, __shfl_xor_sync(0xffffffffu, sb, 1));
                    ab = add(ab, __shfl_xor_sync(0xffffffffu, ab, 1));
                    sa = add(sa, __shfl_xor_sync(0xffffffffu, sa, 2));
                    sb = add(sb, __shfl_xor_sync(0xffffffffu, sb, 2));
                    ab = add(ab, __shfl_xor_sync(0xffffffffu, ab, 2));
                    if (q == 0 && r < nrow) {
                        const double gam = mul(sub(co[2 * k + 1], ab), ialpha);
                        const double vk = mul(sub(u[e], sa), ialpha);
                        Vk[e] = vk;
                        un[e] = mul(sub(sub(wv[e], sb), mul(vk, gam)), ialpha);
                    }
                }
                __syncthreads();
                ++sy.nbar;
                if (tid == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.gbar) : "memory");
            }
            stamp(a, nstep, 5);
            if (wid == 0) {
                if (k > 0 && lane == 0) {
                    const double* __restrict__ hf = Hf + (j & 1) * ld;
                    double* __restrict__ hc = H + (long long)j * ld;
                    const double* __restrict__ cr = cs;
                    const double* __restrict__ sr = sn;
                    double hi = add(hf[0], co[0]);
                    for (int i = 0; i < j; ++i) {
                        const double hn = add(hf[i + 1], co[i + 1]);
                        const double c = cr[i], sv = sr[i];
                        hc[i] = add(mul(c, hi), mul(sv, hn));
                        hi = add(mul(-sv, hi), mul(c, hn));
                    }
                    const double h1 = alpha;
                    const double rad = hypot(hi, h1);
                    double est = 0.0;
                    int isdead = 0;
                    if (rad == 0.0) {
                        isdead = 1;
                    } else {
                        cs[j] = hi / rad;
                        sn[j] = h1 / rad;
                        hc[j] = rad;
                        hc[j + 1] = 0.0;
                        gg[j + 1] = mul(-sn[j], gg[j]);
                        gg[j] = mul(cs[j], gg[j]);
                        est = fabs(gg[j + 1]) / bnorm;
                        if (cta == 0 && hlen < a.hist_cap) a.hist[hlen] = est;
                    }
                    sc[0] = isdead;
                    sc[1] = est;
                }
            } else if (wid == 1) {
                if (k > 0) {
                    const double* hf = Hf + (j & 1) * ld;
                    double* hr = Hr + (long long)j * ld;
                    for (int i = lane; i <= k; i += 32) hr[i] = i < k ? add(hf[i], co[i]) : alpha;
                    __syncwarp();
                }
                if (more) {
                    double* hf = Hf + (k & 1) * ld;
                    for (int i = lane; i <= k; i += 32) {
                        double t = 0.0;
                        for (int jj = i > 0 ? i - 1 : 0; jj < k; ++jj)
                            t = add(t, mul(Hr[(long long)jj * ld + i], co[jj]));
                        double bi;
                        if (i < k) {
                            bi = co[k + 1 + i];
                        } else {  // g, summed as the sweep's quads do
                            double ab4[4];
                            for (int q = 0; q < 4; ++q) {
                                ab4[q] = 0.0;
                                for (int ii = q; ii < k; ii += 4) ab4[q] = add(ab4[q], mul(co[ii], co[k + 1 + ii]));
                            }
                            const double ab = add(add(ab4[0], ab4[1]), add(ab4[2], ab4[3]));
                            bi = mul(sub(co[2 * k + 1], ab), ialpha);
                        }
                        hf[i] = mul(sub(bi, t), ialpha);
                    }
                }
            }
            if (more && tid == 0) {  // wait for every CTA's u_{k+1}
                const unsigned long long target = sy.nbar * (unsigned long long)G;
                long long spins = 0;
                unsigned long long v;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.gbar) : "memory");
                    if (++spins > kSpinCap) asm volatile("trap;");
                } while (v < target);
            }
            __syncthreads();
            stamp(a, nstep, 6);
            ++nstep;
            if (k > 0) {
                total += 1;
                if (sc[0] != 0.0) {  // column added nothing (solver.py:483-487)
                    dead = true;
                    used = j;
                    break;
                }
                used = j + 1;
                const double est = sc[1];
                ++hlen;
                if (alpha < tiny) {  // breakdown (solver.py:497-499)
                    broke = true;
                    break;
                }
                if (est <= a.tol || total >= a.cap) break;
            }
            if (!more) break;
        }

        if (used > 0) {  // y = R^-1 g ; x += M^-1 (V y)   (solver.py:504-511)
            if (tid == 0) {
                for (int i = used - 1; i >= 0; --i) {
                    double d = 0.0;
                    for (int j = i + 1; j < used; ++j) d = add(d, mul(H[(long long)j * ld + i], yy[j]));
                    yy[i] = sub(gg[i], d) / H[(long long)i * ld + i];
                }
            }
            __syncthreads();
            for (int e = lo + tid; e < hi; e += bd) {
                double s = 0.0;
                for (int i = 0; i < used; ++i) s = add(s, mul(vrow(i)[e], yy[i]));
                if (PRE) s = mul(a.minv[e], s);
                a.x[e] = add(a.x[e], s);
            }
        }
        if (cta == 0 && tid == 0 && cycles < a.cyc_cap) a.cyc[cycles] = hlen - hstart;
        ++cycles;
        have_prev = true;
        prev_start = cycle_start;
        sy.barrier();  // x final everywhere before the next SpMV

        if (broke || dead) {  // solver.py:516-524
            rel = true_residual();
            if (rel <= a.tol) {
                converged = true;
            } else {
                status = RAFEM_ERR_BREAKDOWN;
            }
            break;
        }
    }
    if (cta == 0 && tid == 0) write_result(a.res, total, cycles, hlen, rel, converged, latched && !converged, status);
}

// ---------------------------------------------------------------------------
// Jacobi-preconditioned CG in the single-reduction (Chronopoulos-Gear)
// form: per iteration ONE fused pass computes the owner updates
//     p = u + beta p,  s = w + beta s,  x += alpha p,  r -= alpha s,
//     u = M^-1 r,      w = A u,         (r.u, w.u, r.r)
// and ONE barrier publishes the three dots.  The SpMV operand u_j is
// formed on the fly in the gather from the previous iteration's r, w, s
// (final after the last barrier) with exactly the owner's operation
// sequence, so owner and gatherers agree bit for bit.  Not in the
// reference (which ships GMRES only); used for the SPD FEM systems under
// its own backend name.  Converged only when the TRUE residual meets the
// tolerance: a recursive-residual exit re-enters at the top with
// r = b - A x and restarts the recurrence if needed (solver.py:437-450).

// u_j = M_j (r_j - alpha (w_j + beta s_j)); mode 0: u = M r; mode 1: no s term.
template <bool PRE>
struct SrcCgU {
    static constexpr int kChunk2 = 2;
    const double* r;
    const double* w;
    const double* s;
    const double* minv;
    double alpha, beta;
    int mode;
    RF_DEV double at(int j) const {
        double t = __ldca(r + j);
        if (mode) {
            const double sw = mode == 2 ? add(__ldca(w + j), mul(beta, __ldca(s + j))) : __ldca(w + j);
            t = sub(t, mul(alpha, sw));
        }
        return PRE ? mul(__ldg(minv + j), t) : t;
    }
    RF_DEV double2 at2(int c) const {
        double2 t = __ldca(reinterpret_cast<const double2*>(r) + c);
        if (mode) {
            double2 sw = __ldca(reinterpret_cast<const double2*>(w) + c);
            if (mode == 2) {
                const double2 ss = __ldca(reinterpret_cast<const double2*>(s) + c);
                sw.x = add(sw.x, mul(beta, ss.x));
                sw.y = add(sw.y, mul(beta, ss.y));
            }
            t.x = sub(t.x, mul(alpha, sw.x));
            t.y = sub(t.y, mul(alpha, sw.y));
        }
        if (PRE) {
            const double2 mv = __ldg(reinterpret_cast<const double2*>(minv) + c);
            t.x = mul(mv.x, t.x);
            t.y = mul(mv.y, t.y);
        }
        return t;
    }
};

// Uniform (identical in every CTA) outcome of one PCG solve.
struct PcgOut {
    long long total;
    double rel;
    int converged;
    int status;
};

// The PCG iteration proper, after ||b|| is known.  `co`/`red` are the
// caller's shared scratch; `par` its partial-buffer parity.
template <int W, bool PRE, class Mode, class R>
RF_DEV PcgOut pcg_core(const KArgs& a, const R& rows, Sync<Mode>& sy, double bnorm, double* co, double* red,
                       int& par) {
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const long long pstride = 8LL * G;
    // ping-pong r, w, s (gathered); p and x are owner-only.  Selected with
    // ternaries, not arrays, so nothing is indexed dynamically (no stack).
    auto rb = [&](int i) { return i ? a.z : a.r; };
    auto wb = [&](int i) { return i ? a.w1 : a.w0; };
    auto sb = [&](int i) { return i ? a.q : a.p1; };
    double* p = a.p0;

    long long total = 0, cycles = 0, hlen = 0;
    bool converged = false;
    double rel = INFINITY;
    int status = RAFEM_OK;
    int cur = 0;

    auto round = [&](double (&v)[3]) {
        double* P = a.partial + par * pstride;
        stamp(a, total, 1);
        sy.template reduce<3>(v, 3, P, co, red);
        stamp(a, total, 4);
        par ^= 1;
    };

    while (true) {
        {  // r = b - A x ; r.r
            double v[3] = {0.0, 0.0, 0.0};
            double* r = rb(cur);
            spmv_team<W>(rows, g0, g1, a.team, SrcPlain{a.x}, [&](int g, const double* y) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    const int e = W * g + w;
                    const double re = sub(a.b[e], y[w]);
                    r[e] = re;
                    v[2] = add(v[2], mul(re, re));
                }
            });
            round(v);
        }
        rel = sqrt(co[2]) / bnorm;
        if (rel <= a.tol) {
            converged = true;
            break;
        }
        if (total >= a.cap) break;
        double gamma, alpha, beta = 0.0;
        {  // w = A u, u = M^-1 r ; (r.u, w.u)
            double v[3] = {0.0, 0.0, 0.0};
            const double* r = rb(cur);
            double* w = wb(cur);
            const SrcCgU<PRE> src{r, nullptr, nullptr, a.minv, 0.0, 0.0, 0};
            spmv_team<W>(rows, g0, g1, a.team, src, [&](int g, const double* y) {
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int e = W * g + k;
                    const double ue = src.at(e);
                    w[e] = y[k];
                    v[0] = add(v[0], mul(r[e], ue));
                    v[1] = add(v[1], mul(y[k], ue));
                }
            });
            round(v);
            gamma = co[0];
            if (!(gamma > 0.0) || !(co[1] > 0.0) || !isfinite(gamma) || !isfinite(co[1])) {
                status = RAFEM_ERR_BREAKDOWN;  // not SPD under this preconditioner
                break;
            }
            alpha = gamma / co[1];
        }
        const long long hstart = hlen;
        int mode = 1;
        while (true) {
            stamp(a, total, 0);
            const double* ro = rb(cur);
            const double* wo = wb(cur);
            const double* so = sb(cur);
            double* rn = rb(cur ^ 1);
            double* wn = wb(cur ^ 1);
            double* sn = sb(cur ^ 1);
            double v[3] = {0.0, 0.0, 0.0};
            const SrcCgU<PRE> src{ro, wo, so, a.minv, alpha, beta, mode};
            // owner-row operands are loaded before the slot loop (prefetch)
            struct Own {
                double r[W], w[W], s[W], m[W], p[W], x[W];
            };
            auto pre = [&](int g) {
                Own o;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int e = W * g + k;
                    o.r[k] = ro[e];
                    o.w[k] = wo[e];
                    o.s[k] = mode == 2 ? so[e] : 0.0;
                    o.m[k] = PRE ? __ldcg(a.minv + e) : 1.0;
                    o.p[k] = mode == 2 ? p[e] : 0.0;
                    o.x[k] = a.x[e];
                }
                return o;
            };
            spmv_team2<W>(rows, g0, g1, a.team, src, pre, [&](int g, const double* y, const Own& o) {
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int e = W * g + k;
                    const double s_n = mode == 2 ? add(o.w[k], mul(beta, o.s[k])) : o.w[k];
                    const double u_o = PRE ? mul(o.m[k], o.r[k]) : o.r[k];
                    const double p_n = mode == 2 ? add(u_o, mul(beta, o.p[k])) : u_o;
                    a.x[e] = add(o.x[k], mul(alpha, p_n));
                    p[e] = p_n;
                    const double r_n = sub(o.r[k], mul(alpha, s_n));
                    const double u_n = PRE ? mul(o.m[k], r_n) : r_n;
                    rn[e] = r_n;
                    wn[e] = y[k];
                    sn[e] = s_n;
                    v[0] = add(v[0], mul(r_n, u_n));
                    v[1] = add(v[1], mul(y[k], u_n));
                    v[2] = add(v[2], mul(r_n, r_n));
                }
            });
            round(v);
            cur ^= 1;
            ++total;
            const double est = sqrt(co[2]) / bnorm;
            if (cta == 0 && tid == 0 && hlen < a.hist_cap) a.hist[hlen] = est;
            ++hlen;
            if (est <= a.tol || total >= a.cap) break;
            const double gnew = co[0];
            const double bnew = gnew / gamma;
            const double den = co[1] - bnew * gnew / alpha;
            if (!(gnew > 0.0) || !(den > 0.0) || !isfinite(den)) {
                status = RAFEM_ERR_BREAKDOWN;
                break;
            }
            alpha = gnew / den;
            beta = bnew;
            gamma = gnew;
            mode = 2;
        }
        if (cta == 0 && tid == 0 && cycles < a.cyc_cap) a.cyc[cycles] = hlen - hstart;
        ++cycles;
        if (status != RAFEM_OK) break;
    }
    if (a.res && cta == 0 && tid == 0) write_result(a.res, total, cycles, hlen, rel, converged, false, status);
    return PcgOut{total, rel, converged ? 1 : 0, status};
}

// ---------------------------------------------------------------------------
// Pipelined PCG (Ghysels & Vanroose) for paper-scale systems: ONE grid
// barrier per iteration, and the all-reduce of that iteration's dot
// products is gathered WHILE the SpMV runs, because the SpMV operand
// m = M^-1 w does not depend on it:
//
//   (after barrier i)  gather (r_i.u_i, w_i.u_i, r_i.r_i)  ||  n_i = A m_i
//   alpha_i, beta_i from the gathered scalars (same recurrence as pcg_core)
//   z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p
//   x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z, m' = M^-1 w
//   publish (r.u, w.u, r.r) of the new vectors -> barrier i+1
//
// m is double-buffered (neighbours gather m_i while its owner writes
// m_{i+1}); every other vector is owner-only.  Same contract as pcg_core:
// one history entry per update, converged only on the TRUE residual (the
// head recomputes r, u, w, m from x), breakdown -> RAFEM_ERR_BREAKDOWN.

constexpr int kPipeRows = 128;  // max node rows per CTA (y and the owner vectors staged in smem)

// bnorm < 0: ||b|| (and, with zflag, the zero-diagonal flag of the Jacobi
// setup) are folded into the first head reduction instead of a separate
// round; a raised flag returns RAFEM_ERR_INVALID, b == 0 gives x = 0.
// x0_gather: where the FIRST head gathers the initial guess from (a copy of
// x that is already complete on every CTA), so the caller's owner-only copy
// into x needs no barrier of its own; later heads gather x itself.
template <bool PRE, class Mode, class R>
RF_DEV PcgOut pcg_pipe_core(const KArgs& a, const R& rows, Sync<Mode>& sy, double bnorm, double* co, double* red,
                            int& par, const int* zflag = nullptr, const double* x0_gather = nullptr,
                            const double* xold = nullptr, double* dmax = nullptr, const double* r_pre = nullptr) {
    __shared__ double2 ybuf[kPipeRows];
    // owner-only recurrence vectors live in shared memory (indexed by the
    // global dof, offset by the CTA's first dof); u is mirrored to global
    // memory only when a head's SpMV gathers it
    __shared__ double s_r[2 * kPipeRows], s_u[2 * kPipeRows], s_w[2 * kPipeRows], s_z[2 * kPipeRows],
        s_q[2 * kPipeRows], s_s[2 * kPipeRows], s_p[2 * kPipeRows], s_x[2 * kPipeRows], s_m[2 * kPipeRows],
        s_mv[2 * kPipeRows], s_y[2 * kPipeRows];
    __shared__ double s_omega;
    __shared__ unsigned s_inmask[kPipeRows];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const int lo = 2 * g0, hi = 2 * g1;
    const long long pstride = 8LL * G;
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    double* x = a.x;
    double* r = s_r - lo;
    double* u = s_u - lo;
    double* ug = a.z;  // global copy of u for the head's gather
    double* w = s_w - lo;
    double* z = s_z - lo;
    double* q = s_q - lo;
    double* sv = s_s - lo;
    double* p = s_p - lo;
    auto mb = [&](int i) { return i ? a.e1 : a.w1; };
    double* xs = s_x - lo;   // owner copy of x (written through to HBM)
    double* ms = s_m - lo;   // owner copy of the current m
    double* mvs = s_mv - lo; // owner Jacobi inverse diagonal
    for (int e = lo + tid; e < hi; e += blockDim.x) mvs[e] = PRE ? __ldcg(a.minv + e) : 1.0;
    __syncthreads();
    auto M = [&](int e) { return mvs[e]; };
    // Block-Jacobi (a.block): M^-1 = D^-1 + omega D^-1 (D - A_cc) D^-1 on this
    // CTA's diagonal block A_cc, i.e. one Neumann step of the block solve:
    // m = y + omega D^-1 (w - A_cc y), y = D^-1 w.  SPD when omega < 1 /
    // (lambda_max(D^-1/2 A_cc D^-1/2) - 1); omega comes from the block's
    // Gershgorin bound (1 for the FEM blocks, whose bound stays below 2).
    const bool blk = PRE && a.block;
    double* yl = s_y - lo;
    const int nr = g1 - g0;
    if (blk) {
        // in-block slots of each own row as a bit mask (rows have <= 32 slots
        // here), and the block's Gershgorin bound of D^-1/2 A_cc D^-1/2
        // a team of lanes per row (slots l, l + bt, ...), D^-1/2 staged once
        double gmax = 0.0;
        for (int e = lo + tid; e < hi; e += blockDim.x) s_y[e - lo] = sqrt(mvs[e]);
        __syncthreads();
        const double* sq = s_y - lo;
        int bt = 1;
        while (bt < 8 && ((nr * bt * 2 + 31) & ~31) <= (int)blockDim.x) bt *= 2;
        for (int base = 0; base < nr * bt; base += blockDim.x) {
            const int q = base + tid, rr = q / bt, l0 = q & (bt - 1);
            unsigned mask = 0;
            double gv = 0.0, gt = 0.0;
            if (rr < nr) {
                const int g = g0 + rr, sb = rows.start(g), deg = rows.start(g + 1) - sb;
                for (int l = l0; l < deg && l < 32; l += bt) {
                    const int c = rows.column(sb + l);
                    if (c < g0 || c >= g1) continue;
                    mask |= 1u << l;
                    const double2 v = rows.value2(sb + l);
                    gv = add(gv, mul(fabs(v.x), mul(sq[2 * g], sq[2 * c])));
                    gt = add(gt, mul(fabs(v.y), mul(sq[2 * g + 1], sq[2 * c + 1])));
                }
            }
            for (int o = bt >> 1; o > 0; o >>= 1) {  // (whole warps: bt divides 32)
                mask |= __shfl_xor_sync(0xffffffffu, mask, o);
                gv = add(gv, __shfl_xor_sync(0xffffffffu, gv, o));
                gt = add(gt, __shfl_xor_sync(0xffffffffu, gt, o));
            }
            if (rr < nr && l0 == 0) {
                s_inmask[rr] = mask;
                gmax = fmax(gmax, fmax(gv, gt));
            }
        }
        gmax = block_max(gmax, red);
        if (tid == 0) s_omega = gmax > 1.98 ? 0.98 / (gmax - 1.0) : 1.0;
        __syncthreads();
    }
    const double omega = blk ? s_omega : 0.0;
    // dst (owner dofs, smem) = M^-1 src; also to dst_g when given.  y = D^-1 src
    // is expected in yl already when y_ready (the caller fused it).
    // The block step's rows run on the threads below `nthr` (whole warps), a
    // team of bt lanes per row: lane l takes the in-block slots l, l + bt, ...
    // of its row in stored order and the team combines them with a fixed
    // xor-butterfly, so the result is deterministic (bt == 1 is the plain
    // left-to-right row sum).
    auto block_rows = [&](const double* src, double* dst, double* dst_g, int nthr) {
        int bt = 1;
        while (bt < 8 && ((nr * bt * 2 + 31) & ~31) <= nthr) bt *= 2;
        if (tid < ((nr * bt + 31) & ~31)) {
            const int rr = tid / bt, l = tid & (bt - 1);
            double av = 0.0, at = 0.0;
            if (rr < nr) {
                const int sb = rows.start(g0 + rr);
                const unsigned pat = bt == 1 ? 0xffffffffu : bt == 2 ? 0x55555555u : bt == 4 ? 0x11111111u : 0x01010101u;
                unsigned mask = s_inmask[rr] & (pat << l);
                while (mask) {
                    const int k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const int c = rows.column(sb + k);
                    const double2 v = rows.value2(sb + k);
                    av = add(av, mul(v.x, yl[2 * c]));
                    at = add(at, mul(v.y, yl[2 * c + 1]));
                }
            }
            for (int o = bt >> 1; o > 0; o >>= 1) {
                av = add(av, __shfl_xor_sync(0xffffffffu, av, o));
                at = add(at, __shfl_xor_sync(0xffffffffu, at, o));
            }
            if (rr < nr && l == 0) {
                const int e0 = 2 * (g0 + rr);
                const double d0 = add(yl[e0], mul(omega, mul(mvs[e0], sub(src[e0], av))));
                const double d1 = add(yl[e0 + 1], mul(omega, mul(mvs[e0 + 1], sub(src[e0 + 1], at))));
                dst[e0] = d0;
                dst[e0 + 1] = d1;
                if (dst_g) {
                    dst_g[e0] = d0;
                    dst_g[e0 + 1] = d1;
                }
            }
        }
    };
    // dst (owner dofs, smem) = M^-1 src; also to dst_g when given.
    auto apply_block = [&](const double* src, double* dst, double* dst_g) {
        for (int e = lo + tid; e < hi; e += blockDim.x) yl[e] = mul(mvs[e], src[e]);
        __syncthreads();
        block_rows(src, dst, dst_g, blockDim.x);
        __syncthreads();
    };

    long long total = 0, cycles = 0, hlen = 0;
    bool converged = false;
    double rel = INFINITY;
    int status = RAFEM_OK;
    int cur = 0;  // m buffer gathered by the next SpMV

    auto publish3 = [&](double (&v)[3]) {
        block_sum<3>(v, red);
        if (tid == 0) {
            double* P = a.partial + par * pstride;
#pragma unroll
            for (int j = 0; j < 3; ++j) P[(long long)j * G + cta] = v[j];
        }
    };
    // the last warps fold the published partials while the others start the SpMV
    auto gather3 = [&]() {
        const int gw = warp - (nwarps - 3);
        if (gw >= 0) {
            const double s = reduce_partials_warp(a.partial + par * pstride + (long long)gw * G, G);
            if (lane == 0) co[gw] = s;
        }
    };

    bool first_head = true;
    while (true) {
        {  // head: r = b - A x, u = M r ; then w = A u, m = M w ; partials of (r.u, w.u, r.r)
            const bool with_b = bnorm < 0.0;
            double v[3] = {0.0, 0.0, 0.0};
            const double* xg = x0_gather ? x0_gather : x;
            x0_gather = nullptr;
            if (r_pre) {  // the caller's exact r = b - A x of the start (no product here)
                for (int e = lo + tid; e < hi; e += blockDim.x) {
                    const double be = a.b[e];
                    const double re = r_pre[e];
                    r[e] = re;
                    if (!blk) {
                        const double ue = PRE ? mul(M(e), re) : re;
                        u[e] = ue;
                        ug[e] = ue;
                    }
                    v[2] = add(v[2], mul(re, re));
                    if (with_b) v[0] = add(v[0], mul(be, be));
                }
                r_pre = nullptr;
            } else {
                spmv_team<2>(rows, g0, g1, a.team, SrcPlain{xg}, [&](int g, const double* y) {
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        const int e = 2 * g + k;
                        const double be = a.b[e];
                        const double re = sub(be, y[k]);
                        r[e] = re;
                        if (!blk) {
                            const double ue = PRE ? mul(M(e), re) : re;
                            u[e] = ue;
                            ug[e] = ue;
                        }
                        v[2] = add(v[2], mul(re, re));
                        if (with_b) v[0] = add(v[0], mul(be, be));
                    }
                });
            }
            // later heads usually end the solve: their block step waits until
            // the true residual says the iteration continues
            if (blk && first_head) {
                __syncthreads();
                apply_block(r, u, ug);
            }
            if (with_b && zflag && tid == 0) v[1] = (double)*zflag;
            if (xold) {
                // the corrector delta of this iterate against xold (fem.py:527-528)
                // rides on the head's reduction: max over CTAs by a fourth warp
                double dm = 0.0;
                for (int e = lo + tid; e < hi; e += blockDim.x) {
                    const double xe = x[e], xo = xold[e];
                    xs[e] = xe;  // owner copy (synced below)
                    const double d = fabs(sub(xe, xo)) / fmax(1.0, fabs(xo));
                    dm = (d > dm || d != d) ? d : dm;
                }
                double* P = a.partial + par * pstride;
                dm = block_max(dm, red);
                if (tid == 0) P[3LL * G + cta] = dm;
                publish<3>(v, 3, P, 0, G, red);
                sy.barrier();
                if (warp < 3) {
                    const double s = reduce_partials_warp(P + (long long)warp * G, G);
                    if (lane == 0) co[warp] = s;
                } else if (warp == 3) {
                    const double mx = reduce_max_partials_warp(P + 3LL * G, G);
                    if (lane == 0) co[3] = mx;
                }
                __syncthreads();
                *dmax = co[3];
            } else {
                for (int e = lo + tid; e < hi; e += blockDim.x) xs[e] = x[e];  // owner copy (synced below)
                sy.template reduce<3>(v, 3, a.partial + par * pstride, co, red);
            }
            par ^= 1;
            if (with_b) {
                if (co[1] > 0.0) return PcgOut{0, INFINITY, 0, RAFEM_ERR_INVALID};
                bnorm = sqrt(co[0]);
                if (bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
                    for (int e = lo + tid; e < hi; e += blockDim.x) x[e] = 0.0;
                    __syncthreads();
                    if (dmax) *dmax = -1.0;  // x changed after the head: the caller computes the delta
                    return PcgOut{0, 0.0, 1, RAFEM_OK};
                }
            }
        }
        rel = sqrt(co[2]) / bnorm;
        if (rel <= a.tol) {
            converged = true;
            break;
        }
        if (total >= a.cap) break;
        if (blk && !first_head) {  // restart on the true residual: u = M r, visible to the SpMV below
            __syncthreads();
            apply_block(r, u, ug);
            sy.barrier();
        }
        first_head = false;
        {
            double v[3] = {0.0, 0.0, 0.0};
            double* m = mb(cur);
            spmv_team<2>(rows, g0, g1, a.team, SrcPlain{ug}, [&](int g, const double* y) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int e = 2 * g + k;
                    const double ue = u[e], re = r[e];
                    w[e] = y[k];
                    if (!blk) {
                        const double me = PRE ? mul(M(e), y[k]) : y[k];
                        m[e] = me;
                        ms[e] = me;
                    }
                    v[0] = add(v[0], mul(re, ue));
                    v[1] = add(v[1], mul(y[k], ue));
                    v[2] = add(v[2], mul(re, re));
                }
            });
            if (blk) {
                __syncthreads();
                apply_block(w, ms, m);
            }
            publish3(v);
            sy.barrier();
        }
        // alpha_{i+1} = gn / (dn - beta gn / alpha_i), beta = gn / gamma, is
        // evaluated as gn / (dn - (gn * ig) * gn) with ig = 1 / (gamma alpha_i):
        // one division per iteration (not three plus a square root), all
        // scalars from q = 1 / (gn den) (below).
        // The convergence test compares squared norms; the history keeps the
        // squared estimates and is rescaled once after the solve.
        double alpha = 0.0, ig = 0.0, igam = 0.0;
        bool first = true;
        const long long hstart = hlen;
        const double thr = mul(mul(a.tol, bnorm), mul(a.tol, bnorm));
        while (true) {
            // n = A m (gathered) || fold the partials of the current vectors.
            // The folding warps issue their partial loads first and add them
            // up after their own share of the SpMV, so the fold's round trip
            // hides under the SpMV's (same order as reduce_partials_warp).
            constexpr int kFold = 5;  // partials per lane in flight: G <= 160
            stamp(a, total, 0);
            const int gw = warp - (nwarps - 3);
            double pv[kFold];
            if (gw >= 0) {
                if (G <= 32 * kFold) {
                    const double* src = a.partial + par * pstride + (long long)gw * G;
#pragma unroll
                    for (int j = 0; j < kFold; ++j) pv[j] = lane + 32 * j < G ? __ldcg(src + lane + 32 * j) : 0.0;
                } else {
                    gather3();
                }
            }
            const double* m = mb(cur);
            spmv_team<2>(rows, g0, g1, a.team, SrcPlain{m}, [&](int g, const double* y) {
                ybuf[g - g0] = make_double2(y[0], y[1]);
            });
            if (gw >= 0 && G <= 32 * kFold) {
                double sacc = 0.0;
#pragma unroll
                for (int j = 0; j < kFold; ++j)
                    if (lane + 32 * j < G) sacc = add(sacc, pv[j]);
                sacc = warp_sum(sacc);
                if (lane == 0) co[gw] = sacc;
            }
            __syncthreads();
            stamp(a, total, 1);
            par ^= 1;
            const double gn = co[0], dn = co[1];
            double beta = 0.0, den = dn;
            if (first) {
                if (!(gn > 0.0) || !(dn > 0.0) || !isfinite(gn) || !isfinite(dn)) {
                    status = RAFEM_ERR_BREAKDOWN;
                    break;
                }
            } else {
                ++total;
                const double rr = co[2];
                if (cta == 0 && tid == 0 && hlen < a.hist_cap) a.hist[hlen] = rr;
                ++hlen;
                if (rr <= thr || total >= a.cap) break;
                beta = gn * igam;
                den = fma(-(gn * ig), gn, dn);
                if (!(gn > 0.0) || !(den > 0.0) || !isfinite(den)) {
                    status = RAFEM_ERR_BREAKDOWN;
                    break;
                }
            }
            // ONE division per iteration: with q = 1 / (gn den),
            // alpha = gn / den = gn^2 q, 1 / gn = den q and 1 / (gn alpha) =
            // den / gn^2 (the next iteration's beta and den).  Two more
            // divisions after the update were 11.5 % of the simulation
            // kernel's stall samples (ncu r2f, scripts/sass_line_stalls.py).
            {
                const double q = 1.0 / (gn * den);
                alpha = (gn * gn) * q;
                igam = den * q;
                ig = (den * igam) * igam;
            }
            double* mn = mb(cur ^ 1);
            double v[3] = {0.0, 0.0, 0.0};
            stamp(a, total, 6);
            for (int e = lo + tid; e < hi; e += blockDim.x) {
                const double ne = (e & 1) ? ybuf[(e >> 1) - g0].y : ybuf[(e >> 1) - g0].x;
                const double me = ms[e], we = w[e], ue = u[e];
                double ze = ne, qe = me, se = we, pe = ue;
                if (!first) {
                    ze = add(ne, mul(beta, z[e]));
                    qe = add(me, mul(beta, q[e]));
                    se = add(we, mul(beta, sv[e]));
                    pe = add(ue, mul(beta, p[e]));
                }
                z[e] = ze;
                q[e] = qe;
                sv[e] = se;
                p[e] = pe;
                const double xn = add(xs[e], mul(alpha, pe));
                xs[e] = xn;
                x[e] = xn;
                const double rn = sub(r[e], mul(alpha, se));
                const double un = sub(ue, mul(alpha, qe));
                const double wn = sub(we, mul(alpha, ze));
                r[e] = rn;
                u[e] = un;
                w[e] = wn;
                if (!blk) {
                    const double mne = PRE ? mul(M(e), wn) : wn;
                    mn[e] = mne;
                    ms[e] = mne;
                } else {
                    yl[e] = mul(M(e), wn);  // y = D^-1 w for the block step below
                }
                v[0] = add(v[0], mul(rn, un));
                v[1] = add(v[1], mul(wn, un));
                v[2] = add(v[2], mul(rn, rn));
            }
            stamp(a, total, 7);
            // the CTA's dot partials: groups of 4 lanes pre-combine theirs
            // (owner dofs sit on threads < 2 * kPipeRows), the 64 group sums
            // per value go through shared memory (`red`, 256 doubles, is not
            // used inside the iteration), and the last three warps each fold
            // one value while the other warps run the block step
            double* tv = red;  // 3 x 64 doubles
            if (tid < 2 * kPipeRows) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    v[j] = add(v[j], __shfl_xor_sync(0xffffffffu, v[j], 1));
                    v[j] = add(v[j], __shfl_xor_sync(0xffffffffu, v[j], 2));
                }
                if ((lane & 3) == 0)
#pragma unroll
                    for (int j = 0; j < 3; ++j) tv[j * (kPipeRows / 2) + (tid >> 2)] = v[j];
            }
            for (int i = blockDim.x + tid; i < 2 * kPipeRows; i += blockDim.x)  // (narrow CTAs)
                if ((i & 3) == 0)
#pragma unroll
                    for (int j = 0; j < 3; ++j) tv[j * (kPipeRows / 2) + (i >> 2)] = 0.0;
            __syncthreads();  // y (block step) and the partials are complete
            stamp(a, total, 2);
            {
                const int gw = warp - (nwarps - 3);
                if (gw >= 0) {
                    const double* t = tv + gw * (kPipeRows / 2) + lane * (kPipeRows / 64);
                    double sacc = 0.0;
#pragma unroll
                    for (int k = 0; k < kPipeRows / 64; ++k) sacc = add(sacc, t[k]);
                    sacc = warp_sum(sacc);
                    if (lane == 0) a.partial[par * pstride + (long long)gw * G + cta] = sacc;
                } else if (blk) {
                    block_rows(w, ms, mn, (nwarps - 3) * 32);
                }
            }
            stamp(a, total, 3);
            cur ^= 1;
            first = false;
            stamp(a, total, 4);
            sy.barrier();
            stamp(a, total, 5);
        }
        if (cta == 0 && tid == 0 && cycles < a.cyc_cap) a.cyc[cycles] = hlen - hstart;
        if (cta == 0) {  // squared estimates of this cycle -> relative residuals
            __syncthreads();
            for (long long h = hstart + tid; h < hlen && h < a.hist_cap; h += blockDim.x)
                a.hist[h] = sqrt(a.hist[h]) / bnorm;
        }
        ++cycles;
        if (status != RAFEM_OK) break;
    }
    if (a.res && cta == 0 && tid == 0) write_result(a.res, total, cycles, hlen, rel, converged, false, status);
    return PcgOut{total, rel, converged ? 1 : 0, status};
}

template <int W, bool PRE, class Mode, class R>
RF_DEV void pcg_body(const KArgs& a, const R& rows) {
    __shared__ double red[32 * 8];
    __shared__ double co[8];
    const int g0 = a.gpart[blockIdx.x], g1 = a.gpart[blockIdx.x + 1];
    int par = 0;
    Sync<Mode> sy{a};
    const double bnorm = prologue<Mode>(a, sy, W * g0, W * g1, co, red, par, 8LL * gridDim.x);
    if (bnorm < 0.0) return;
    if constexpr (W == 2) {
        if (a.pipe) {
            pcg_pipe_core<PRE, Mode>(a, rows, sy, bnorm, co, red, par);
            return;
        }
    }
    pcg_core<W, PRE, Mode>(a, rows, sy, bnorm, co, red, par);
}


// ---------------------------------------------------------------------------
// Streaming PCG for systems far larger than L2 (paired W = 2 layout).
//
// At paper scale the solve is barrier-latency bound and the single-barrier
// form above wins; at >= 1M dofs every iteration is an HBM sweep and the
// on-the-fly operand of pcg_core (four gathered vectors per slot) makes the
// SpMV gather-bound.  This variant materialises u = M^-1 r, so each slot
// gathers ONE double2, and streams the CTA's matrix rows through shared
// memory with TMA bulk copies (TmaSweep below), one thread per node row,
// every gather of a row in flight before its left-to-right accumulation.
// Same Chronopoulos-Gear recurrence, same history / restart / breakdown
// semantics as pcg_core; two grid barriers per iteration instead of one,
// which is ~2 % of an iteration at these sizes.

constexpr int KS = 256;  // threads of the streaming kernels (one node row each per tile)
constexpr int kSweepStages = 2;

// Pipelined sweep over this CTA's node rows [g0, g1) in tiles of KS rows.
// Tile loads are counted over the kernel's lifetime so the mbarrier
// phases stay consistent across sweeps; prefetch() issues the next sweep's
// first tiles early (e.g. before a grid barrier: the matrix is constant).
struct TmaSweep {
    const MatView* A;
    unsigned long long* bar;
    unsigned char* sm;
    int bufbytes, valcap;
    int g0, g1, ntiles;
    unsigned base;  // tiles consumed before the current sweep
    bool pending;   // first tiles of the next sweep already issued
    unsigned long long pol;

    RF_DEV void issue(int j) const {  // tile j of the sweep starting at `base` (thread 0)
        const unsigned k = base + (unsigned)j;
        const int b = (int)(k % kSweepStages);
        const int r0 = g0 + j * KS, r1 = min(g1, r0 + KS);
        const int s0 = __ldg(A->rp + r0), s1 = __ldg(A->rp + r1);
        const int sa = s0 & ~3, se = (s1 + 3) & ~3;
        unsigned char* dst = sm + (size_t)b * bufbytes;
        const unsigned vb = 16u * (unsigned)(s1 - s0), cb = 4u * (unsigned)(se - sa);
        mbar_expect_tx(&bar[b], vb + cb);
        if (vb) tma_load_1d_hint(dst, A->val + 2LL * s0, vb, &bar[b], pol);
        if (cb) tma_load_1d_hint(dst + (size_t)valcap * 16, A->col + sa, cb, &bar[b], pol);
    }
    RF_DEV void prefetch() {
        if (!pending && threadIdx.x == 0) {
            fence_proxy_async();
            for (int j = 0; j < kSweepStages && j < ntiles; ++j) issue(j);
        }
        pending = true;
    }
    // wait out tiles issued by prefetch() when no sweep follows
    RF_DEV void drain() {
        if (pending)
            for (int j = 0; j < kSweepStages && j < ntiles; ++j) {
                const unsigned k = base + (unsigned)j;
                mbar_wait(&bar[k % kSweepStages], (k / kSweepStages) & 1u);
            }
        pending = false;
    }
    // y = A src over this CTA's rows; epi(g, yV, yT) for every owned row.
    template <int CH = 16, class Src, class Epi>
    RF_DEV void run(const Src& src, Epi&& epi) {
        prefetch();
        for (int j = 0; j < ntiles; ++j) {
            const unsigned k = base + (unsigned)j;
            const int b = (int)(k % kSweepStages);
            const int r0 = g0 + j * KS, r1 = min(g1, r0 + KS);
            const int r = r0 + threadIdx.x;
            int a0 = 0, a1 = 0;
            if (r < r1) {
                a0 = __ldg(A->rp + r);
                a1 = __ldg(A->rp + r + 1);
            }
            const int s0 = __ldg(A->rp + r0);
            const int sa = s0 & ~3;
            mbar_wait(&bar[b], (k / kSweepStages) & 1u);
            const double2* sv = reinterpret_cast<const double2*>(sm + (size_t)b * bufbytes);
            const int* sc = reinterpret_cast<const int*>(sm + (size_t)b * bufbytes + (size_t)valcap * 16);
            if (r < r1) {
                double av = 0.0, at = 0.0;
                for (int s = a0; s < a1; s += CH) {
                    int c[CH];
                    double2 xv[CH];
#pragma unroll
                    for (int q = 0; q < CH; ++q)
                        if (s + q < a1) c[q] = sc[s + q - sa];
#pragma unroll
                    for (int q = 0; q < CH; ++q)
                        if (s + q < a1) xv[q] = src.at2(c[q]);
#pragma unroll
                    for (int q = 0; q < CH; ++q)
                        if (s + q < a1) {
                            const double2 vv = sv[s + q - s0];
                            av = add(av, mul(vv.x, xv[q].x));
                            at = add(at, mul(vv.y, xv[q].y));
                        }
                }
                epi(r, av, at);
            }
            __syncthreads();  // stage b fully read
            if (threadIdx.x == 0 && j + kSweepStages < ntiles) {
                fence_proxy_async();
                issue(j + kSweepStages);
            }
        }
        base += (unsigned)ntiles;
        pending = false;
    }
};

RF_DEV TmaSweep make_sweep(const MatView& A, unsigned char* sm, unsigned long long* bar, int g0, int g1,
                           int bufbytes, int valcap) {
    if (threadIdx.x == 0) {
        for (int b = 0; b < kSweepStages; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
    __syncthreads();
    TmaSweep t;
    t.A = &A;
    t.bar = bar;
    t.sm = sm;
    t.bufbytes = bufbytes;
    t.valcap = valcap;
    t.g0 = g0;
    t.g1 = g1;
    t.ntiles = g1 > g0 ? (g1 - g0 + KS - 1) / KS : 0;
    t.base = 0;
    t.pending = false;
    t.pol = l2_policy_evict_first();
    return t;
}

// Gathered operand inside a persistent kernel: coherent L1-cached loads
// (never ld.global.nc: the vector is rewritten between sweeps).
struct SrcVec2 {
    const double* v;
    RF_DEV double2 at2(int c) const { return __ldca(reinterpret_cast<const double2*>(v) + c); }
};

// Phase A of pcg_stream_kernel (owner rows, no gathers): p = u + beta p,
// s = w + beta s, x += alpha p, r -= alpha s, u = M r; partials r.u, r.r
// into v[0], v[2].  Kept out of line so its U-deep load batches get their
// own register budget instead of competing with the inlined sweeps.
template <bool PRE, int U>
__device__ __noinline__ double2 phase_a(int g0, int g1, bool first, double alpha, double beta,
                                        double2* __restrict__ x, double2* __restrict__ r, double2* __restrict__ u,
                                        double2* __restrict__ w, double2* __restrict__ s, double2* __restrict__ p,
                                        const double2* __restrict__ mv) {
    const int tid = threadIdx.x;
    double v[3] = {0.0, 0.0, 0.0};
    auto M = [&](int g) { return PRE ? __ldg(mv + g) : make_double2(1.0, 1.0); };
    // U nodes per thread per trip: 7U independent 16-B loads in
    // flight per thread (one CTA of 256 threads per SM is too few
    // warps to cover HBM latency one node at a time)
    for (int gb = g0 + tid; gb < g1; gb += U * KS) {
        double2 uo[U], wo[U], m[U], po[U], so[U], xo[U], ro[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int g = gb + k * KS;
            if (g < g1) {
                uo[k] = u[g];
                wo[k] = w[g];
                m[k] = M(g);
                xo[k] = x[g];
                ro[k] = r[g];
                if (!first) {
                    po[k] = p[g];
                    so[k] = s[g];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int g = gb + k * KS;
            if (g < g1) {
                double2 pn = uo[k], sn = wo[k];
                if (!first) {
                    pn = make_double2(add(uo[k].x, mul(beta, po[k].x)), add(uo[k].y, mul(beta, po[k].y)));
                    sn = make_double2(add(wo[k].x, mul(beta, so[k].x)), add(wo[k].y, mul(beta, so[k].y)));
                }
                x[g] = make_double2(add(xo[k].x, mul(alpha, pn.x)), add(xo[k].y, mul(alpha, pn.y)));
                const double2 rn =
                    make_double2(sub(ro[k].x, mul(alpha, sn.x)), sub(ro[k].y, mul(alpha, sn.y)));
                const double2 un = PRE ? make_double2(mul(m[k].x, rn.x), mul(m[k].y, rn.y)) : rn;
                p[g] = pn;
                s[g] = sn;
                r[g] = rn;
                u[g] = un;
                v[0] = add(add(v[0], mul(rn.x, un.x)), mul(rn.y, un.y));
                v[2] = add(add(v[2], mul(rn.x, rn.x)), mul(rn.y, rn.y));
            }
        }
    }
    return make_double2(v[0], v[2]);
}

template <bool PRE, int CH, int U>
__global__ void __launch_bounds__(KS, 1) pcg_stream_kernel(KArgs a, int bufbytes, int valcap) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ __align__(8) unsigned long long bar[kSweepStages];
    __shared__ double red[32 * 8];
    __shared__ double co[8];
    const int cta = blockIdx.x, tid = threadIdx.x;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const long long pstride = 8LL * gridDim.x;
    int par = 0;
    Sync<GridMode> sy{a};
    TmaSweep sw = make_sweep(a.A, dsm, bar, g0, g1, bufbytes, valcap);
    sw.prefetch();  // overlaps the ||b|| reduction
    const double bnorm = prologue<GridMode>(a, sy, 2 * g0, 2 * g1, co, red, par, pstride);
    if (bnorm < 0.0) {
        sw.drain();  // no bulk copy may outlive the CTA
        return;
    }
    double2* x = reinterpret_cast<double2*>(a.x);
    const double2* b = reinterpret_cast<const double2*>(a.b);
    const double2* mv = reinterpret_cast<const double2*>(a.minv);
    double2* r = reinterpret_cast<double2*>(a.r);
    double2* u = reinterpret_cast<double2*>(a.z);
    double2* w = reinterpret_cast<double2*>(a.w0);
    double2* s = reinterpret_cast<double2*>(a.p1);
    double2* p = reinterpret_cast<double2*>(a.p0);
    auto M = [&](int g) { return PRE ? __ldg(mv + g) : make_double2(1.0, 1.0); };
    auto round = [&](double (&v)[3], int nv) {
        sy.template reduce<3>(v, nv, a.partial + par * pstride, co, red);
        par ^= 1;
    };

    long long total = 0, cycles = 0, hlen = 0;
    bool converged = false;
    double rel = INFINITY;
    int status = RAFEM_OK;
    while (true) {
        double gamma, alpha, beta = 0.0;
        {  // r = b - A x, u = M r ; (r.u, -, r.r)
            double v[3] = {0.0, 0.0, 0.0};
            sw.template run<CH>(SrcVec2{a.x}, [&](int g, double yv, double yt) {
                const double2 bb = b[g], m = M(g);
                const double2 rr = make_double2(sub(bb.x, yv), sub(bb.y, yt));
                const double2 uu = PRE ? make_double2(mul(m.x, rr.x), mul(m.y, rr.y)) : rr;
                r[g] = rr;
                u[g] = uu;
                v[0] = add(add(v[0], mul(rr.x, uu.x)), mul(rr.y, uu.y));
                v[2] = add(add(v[2], mul(rr.x, rr.x)), mul(rr.y, rr.y));
            });
            sw.prefetch();
            round(v, 3);
        }
        rel = sqrt(co[2]) / bnorm;
        if (rel <= a.tol) {
            converged = true;
            break;
        }
        if (total >= a.cap) break;
        gamma = co[0];
        {  // w = A u ; (w.u)
            double v[3] = {0.0, 0.0, 0.0};
            sw.template run<CH>(SrcVec2{a.z}, [&](int g, double yv, double yt) {
                const double2 uu = __ldca(u + g);
                w[g] = make_double2(yv, yt);
                v[0] = add(add(v[0], mul(yv, uu.x)), mul(yt, uu.y));
            });
            round(v, 1);
            if (!(gamma > 0.0) || !(co[0] > 0.0) || !isfinite(gamma) || !isfinite(co[0])) {
                status = RAFEM_ERR_BREAKDOWN;
                break;
            }
            alpha = gamma / co[0];
        }
        const long long hstart = hlen;
        bool first = true;
        while (true) {
            double v[3] = {0.0, 0.0, 0.0};
            // phase A (owner rows): p = u + beta p, s = w + beta s, x += alpha p,
            // r -= alpha s, u = M r ; partials (r.u, -, r.r)
            {
                const double2 pa = phase_a<PRE, U>(g0, g1, first, alpha, beta, x, r, u, w, s, p, mv);
                v[0] = pa.x;
                v[2] = pa.y;
            }
            sw.prefetch();
            sy.barrier();
            // phase B: w = A u ; partial (w.u)
            sw.template run<CH>(SrcVec2{a.z}, [&](int g, double yv, double yt) {
                const double2 uu = __ldca(u + g);
                w[g] = make_double2(yv, yt);
                v[1] = add(add(v[1], mul(yv, uu.x)), mul(yt, uu.y));
            });
            sw.prefetch();
            round(v, 3);
            ++total;
            const double est = sqrt(co[2]) / bnorm;
            if (cta == 0 && tid == 0 && hlen < a.hist_cap) a.hist[hlen] = est;
            ++hlen;
            if (est <= a.tol || total >= a.cap) break;
            const double gnew = co[0];
            const double bnew = gnew / gamma;
            const double den = co[1] - bnew * gnew / alpha;
            if (!(gnew > 0.0) || !(den > 0.0) || !isfinite(den)) {
                status = RAFEM_ERR_BREAKDOWN;
                break;
            }
            alpha = gnew / den;
            beta = bnew;
            gamma = gnew;
            first = false;
        }
        if (cta == 0 && tid == 0 && cycles < a.cyc_cap) a.cyc[cycles] = hlen - hstart;
        ++cycles;
        if (status != RAFEM_OK) break;
    }
    sw.drain();
    if (a.res && cta == 0 && tid == 0) write_result(a.res, total, cycles, hlen, rel, converged, false, status);
}

// ---------------------------------------------------------------------------
// kernels

// A CTA's matrix slice staged in shared memory (constant for the solve):
// dynamic smem = [Hessenberg scratch | value slice | column slice | rp slice]
template <int W>
RF_DEV Rows<W, true, false> cluster_rows(const KArgs& a, double* dyn) {
    const int g0 = a.gpart[blockIdx.x], g1 = a.gpart[blockIdx.x + 1];
    const int ns = __ldg(a.A.rp + g1) - __ldg(a.A.rp + g0);
    double* sval = dyn + a.hess_smem;
    int* scol = reinterpret_cast<int*>(sval + (long long)W * ns);
    int* srp = scol + ((ns + 3) & ~3);
    stage_slice<W>(a.A, g0, g1, sval, scol, srp);
    return Rows<W, true, false>{srp, scol, sval, g0};
}

// Grid mode; MS selects the matrix source: 0 read-only global loads,
// 1 evict-first streaming loads (matrix larger than L2), 2 slice in smem.
template <int W, bool PRE, int MS>
__global__ void __launch_bounds__(KT, 1) gmres_grid_kernel(KArgs a) {
    extern __shared__ __align__(16) double dyn[];
    if constexpr (MS == 2) {
        const auto rows = cluster_rows<W>(a, dyn);
        gmres_body<W, PRE, GridMode>(a, rows, dyn);
    } else {
        const Rows<W, false, MS == 1> rows{a.A.rp, a.A.col, a.A.val, 0};
        gmres_body<W, PRE, GridMode>(a, rows, dyn);
    }
}

template <int W, bool PRE, int MS>
__global__ void __launch_bounds__(KT, 1) pcg_grid_kernel(KArgs a) {
    extern __shared__ __align__(16) double dyn[];
    if constexpr (MS == 2) {
        const auto rows = cluster_rows<W>(a, dyn);
        pcg_body<W, PRE, GridMode>(a, rows);
    } else {
        const Rows<W, false, MS == 1> rows{a.A.rp, a.A.col, a.A.val, 0};
        pcg_body<W, PRE, GridMode>(a, rows);
    }
}

template <int W, bool PRE>
__global__ void __launch_bounds__(KT, 1) gmres_cluster_kernel(KArgs a) {
    extern __shared__ __align__(16) double dyn[];
    const auto rows = cluster_rows<W>(a, dyn);
    gmres_body<W, PRE, ClusterMode>(a, rows, dyn);
}

template <int W, bool PRE>
__global__ void __launch_bounds__(KTC, 1) pcg_cluster_kernel(KArgs a) {
    extern __shared__ __align__(16) double dyn[];
    const auto rows = cluster_rows<W>(a, dyn);
    pcg_body<W, PRE, ClusterMode>(a, rows);
}

// Balanced partition of row groups: CTA c starts at the first group whose
// weight prefix (slots + groups) reaches c/G of the total.
__global__ void partition_kernel(const int* rp, int ngroups, int G, int* gpart, int by_rows) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > G) return;
    if (c == 0) {
        gpart[0] = 0;
        return;
    }
    if (c == G) {
        gpart[G] = ngroups;
        return;
    }
    if (by_rows) {
        gpart[c] = (int)((long long)ngroups * c / G);
        return;
    }
    const long long total = (long long)rp[ngroups] + ngroups;
    const long long target = (total * c + G - 1) / G;
    int lo = 0, hi = ngroups;  // first g with rp[g] + g >= target
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((long long)rp[mid] + mid >= target)
            hi = mid;
        else
            lo = mid + 1;
    }
    gpart[c] = lo;
}

// minv = 1 / stored diagonal (solver.py:413-418, sparse.py:121-128).
template <int W>
__global__ void jacobi_kernel(MatView A, double* minv, int* flag) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= A.ngroups) return;
    double d[W];
#pragma unroll
    for (int w = 0; w < W; ++w) d[w] = 0.0;
    for (int s = A.rp[g]; s < A.rp[g + 1]; ++s) {
        if (A.col[s] == g) {
#pragma unroll
            for (int w = 0; w < W; ++w) d[w] = A.val[(long long)s * W + w];
        }
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
        if (d[w] == 0.0) atomicOr(flag, 1);
        minv[W * g + w] = 1.0 / d[w];
    }
}

template <int W, bool STREAM>
__global__ void __launch_bounds__(256) spmv_kernel(MatView A, const double* __restrict__ x,
                                                   double* __restrict__ y) {
    const int g0 = blockIdx.x * blockDim.x;
    const int g1 = min(A.ngroups, g0 + (int)blockDim.x);
    const Rows<W, false, STREAM> rows{A.rp, A.col, A.val, 0};
    spmv_groups<W>(rows, g0, g1, SrcPlain{x}, [&](int g, const double* yy) {
        if (W == 1) {
            y[g] = yy[0];
        } else {
            reinterpret_cast<double2*>(y)[g] = make_double2(yy[0], yy[1]);
        }
    });
}

// Bandwidth-bound SpMV for paired matrices larger than L2: each CTA walks
// tiles of `tr` node rows; one elected thread streams a tile's contiguous
// slot data (double2 values + int32 columns) into shared memory with 1-D
// TMA bulk copies completing on an mbarrier, double-buffered so the next
// tile's copy overlaps this tile's compute.  Threads then sum their row left
// to right from shared memory (bit-identical to sparse.py:217-218) while the
// x gathers hit L2.  The matrix never passes through registers on its way
// in, and no thread waits on a column load before issuing its gathers.
__global__ void __launch_bounds__(256, 1) spmv_tma_kernel(MatView A, const double* __restrict__ x,
                                                          double* __restrict__ y, int tr, int valcap,
                                                          int bufbytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[2];
    const int N = A.ngroups;
    const int tiles = (N + tr - 1) / tr;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int t, int b) {
        const int r0 = t * tr, r1 = min(N, r0 + tr);
        const int s0 = __ldg(A.rp + r0), s1 = __ldg(A.rp + r1);
        const int sa = s0 & ~3, se = (s1 + 3) & ~3;
        unsigned char* base = sm + (size_t)b * bufbytes;
        const unsigned vb = 16u * (unsigned)(s1 - s0), cb = 4u * (unsigned)(se - sa);
        mbar_expect_tx(&bar[b], vb + cb);
        if (vb) tma_load_1d(base, A.val + 2LL * s0, vb, &bar[b]);
        if (cb) tma_load_1d(base + (size_t)valcap * 16, A.col + sa, cb, &bar[b]);
    };
    int i = 0;
    if (threadIdx.x == 0 && (int)blockIdx.x < tiles) issue(blockIdx.x, 0);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        const int tn = t + gridDim.x;
        if (threadIdx.x == 0 && tn < tiles) {
            fence_proxy_async();  // earlier generic reads of buffer b^1 before the async overwrite
            issue(tn, b ^ 1);
        }
        mbar_wait(&bar[b], (unsigned)(i >> 1) & 1u);
        const int r0 = t * tr, r1 = min(N, r0 + tr);
        const int s0 = __ldg(A.rp + r0);
        const int sa = s0 & ~3;
        const double2* sv = reinterpret_cast<const double2*>(sm + (size_t)b * bufbytes);
        const int* sc = reinterpret_cast<const int*>(sm + (size_t)b * bufbytes + (size_t)valcap * 16);
        for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            const int a0 = __ldg(A.rp + r), a1 = __ldg(A.rp + r + 1);
            double av = 0.0, at = 0.0;
            for (int s = a0; s < a1; s += 4) {
                double2 xv[4], vv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (s + j < a1) {
                        vv[j] = sv[s + j - s0];
                        xv[j] = __ldg(x2 + sc[s + j - sa]);
                    }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (s + j < a1) {
                        av = add(av, mul(vv[j].x, xv[j].x));
                        at = add(at, mul(vv[j].y, xv[j].y));
                    }
            }
            reinterpret_cast<double2*>(y)[r] = make_double2(av, at);
        }
        __syncthreads();
    }
}

// Deeper pipeline of the same idea: ST stages of NT-row tiles (one thread
// per node row), so ST-1 tile loads stay in flight while a tile is summed,
// and each row issues up to CH operand gathers before its first
// accumulation (a Kuhn-mesh row has <= 15 slots: one L2 round trip per
// row instead of one per 4 slots).  The accumulation order is still the
// row's stored order, left to right, so y stays bit-identical to
// sparse.py:217-218.  HINT marks the streamed matrix evict-first in L2 so
// the gathered x keeps its lines.
//
// CLS: the matrix has stencil classes (MatView::cls): a row's columns are
// row + cls_off[class][k], so only the values are streamed (16 of the 20
// bytes per slot) and the columns come from a shared-memory table.
template <int NT, int ST, int CH, bool HINT, bool CLS>
__global__ void __launch_bounds__(NT, 1) spmv_tma_pipe_kernel(MatView A, const double* __restrict__ x,
                                                              double* __restrict__ y, int valcap, int bufbytes,
                                                              int xpf) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[ST];
    int* soff = reinterpret_cast<int*>(sm + (size_t)ST * bufbytes);  // CLS: the class table after the stages
    const int N = A.ngroups;
    const int tiles = (N + NT - 1) / NT;
    const int mine = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (CLS)
        for (int k = threadIdx.x; k < A.ncls * kClsWidth; k += NT) soff[k] = __ldg(A.cls_off + k);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
    __syncthreads();
    unsigned long long pol = 0;
    if (HINT) pol = l2_policy_evict_first();
    auto issue = [&](int i) {  // i-th tile of this CTA into stage i % ST
        const int t = blockIdx.x + i * gridDim.x;
        const int b = i % ST;
        const int r0 = t * NT, r1 = min(N, r0 + NT);
        const int s0 = __ldg(A.rp + r0), s1 = __ldg(A.rp + r1);
        const int sa = s0 & ~3, se = (s1 + 3) & ~3;
        unsigned char* base = sm + (size_t)b * bufbytes;
        const unsigned vb = 16u * (unsigned)(s1 - s0), cb = CLS ? 0u : 4u * (unsigned)(se - sa);
        mbar_expect_tx(&bar[b], vb + cb);
        if (HINT) {
            if (vb) tma_load_1d_hint(base, A.val + 2LL * s0, vb, &bar[b], pol);
            if (cb) tma_load_1d_hint(base + (size_t)valcap * 16, A.col + sa, cb, &bar[b], pol);
        } else {
            if (vb) tma_load_1d(base, A.val + 2LL * s0, vb, &bar[b]);
            if (cb) tma_load_1d(base + (size_t)valcap * 16, A.col + sa, cb, &bar[b]);
        }
        // the tile's own x rows into L2 a tile-time before its gathers need
        // them: a wave of tiles gathers mostly within the wave's own rows
        // (box stencils reach one plane), so a cold x is not a DRAM round
        // trip per tile
        if (xpf && r1 > r0) prefetch_l2_bulk(x + 2LL * r0, 16u * (unsigned)(r1 - r0));
    };
    // programmatic dependent launch (no-ops otherwise): let the next kernel
    // in the stream start its prologue as this grid's CTAs retire, and
    // stream this grid's first matrix tiles (constant data) before waiting
    // for the previous kernel, which may still be writing x or reading y
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0)
        for (int i = 0; i < ST && i < mine; ++i) issue(i);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int i = 0; i < mine; ++i) {
        const int b = i % ST;
        const int t = blockIdx.x + i * gridDim.x;
        const int r0 = t * NT, r1 = min(N, r0 + NT);
        const int r = r0 + threadIdx.x;
        int a0 = 0, a1 = 0, cid = 0;
        if (r < r1) {
            a0 = __ldg(A.rp + r);
            a1 = __ldg(A.rp + r + 1);
            if (CLS) cid = __ldg(A.cls + r);
        }
        const int s0 = __ldg(A.rp + r0);
        const int sa = s0 & ~3;
        mbar_wait(&bar[b], (unsigned)(i / ST) & 1u);
        const double2* sv = reinterpret_cast<const double2*>(sm + (size_t)b * bufbytes);
        const int* sc = reinterpret_cast<const int*>(sm + (size_t)b * bufbytes + (size_t)valcap * 16);
        const int* so = soff + cid * kClsWidth - a0;  // CLS: column of slot s is r + so[s]
        if (r < r1) {
            double av = 0.0, at = 0.0;
            for (int s = a0; s < a1; s += CH) {
                int c[CH];
                double2 xv[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (s + j < a1) c[j] = CLS ? r + so[s + j] : sc[s + j - sa];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (s + j < a1) xv[j] = __ldg(x2 + c[j]);
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (s + j < a1) {
                        const double2 vv = sv[s + j - s0];
                        av = add(av, mul(vv.x, xv[j].x));
                        at = add(at, mul(vv.y, xv[j].y));
                    }
            }
            __stcs(reinterpret_cast<double2*>(y) + r, make_double2(av, at));  // evict-first: keep x in L2
        }
        __syncthreads();  // every thread is done with stage b
        if (threadIdx.x == 0 && i + ST < mine) {
            fence_proxy_async();  // generic reads of stage b before the async overwrite
            issue(i + ST);
        }
    }
}

// delta = max |xn - xo| / max(1, |xo|)  (fem.py:527-528); nonnegative
// doubles order like their bit patterns, so an integer atomicMax is an
// exact, order-independent max.
__global__ void delta_kernel(const double* xn, const double* xo, int n, unsigned long long* out) {
    __shared__ double red[32];
    double v = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double o = xo[i];
        const double d = fabs(sub(xn[i], o)) / fmax(1.0, fabs(o));
        v = (d > v || d != d) ? d : v;
    }
    v = block_max(v, red);
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------------------
// host launchers

// Per row-block boundary c <= G: gpart[c], rp[gpart[c]] and, with the
// optional arrays, inc_ptr[gpart[c]] and slot_ptr[rp[gpart[c]]]; `nout`
// of these rows (each G + 1 ints) are written to out.
__global__ void block_bounds_kernel(const int* gpart, int G, const int* rp, const int* inc_ptr, const int* slot_ptr,
                                    int* out, int nout) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > G) return;
    const int g = gpart[c], s = rp[g];
    const int n = G + 1;
    out[c] = g;
    out[n + c] = s;
    if (nout > 2) out[2 * n + c] = inc_ptr ? inc_ptr[g] : 0;
    if (nout > 3) out[3 * n + c] = slot_ptr ? slot_ptr[s] : 0;
}

// The grid-barrier counter lives after the 2 x G x 8 barrier slots of
// ws_flags.  Opt-in (RAFEM_CNT_SYNC=1): in the microbenchmark it beats
// cooperative_groups' grid sync by 0.8 us per round when every CTA has
// just written global data, but inside the fused simulation it measured
// 4.71 vs 4.60 us per PCG iteration (r1j), so the default stays cg.
static unsigned long long* grid_counter(rafem_ctx*, unsigned long long* flags, int G) {
    const char* e = getenv("RAFEM_CNT_SYNC");
    return !(e && e[0] == '1') ? nullptr : flags + 2 * 8 * (size_t)std::max(G, 1);
}

int jacobi_minv(rafem_ctx* ctx, const MatView& A, double* minv_dev, int* flag_dev) {
    RF_CUDA_TRY(ctx, cudaMemsetAsync(flag_dev, 0, sizeof(int), ctx->stream));
    const int blocks = (A.ngroups + 255) / 256;
    if (blocks > 0) {
        if (A.W == 1)
            jacobi_kernel<1><<<blocks, 256, 0, ctx->stream>>>(A, minv_dev, flag_dev);
        else
            jacobi_kernel<2><<<blocks, 256, 0, ctx->stream>>>(A, minv_dev, flag_dev);
        ctx->launches++;
        RF_CUDA_TRY(ctx, cudaGetLastError());
    }
    return RAFEM_OK;
}

// Pipelined TMA SpMV launch; RAFEM_ERR_UNSUPPORTED when no configuration
// fits the row degree (the caller then uses the two-stage kernel).
// RAFEM_SPMV_CFG="NT,ST,HINT[,CPS]" selects a configuration and CTAs per SM
// (tuning only).
struct PipeCfg {
    int nt, st, hint;
    const void* fn;
    const void* fn_cls;
};
template <int NT, int ST, int HINT>
static PipeCfg pipe_cfg() {
    return {NT, ST, HINT, (const void*)spmv_tma_pipe_kernel<NT, ST, 16, HINT != 0, false>,
            (const void*)spmv_tma_pipe_kernel<NT, ST, 16, HINT != 0, true>};
}
static int spmv_pipe_launch(rafem_ctx* ctx, const MatView& A, const double* x_dev, double* y_dev) {
    static const PipeCfg cfgs[] = {pipe_cfg<256, 2, 1>(), pipe_cfg<128, 4, 1>(), pipe_cfg<192, 3, 1>(),
                                   pipe_cfg<256, 3, 1>(), pipe_cfg<384, 2, 1>(), pipe_cfg<512, 2, 1>(),
                                   pipe_cfg<128, 3, 1>(), pipe_cfg<96, 4, 1>(),  pipe_cfg<128, 2, 1>(),
                                   pipe_cfg<64, 4, 1>(),  pipe_cfg<192, 2, 1>()};
    int cps = 1;  // CTAs per SM
    const char* nc = getenv("RAFEM_NO_CLASSES");
    const bool cls = A.cls && A.ncls > 0 && A.maxdeg <= kClsWidth && !(nc && nc[0] == '1');
    auto buf_bytes = [&](int t) {
        return t * A.maxdeg * 16 + (cls ? 0 : ((t * A.maxdeg + 8) * 4 + 15) / 16 * 16);
    };
    const size_t tab = cls ? sizeof(int) * (size_t)A.ncls * kClsWidth : 0;
    const size_t budget = kSmemBudget - tab;
    // default: the widest configuration whose stages fit (measured on B200,
    // cold L2: 384 x 2 with stencil classes 411 us at 16M dofs, 256 x 2 521 us)
    // (measured r1j, cold L2: two CTAs per SM of 192 x 2 405 us at 16M dofs,
    // 36.9 us at 1M; one CTA of 384 x 2 416 / 37.6 us)
    auto fits = [&](int i, int k) {
        const size_t sm = (size_t)cfgs[i].st * buf_bytes(cfgs[i].nt);
        return sm <= budget && (size_t)k * (sm + tab + 1024) <= 228 * 1024;
    };
    int want = -1;
    for (auto [i, k] : {std::pair{10, 2}, std::pair{4, 1}, std::pair{0, 1}, std::pair{1, 1}}) {
        if (fits(i, k)) {
            want = i;
            cps = k;
            break;
        }
    }
    if (want < 0) return RAFEM_ERR_UNSUPPORTED;
    if (const char* env = getenv("RAFEM_SPMV_CFG")) {
        int nt = 0, st = 0, hint = 1, ec = 1;
        if (sscanf(env, "%d,%d,%d,%d", &nt, &st, &hint, &ec) >= 2) {
            cps = std::max(1, ec);
            want = -1;
            for (int i = 0; i < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++i)
                if (cfgs[i].nt == nt && cfgs[i].st == st && cfgs[i].hint == hint) want = i;
            if (want < 0) return RAFEM_ERR_UNSUPPORTED;
        }
    }
    const PipeCfg& c = cfgs[want];
    const void* fn = cls ? c.fn_cls : c.fn;
    const size_t smem = (size_t)c.st * buf_bytes(c.nt) + tab;
    if (smem > kSmemBudget) return RAFEM_ERR_UNSUPPORTED;
    RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int tiles = (A.ngroups + c.nt - 1) / c.nt;
    if ((size_t)cps * (smem + 1024) > 228 * 1024) return RAFEM_ERR_UNSUPPORTED;
    const int grid = std::min(tiles, ctx->sm_count * cps);
    int valcap = c.nt * A.maxdeg, bufbytes = buf_bytes(c.nt);
    MatView Av = A;
    const double* xp = x_dev;
    double* yp = y_dev;
    // per-tile bulk L2 prefetch of the tile's own x rows (default on;
    // RAFEM_XPF=0 turns it off) — measured r2h, cold L2, 192 x 2 tiles, three
    // runs: C3 36.9 -> 35.4-35.7 us, C4 400.4 -> 388.0-388.5 us (an earlier
    // r2b sweep had C4 slower, 401 -> 416; profiles/r2h_spmv_xpf.txt)
    // (a per-gather L2 prefetch of the next tile's columns — computable from
    // the stencil classes before its matrix tile lands — measured slower at
    // C3: 38.9 vs 37.5 us; profiles/r2b_spmv_x_prefetch_sweep.txt)
    const char* xe = getenv("RAFEM_XPF");
    int xpf = (xe && xe[0] == '0') ? 0 : 1;
    void* args[] = {&Av, &xp, &yp, &valcap, &bufbytes, &xpf};
    if (ctx->spmv_pdl) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(c.nt);
        lc.dynamicSmemBytes = smem;
        lc.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        RF_CUDA_TRY(ctx, cudaLaunchKernelExC(&lc, fn, args));
    } else {
        RF_CUDA_TRY(ctx, cudaLaunchKernel(fn, dim3(grid), dim3(c.nt), args, smem, ctx->stream));
    }
    ctx->launches++;
    return RAFEM_OK;
}

static bool streams_matrix(const MatView& A) { return A.slots * (4 + 8LL * A.W) > (48LL << 20); }

int spmv_launch(rafem_ctx* ctx, const MatView& A, const double* x_dev, double* y_dev) {
    const int blocks = (A.ngroups + 255) / 256;
    if (blocks == 0) return RAFEM_OK;
    const bool stream = streams_matrix(A);
    const char* no_tma = getenv("RAFEM_NO_TMA_SPMV");
    if (A.W == 2 && stream && A.maxdeg > 0 && !(no_tma && no_tma[0] == '1')) {
        if (int rc = spmv_pipe_launch(ctx, A, x_dev, y_dev); rc != RAFEM_ERR_UNSUPPORTED) return rc;
        int tr = 256;
        // per buffer: tr*maxdeg double2 values + (tr*maxdeg + 8) int32 columns, two buffers
        auto buf_bytes = [&](int t) { return t * A.maxdeg * 16 + ((t * A.maxdeg + 8) * 4 + 15) / 16 * 16; };
        while (tr > 32 && 2 * (size_t)buf_bytes(tr) > kSmemBudget) tr /= 2;
        if (2 * (size_t)buf_bytes(tr) <= kSmemBudget) {
            const int valcap = tr * A.maxdeg;
            const size_t smem = 2 * (size_t)buf_bytes(tr);
            RF_CUDA_TRY(ctx, cudaFuncSetAttribute(spmv_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int tiles = (A.ngroups + tr - 1) / tr;
            const int grid = std::min(tiles, ctx->sm_count);
            spmv_tma_kernel<<<grid, 256, smem, ctx->stream>>>(A, x_dev, y_dev, tr, valcap, buf_bytes(tr));
            ctx->launches++;
            RF_CUDA_TRY(ctx, cudaGetLastError());
            return RAFEM_OK;
        }
    }
    if (A.W == 1) {
        if (stream)
            spmv_kernel<1, true><<<blocks, 256, 0, ctx->stream>>>(A, x_dev, y_dev);
        else
            spmv_kernel<1, false><<<blocks, 256, 0, ctx->stream>>>(A, x_dev, y_dev);
    } else {
        if (stream)
            spmv_kernel<2, true><<<blocks, 256, 0, ctx->stream>>>(A, x_dev, y_dev);
        else
            spmv_kernel<2, false><<<blocks, 256, 0, ctx->stream>>>(A, x_dev, y_dev);
    }
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int vec_delta_launch(rafem_ctx* ctx, const double* xn, const double* xo, int n, double* out_dev) {
    RF_CUDA_TRY(ctx, cudaMemsetAsync(out_dev, 0, sizeof(double), ctx->stream));
    const int blocks = std::max(1, std::min((n + 255) / 256, ctx->sm_count * 4));
    delta_kernel<<<blocks, 256, 0, ctx->stream>>>(xn, xo, n, reinterpret_cast<unsigned long long*>(out_dev));
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

template <int W, bool PRE, int MS>
static const void* grid_kernel_ms(bool gmres) {
    return gmres ? (const void*)gmres_grid_kernel<W, PRE, MS> : (const void*)pcg_grid_kernel<W, PRE, MS>;
}
template <int W, bool PRE>
static const void* grid_kernel(bool gmres, int ms) {
    if (ms == 2) return grid_kernel_ms<W, PRE, 2>(gmres);
    return ms == 1 ? grid_kernel_ms<W, PRE, 1>(gmres) : grid_kernel_ms<W, PRE, 0>(gmres);
}
template <int W, bool PRE>
static const void* cluster_kernel(bool gmres) {
    return gmres ? (const void*)gmres_cluster_kernel<W, PRE> : (const void*)pcg_cluster_kernel<W, PRE>;
}
static const void* select_grid(bool gmres, int W, bool pre, int ms) {
    if (W == 1) return pre ? grid_kernel<1, true>(gmres, ms) : grid_kernel<1, false>(gmres, ms);
    return pre ? grid_kernel<2, true>(gmres, ms) : grid_kernel<2, false>(gmres, ms);
}
static const void* select_cluster(bool gmres, int W, bool pre) {
    if (W == 1) return pre ? cluster_kernel<1, true>(gmres) : cluster_kernel<1, false>(gmres);
    return pre ? cluster_kernel<2, true>(gmres) : cluster_kernel<2, false>(gmres);
}

// Partition for G CTAs (device) and, for the cluster path, the largest
// per-CTA slice in bytes (host).  Cached per pattern id.
struct PartInfo {
    int* gpart = nullptr;
    size_t max_slice = 0;
    int max_groups = 0;
};

// by_rows: equal row-group counts (ceil(ngroups / G) at most per CTA) for
// the pipelined PCG, whose SpMV phase costs one team pass per 256 / team
// rows: a slot-balanced split hands the CTAs with many short boundary rows
// a second pass (measured: 79-row CTAs set the iteration time at mesh B).
// The pipelined PCG runs (RAFEM_PIPE=0 selects the single-reduction kernel)
static bool pipe_rows(bool gm, int W, int ngroups, int G) {
    const char* pe = getenv("RAFEM_PIPE");
    return !gm && W == 2 && (ngroups + G - 1) / G <= kPipeRows && !(pe && pe[0] == '0');
}

static int partition(rafem_ctx* ctx, const MatView& A, int G, bool need_slice, PartInfo& out,
                     bool by_rows = false) {
    // cache hit?
    for (auto& e : ctx->part_cache) {
        if (A.pattern_id && e.pattern_id == A.pattern_id && e.G == G && e.rp == A.rp && e.by_rows == by_rows &&
            (!need_slice || e.max_slice > 0)) {
            out.gpart = e.gpart;
            out.max_slice = e.max_slice;
            out.max_groups = e.max_groups;
            return RAFEM_OK;
        }
    }
    int* gpart = nullptr;
    if (A.pattern_id) {
        RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&gpart, sizeof(int) * (G + 1)));
    } else {
        if (int rc = ensure(ctx, ctx->ws_part, sizeof(int) * (size_t)(G + 1))) return rc;
        gpart = static_cast<int*>(ctx->ws_part.p);
    }
    partition_kernel<<<(G + 1 + 127) / 128, 128, 0, ctx->stream>>>(A.rp, A.ngroups, G, gpart, by_rows ? 1 : 0);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    size_t max_slice = 0;
    int max_groups = 0;
    if (need_slice) {
        // the block boundaries and their row starts in one copy (gathered on
        // the device: G + 1 single-int copies cost ~1 ms of driver calls)
        std::vector<int> hb(2 * (G + 1));
        int* db = nullptr;
        RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&db), sizeof(int) * 2 * (G + 1)));
        block_bounds_kernel<<<(G + 1 + 127) / 128, 128, 0, ctx->stream>>>(gpart, G, A.rp, nullptr, nullptr, db, 2);
        ctx->launches++;
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(hb.data(), db, sizeof(int) * 2 * (G + 1), cudaMemcpyDeviceToHost, ctx->stream));
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        dfree(ctx, db);
        const int* hp = hb.data();
        const int* hr = hb.data() + (G + 1);
        for (int c = 0; c < G; ++c) {
            const size_t ns = (size_t)(hr[c + 1] - hr[c]);
            const size_t ng = (size_t)(hp[c + 1] - hp[c]);
            const size_t bytes = ns * 8 * A.W + ((ns + 3) & ~(size_t)3) * 4 + (ng + 1) * 4;
            max_slice = std::max(max_slice, bytes);
            max_groups = std::max(max_groups, (int)ng);
        }
        max_slice = (max_slice + 15) / 16 * 16;
    }
    if (A.pattern_id) ctx->part_cache.push_back({A.pattern_id, A.rp, G, gpart, max_slice, max_groups, by_rows});
    out.gpart = gpart;
    out.max_slice = max_slice;
    out.max_groups = max_groups;
    return RAFEM_OK;
}

int krylov_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, const double* x0_dev,
                 double* x_dev, const double* minv_dev, const rafem_solver_params& p,
                 KResult* res_dev, int* flag_dev, cudaEvent_t ev_start, cudaEvent_t ev_stop) {
    const int n = A.ngroups * A.W;
    const bool gm = p.method != RAFEM_METHOD_PCG;
    const int m = gm ? p.restart_m : 1;
    const bool pre = p.precondition != RAFEM_PRECOND_NONE;  // block-Jacobi needs the point inverse too
    const bool stream = streams_matrix(A);

    // x starts at x0 (or zero); the kernel never touches x before the first
    // true-residual test, so an exact x0 comes back bitwise (solver.py:448-450)
    if (x0_dev) {
        if (x0_dev != x_dev)
            RF_CUDA_TRY(ctx, cudaMemcpyAsync(x_dev, x0_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        RF_CUDA_TRY(ctx, cudaMemsetAsync(x_dev, 0, sizeof(double) * n, ctx->stream));
    }

    // rotated H, cs, sn, g, y, 2m + 4 reduction results, raw H, two
    // first-pass columns and the gather scratch (gmres_1r_body)
    const long long hess_doubles = gm ? 2LL * (m + 1) * m + 5LL * m + 5 + m + 2LL * (m + 1) + 512 : 0;
    const size_t hess_bytes = (size_t)hess_doubles * 8;

    static const bool timing = [] { const char* e = getenv("RAFEM_HOST_TIMING"); return e && e[0] == '1'; }();
    auto now_us = [] {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double k0 = timing ? now_us() : 0.0;
    // ---- choose the execution mode
    // paper-scale PCG and GMRES: the cluster-resident engine (cluster.cu)
    // when the system fits one cluster's shared memory
    {
        const int crc = cluster_pcg_solve(ctx, A, b_dev, x_dev, minv_dev, p, res_dev, flag_dev, ev_start, ev_stop);
        if (timing && crc != RAFEM_ERR_UNSUPPORTED) std::fprintf(stderr, "  cluster engine %.1f us\n", now_us() - k0);
        if (crc != RAFEM_ERR_UNSUPPORTED) return crc;
    }
    const double k1 = timing ? now_us() : 0.0;
    const void* fn = nullptr;
    size_t smem = 0;
    bool cluster = false, hess_global = false;
    int stream_buf = 0, stream_valcap = 0;
    long long vs_off = 0;
    int vs_ld = 0;
    PartInfo part;
    int G = 0;
    // Grid mode over every SM is the default: measured on B200 (mesh-B
    // analog) a 148-CTA grid with team SpMV beats one 16-CTA cluster by
    // 2.5x despite the costlier barrier.  RAFEM_SOLVER_MODE=cluster selects
    // the cluster-resident variant for experiments.
    const char* force = getenv("RAFEM_SOLVER_MODE");
    const bool try_cluster = p.grid_ctas <= 0 && (force && force[0] == 'c') &&
                             A.slots * (4 + 8LL * A.W) <= (long long)kMaxCluster * (200 << 10);
    if (try_cluster) {
        int C = (int)std::min<long long>(kMaxCluster, std::max<long long>(1, (A.ngroups + 255) / 256));
        if (int rc = partition(ctx, A, C, true, part)) return rc;
        const size_t need = (size_t)((hess_doubles + 1) / 2 * 2) * 8 + part.max_slice;
        if (need <= kSmemBudget) {
            fn = select_cluster(gm, A.W, pre);
            RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(gm ? KT : KTC);
            cfg.dynamicSmemBytes = need;
            cfg.stream = ctx->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters >= 1) {
                cluster = true;
                smem = need;
                G = C;
            }
            cudaGetLastError();
        }
    }
    int ms = stream ? 1 : 0;
    int threads = KT;
    const char* no_sp = getenv("RAFEM_NO_STREAM_PCG");
    if (!cluster && !gm && A.W == 2 && stream && A.maxdeg > 0 && p.grid_ctas <= 0 && !(no_sp && no_sp[0] == '1')) {
        const int bufbytes = KS * A.maxdeg * 16 + ((KS * A.maxdeg + 8) * 4 + 15) / 16 * 16;
        const size_t need = (size_t)kSweepStages * bufbytes;
        if (need <= kSmemBudget) {
            const char* us = getenv("RAFEM_STREAM_U");
            const int uu = us ? atoi(us) : 4;
            if (uu == 1)
                fn = pre ? (const void*)pcg_stream_kernel<true, 12, 1> : (const void*)pcg_stream_kernel<false, 12, 1>;
            else if (uu == 4)
                fn = pre ? (const void*)pcg_stream_kernel<true, 12, 4> : (const void*)pcg_stream_kernel<false, 12, 4>;
            else
                fn = pre ? (const void*)pcg_stream_kernel<true, 12, 2> : (const void*)pcg_stream_kernel<false, 12, 2>;
            RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
            int occ = 0;
            RF_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, KS, need));
            if (occ >= 1) {
                G = std::max(1, std::min(ctx->sm_count, A.ngroups));
                if (int rc = partition(ctx, A, G, false, part)) return rc;
                smem = need;
                threads = KS;
                ms = 3;
                stream_buf = bufbytes;
                stream_valcap = KS * A.maxdeg;
            } else {
                fn = nullptr;
            }
        }
    }
    if (!cluster && ms != 3) {
        // one CTA per SM (the kernels are register-bound to 1 CTA/SM)
        int want = p.grid_ctas > 0 ? p.grid_ctas : ctx->sm_count;
        want = std::max(1, std::min(want, A.ngroups));
        G = want;
        // stage the matrix slice in smem when it fits next to the Hessenberg scratch
        const bool small = A.slots * (4 + 8LL * A.W) <= (long long)G * (160 << 10);
        if (int rc = partition(ctx, A, G, small, part, pipe_rows(gm, A.W, A.ngroups, G))) return rc;
        const size_t hs_al = (size_t)((hess_doubles + 1) / 2 * 2) * 8;
        if (small && hs_al + part.max_slice <= kSmemBudget) {
            ms = 2;
            smem = hs_al + part.max_slice;
            // GMRES: the CTA's own rows of the Krylov basis in shared memory too
            const char* nv = getenv("RAFEM_NO_SMEM_BASIS");
            const size_t vs_bytes = (size_t)(m + 1) * A.W * part.max_groups * sizeof(double);
            if (gm && smem + vs_bytes <= kSmemBudget && !(nv && nv[0] == '1')) {
                vs_off = (long long)(smem / sizeof(double));
                vs_ld = A.W * part.max_groups;
                smem += vs_bytes;
            }
        } else if (hess_bytes <= 160 * 1024) {
            smem = hess_bytes;
        } else {
            hess_global = true;
        }
        fn = select_grid(gm, A.W, pre, ms);
        // opt in whenever dynamic smem is used: without it static + dynamic
        // must stay within 48 KB, which a dynamic size just under 48 KB breaks
        if (smem > 0)
            RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        RF_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, KT, smem));
        if (occ < 1) return rafem_fail(ctx, RAFEM_ERR_CUDA, "cannot size the cooperative solver grid");
        if (G > occ * ctx->sm_count) return rafem_fail(ctx, RAFEM_ERR_INVALID, "grid_ctas exceeds co-resident CTAs");
    }

    const double k2 = timing ? now_us() : 0.0;
    // ---- workspace
    const long long ldv = ((long long)n + 31) / 32 * 32;
    if (gm) {
        if (int rc = ensure(ctx, ctx->ws_basis, sizeof(double) * (size_t)(m + 1) * ldv)) return rc;
    }
    if (int rc = ensure(ctx, ctx->ws_vec, sizeof(double) * (size_t)10 * ldv)) return rc;
    if (int rc = ensure(ctx, ctx->ws_partial, sizeof(double) * (size_t)2 * (2 * std::max(m, 6) + 4) * G)) return rc;
    if (hess_global) {
        if (int rc = ensure(ctx, ctx->ws_hess, sizeof(double) * (size_t)hess_doubles * G)) return rc;
    }
    const long long hist_cap = std::min<long long>(p.max_total_iters > 0 ? p.max_total_iters : 10LL * n, 1LL << 20) + 1;
    const long long cyc_cap = hist_cap;
    if (int rc = ensure(ctx, ctx->ws_hist, sizeof(double) * (size_t)hist_cap)) return rc;
    if (int rc = ensure(ctx, ctx->ws_cyc, sizeof(long long) * (size_t)cyc_cap)) return rc;

    double* vec = static_cast<double*>(ctx->ws_vec.p);
    KArgs a{};
    a.A = A;
    a.gpart = part.gpart;
    a.ldv = ldv;
    a.b = b_dev;
    a.x = x_dev;
    a.minv = pre ? minv_dev : nullptr;
    a.V = gm ? static_cast<double*>(ctx->ws_basis.p) : nullptr;
    a.w0 = vec;
    a.w1 = vec + ldv;
    a.r = vec + 2 * ldv;
    a.z = vec + 3 * ldv;
    a.p0 = vec + 4 * ldv;
    a.p1 = vec + 5 * ldv;
    a.q = vec + 6 * ldv;
    a.e0 = vec + 7 * ldv;
    a.e1 = vec + 8 * ldv;
    a.e2 = vec + 9 * ldv;
    a.partial = static_cast<double*>(ctx->ws_partial.p);
    a.hess = hess_global ? static_cast<double*>(ctx->ws_hess.p) : nullptr;
    a.hess_stride = hess_doubles;
    a.hess_smem = ((cluster || ms == 2) && gm) ? (hess_doubles + 1) / 2 * 2 : 0;  // keep the slice 16-B aligned
    a.vs_off = vs_off;
    a.vs_ld = vs_ld;
    {
        const char* c2 = getenv("RAFEM_GMRES_CGS2");  // the three-synchronisation CGS2 step
        a.gm1r = (gm && vs_off && !cluster && threads == 512 && !(c2 && c2[0] == '1')) ? 1 : 0;
    }
    a.m = m;
    a.tol = p.tolerance;
    a.cap = p.max_total_iters > 0 ? p.max_total_iters : 10LL * n;
    a.hist = static_cast<double*>(ctx->ws_hist.p);
    a.hist_cap = hist_cap;
    a.cyc = static_cast<long long*>(ctx->ws_cyc.p);
    a.cyc_cap = cyc_cap;
    a.res = res_dev;
    a.flag = flag_dev;
    {  // barrier / all-reduce slots: zeroed once, distinguished per launch by the epoch
        const size_t fb = sizeof(unsigned long long) * (2 * 8 * (size_t)std::max(G, 1) + 8);
        if (ctx->ws_flags.bytes < fb) {
            if (int rc = ensure(ctx, ctx->ws_flags, fb)) return rc;
            RF_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ws_flags.p, 0, ctx->ws_flags.bytes, ctx->stream));
        }
        ctx->epoch = ctx->epoch % 0xffffu + 1;
        a.flags = static_cast<unsigned long long*>(ctx->ws_flags.p);
        a.epoch = ctx->epoch;
        a.gbar = grid_counter(ctx, a.flags, G);
        // the one-reduce GMRES splits its per-step barrier (arrive / wait) on the counter
        if (!a.gbar && a.gm1r) a.gbar = a.flags + 2 * 8 * (size_t)std::max(G, 1);
        if (a.gbar) RF_CUDA_TRY(ctx, cudaMemsetAsync(a.gbar, 0, sizeof(unsigned long long), ctx->stream));
    }
    if (ctx->trace_on) {
        if (int rc = ensure(ctx, ctx->ws_trace, sizeof(long long) * 8 * 4096)) return rc;
        RF_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ws_trace.p, 0, sizeof(long long) * 8 * 4096, ctx->stream));
        a.trace = static_cast<long long*>(ctx->ws_trace.p);
        a.trace_cap = 8 * 4096;
    }
    {
        const int rows_per_cta = (A.ngroups + G - 1) / G;
        const int threads = (cluster && !gm) ? KTC : KT;
        int team = 1;
        // measured on B200 (probe_trace.py): the largest team with rows * team <= threads / 4
        // (mesh B: 4 lanes, 1.8 us SpMV phase vs 2.6 with 8; mesh A: 8 lanes)
        while (team < 16 && rows_per_cta * team * 4 <= threads) team *= 2;
        if (const char* env = getenv("RAFEM_TEAM")) team = std::max(1, std::min(32, atoi(env)));
        a.team = team;
        ctx->last_team = team;
    }
    {
        // pipelined PCG for paper-scale systems (<= kPipeRows rows per CTA):
        // RAFEM_PIPE=0 selects the single-reduction Chronopoulos-Gear kernel
        const char* pe = getenv("RAFEM_PIPE");
        const int rows_per_cta = (A.ngroups + G - 1) / G;
        a.pipe = (!gm && A.W == 2 && !cluster && ms != 3 && rows_per_cta <= kPipeRows && !(pe && pe[0] == '0'))
                     ? 1 : 0;
        a.block = (a.pipe && p.precondition == RAFEM_PRECOND_BLOCK_JACOBI && A.maxdeg > 0 && A.maxdeg <= 32) ? 1 : 0;
        ctx->last_precond = a.block ? RAFEM_PRECOND_BLOCK_JACOBI : (pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE);
    }
    if (cluster) smem = (size_t)a.hess_smem * 8 + part.max_slice;
    const double k3 = timing ? now_us() : 0.0;
    void* args[] = {&a};
    void* sargs[] = {&a, &stream_buf, &stream_valcap};
    if (ev_start) RF_CUDA_TRY(ctx, cudaEventRecord(ev_start, ctx->stream));
    if (cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(gm ? KT : KTC);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RF_CUDA_TRY(ctx, cudaLaunchKernelExC(&cfg, fn, args));
        ctx->last_mode = 1;
    } else {
        RF_CUDA_TRY(ctx, cudaLaunchCooperativeKernel(fn, dim3(G), dim3(threads), ms == 3 ? sargs : args, smem,
                                                     ctx->stream));
        ctx->last_mode = ms == 3 ? 3 : 0;
    }
    if (ev_stop) RF_CUDA_TRY(ctx, cudaEventRecord(ev_stop, ctx->stream));
    ctx->last_ctas = G;
    ctx->launches++;
    if (timing)
        std::fprintf(stderr, "  krylov_solve: cluster attempt %.1f, mode %.1f, workspace + args %.1f, launch %.1f us\n",
                     k1 - k0, k2 - k1, k3 - k2, now_us() - k3);
    return RAFEM_OK;
}

int krylov_read_history(rafem_ctx* ctx, const KResult& r, double* hist, long long hist_cap,
                        long long* cyc, long long cyc_cap) {
    if (hist && hist_cap > 0 && r.hist_len > 0) {
        const long long nh = std::min<long long>(std::min<long long>(r.hist_len, hist_cap),
                                                 (long long)(ctx->ws_hist.bytes / sizeof(double)));
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(hist, ctx->ws_hist.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (cyc && cyc_cap > 0 && r.cycles > 0) {
        const long long nc = std::min<long long>(std::min<long long>(r.cycles, cyc_cap),
                                                 (long long)(ctx->ws_cyc.bytes / sizeof(long long)));
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(cyc, ctx->ws_cyc.p, sizeof(long long) * nc, cudaMemcpyDeviceToHost, ctx->stream));
    }
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

}  // namespace rafem

// ---------------------------------------------------------------------------
// fused device-resident simulation (simulate_dev.cuh)

#include "simulate_dev.cuh"

namespace rafem {

int simulate_fused(rafem_system* s, const rafem_sim_params* p, SimDevOut* out, double* rec_x_dev,
                   double* rec_time_dev, double* rec_dt_dev, int* rec_iters_dev, long long rec_cap,
                   double* final_x_dev, float* ms, const SimStream* stream) {
    {  // paper-scale meshes: the cluster-resident simulation (cluster.cu)
        const int crc = simulate_cluster(s, p, out, rec_x_dev, rec_time_dev, rec_dt_dev, rec_iters_dev, rec_cap,
                                         final_x_dev, ms, stream);
        if (crc != RAFEM_ERR_UNSUPPORTED) return crc;
    }
    rafem_mesh* mesh = s->mesh;
    rafem_ctx* ctx = mesh->ctx;
    const int N = mesh->N;
    if (N == 0 || mesh->M == 0) return RAFEM_ERR_UNSUPPORTED;
    MatView A;
    A.rp = mesh->rp;
    A.col = mesh->col;
    A.val = s->val2;
    A.ngroups = N;
    A.W = 2;
    A.slots = mesh->slots;
    A.pattern_id = mesh->id;
    A.maxdeg = mesh->maxdeg;
    if (mesh->maxdeg > 32) return RAFEM_ERR_UNSUPPORTED;
    const bool pre = p->solver.precondition != RAFEM_PRECOND_NONE;
    // 256 threads per CTA: rows * team <= 256 holds at paper scale, the PCG
    // iteration is as fast as with 512 (measured), and the 255-register cap
    // leaves room for the thread-per-slot fill and the pipelined PCG's
    // shared-memory vectors.
    const int nt = 256;
    if (!mesh->slot_lists_tried)
        if (int rc = mesh_slot_lists(mesh)) return rc;
    const void* fn = pre ? (const void*)simulate_kernel<true, 256, false> : (const void*)simulate_kernel<false, 256, false>;
    const void* fn_lean = pre ? (const void*)simulate_kernel<true, 256, true> : (const void*)simulate_kernel<false, 256, true>;
    // one CTA per SM (RAFEM_SIM_CTAS overrides, for experiments)
    int gsim = ctx->sm_count;
    if (const char* e = getenv("RAFEM_SIM_CTAS")) gsim = std::max(1, std::min(ctx->sm_count, atoi(e)));
    const bool pipe = pipe_rows(false, 2, N, std::max(1, std::min(gsim, N)));
    const int G = std::max(1, std::min(gsim, N));
    PartInfo part;
    if (A.slots * 20LL > (long long)G * (150 << 10)) return RAFEM_ERR_UNSUPPORTED;
    if (int rc = partition(ctx, A, G, true, part, pipe_rows(false, 2, N, G))) return rc;
    cudaFuncAttributes fa, fa_lean;
    RF_CUDA_TRY(ctx, cudaFuncGetAttributes(&fa, fn));
    RF_CUDA_TRY(ctx, cudaFuncGetAttributes(&fa_lean, fn_lean));
    size_t smem = part.max_slice;
    if (smem + fa.sharedSizeBytes > 227 * 1024) return RAFEM_ERR_UNSUPPORTED;
    // room to stage each CTA's assembly index data (simulate_dev.cuh)
    int stage_fill = 0;
    size_t gal_scratch_min = ~(size_t)0;  // doubles of contribution scratch on the smallest CTA
    if (mesh->slot_src && !(getenv("RAFEM_NO_STAGE_FILL") && getenv("RAFEM_NO_STAGE_FILL")[0] == '1')) {
        // per block: row, slot, incidence and contributor-list boundaries,
        // gathered on the device and copied once
        const int n1 = G + 1;
        std::vector<int> hb(4 * (size_t)n1);
        int* db = nullptr;
        RF_CUDA_TRY(ctx, dmalloc(ctx, reinterpret_cast<void**>(&db), sizeof(int) * 4 * (size_t)n1));
        block_bounds_kernel<<<(n1 + 127) / 128, 128, 0, ctx->stream>>>(part.gpart, G, mesh->rp, mesh->inc_ptr,
                                                                       mesh->slot_ptr, db, 4);
        ctx->launches++;
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(hb.data(), db, sizeof(int) * 4 * (size_t)n1, cudaMemcpyDeviceToHost,
                                         ctx->stream));
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        dfree(ctx, db);
        const int *hg = hb.data(), *hrs = hb.data() + n1, *hip = hb.data() + 2 * n1, *hsp = hb.data() + 3 * n1;
        size_t need = 0, need2 = 0;
        for (int c = 0; c < G; ++c) {
            const size_t nr = (size_t)(hg[c + 1] - hg[c]);
            const size_t ns = (size_t)(hrs[c + 1] - hrs[c]);
            const size_t nsrc = (size_t)(hsp[c + 1] - hsp[c]);
            const size_t ninc = (size_t)(hip[c + 1] - hip[c]);
            const size_t slice = ns * 16 + ((ns + 3) & ~(size_t)3) * 4 + (nr + 1) * 4;
            const size_t extra = (ns + 1) * 4 + nsrc * 4 + (nr + 1) * 4 + ninc * 4 + nr * 4 + ns + 2 * nr + 8 + 8 * nr;
            need = std::max(need, slice + extra);
            // + the pass's contributions and loads, copied in by cp.async
            need2 = std::max(need2, slice + extra + 32 + nsrc * 16 + ninc * 8);
        }
        need = (need + 15) / 16 * 16;
        need2 = (need2 + 15) / 16 * 16;
        for (int c = 0; c < G; ++c) gal_scratch_min = std::min(gal_scratch_min, 2 * (size_t)(hsp[c + 1] - hsp[c]));
        const char* nsc = getenv("RAFEM_NO_STAGE_CONTRIB");
        const char* nl = getenv("RAFEM_NO_LEAN_SIM");
        if (pipe && need2 + fa_lean.sharedSizeBytes <= 227 * 1024 && !(nsc && nsc[0] == '1') &&
            !(nl && nl[0] == '1')) {
            smem = std::max(smem, need2);
            stage_fill = 2;
            fn = fn_lean;  // pipelined PCG + cp.async fill, nothing else compiled in
        } else if (need2 + fa.sharedSizeBytes <= 227 * 1024 && !(nsc && nsc[0] == '1')) {
            smem = std::max(smem, need2);
            stage_fill = 2;
        } else if (need + fa.sharedSizeBytes <= 227 * 1024) {
            smem = std::max(smem, need);
            stage_fill = 1;
        }
    }
    RF_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    RF_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, smem));
    if (occ < 1 || G > occ * ctx->sm_count) return RAFEM_ERR_UNSUPPORTED;

    const long long n2 = 2LL * N;
    const long long ldv = (n2 + 31) / 32 * 32;
    if (int rc = ensure(ctx, ctx->ws_vec, sizeof(double) * (size_t)10 * ldv)) return rc;
    // partials: two parity buffers of 8 x G, then the Galerkin start's
    // nv (nv + 3) / 2 x G
    if (int rc = ensure(ctx, ctx->ws_partial,
                        sizeof(double) * ((size_t)(16 + kGalMax + kGalMax * (kGalMax + 1) / 2) * G +
                                          kGalMax + kGalMax * (kGalMax + 1) / 2)))
        return rc;
    if (int rc = ensure(ctx, ctx->ws_simout, sizeof(SimDevOut))) return rc;
    {
        const size_t fb = sizeof(unsigned long long) * (2 * 8 * (size_t)G + 8);
        if (ctx->ws_flags.bytes < fb) {
            if (int rc = ensure(ctx, ctx->ws_flags, fb)) return rc;
            RF_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ws_flags.p, 0, ctx->ws_flags.bytes, ctx->stream));
        }
        ctx->epoch = ctx->epoch % 0xffffu + 1;
    }
    double* vec = static_cast<double*>(ctx->ws_vec.p);
    SimArgs S{};
    KArgs& a = S.k;
    a.A = A;
    a.gpart = part.gpart;
    a.ldv = ldv;
    a.minv = pre ? s->minv : nullptr;
    a.w0 = vec;
    a.w1 = vec + ldv;
    a.r = vec + 2 * ldv;
    a.z = vec + 3 * ldv;
    a.p0 = vec + 4 * ldv;
    a.p1 = vec + 5 * ldv;
    a.q = vec + 6 * ldv;
    a.e0 = vec + 7 * ldv;
    a.e1 = vec + 8 * ldv;
    a.e2 = vec + 9 * ldv;
    a.partial = static_cast<double*>(ctx->ws_partial.p);
    a.m = 1;
    a.tol = p->solver.tolerance;
    a.cap = p->solver.max_total_iters > 0 ? p->solver.max_total_iters : 10LL * n2;
    a.flags = static_cast<unsigned long long*>(ctx->ws_flags.p);
    a.epoch = ctx->epoch;
    a.gbar = grid_counter(ctx, a.flags, G);
    if (a.gbar) RF_CUDA_TRY(ctx, cudaMemsetAsync(a.gbar, 0, sizeof(unsigned long long), ctx->stream));
    {
        const int rows_per_cta = (N + G - 1) / G;
        int team = 1;
        // see krylov_solve: the largest team with rows * team <= 256 lanes
        while (team < 16 && rows_per_cta * team * 2 <= 256) team *= 2;
        if (const char* env = getenv("RAFEM_TEAM")) team = std::max(1, std::min(32, atoi(env)));
        a.team = team;
        ctx->last_team = team;
    }
    {
        a.pipe = pipe ? 1 : 0;
        a.block = (a.pipe && p->solver.precondition == RAFEM_PRECOND_BLOCK_JACOBI && mesh->maxdeg <= 32) ? 1 : 0;
        ctx->last_precond = a.block ? RAFEM_PRECOND_BLOCK_JACOBI : (pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE);
    }
    // slot-major element outputs for the cp.async fill (RAFEM_NO_SLOT_MAJOR=1: tet-major)
    const char* nsm = getenv("RAFEM_NO_SLOT_MAJOR");
    const bool slot_major = stage_fill == 2 && !(nsm && nsm[0] == '1');
    if (slot_major)
        if (int rc = mesh_slot_positions(mesh)) return rc;
    S.m = asm_mesh(mesh);
    if (!slot_major) {
        S.m.cpos = nullptr;
        S.m.lpos = nullptr;
    }
    S.stage_fill = stage_fill;
    {
        const char* nv = getenv("RAFEM_NO_VX0");
        S.vx0 = !(nv && nv[0] == '1');
    }
    {
        // Galerkin solver start (pipelined PCG with staged contributions, whose
        // scratch holds the (2k + 1) x 2 rows-per-CTA doubles it needs)
        int K = 14;  // window (mesh-B run, r2d: 10 22.34, 12 22.23, 14 22.00, 16 22.06 ms; r2c before the CTA-wide solve: 8 26.3, 10 23.1, 12 23.2, 14 23.6, 16 24.4)
        if (const char* ge = getenv("RAFEM_GALERKIN_K")) K = std::max(0, std::min(kGalMax, atoi(ge)));
        if (!(stage_fill == 2 && fn == fn_lean) || !pipe) K = 0;
        if (K > 0 && gal_scratch_min < (size_t)(2 * K + 1) * 2 * part.max_groups) K = 0;
        if (K > 0) {
            if (int rc = ensure(ctx, ctx->ws_gal, sizeof(double) * (size_t)(K + 1) * n2)) return rc;
            S.gal_d = static_cast<double*>(ctx->ws_gal.p);
            S.gal_xl = S.gal_d + (size_t)K * n2;
        }
        S.gal_k = K;
        if (const char* gd = getenv("RAFEM_GAL_DBG")) S.gal_dbg = atoi(gd);
    }
    if (int rc = system_contrib(s)) return rc;
    S.contrib = reinterpret_cast<double2*>(s->contrib);
    S.load = s->load;
    S.rhs = s->rhs;
    S.diag_raw = s->diagpart;
    S.xs = s->xs;
    S.final_x = final_x_dev;
    S.n2 = n2;
    S.p = *p;
    S.rec_x = rec_x_dev;
    S.rec_time = rec_time_dev;
    S.rec_dt = rec_dt_dev;
    S.rec_iters = rec_iters_dev;
    S.rec_cap = rec_cap;
    S.out = static_cast<SimDevOut*>(ctx->ws_simout.p);
    if (ctx->trace_on) {  // per-pass phase stamps (rafem_get_trace)
        if (int rc = ensure(ctx, ctx->ws_trace, sizeof(long long) * 8 * 4096)) return rc;
        RF_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ws_trace.p, 0, sizeof(long long) * 8 * 4096, ctx->stream));
        S.ptrace = static_cast<long long*>(ctx->ws_trace.p);
        S.ptrace_cap = 8 * 4096;
    }
    if (stream) {
        S.ring = stream->ring;
        S.ring_slots = stream->slots;
        S.prog = stream->prog;
        S.cons = stream->cons;
    }
    void* args[] = {&S};
    RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    RF_CUDA_TRY(ctx, cudaLaunchCooperativeKernel(fn, dim3(G), dim3(nt), args, smem, ctx->stream));
    RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->launches++;
    ctx->last_mode = 2;
    ctx->last_ctas = G;
    if (stream && stream->pump) {  // consume records while the kernel runs
        if (int rc = stream->pump(stream->user)) return rc;
    }
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->ws_simout.p, sizeof(SimDevOut), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ms) cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1);
    return RAFEM_OK;
}

}  // namespace rafem
