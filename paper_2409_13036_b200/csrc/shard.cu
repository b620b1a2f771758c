// shard.cu — kernel-per-phase PCG over one row block ("shard") of the FEM
// system, for meshes far larger than L2 and for the row-block partition
// across GPUs.
//
// Reference semantics: the PCG contract of pcg_core (krylov.cu) — the
// Chronopoulos-Gear recurrence, true-residual restarts (solver.py:437-450),
// one history entry per iteration, breakdown -> GmresBreakdownError — on a
// system whose rows are owned by `nranks` shards.  A shard's matrix holds
// its owned node rows; columns index an extended vector
//   [owned nodes 0 .. n_own) ++ [ghost nodes n_own .. n_ext)
// whose ghost part is refreshed by a halo exchange before every SpMV.
//
// One iteration is two kernels with the collectives between them:
//
//   kp_update (owner rows: p, s, x, r, u updates; partials r.u, r.r)
//   [pack u -> halo exchange]                       (host: NCCL / P2P)
//   kp_spmv   (w = A u through the TMA pipeline; partial w.u; the last CTA
//              folds every partial into this shard's (r.u, w.u, r.r) slot)
//   [all-gather of the per-shard slots]             (host: NCCL)
//
// Every scalar decision is taken inside kp_update: all its CTAs reduce the
// gathered shard slots in rank order and run the same recurrence on the
// same bits, so all shards and all CTAs agree without any further
// communication.  CTA 0 writes the new solver state into the other half of
// a double-buffered state block (readers of the current half never race
// the writer).  Once the state says stop, every kernel is a no-op until the
// host, which looks at the state only every `batch` iterations, runs the
// true-residual head (kp_head + kp_spmv + kp_update(first)).  Nothing here
// uses float atomics: results are bitwise reproducible for a fixed shard
// count and launch shape.
#include "common.cuh"
#include "internal.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

namespace rafem {

// threads per CTA of the SpMV kernels = node rows per tile: with
// stencil-class columns 192, two CTAs per SM (values-only stages fit twice
// per CTA; measured on the streaming SpMV, r1j: 405 vs 416 us at 16M dofs
// for one 384-row CTA per SM), else 256 at one CTA per SM
template <bool CLS>
__host__ __device__ constexpr int kpt() { return CLS ? 192 : 256; }
template <bool CLS>
__host__ __device__ constexpr int kpc() { return CLS ? 2 : 1; }  // SpMV CTAs per SM

// Programmatic dependent launch: every phase kernel lets the next one in
// the stream be scheduled as soon as all its CTAs have started, and waits
// for the previous one (completion and memory) before touching anything
// mutable, so a phase's launch latency hides under its predecessor's tail.
// No-ops unless the launch carries the PDL attribute (kp_go).
RF_DEV void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
constexpr int KPU = 256;      // threads per CTA of the update kernel
constexpr int kKpStages = 2;  // TMA pipeline depth

struct KPState {
    int done, converged, status, need_head;
    long long total, hlen, cycles, hstart;
    double bnorm, alpha, beta, gamma, rel;
};

// Device-initiated data plane (rafem_kp_ipc_connect): every shard maps its
// peers' kp blocks (CUDA IPC; NVLink peer memory across GPUs) and the phase
// kernels move the halo and the scalar slots themselves — remote stores,
// then a system-scope release of a per-(kind, sender) sequence word in the
// receiver's flag block; consumers acquire it at kernel start.  No host
// collective and no host round trip per iteration.
constexpr int kIpcRanks = 8;  // shards per job on this path (one node)
constexpr int kIpcKinds = 4;  // 0 halo of x, 1 halo of u, 2 scalar slots
enum { kIpcX = 0, kIpcU = 1, kIpcS = 2 };
struct KPIpc {
    int rank, nranks, nseg;
    unsigned send_mask, recv_mask, slot_mask;       // halo peers I send to / receive from; slot peers
    int seg_start[kIpcRanks + 1];                   // send-index ranges per neighbour
    int seg_peer[kIpcRanks];
    double2* seg_dst[2][kIpcRanks];                 // [x | u] ghost range of me in the peer's vector
    double* slot_dst[kIpcRanks];                    // peer's rank_part + 4 * rank
    unsigned long long* peer_flags[kIpcRanks];      // peer's flag block
    unsigned long long* my_flags;                   // kinds x ranks sequence words
};

struct KPArgs {
    MatView A;  // owned node rows; columns into the extended vector
    int n_own;
    double2* x;  // extended
    double2* u;  // extended
    double2* r;
    double2* w;
    double2* s;
    double2* p;
    const double2* b;
    const double2* minv;  // null: no preconditioner
    double* partA;        // (r.u, r.r) per CTA of the writer
    double* partB;        // (w.u) per CTA of kp_spmv
    double* rank_part;    // nranks x 4
    int nranks, rank;
    unsigned* counter;    // last-CTA ticket
    KPState* st;          // [2]
    double* hist;
    long long hist_cap;
    long long* cyc;
    long long cyc_cap;
    double tol;
    long long cap;
    const int* send_idx;
    double2* send_buf;
    int n_send;
    int bufbytes, valcap;  // TMA tile buffers
    const KPIpc* ipc;      // device-initiated halo / slots (null: the host's collectives)
    unsigned long long seq_wait, seq_push;  // sequence numbers of this launch's exchange
    int xpf;               // SpMV: bulk L2 prefetch of each tile's own source rows (RAFEM_KP_XPF=0: off)
};

RF_DEV bool kp_stopped(const KPState& s) { return s.done || s.need_head; }

// ---- the TMA-pipelined SpMV shared by kp_head and kp_spmv ---------------
// Tiles of KPT owned rows are dealt round-robin to the CTAs; each tile's
// contiguous slot data (double2 values + int32 columns) arrives by 1-D bulk
// copy into a double-buffered smem stage (evict-first in L2), and every
// thread sums its row left to right with all of the row's gathers issued
// before the first accumulation.
// CLS: stencil classes (MatView::cls) — only values are streamed, columns
// come from the class table in shared memory.
template <bool CLS, class Epi>
RF_DEV void kp_sweep(const KPArgs& a, const double2* __restrict__ src, unsigned char* sm,
                     unsigned long long* bar, Epi&& epi) {
    __shared__ int soff[CLS ? kMaxClasses * kClsWidth : 1];
    const int N = a.n_own;
    constexpr int KPT = kpt<CLS>();
    const int tiles = (N + KPT - 1) / KPT;
    const int mine = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (CLS)
        for (int k = threadIdx.x; k < a.A.ncls * kClsWidth; k += blockDim.x) soff[k] = __ldg(a.A.cls_off + k);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kKpStages; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const unsigned long long pol = l2_policy_evict_first();
    auto issue = [&](int i) {
        const int t = blockIdx.x + i * gridDim.x;
        const int b = i % kKpStages;
        const int r0 = t * KPT, r1 = min(N, r0 + KPT);
        const int s0 = __ldg(a.A.rp + r0), s1 = __ldg(a.A.rp + r1);
        const int sa = s0 & ~3, se = (s1 + 3) & ~3;
        unsigned char* dst = sm + (size_t)b * a.bufbytes;
        const unsigned vb = 16u * (unsigned)(s1 - s0), cb = CLS ? 0u : 4u * (unsigned)(se - sa);
        mbar_expect_tx(&bar[b], vb + cb);
        if (vb) tma_load_1d_hint(dst, a.A.val + 2LL * s0, vb, &bar[b], pol);
        if (cb) tma_load_1d_hint(dst + (size_t)a.valcap * 16, a.A.col + sa, cb, &bar[b], pol);
        // the tile's own source rows into L2 ahead of its gathers (as the
        // standalone SpMV does); L2 is the point of coherence, so a prefetch
        // issued before the previous kernel's writes land stays correct
        if (a.xpf && r1 > r0) prefetch_l2_bulk(src + r0, 16u * (unsigned)(r1 - r0));
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < kKpStages && i < mine; ++i) issue(i);
    for (int i = 0; i < mine; ++i) {
        const int b = i % kKpStages;
        const int t = blockIdx.x + i * gridDim.x;
        const int r0 = t * KPT, r1 = min(N, r0 + KPT);
        const int r = r0 + threadIdx.x;
        int a0 = 0, a1 = 0, cid = 0;
        if (r < r1) {
            a0 = __ldg(a.A.rp + r);
            a1 = __ldg(a.A.rp + r + 1);
            if (CLS) cid = __ldg(a.A.cls + r);
        }
        const int s0 = __ldg(a.A.rp + r0);
        const int sa = s0 & ~3;
        mbar_wait(&bar[b], (unsigned)(i / kKpStages) & 1u);
        const double2* sv = reinterpret_cast<const double2*>(sm + (size_t)b * a.bufbytes);
        const int* sc = reinterpret_cast<const int*>(sm + (size_t)b * a.bufbytes + (size_t)a.valcap * 16);
        const int* so = soff + cid * kClsWidth - a0;
        if (r < r1) {
            double av = 0.0, at = 0.0;
            for (int s = a0; s < a1; s += 16) {
                int c[16];
                double2 xv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (s + q < a1) c[q] = CLS ? r + so[s + q] : sc[s + q - sa];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (s + q < a1) xv[q] = __ldg(src + c[q]);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (s + q < a1) {
                        const double2 vv = sv[s + q - s0];
                        av = add(av, mul(vv.x, xv[q].x));
                        at = add(at, mul(vv.y, xv[q].y));
                    }
            }
            epi(r, av, at);
        }
        __syncthreads();
        if (threadIdx.x == 0 && i + kKpStages < mine) {
            fence_proxy_async();
            issue(i + kKpStages);
        }
    }
}

// Store this CTA's block-reduced partials at part[cta * NV + j].
template <int NV>
RF_DEV void kp_publish(double (&v)[NV], double* part, double* red) {
    block_sum<NV>(v, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) part[blockIdx.x * NV + j] = v[j];
}

// Last-CTA ticket: true in exactly one CTA, after every CTA's partials are
// visible.  The ticket resets itself for the next launch.
RF_DEV bool kp_last_cta(unsigned* counter) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(counter, 1u);
        last = t == gridDim.x - 1;
        if (last) *counter = 0u;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// Sum of part[j], part[j + stride], ... over `n` entries, fixed order (one warp).
RF_DEV double kp_fold(const double* part, int n, int stride, int j) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s = add(s, __ldcg(part + (long long)c * stride + j));
    return warp_sum(s);
}

// ---- device-initiated exchange (KPIpc) ------------------------------------
RF_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
RF_DEV void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
RF_DEV unsigned long long global_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// thread 0 of the CTA waits until every rank in `mask` has published
// sequence >= seq for `kind`; the CTA's barrier then orders its reads after
// the acquire.  A peer silent for 60 s traps instead of hanging the GPU.
RF_DEV void ipc_wait(const KPIpc* ipc, int kind, unsigned mask, unsigned long long seq) {
    if (threadIdx.x == 0) {
        const unsigned long long t0 = global_timer();
        for (int r = 0; r < ipc->nranks; ++r) {
            if (!((mask >> r) & 1u)) continue;
            const unsigned long long* f = ipc->my_flags + kind * kIpcRanks + r;
            while (ld_acquire_sys(f) < seq) {
                if (global_timer() - t0 > 60000000000ULL) asm volatile("trap;");
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
}
// one thread, after the data it announces is written (and fenced at
// system scope by every writer): publish `seq` to every rank in `mask`
RF_DEV void ipc_signal(const KPIpc* ipc, int kind, unsigned mask, unsigned long long seq) {
    __threadfence_system();
    for (int r = 0; r < ipc->nranks; ++r)
        if ((mask >> r) & 1u) st_release_sys(ipc->peer_flags[r] + kind * kIpcRanks + ipc->rank, seq);
}
// the shard's 4 slot values to every peer's rank_part, then the signal
// Slot regions alternate with the sequence parity: a peer two exchanges
// ahead cannot exist (its next slot needs this shard's next halo, sent only
// after this shard's update consumed the current slots), so two regions of
// nranks x 4 doubles keep a fast peer from overwriting unread values.
RF_DEV double* slot_region(const KPArgs& a, unsigned long long seq) {
    return a.rank_part + (a.ipc ? 4LL * a.nranks * (long long)(seq & 1ULL) : 0LL);
}
RF_DEV void ipc_push_slots(const KPIpc* ipc, const double* o, unsigned long long seq) {
    const long long par = 4LL * ipc->nranks * (long long)(seq & 1ULL);
    for (int r = 0; r < ipc->nranks; ++r)
        if ((ipc->slot_mask >> r) & 1u)
            for (int j = 0; j < 4; ++j) ipc->slot_dst[r][par + j] = o[j];
    ipc_signal(ipc, kIpcS, ipc->slot_mask, seq);
}
// last-CTA ticket whose writers fenced at system scope (remote stores)
RF_DEV bool kp_last_cta_sys(unsigned* counter) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned t = atomicAdd(counter, 1u);
        last = t == gridDim.x - 1;
        if (last) *counter = 0u;
    }
    __syncthreads();
    return last;
}

// ---- kernels --------------------------------------------------------------

// ||b||^2 partial of this shard -> rank_part[rank].x
__global__ void __launch_bounds__(KPU) kp_bnorm_kernel(KPArgs a) {
    pdl_begin();
    __shared__ double red[32];
    double v[1] = {0.0};
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < a.n_own; g += gridDim.x * blockDim.x) {
        const double2 bb = a.b[g];
        v[0] = add(add(v[0], mul(bb.x, bb.x)), mul(bb.y, bb.y));
    }
    kp_publish<1>(v, a.partA, red);
    if (kp_last_cta(a.counter) && threadIdx.x < 32) {
        const double s = kp_fold(a.partA, gridDim.x, 1, 0);
        if (threadIdx.x == 0) {
            double* o = slot_region(a, a.seq_push) + 4LL * a.rank;
            o[0] = s;
            o[1] = o[2] = o[3] = 0.0;
            if (a.ipc) ipc_push_slots(a.ipc, o, a.seq_push);
        }
    }
}

// bnorm from the gathered shard slots; initial state in st[0]
__global__ void kp_bnorm_finish_kernel(KPArgs a) {
    pdl_begin();
    if (a.ipc) ipc_wait(a.ipc, kIpcS, a.ipc->slot_mask, a.seq_wait);
    if (threadIdx.x != 0) return;
    double s = 0.0;
    const double* rp = slot_region(a, a.seq_wait);
    for (int q = 0; q < a.nranks; ++q) s = add(s, rp[4LL * q]);
    KPState st{};
    st.bnorm = sqrt(s);
    st.rel = INFINITY;
    st.status = RAFEM_OK;
    if (st.bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
        st.done = 1;
        st.converged = 1;
        st.rel = 0.0;
    }
    a.st[0] = st;
    a.st[1] = st;
}

// head: r = b - A x, u = M r ; partials (r.u, r.r) -> partA
template <bool PRE, bool CLS>
__global__ void __launch_bounds__(kpt<CLS>(), kpc<CLS>()) kp_head_kernel(KPArgs a, int idx) {
    pdl_begin();
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[kKpStages];
    __shared__ double red[64];
    if (a.st[idx].done) return;
    if (a.ipc) ipc_wait(a.ipc, kIpcX, a.ipc->recv_mask, a.seq_wait);
    double v[2] = {0.0, 0.0};
    kp_sweep<CLS>(a, a.x, sm, bar, [&](int g, double yv, double yt) {
        const double2 bb = a.b[g];
        const double2 rr = make_double2(sub(bb.x, yv), sub(bb.y, yt));
        double2 uu = rr;
        if (PRE) {
            const double2 m = __ldg(a.minv + g);
            uu = make_double2(mul(m.x, rr.x), mul(m.y, rr.y));
        }
        a.r[g] = rr;
        a.u[g] = uu;
        v[0] = add(add(v[0], mul(rr.x, uu.x)), mul(rr.y, uu.y));
        v[1] = add(add(v[1], mul(rr.x, rr.x)), mul(rr.y, rr.y));
    });
    kp_publish<2>(v, a.partA, red);
}

// w = A u ; partial (w.u); last CTA folds (r.u, r.r) of the preceding
// writer (ga CTAs) and (w.u) into rank_part[rank]
template <bool CLS>
__global__ void __launch_bounds__(kpt<CLS>(), kpc<CLS>()) kp_spmv_kernel(KPArgs a, int idx, int after_head, int ga) {
    pdl_begin();
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[kKpStages];
    __shared__ double red[32];
    const KPState& st = a.st[idx];
    if (st.done || (!after_head && st.need_head)) return;
    if (a.ipc) ipc_wait(a.ipc, kIpcU, a.ipc->recv_mask, a.seq_wait);
    double v[1] = {0.0};
    kp_sweep<CLS>(a, a.u, sm, bar, [&](int g, double yv, double yt) {
        const double2 uu = a.u[g];
        __stcs(a.w + g, make_double2(yv, yt));  // evict-first: keep the gathered u in L2
        v[0] = add(add(v[0], mul(yv, uu.x)), mul(yt, uu.y));
    });
    kp_publish<1>(v, a.partB, red);
    if (kp_last_cta(a.counter) && threadIdx.x < 32) {
        const double ru = kp_fold(a.partA, ga, 2, 0);
        const double rr = kp_fold(a.partA, ga, 2, 1);
        const double wu = kp_fold(a.partB, gridDim.x, 1, 0);
        if (threadIdx.x == 0) {
            double* o = slot_region(a, a.seq_push) + 4LL * a.rank;
            o[0] = ru;
            o[1] = wu;
            o[2] = rr;
            o[3] = 0.0;
            if (a.ipc) ipc_push_slots(a.ipc, o, a.seq_push);
        }
    }
}

// Owner update.  Reads st[idx], writes st[idx ^ 1].  first != 0: right
// after a head (true residual check, then the first step of a cycle).
template <bool PRE, int U>
__global__ void __launch_bounds__(KPU) kp_update_kernel(KPArgs a, int idx, int first) {
    pdl_begin();
    __shared__ double red[64];
    __shared__ double co[3];
    KPState S = a.st[idx];
    const bool was_stopped = S.done || (!first && S.need_head);
    if (a.ipc && !was_stopped) ipc_wait(a.ipc, kIpcS, a.ipc->slot_mask, a.seq_wait);
    if (threadIdx.x < 32) {  // gathered shard slots, rank order
        double t[3] = {0.0, 0.0, 0.0};
        if (threadIdx.x == 0) {
            const double* rp = slot_region(a, a.seq_wait);
            for (int q = 0; q < a.nranks; ++q)
                for (int j = 0; j < 3; ++j) t[j] = add(t[j], rp[4LL * q + j]);
        }
        if (threadIdx.x == 0) {
            co[0] = t[0];
            co[1] = t[1];
            co[2] = t[2];
        }
    }
    __syncthreads();
    const double gn = co[0], dn = co[1], rrn = co[2];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    bool step = false;
    double alpha = S.alpha, beta = 0.0;
    if (!was_stopped) {
        if (first) {
            S.need_head = 0;
            S.rel = sqrt(rrn) / S.bnorm;
            if (S.rel <= a.tol) {
                S.done = 1;
                S.converged = 1;
            } else if (S.total >= a.cap) {
                S.done = 1;
            } else if (!(gn > 0.0) || !(dn > 0.0) || !isfinite(gn) || !isfinite(dn)) {
                S.status = RAFEM_ERR_BREAKDOWN;  // not SPD under this preconditioner
                S.done = 1;
            } else {
                S.gamma = gn;
                S.alpha = alpha = gn / dn;
                S.beta = 0.0;
                S.hstart = S.hlen;
                step = true;
            }
        } else {
            S.total += 1;
            const double est = sqrt(rrn) / S.bnorm;
            if (lead && S.hlen < a.hist_cap) a.hist[S.hlen] = est;
            S.hlen += 1;
            bool close = false;
            if (est <= a.tol || S.total >= a.cap) {
                S.need_head = 1;
                close = true;
            } else {
                const double bnew = gn / S.gamma;
                const double den = dn - bnew * gn / S.alpha;
                if (!(gn > 0.0) || !(den > 0.0) || !isfinite(den)) {
                    S.status = RAFEM_ERR_BREAKDOWN;
                    S.done = 1;
                    close = true;
                } else {
                    S.alpha = alpha = gn / den;
                    S.beta = beta = bnew;
                    S.gamma = gn;
                    step = true;
                }
            }
            if (close) {
                if (lead && S.cycles < a.cyc_cap) a.cyc[S.cycles] = S.hlen - S.hstart;
                S.cycles += 1;
            }
        }
    }
    if (lead) a.st[idx ^ 1] = S;
    if (!step) return;
    // p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s, u = M r
    const bool fst = first != 0;
    double v[2] = {0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    for (int gb = blockIdx.x * blockDim.x + threadIdx.x; gb < a.n_own; gb += U * stride) {
        double2 uo[U], wo[U], po[U], so[U], xo[U], ro[U], m[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int g = gb + k * stride;
            if (g < a.n_own) {
                uo[k] = a.u[g];
                wo[k] = a.w[g];
                xo[k] = a.x[g];
                ro[k] = a.r[g];
                m[k] = PRE ? __ldg(a.minv + g) : make_double2(1.0, 1.0);
                if (!fst) {
                    po[k] = a.p[g];
                    so[k] = a.s[g];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int g = gb + k * stride;
            if (g < a.n_own) {
                double2 pn = uo[k], sn = wo[k];
                if (!fst) {
                    pn = make_double2(add(uo[k].x, mul(beta, po[k].x)), add(uo[k].y, mul(beta, po[k].y)));
                    sn = make_double2(add(wo[k].x, mul(beta, so[k].x)), add(wo[k].y, mul(beta, so[k].y)));
                }
                a.x[g] = make_double2(add(xo[k].x, mul(alpha, pn.x)), add(xo[k].y, mul(alpha, pn.y)));
                const double2 rn = make_double2(sub(ro[k].x, mul(alpha, sn.x)), sub(ro[k].y, mul(alpha, sn.y)));
                const double2 un = PRE ? make_double2(mul(m[k].x, rn.x), mul(m[k].y, rn.y)) : rn;
                a.p[g] = pn;
                a.s[g] = sn;
                a.r[g] = rn;
                a.u[g] = un;
                v[0] = add(add(v[0], mul(rn.x, un.x)), mul(rn.y, un.y));
                v[1] = add(add(v[1], mul(rn.x, rn.x)), mul(rn.y, rn.y));
            }
        }
    }
    kp_publish<2>(v, a.partA, red);
}

// send_buf[k] = vec[send_idx[k]] (halo values the neighbours need)
__global__ void kp_pack_kernel(KPArgs a, int idx, int which, int force) {
    pdl_begin();
    const KPState& st = a.st[idx];
    if (st.done || (!force && st.need_head)) return;
    const double2* v = which ? a.u : a.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n_send; k += gridDim.x * blockDim.x)
        a.send_buf[k] = v[__ldg(a.send_idx + k)];
}

// halo push: every send entry straight into the neighbour's ghost range
// (remote store through the peer mapping), then one release per neighbour
__global__ void kp_ipc_push_kernel(KPArgs a, int idx, int which, int force) {
    const KPState& st = a.st[idx];
    if (st.done || (!force && st.need_head)) return;
    const KPIpc* ipc = a.ipc;
    const double2* v = which ? a.u : a.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n_send; k += gridDim.x * blockDim.x) {
        int sg = 0;
        while (sg + 1 < ipc->nseg && k >= ipc->seg_start[sg + 1]) ++sg;
        ipc->seg_dst[which][sg][k - ipc->seg_start[sg]] = v[__ldg(a.send_idx + k)];
    }
    if (kp_last_cta_sys(a.counter) && threadIdx.x == 0) ipc_signal(ipc, which ? kIpcU : kIpcX, ipc->send_mask, a.seq_push);
}

}  // namespace rafem

using namespace rafem;

// ---------------------------------------------------------------------------
// host side

struct rafem_kp {
    bool pdl = false;  // phase kernels launched with programmatic dependent launch (kp_go)
    rafem_system* sys = nullptr;
    rafem_ctx* ctx = nullptr;
    KPArgs a{};
    int n_ext = 0;
    int ga = 1;        // CTAs of the last partA writer
    int g_spmv = 1;    // CTAs of the SpMV kernels
    int g_upd = 1;     // CTAs of the update kernel
    int idx = 0;       // current state half
    size_t smem = 0;
    bool pre = true;
    void* block = nullptr;  // one allocation for every vector and scratch
    void* sendb = nullptr;
    int* sidx = nullptr;
    int* flag = nullptr;
    int launches_at_begin = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // device-initiated data plane (rafem_kp_ipc_connect)
    size_t off_x = 0, off_u = 0, off_rp = 0, off_fl = 0;  // byte offsets in `block` (exported)
    KPIpc* ipc_dev = nullptr;
    void* peer_base[kIpcRanks] = {};
    unsigned long long seq[kIpcKinds] = {};
};

namespace {

int kp_launch_check(rafem_ctx* ctx) {
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

}  // namespace

// Phase kernel launch, with the programmatic-dependent-launch attribute
// when `pdl` (rafem_kp::pdl: shards below 2M owned nodes — measured r1n,
// 1M dofs 45.4 vs 47.5 us per iteration, while at 16M dofs the early
// resident dependents cost 693 vs 654 us; RAFEM_NO_PDL=1: never).
template <typename... P, typename... A>
static void kp_go(bool pdl, void (*fn)(P...), int grid, int block, size_t smem, cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&lc, fn, std::forward<A>(args)...);
}

extern "C" {

int rafem_kp_create(rafem_system* sys, int64_t n_owned, int64_t n_ext, int32_t nranks, int32_t rank,
                    rafem_kp** out) {
    if (!sys || !out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    rafem_mesh* m = sys->mesh;
    rafem_ctx* ctx = m->ctx;
    if (n_owned < 1 || n_owned > m->N || n_ext < n_owned || n_ext > m->N || nranks < 1 || rank < 0 || rank >= nranks)
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "kp_create: bad shard shape");
    if (m->maxdeg < 1) return rafem_fail(ctx, RAFEM_ERR_INVALID, "kp_create: empty pattern");
    if (!m->cls_tried) mesh_stencil_classes(m);  // none on unstructured / renumbered shards
    const char* nc = getenv("RAFEM_NO_CLASSES");
    const bool cls = m->cls && m->ncls > 0 && m->maxdeg <= kClsWidth && !(nc && nc[0] == '1');
    const int KPT = cls ? kpt<true>() : kpt<false>();
    const int bufbytes = KPT * m->maxdeg * 16 + (cls ? 0 : ((KPT * m->maxdeg + 8) * 4 + 15) / 16 * 16);
    const size_t smem = (size_t)kKpStages * bufbytes;
    if (smem > 200 * 1024 + (cls ? 0 : 16 * 1024))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "kp_create: rows too long for the TMA tile buffers");
    rafem_kp* k = new rafem_kp();
    k->sys = sys;
    k->ctx = ctx;
    k->n_ext = (int)n_ext;
    k->smem = smem;
    const int tiles = (int)((n_owned + KPT - 1) / KPT);
    k->g_spmv = std::max(1, std::min(tiles, (cls ? kpc<true>() : kpc<false>()) * ctx->sm_count));
    {
        const char* e = getenv("RAFEM_NO_PDL");
        k->pdl = n_owned < (2LL << 20) && !(e && e[0] == '1');
    }
    k->g_upd = std::max(1, std::min((int)((n_owned + KPU - 1) / KPU), 4 * ctx->sm_count));
    const int gmax = std::max(k->g_spmv, k->g_upd);
    // layout: x_ext, u_ext (n_ext), r, w, s, p, b, minv (n_own) double2; partA 2*gmax, partB gmax,
    // rank_part 4*nranks, state 2, counter, flag
    const size_t v2 = sizeof(double2);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
    const size_t ox = take(v2 * n_ext), ou = take(v2 * n_ext);
    const size_t orr = take(v2 * n_owned), ow = take(v2 * n_owned), os = take(v2 * n_owned), op = take(v2 * n_owned);
    const size_t ob = take(v2 * n_owned), om = take(v2 * n_owned);
    const size_t opa = take(sizeof(double) * 2 * gmax), opb = take(sizeof(double) * gmax);
    const size_t orp = take(sizeof(double) * 8 * nranks), ost = take(sizeof(KPState) * 2);
    const size_t oc = take(sizeof(unsigned)), of = take(sizeof(int));
    const size_t ofl = take(sizeof(unsigned long long) * kIpcKinds * kIpcRanks);  // zeroed with the block
    cudaError_t e = cudaMalloc(&k->block, off);
    if (e != cudaSuccess) {
        delete k;
        return rafem_fail_cuda(ctx, e, "cudaMalloc(kp)", __FILE__, __LINE__);
    }
    char* base = static_cast<char*>(k->block);
    cudaMemsetAsync(k->block, 0, off, ctx->stream);
    KPArgs& a = k->a;
    a.A.rp = m->rp;
    a.A.col = m->col;
    a.A.val = sys->val2;
    a.A.ngroups = (int)n_owned;
    a.A.W = 2;
    a.A.slots = m->slots;
    a.A.maxdeg = m->maxdeg;
    if (cls) {
        a.A.cls = m->cls;
        a.A.cls_off = m->cls_off;
        a.A.ncls = m->ncls;
    }
    a.n_own = (int)n_owned;
    a.x = reinterpret_cast<double2*>(base + ox);
    a.u = reinterpret_cast<double2*>(base + ou);
    a.r = reinterpret_cast<double2*>(base + orr);
    a.w = reinterpret_cast<double2*>(base + ow);
    a.s = reinterpret_cast<double2*>(base + os);
    a.p = reinterpret_cast<double2*>(base + op);
    a.b = reinterpret_cast<double2*>(base + ob);
    a.minv = reinterpret_cast<double2*>(base + om);
    a.partA = reinterpret_cast<double*>(base + opa);
    a.partB = reinterpret_cast<double*>(base + opb);
    a.rank_part = reinterpret_cast<double*>(base + orp);
    a.st = reinterpret_cast<KPState*>(base + ost);
    a.counter = reinterpret_cast<unsigned*>(base + oc);
    k->flag = reinterpret_cast<int*>(base + of);
    k->off_x = ox;
    k->off_u = ou;
    k->off_rp = orp;
    k->off_fl = ofl;
    a.nranks = nranks;
    a.rank = rank;
    a.bufbytes = bufbytes;
    a.valcap = KPT * m->maxdeg;
    {
        const char* xe = getenv("RAFEM_KP_XPF");
        a.xpf = (xe && xe[0] == '0') ? 0 : 1;
    }
    cudaEventCreate(&k->e0);
    cudaEventCreate(&k->e1);
    for (const void* fn : {(const void*)kp_head_kernel<true, false>, (const void*)kp_head_kernel<false, false>,
                           (const void*)kp_spmv_kernel<false>, (const void*)kp_head_kernel<true, true>,
                           (const void*)kp_head_kernel<false, true>, (const void*)kp_spmv_kernel<true>}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            rafem_kp_destroy(k);
            return rafem_fail_cuda(ctx, e, "cudaFuncSetAttribute(kp)", __FILE__, __LINE__);
        }
    }
    *out = k;
    return RAFEM_OK;
}

void rafem_kp_destroy(rafem_kp* k) {
    if (!k) return;
    if (k->ctx) cudaStreamSynchronize(k->ctx->stream);
    for (void* pb : k->peer_base)
        if (pb) cudaIpcCloseMemHandle(pb);
    if (k->ipc_dev) cudaFree(k->ipc_dev);
    if (k->block) cudaFree(k->block);
    if (k->sendb) cudaFree(k->sendb);
    if (k->sidx) cudaFree(k->sidx);
    if (k->e0) cudaEventDestroy(k->e0);
    if (k->e1) cudaEventDestroy(k->e1);
    delete k;
}

int rafem_kp_set_halo(rafem_kp* k, const int32_t* send_idx, int64_t n_send) {
    if (!k || n_send < 0) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    if (k->sendb) cudaFree(k->sendb);
    if (k->sidx) cudaFree(k->sidx);
    k->sendb = nullptr;
    k->sidx = nullptr;
    for (int64_t i = 0; i < n_send; ++i)
        if (send_idx[i] < 0 || send_idx[i] >= k->a.n_own)
            return rafem_fail(ctx, RAFEM_ERR_INVALID, "kp_set_halo: send index outside the owned rows");
    const size_t ns = (size_t)std::max<int64_t>(n_send, 1);
    RF_CUDA_TRY(ctx, cudaMalloc(&k->sendb, sizeof(double2) * ns));
    RF_CUDA_TRY(ctx, cudaMalloc(&k->sidx, sizeof(int) * ns));
    if (n_send)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(k->sidx, send_idx, sizeof(int) * n_send, cudaMemcpyHostToDevice, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    k->a.send_idx = k->sidx;
    k->a.send_buf = static_cast<double2*>(k->sendb);
    k->a.n_send = (int)n_send;
    return RAFEM_OK;
}

// device pointers the host-side collectives read / write
int rafem_kp_buffers(rafem_kp* k, void** x_ext, void** u_ext, void** send_buf, void** rank_part) {
    if (!k) return RAFEM_ERR_INVALID;
    if (x_ext) *x_ext = k->a.x;
    if (u_ext) *u_ext = k->a.u;
    if (send_buf) *send_buf = k->a.send_buf;
    if (rank_part) *rank_part = k->a.rank_part;
    return RAFEM_OK;
}

}  // extern "C"

// b: host array, or NULL for the assembled rhs of the shard's system;
// x0: host array, NULL = zero, or (keep_x) the owned part of a.x as the
// caller's device code left it (the device-resident shard time loop)
static int kp_begin_impl(rafem_kp* k, const double* b, const double* x0, bool keep_x,
                         const rafem_solver_params* p) {
    if (!k || !p) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    if (p->method != RAFEM_METHOD_PCG) return rafem_fail(ctx, RAFEM_ERR_INVALID, "kp solver is PCG only");
    if (!(p->tolerance > 0.0 && p->tolerance < 1.0))
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "tolerance must lie in (0, 1)");
    KPArgs& a = k->a;
    const size_t nb = sizeof(double2) * a.n_own;
    if (b)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync((void*)a.b, b, nb, cudaMemcpyHostToDevice, ctx->stream));
    else
        RF_CUDA_TRY(ctx, cudaMemcpyAsync((void*)a.b, k->sys->rhs, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (x0)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(a.x, x0, nb, cudaMemcpyHostToDevice, ctx->stream));
    else if (!keep_x)
        RF_CUDA_TRY(ctx, cudaMemsetAsync(a.x, 0, nb, ctx->stream));
    k->pre = p->precondition != RAFEM_PRECOND_NONE;  // block-Jacobi: point Jacobi on this engine
    if (k->pre) {
        MatView own = a.A;
        if (int rc = jacobi_minv(ctx, own, const_cast<double*>(reinterpret_cast<const double*>(a.minv)), k->flag))
            return rc;
        int hf = 0;
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(&hf, k->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        if (hf) return rafem_fail(ctx, RAFEM_ERR_INVALID, "zero diagonal entry: Jacobi preconditioner undefined");
    }
    const long long n = 2LL * a.n_own;
    a.tol = p->tolerance;
    a.cap = p->max_total_iters > 0 ? p->max_total_iters : 10LL * n;
    const long long hc = std::min<long long>(a.cap, 1LL << 20) + 1;
    if (int rc = ensure(ctx, ctx->ws_hist, sizeof(double) * (size_t)hc)) return rc;
    if (int rc = ensure(ctx, ctx->ws_cyc, sizeof(long long) * (size_t)hc)) return rc;
    a.hist = static_cast<double*>(ctx->ws_hist.p);
    a.hist_cap = hc;
    a.cyc = static_cast<long long*>(ctx->ws_cyc.p);
    a.cyc_cap = hc;
    k->idx = 0;
    RF_CUDA_TRY(ctx, cudaEventRecord(k->e0, ctx->stream));
    if (a.ipc) a.seq_push = ++k->seq[kIpcS];
    kp_bnorm_kernel<<<k->g_upd, KPU, 0, ctx->stream>>>(a);
    return kp_launch_check(ctx);
}

extern "C" {

int rafem_kp_begin(rafem_kp* k, const double* b, const double* x0, const rafem_solver_params* p) {
    return kp_begin_impl(k, b, x0, false, p);
}

// Phase launches (asynchronous).  what: 0 bnorm-finish, 1 head, 2 spmv after
// head, 3 spmv, 4 update(first), 5 update, 6 pack x, 7 pack u after head,
// 8 pack u.
int rafem_kp_launch(rafem_kp* k, int32_t what) {
    if (!k) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    KPArgs& a = k->a;
    cudaStream_t st = ctx->stream;
    if (a.ipc) {  // this launch's exchange: wait for / publish the kind's next sequence number
        if (what == 0 || what == 4 || what == 5) a.seq_wait = k->seq[kIpcS];
        if (what == 1) a.seq_wait = k->seq[kIpcX];
        if (what == 2 || what == 3) {
            a.seq_wait = k->seq[kIpcU];
            a.seq_push = ++k->seq[kIpcS];
        }
        if (what == 6) a.seq_push = ++k->seq[kIpcX];
        if (what == 7 || what == 8) a.seq_push = ++k->seq[kIpcU];
    }
    switch (what) {
        case 0:
            kp_go(k->pdl, kp_bnorm_finish_kernel, 1, 32, 0, st, a);
            k->idx = 0;
            break;
        case 1:
            if (a.A.cls) {
                if (k->pre)
                    kp_go(k->pdl, kp_head_kernel<true, true>, k->g_spmv, kpt<true>(), k->smem, st, a, k->idx);
                else
                    kp_go(k->pdl, kp_head_kernel<false, true>, k->g_spmv, kpt<true>(), k->smem, st, a, k->idx);
            } else {
                if (k->pre)
                    kp_go(k->pdl, kp_head_kernel<true, false>, k->g_spmv, kpt<false>(), k->smem, st, a, k->idx);
                else
                    kp_go(k->pdl, kp_head_kernel<false, false>, k->g_spmv, kpt<false>(), k->smem, st, a, k->idx);
            }
            k->ga = k->g_spmv;
            break;
        case 2:
        case 3:
            if (a.A.cls)
                kp_go(k->pdl, kp_spmv_kernel<true>, k->g_spmv, kpt<true>(), k->smem, st, a, k->idx, (int)(what == 2), k->ga);
            else
                kp_go(k->pdl, kp_spmv_kernel<false>, k->g_spmv, kpt<false>(), k->smem, st, a, k->idx, (int)(what == 2), k->ga);
            break;
        case 4:
        case 5:
            if (k->pre)
                kp_go(k->pdl, kp_update_kernel<true, 2>, k->g_upd, KPU, 0, st, a, k->idx, (int)(what == 4));
            else
                kp_go(k->pdl, kp_update_kernel<false, 2>, k->g_upd, KPU, 0, st, a, k->idx, (int)(what == 4));
            k->idx ^= 1;
            k->ga = k->g_upd;
            break;
        case 6:
        case 7:
        case 8:
            if (a.n_send <= 0) return RAFEM_OK;
            if (a.ipc)  // straight into the neighbours' ghost ranges
                kp_ipc_push_kernel<<<std::max(1, std::min((a.n_send + 255) / 256, 4 * ctx->sm_count)), 256, 0, st>>>(
                    a, k->idx, what != 6, what != 8);
            else
                kp_pack_kernel<<<std::max(1, std::min((a.n_send + 255) / 256, 4 * ctx->sm_count)), 256, 0, st>>>(
                    a, k->idx, what != 6, what != 8);
            break;
        default:
            return rafem_fail(ctx, RAFEM_ERR_INVALID, "kp_launch: unknown phase");
    }
    return kp_launch_check(ctx);
}

// Single-shard driver: `iters` SPMV + UPDATE pairs back to back (no host
// round trip), for nranks == 1.
int rafem_kp_iterate(rafem_kp* k, int32_t iters) {
    if (!k || (k->a.nranks != 1 && !k->a.ipc)) return RAFEM_ERR_INVALID;
    for (int i = 0; i < iters; ++i) {
        if (k->a.ipc)  // the halo of u goes out by itself (device-initiated)
            if (int rc = rafem_kp_launch(k, RAFEM_KP_PACK_U)) return rc;
        if (int rc = rafem_kp_launch(k, 3)) return rc;  // w = A u (u from the last update)
        if (int rc = rafem_kp_launch(k, 5)) return rc;
    }
    return RAFEM_OK;
}

// ---- device-initiated data plane ------------------------------------------
int rafem_kp_ipc_export(rafem_kp* k, void* handle, int64_t* offsets) {
    if (!k || !handle || !offsets) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    cudaIpcMemHandle_t h;
    RF_CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, k->block));
    std::memcpy(handle, &h, sizeof(h));
    offsets[0] = (int64_t)k->off_x;
    offsets[1] = (int64_t)k->off_u;
    offsets[2] = (int64_t)k->off_rp;
    offsets[3] = (int64_t)k->off_fl;
    return RAFEM_OK;
}

int rafem_kp_ipc_connect(rafem_kp* k, const void* handles, const int64_t* offsets, int32_t nseg,
                         const int32_t* seg_peer, const int64_t* seg_start, const int64_t* seg_dst_node,
                         int32_t n_recv_peers, const int32_t* recv_peers) {
    if (!k || !handles || !offsets || nseg < 0 || n_recv_peers < 0) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    KPArgs& a = k->a;
    const int R = a.nranks, me = a.rank;
    if (R < 2 || R > kIpcRanks || nseg > kIpcRanks)
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "ipc: 2..8 shards with at most 8 neighbours");
    if (nseg && seg_start[nseg] != a.n_send) return rafem_fail(ctx, RAFEM_ERR_INVALID, "ipc: send segments != halo");
    KPIpc h{};
    h.rank = me;
    h.nranks = R;
    h.nseg = nseg;
    char* base[kIpcRanks] = {};
    const cudaIpcMemHandle_t* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int r = 0; r < R; ++r) {
        if (r == me) {
            base[r] = static_cast<char*>(k->block);
            continue;
        }
        if (!k->peer_base[r]) {
            void* pb = nullptr;
            RF_CUDA_TRY(ctx, cudaIpcOpenMemHandle(&pb, hs[r], cudaIpcMemLazyEnablePeerAccess));
            k->peer_base[r] = pb;
        }
        base[r] = static_cast<char*>(k->peer_base[r]);
        h.slot_mask |= 1u << r;
        h.slot_dst[r] = reinterpret_cast<double*>(base[r] + offsets[4 * r + 2]) + 4LL * me;
        h.peer_flags[r] = reinterpret_cast<unsigned long long*>(base[r] + offsets[4 * r + 3]);
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
        const int q = seg_peer[sgi];
        if (q < 0 || q >= R || q == me) return rafem_fail(ctx, RAFEM_ERR_INVALID, "ipc: bad neighbour");
        h.seg_peer[sgi] = q;
        h.seg_start[sgi] = (int)seg_start[sgi];
        h.seg_dst[0][sgi] = reinterpret_cast<double2*>(base[q] + offsets[4 * q + 0]) + seg_dst_node[sgi];
        h.seg_dst[1][sgi] = reinterpret_cast<double2*>(base[q] + offsets[4 * q + 1]) + seg_dst_node[sgi];
        h.send_mask |= 1u << q;
    }
    h.seg_start[nseg] = (int)(nseg ? seg_start[nseg] : 0);
    for (int i = 0; i < n_recv_peers; ++i) {
        if (recv_peers[i] < 0 || recv_peers[i] >= R || recv_peers[i] == me)
            return rafem_fail(ctx, RAFEM_ERR_INVALID, "ipc: bad receive peer");
        h.recv_mask |= 1u << recv_peers[i];
    }
    h.my_flags = reinterpret_cast<unsigned long long*>(base[me] + k->off_fl);
    if (!k->ipc_dev) RF_CUDA_TRY(ctx, cudaMalloc(&k->ipc_dev, sizeof(KPIpc)));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(k->ipc_dev, &h, sizeof(KPIpc), cudaMemcpyHostToDevice, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    a.ipc = k->ipc_dev;
    return RAFEM_OK;
}

// Current solver state (synchronises the stream).  flags: bit0 done,
// bit1 need_head, bit2 converged.
int rafem_kp_state(rafem_kp* k, int32_t* flags, int64_t* iterations, double* rel) {
    if (!k) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    KPState s;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&s, k->a.st + k->idx, sizeof(s), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (flags) *flags = (s.done ? 1 : 0) | (s.need_head ? 2 : 0) | (s.converged ? 4 : 0);
    if (iterations) *iterations = s.total;
    if (rel) *rel = s.rel;
    return RAFEM_OK;
}

int rafem_kp_finish(rafem_kp* k, double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap,
                    int64_t* cycle_lens, int64_t cycle_cap) {
    if (!k) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = k->ctx;
    RF_CUDA_TRY(ctx, cudaEventRecord(k->e1, ctx->stream));
    KPState s;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&s, k->a.st + k->idx, sizeof(s), cudaMemcpyDeviceToHost, ctx->stream));
    if (x_out) {
        if (s.bnorm == 0.0 && s.done) RF_CUDA_TRY(ctx, cudaMemsetAsync(k->a.x, 0, sizeof(double2) * k->a.n_own, ctx->stream));
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(x_out, k->a.x, sizeof(double2) * k->a.n_own, cudaMemcpyDeviceToHost, ctx->stream));
    }
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    // the bnorm == 0 state was read before the memset: report x = 0
    if (s.bnorm == 0.0 && s.done && x_out) std::memset(x_out, 0, sizeof(double2) * k->a.n_own);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, k->e0, k->e1);
    if (st) {
        st->iterations = s.total;
        st->restarts = s.cycles > 0 ? s.cycles - 1 : 0;
        st->final_relative_residual = s.rel;
        st->converged = s.converged;
        st->stagnated = 0;
        st->cycles = s.cycles;
        st->history_len = s.hlen;
        st->device_ms = ms;
    }
    KResult r{};
    r.hist_len = s.hlen;
    r.cycles = s.cycles;
    if (int rc = krylov_read_history(ctx, r, hist, hist_cap, reinterpret_cast<long long*>(cycle_lens), cycle_cap))
        return rc;
    return s.status;
}

}  // extern "C"

namespace rafem {

// Single-shard PCG on an assembled system, used by rafem_system_solve for
// PCG on systems whose matrix is far larger than L2: >= 1 GB (measured on
// B200 at 16M dofs: 771 us per iteration vs 1043 us for the persistent
// streaming kernel), and from the streaming size (48 MB) up when the
// pattern has stencil classes, whose values-only tiles run two CTAs per SM
// (r1n, 1M dofs: 47.4 vs 50.5 us per iteration).  Otherwise the persistent
// streaming kernel.  RAFEM_KP=0/1 forces it off/on (tests, tuning).
int kp_system_solve(rafem_system* s, const double* b, const double* x0, const rafem_solver_params* p,
                    double* x_out, rafem_solve_stats* st, double* hist, int64_t hist_cap, int64_t* cycle_lens,
                    int64_t cycle_cap) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    if (!p || p->method != RAFEM_METHOD_PCG || p->grid_ctas > 0 || m->N < 1) return RAFEM_ERR_UNSUPPORTED;
    const char* env = getenv("RAFEM_KP");
    bool use = (double)m->slots * 20.0 >= 1.0e9;
    if (!use && !env && (double)m->slots * 20.0 > (double)(48LL << 20)) {
        if (!m->cls_tried) mesh_stencil_classes(m);
        const char* nc = getenv("RAFEM_NO_CLASSES");
        use = m->cls && m->ncls > 0 && m->maxdeg <= kClsWidth && !(nc && nc[0] == '1');
    }
    if (env ? env[0] != '1' : !use) return RAFEM_ERR_UNSUPPORTED;
    if (!(p->tolerance > 0.0 && p->tolerance < 1.0))
        return rafem_fail(ctx, RAFEM_ERR_INVALID, "tolerance must lie in (0, 1)");
    if (!s->kp) {
        if (int rc = rafem_kp_create(s, m->N, m->N, 1, 0, &s->kp)) {
            s->kp = nullptr;
            return rc;  // RAFEM_ERR_UNSUPPORTED: the caller keeps the persistent engine
        }
        if (int rc = rafem_kp_set_halo(s->kp, nullptr, 0)) return rc;
    }
    rafem_kp* k = s->kp;
    k->a.A.val = s->val2;
    if (int rc = rafem_kp_begin(k, b, x0, p)) return rc;
    if (int rc = rafem_kp_launch(k, RAFEM_KP_BNORM_FINISH)) return rc;
    int32_t flags = 0;
    int64_t its = 0;
    double rel = 0.0;
    if (int rc = rafem_kp_state(k, &flags, &its, &rel)) return rc;
    const int batch = 32;
    while (!(flags & 1)) {
        for (int ph : {RAFEM_KP_HEAD, RAFEM_KP_SPMV_AFTER_HEAD, RAFEM_KP_UPDATE_FIRST})
            if (int rc = rafem_kp_launch(k, ph)) return rc;
        if (int rc = rafem_kp_state(k, &flags, &its, &rel)) return rc;
        while (!(flags & 3)) {
            if (int rc = rafem_kp_iterate(k, batch)) return rc;
            if (int rc = rafem_kp_state(k, &flags, &its, &rel)) return rc;
        }
    }
    ctx->last_mode = 4;
    ctx->last_ctas = k->g_spmv;
    ctx->last_precond = p->precondition != RAFEM_PRECOND_NONE ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE;
    const int status = rafem_kp_finish(k, x_out, st, hist, hist_cap, cycle_lens, cycle_cap);
    if (status == RAFEM_ERR_BREAKDOWN)
        return rafem_fail(ctx, RAFEM_ERR_BREAKDOWN, "PCG breakdown: system not SPD under the preconditioner");
    return status;
}

}  // namespace rafem

extern "C" {

// ---- sharded assembly: element + fill, owned-row diagonal sums out -------
int rafem_assemble_partial(rafem_system* s, const double* t_iter, const double* v_iter, const double* t_prev,
                           const rafem_assemble_params* p, int64_t n_owned, double* diag_sums,
                           int64_t* bad_element) {
    if (!s || !p || !diag_sums) return RAFEM_ERR_INVALID;
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    if (!(p->dt > 0.0)) return rafem_fail(ctx, RAFEM_ERR_INVALID, "dt must be positive");
    if (n_owned < 0 || n_owned > m->N) return rafem_fail(ctx, RAFEM_ERR_INVALID, "owned rows out of range");
    const int N = m->N;
    double* pin = static_cast<double*>(pinned(ctx, sizeof(double) * (3 * (size_t)std::max(N, 1) + 4)));
    if (!pin) return rafem_fail(ctx, RAFEM_ERR_CUDA, "pinned staging allocation failed");
    std::memcpy(pin, t_iter, sizeof(double) * N);
    std::memcpy(pin + N, v_iter, sizeof(double) * N);
    std::memcpy(pin + 2 * (size_t)N, t_prev, sizeof(double) * N);
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(s->xin, pin, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
    double* dsum = reinterpret_cast<double*>(s->status) + 96;  // scratch past the pass status
    long long* dbad = reinterpret_cast<long long*>(s->status) + 100;
    if (int rc = assemble_fill_launch(s, s->xin, 1, s->xin + N, 1, s->xin + 2 * (size_t)N, 1, p->dt, dbad)) return rc;
    if (int rc = diag_sums_launch(ctx, s->diagpart, (int)n_owned, 0, dsum, nullptr)) return rc;
    double* hp = pin + 3 * (size_t)std::max(N, 1);
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(hp, dsum, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    long long hb = -1;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&hb, dbad, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    diag_sums[0] = hp[0];
    diag_sums[1] = hp[1];
    if (bad_element) *bad_element = hb;
    if (hb >= 0) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "sigma(T) <= 0 in element %lld", hb);
        return rafem_fail(ctx, RAFEM_ERR_PHYSICS, buf);
    }
    return RAFEM_OK;
}

// equilibration with a given scale (reduced over all shards) + Dirichlet elimination
int rafem_assemble_finish(rafem_system* s, const rafem_assemble_params* p, double scale) {
    if (!s || !p) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = s->mesh->ctx;
    if (int rc = assemble_constrain_launch(s, *p, scale)) return rc;
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    s->scale = scale;
    return RAFEM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Device-resident shard time loop (run_simulation / corrector_step,
// fem.py:463-644, over one row block): the accepted, previous and iterate
// (V, T) states of the shard's extended node set live in HBM; per corrector
// pass the host only moves a halo of 4 doubles per boundary node, the
// equilibration sums, the solver state and the corrector delta (one
// scalar).  Same kernels and arithmetic as the single-GPU per-pass native
// loop (capi.cu simulate_host_loop): predictor_kernel, the fill on strided
// views of the iterate, vec_delta.

namespace rafem {

// send4[k] = (x_it V, x_it T, x_acc V, x_acc T) of owned node idx[k]
__global__ void sl_pack_kernel(const double2* __restrict__ xit, const double2* __restrict__ xacc,
                               const int* __restrict__ idx, int n, double2* __restrict__ send4) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = __ldg(idx + k);
        send4[2 * k] = xit[i];
        send4[2 * k + 1] = xacc[i];
    }
}

// ghost node g (local id n_own + g) <- ghost4[g]
__global__ void sl_unpack_kernel(double2* __restrict__ xit, double2* __restrict__ xacc,
                                 const double2* __restrict__ ghost4, int n_own, int n_ghost) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n_ghost; g += gridDim.x * blockDim.x) {
        xit[n_own + g] = ghost4[2 * g];
        xacc[n_own + g] = ghost4[2 * g + 1];
    }
}

}  // namespace rafem

struct rafem_shard_loop {
    rafem_kp* kp = nullptr;
    rafem_ctx* ctx = nullptr;
    int n_own = 0, n_ext = 0;
    double* block = nullptr;
    double* xacc = nullptr;   // accepted (V, T), extended
    double* xprev = nullptr;  // accepted one step earlier, extended
    double* xit = nullptr;    // corrector iterate x_old, extended
    double* send4 = nullptr;  // 4 doubles per send node
    double* ghost4 = nullptr; // 4 doubles per ghost node
    double* scr = nullptr;    // delta, diag sums, bad element
};

extern "C" {

int rafem_sl_create(rafem_kp* kp, rafem_shard_loop** out) {
    if (!kp || !out) return RAFEM_ERR_INVALID;
    *out = nullptr;
    rafem_ctx* ctx = kp->ctx;
    rafem_shard_loop* l = new rafem_shard_loop();
    l->kp = kp;
    l->ctx = ctx;
    l->n_own = kp->a.n_own;
    l->n_ext = kp->n_ext;
    const size_t ext2 = 2 * (size_t)l->n_ext, s4 = 4 * (size_t)std::max(kp->a.n_send, 1);
    const size_t g4 = 4 * (size_t)std::max(l->n_ext - l->n_own, 1);
    const size_t total = 3 * ext2 + s4 + g4 + 8;
    cudaError_t e = cudaMalloc(&l->block, sizeof(double) * total);
    if (e != cudaSuccess) {
        delete l;
        return rafem_fail_cuda(ctx, e, "cudaMalloc(shard loop)", __FILE__, __LINE__);
    }
    l->xacc = l->block;
    l->xprev = l->xacc + ext2;
    l->xit = l->xprev + ext2;
    l->send4 = l->xit + ext2;
    l->ghost4 = l->send4 + s4;
    l->scr = l->ghost4 + g4;
    *out = l;
    return RAFEM_OK;
}

void rafem_sl_destroy(rafem_shard_loop* l) {
    if (!l) return;
    if (l->ctx) cudaStreamSynchronize(l->ctx->stream);
    if (l->block) cudaFree(l->block);
    delete l;
}

int rafem_sl_buffers(rafem_shard_loop* l, void** send4, void** ghost4) {
    if (!l) return RAFEM_ERR_INVALID;
    if (send4) *send4 = l->send4;
    if (ghost4) *ghost4 = l->ghost4;
    return RAFEM_OK;
}

// T = initial_temp, V = 0 on every node of the extended set (fem.py:573-576)
int rafem_sl_init(rafem_shard_loop* l, double initial_temp) {
    if (!l) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    if (int rc = fill_initial(ctx, l->xacc, l->n_ext, initial_temp)) return rc;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(l->xprev, l->xacc, sizeof(double) * 2 * l->n_ext, cudaMemcpyDeviceToDevice,
                                     ctx->stream));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(l->xit, l->xacc, sizeof(double) * 2 * l->n_ext, cudaMemcpyDeviceToDevice,
                                     ctx->stream));
    return RAFEM_OK;
}

// predictor (fem.py:437-449) on the owned nodes: x_it = (V, T + ratio (T -
// T_prev)); with vx0 the solver start (the kp engine's x) also extrapolates
// V ("Solver start"), else the solve starts from x_it
int rafem_sl_predict(rafem_shard_loop* l, int32_t step, double ratio, int32_t vx0) {
    if (!l) return RAFEM_ERR_INVALID;
    double* xs = vx0 ? reinterpret_cast<double*>(l->kp->a.x) : nullptr;
    return predictor_launch(l->ctx, l->xit, l->xacc, l->xprev, l->n_own, step, ratio, xs);
}

int rafem_sl_pack(rafem_shard_loop* l) {
    if (!l) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    const int n = l->kp->a.n_send;
    if (n == 0) return RAFEM_OK;
    sl_pack_kernel<<<std::min((n + 255) / 256, 4 * ctx->sm_count), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(l->xit), reinterpret_cast<const double2*>(l->xacc), l->kp->a.send_idx, n,
        reinterpret_cast<double2*>(l->send4));
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int rafem_sl_unpack(rafem_shard_loop* l) {
    if (!l) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    const int ng = l->n_ext - l->n_own;
    if (ng == 0) return RAFEM_OK;
    sl_unpack_kernel<<<std::min((ng + 255) / 256, 4 * ctx->sm_count), 256, 0, ctx->stream>>>(
        reinterpret_cast<double2*>(l->xit), reinterpret_cast<double2*>(l->xacc),
        reinterpret_cast<const double2*>(l->ghost4), l->n_own, ng);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

// element + fill from the device iterate (t_it, v_it) and the accepted T
// (fem.py:247-388); owned diagonal sums / bad element out, as
// rafem_assemble_partial.  The caller reduces the sums over the shards and
// calls rafem_assemble_finish.
int rafem_sl_assemble_partial(rafem_shard_loop* l, double dt, double* diag_sums, int64_t* bad_element) {
    if (!l || !diag_sums) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    if (!(dt > 0.0)) return rafem_fail(ctx, RAFEM_ERR_INVALID, "dt must be positive");
    rafem_system* s = l->kp->sys;
    long long* dbad = reinterpret_cast<long long*>(l->scr + 4);
    if (int rc = assemble_fill_launch(s, l->xit + 1, 2, l->xit, 2, l->xacc + 1, 2, dt, dbad)) return rc;
    if (int rc = diag_sums_launch(ctx, s->diagpart, l->n_own, 0, l->scr + 1, nullptr)) return rc;
    double hb[5];
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(hb, l->scr, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    diag_sums[0] = hb[1];
    diag_sums[1] = hb[2];
    long long bad;
    std::memcpy(&bad, hb + 4, sizeof(bad));
    if (bad_element) *bad_element = bad;
    if (bad >= 0) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "sigma(T) <= 0 in element %lld", bad);
        return rafem_fail(ctx, RAFEM_ERR_PHYSICS, buf);
    }
    return RAFEM_OK;
}

// PCG on the shard's assembled system, b = its rhs, x0 = the predictor's
// start (from_start) or x_it; then the usual kp phases (rafem_kp_launch)
int rafem_sl_solve_begin(rafem_shard_loop* l, const rafem_solver_params* p, int32_t from_start) {
    if (!l || !p) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    if (!from_start)
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(l->kp->a.x, l->xit, sizeof(double2) * l->n_own, cudaMemcpyDeviceToDevice,
                                         ctx->stream));
    return kp_begin_impl(l->kp, nullptr, nullptr, true, p);
}

// solve stats + the corrector delta max|x_new - x_old| / max(1, |x_old|)
// over the owned dofs (fem.py:526-528), then x_old <- x_new (fem.py:529-530)
int rafem_sl_solve_end(rafem_shard_loop* l, rafem_solve_stats* st, double* delta) {
    if (!l || !delta) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    rafem_kp* k = l->kp;
    KPState s;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&s, k->a.st + k->idx, sizeof(s), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (s.bnorm == 0.0 && s.done)  // zero rhs: x = 0 (solver.py:425-429)
        RF_CUDA_TRY(ctx, cudaMemsetAsync(k->a.x, 0, sizeof(double2) * l->n_own, ctx->stream));
    const int status = rafem_kp_finish(k, nullptr, st, nullptr, 0, nullptr, 0);
    if (status != RAFEM_OK) return status;
    const double* xn = reinterpret_cast<const double*>(k->a.x);
    if (int rc = vec_delta_launch(ctx, xn, l->xit, 2 * l->n_own, l->scr)) return rc;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(l->xit, xn, sizeof(double2) * l->n_own, cudaMemcpyDeviceToDevice, ctx->stream));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(delta, l->scr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

// accept the step (fem.py:604-607): prev <- acc <- iterate
int rafem_sl_accept(rafem_shard_loop* l) {
    if (!l) return RAFEM_ERR_INVALID;
    double* old_prev = l->xprev;
    l->xprev = l->xacc;
    l->xacc = l->xit;
    l->xit = old_prev;
    return RAFEM_OK;
}

// the owned accepted (V, T) dof vector (2 * n_own doubles, interleaved)
int rafem_sl_download(rafem_shard_loop* l, double* x_out) {
    if (!l || !x_out) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = l->ctx;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(x_out, l->xacc, sizeof(double2) * l->n_own, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

}  // extern "C"
