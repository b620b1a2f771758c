// cluster.cu — cluster-resident engine for paper-scale systems (sm_100a).
//
// One thread-block cluster of C <= 16 CTAs holds the whole node-paired
// system in distributed shared memory: CTA c owns a contiguous block of node
// rows, one THREAD per node row, its matrix rows staged once in its shared
// memory as a warp-sliced ELL (slot l of row t at woff(t/32) + 32 l + t%32,
// so a warp's loads of one slot position are 512 contiguous bytes), columns
// as 16-bit indices into the CTA's local node space [own rows | ghosts].
// The Krylov vectors of a row live in its thread's registers; the only
// vector the SpMV gathers (m = M^-1 w, or x / u in a head) sits in a
// double-buffered local array that owners fill for their own rows and PUSH
// into the ghost slots of every CTA that reads them (st.shared::cluster).
// Each CTA's dot-product partials are pushed the same way into every CTA,
// and ONE split cluster barrier (barrier.cluster.arrive.release /
// wait.acquire) per iteration orders both: no global memory, no grid
// barrier, no L2 round trip inside the iteration.
//
// Reductions are deterministic: fixed xor-butterflies per warp, warps in
// order, CTA partials combined in rank order by every CTA, so all CTAs take
// identical branches and repeat runs are bit-identical.
//
// Reference semantics: the PCG contract of krylov.cu (pcg_pipe_core:
// Ghysels-Vanroose recurrence, history, true-residual restarts, breakdown)
// for the SPD FEM systems of assemble_global (fem.py:325-430); the whole-
// simulation kernel below follows run_simulation / corrector_step
// (fem.py:463-644) exactly as simulate_dev.cuh does.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "assembly_dev.cuh"

namespace rafem {

constexpr int kRPT = 1;      // node rows per thread (2 measured slower: longer serial row work per warp)
constexpr int kCT = 576;     // max threads per CTA (kRPT * kCT node rows)
constexpr int kCDest = 8;    // max other CTAs one row is a ghost of (corner of 8 blocks: 7)
constexpr int kCMax = 16;    // max cluster size (non-portable)
constexpr int kCRegions = 16;

struct CCta {
    int g0, nr, nloc, ell_n;  // (g0 unused: own rows are lgid[lbase .. lbase + nr))
    int ell_base, wbase, lbase, pad;
};

struct CPlan {
    const CCta* cta;
    const int4* warp;        // per warp: own-column section (offset, width), ghost-column section (offset, width)
    const uint16_t* ecol;    // ELL local columns (pads: 0)
    const int* esrc;         // ELL entry -> CSR slot, -1 for pads
    const unsigned* dest;    // N x kCDest: cta << 16 | local index; 0xffffffff none
    const int* lgid;         // per CTA: global node id of every local index (own rows by id, then ghosts)
    const int2* trow;        // per CTA and row (thread order): (global row, local index)
    int C, ell_cap, nloc_cap;
    int rows_cap;            // kRPT * threads per CTA (row slots)
    int ndw;                 // push-target words per row (uint4): 1 or 2
};

// ---------------------------------------------------------------------------
// cluster primitives

RF_DEV unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
RF_DEV void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
RF_DEV void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
RF_DEV void cl_sync() {
    cl_arrive();
    cl_wait();
}
// shared::cta address (u32) -> the same offset in CTA `rank`'s window
RF_DEV unsigned cl_map_u(unsigned local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
RF_DEV unsigned cl_map(const void* local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
RF_DEV void st_cluster2(unsigned addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
// shared::cta accesses by 32-bit address: in a cluster kernel a generic
// pointer into shared memory embeds the CTA's window (SR_CgaCtaId), which
// the compiler re-reads (S2R, tens of cycles) wherever it rematerialises one
RF_DEV double2 lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
RF_DEV void sts2(unsigned a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
RF_DEV unsigned lds_u16(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
RF_DEV uint4 lds_u4(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// 16 bytes into a peer's shared memory, completing 16 transaction bytes on
// the peer's mbarrier (data and signal in one message, no fence)
RF_DEV void st_async2(unsigned addr, double a, double b, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(a), "d"(b), "r"(rbar)
                 : "memory");
}
// (CTA-scope acquire: the peers' st.async data lands in this CTA's shared
// memory through the mbarrier's transaction count, which shared memory
// never caches in L1 — the .cluster form would also invalidate L1 (spill
// reloads would then go to L2 every iteration))
RF_DEV void mbar_wait_cluster(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "XW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra XW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// Shared state of one CTA of the engine (identical in all its threads).
struct CEnv {
    // shared::cta (32-bit) addresses of the arrays the iteration touches (a
    // generic pointer into shared memory in a cluster kernel embeds the CTA
    // window, which the compiler re-reads from SR_CgaCtaId at its uses)
    unsigned mb_s, part_s, xbar_s, ev_s, ec_s, rmv_s, rdest_s, red_s, sc_s, yb_s;
    int nloc_cap;
    int C;
    unsigned rank;
    int nr;             // own node rows
    int ndw;            // push-target words (uint4) per row: 1 (<= 4 targets) or 2 (<= 8)
    // exchanges: every CTA pushes its vector entries into the ghost slots of
    // its readers and its 4 CTA partials into every CTA, each message
    // completing transaction bytes on the receiver's mbarrier xbar[k & 1]
    unsigned xk, xw;    // exchanges begun / waited
    unsigned xbytes;    // bytes a CTA receives per exchange
    int blk;            // block-Jacobi: one Neumann step on the CTA's diagonal block
    double omega;
    // PCG contract
    double tol;
    long long cap;
    double* hist;
    long long hist_cap;
    long long* cyc;
    long long cyc_cap;
    int sit;            // stamp iteration (trace only)
    int abl;            // ablation mask for cost studies (0 in production): 1 own SpMV, 2 ghost SpMV,
                        // 4 halo pushes, 8 breakdown/convergence tests off
    long long* trace;   // optional per-warp phase stamps of CTA 0
    long long trace_cap;
};

// One node row of a thread: the thread owns kRPT rows, warp w's lanes take
// the rows of ELL warp blocks w, w + nwarps, ...
struct CRowC {
    int t;              // local row in thread order (active when < nr)
    int gid, li;        // global node row, local (gathered-vector) index
    int k0, w0, k1, w1; // own-column and ghost-column ELL sections: first entry, widths
};

// per-warp phase stamps of CTA 0 (lane 0 of every warp), iteration E.sit:
// trace[((sit * 32) + warp) * 8 + k]
RF_DEV void c_stamp(const CEnv& E, int k) {
    if (E.trace && E.rank == 0 && (threadIdx.x & 31) == 0) {
        const long long i = ((long long)E.sit * 32 + (threadIdx.x >> 5)) * 8 + k;
        if (i < E.trace_cap) E.trace[i] = clock64();
    }
}

// Partial row sum over one ELL section (left to right over its positions);
// ev, ec: the row's first entry; src: the gathered vector (u32 shared addresses).
RF_DEV void c_spmv_sec(unsigned ev, unsigned ec, int width, unsigned src, double& av, double& at) {
    int l = 0;
#pragma unroll 1
    for (; l + 4 <= width; l += 4) {
        unsigned c[4];
        double2 a[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c[j] = lds_u16(ec + 64u * (l + j));
            a[j] = lds2(ev + 512u * (l + j));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = lds2(src + 16u * c[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            av = fma(a[j].x, v[j].x, av);
            at = fma(a[j].y, v[j].y, at);
        }
    }
#pragma unroll 1
    for (; l < width; ++l) {
        const double2 a = lds2(ev + 512u * l);
        const double2 v = lds2(src + 16u * lds_u16(ec + 64u * l));
        av = fma(a.x, v.x, av);
        at = fma(a.y, v.y, at);
    }
}
RF_DEV unsigned c_buf(const CEnv& E, int buf) { return E.mb_s + 16u * (unsigned)(buf * E.nloc_cap); }
// own-column part of the row's product (needs only this CTA's entries of src)
RF_DEV double2 c_spmv_own(const CEnv& E, const CRowC& rc, unsigned src) {
    double av = 0.0, at = 0.0;
    c_spmv_sec(E.ev_s + 16u * rc.k0, E.ec_s + 2u * rc.k0, rc.w0, src, av, at);
    return make_double2(av, at);
}
// + the ghost-column part (needs the pushed ghost entries)
RF_DEV double2 c_spmv_gh(const CEnv& E, const CRowC& rc, unsigned src, double2 acc) {
    c_spmv_sec(E.ev_s + 16u * rc.k1, E.ec_s + 2u * rc.k1, rc.w1, src, acc.x, acc.y);
    return acc;
}
RF_DEV double2 c_spmv(const CEnv& E, const CRowC& rc, unsigned src) {
    return c_spmv_gh(E, rc, src, c_spmv_own(E, rc, src));
}

// Exchange k (= E.xk) begins: thread 0 arms the CTA's mbarrier with the
// bytes it will receive (peers' messages may already have landed: the
// transaction count then runs negative until this arrive).
RF_DEV void c_xbegin(const CEnv& E, unsigned bytes) {
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(E.xbar_s + 8u * (E.xk & 1)),
                     "r"(bytes)
                     : "memory");
}
RF_DEV void c_xbegin(const CEnv& E) { c_xbegin(E, E.xbytes); }

RF_DEV long long global_ns_c() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A row's entry of buffer `buf`: local store + a push into every CTA that
// holds the row as a ghost (exchange E.xk).
RF_DEV void c_push(const CEnv& E, const CRowC& rc, int buf, double2 v) {
    const unsigned bs = c_buf(E, buf), bar = E.xbar_s + 8u * (E.xk & 1);
    sts2(bs + 16u * rc.li, v);
    if (E.abl & 4) return;
    for (int w = 0; w < E.ndw; ++w) {
        const uint4 d = lds_u4(E.rdest_s + 16u * (E.ndw * rc.t + w));
        const unsigned qs[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned q = qs[k];
            if (q != 0xffffffffu)
                st_async2(cl_map_u(bs + 16u * (q & 0xffffu), q >> 16), v.x, v.y, cl_map_u(bar, q >> 16));
        }
        if (d.w == 0xffffffffu) break;
    }
}

// K-value warp sums with the K butterflies interleaved (every shuffle of a
// level issued before its adds): the same bits per value as warp_sum.
template <int K>
RF_DEV void warp_sum_k(double (&v)[K]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double t[K];
#pragma unroll
        for (int j = 0; j < K; ++j) t[j] = __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
        for (int j = 0; j < K; ++j) v[j] = add(v[j], t[j]);
    }
}

// CTA partials of exchange E.xk (v0..v2 summed; with MAX, v3 max-reduced)
// into part[xk & 1][rank] of every CTA; closes the CTA's side of the
// exchange.  The bar.sync also publishes the own entries of the pushed
// vector inside the CTA.  Second level: warp 0 butterflies the warp
// partials and lane c < C sends the CTA's sums to CTA c.
template <bool MAX>
RF_DEV void c_publish(CEnv& E, double v0, double v1, double v2, double v3) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v[3] = {v0, v1, v2};
    warp_sum_k<3>(v);
    if (MAX) v3 = warp_max(v3);
    if (lane == 0) {
        sts2(E.red_s + 32u * w, make_double2(v[0], v[1]));
        sts2(E.red_s + 32u * w + 16u, make_double2(v[2], v3));
    }
    __syncthreads();
    c_stamp(E, 6);
    if (w == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        double s3 = 0.0;
        if (lane < nw) {
            const double2 a = lds2(E.red_s + 32u * lane);
            const double2 b = lds2(E.red_s + 32u * lane + 16u);
            t[0] = a.x;
            t[1] = a.y;
            t[2] = b.x;
            s3 = b.y;
        }
        warp_sum_k<3>(t);
        if (MAX) s3 = warp_max(s3);
        if (lane < E.C) {
            const unsigned a = cl_map_u(E.part_s + 32u * (16u * (E.xk & 1) + E.rank), (unsigned)lane);
            const unsigned rb = cl_map_u(E.xbar_s + 8u * (E.xk & 1), (unsigned)lane);
            st_async2(a, t[0], t[1], rb);
            st_async2(a + 16, t[2], s3, rb);
        }
    }
    c_stamp(E, 7);
    ++E.xk;
}

// Wait for the oldest outstanding exchange (its ghosts and partials are then
// visible to every thread of the CTA).
RF_DEV void c_xwait(CEnv& E) {
    const unsigned k = E.xw++;
    mbar_wait_cluster(E.xbar_s + 8u * (k & 1), (k >> 1) & 1u);
}

// After the wait: combine the C partials of the last waited exchange.
template <bool MAX>
RF_DEV void c_gather(const CEnv& E, double (&co)[4]) {
    // lane c holds CTA c's partials; one interleaved butterfly: the same bits
    // in every warp of every CTA
    const int lane = threadIdx.x & 31;
    const int par = (E.xw - 1) & 1;
    double t[3] = {0.0, 0.0, 0.0};
    double s3 = 0.0;
    if (lane < E.C) {
        const double2 a = lds2(E.part_s + 32u * (16u * par + lane));
        const double2 b = lds2(E.part_s + 32u * (16u * par + lane) + 16u);
        t[0] = a.x;
        t[1] = a.y;
        t[2] = b.x;
        s3 = b.y;
    }
    warp_sum_k<3>(t);
    co[0] = t[0];
    co[1] = t[1];
    co[2] = t[2];
    co[3] = MAX ? warp_max(s3) : 0.0;
}

RF_DEV double2 d2(double a, double b) { return make_double2(a, b); }

// Krylov vectors of one row (both dofs) in registers.
struct CRow {
    double2 x, r, u, w, z, q, s, p;
};

struct CpcgOut {
    long long total, cycles, hlen;
    double rel;
    int converged;
    int status;
};

// out_j = M^-1 src_j for the thread's rows.  Jacobi: D^-1 src.  Block-Jacobi
// (E.blk): one Neumann step on the CTA's diagonal block A_bb,
// m = y + omega D^-1 (src - A_bb y), y = D^-1 src (the in-block product is
// the own-column ELL section over y); SPD for omega < 1 / (lambda_max(D^-1/2
// A_bb D^-1/2) - 1), omega from the block's Gershgorin bound.  Every thread
// of the CTA must call it (bar.sync inside when blk).
template <bool PRE, int RPT>
RF_DEV void c_prec(const CEnv& E, const CRowC (&rc)[RPT], const double2 (&src)[RPT], double2 (&out)[RPT]) {
    double2 y[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        if (rc[j].t < E.nr) {
            const double2 mv = PRE ? lds2(E.rmv_s + 16u * rc[j].t) : d2(1.0, 1.0);
            y[j] = d2(mv.x * src[j].x, mv.y * src[j].y);
            if (E.blk) sts2(E.yb_s + 16u * rc[j].li, y[j]);
        } else {
            y[j] = d2(0.0, 0.0);
        }
    }
    if (!E.blk) {
#pragma unroll
        for (int j = 0; j < RPT; ++j) out[j] = y[j];
        return;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        if (rc[j].t < E.nr) {
            const double2 t = c_spmv_own(E, rc[j], E.yb_s);
            const double2 mv = lds2(E.rmv_s + 16u * rc[j].t);
            out[j] = d2(fma(E.omega * mv.x, src[j].x - t.x, y[j].x), fma(E.omega * mv.y, src[j].y - t.y, y[j].y));
        } else {
            out[j] = d2(0.0, 0.0);
        }
    }
    __syncthreads();  // y is rewritten by the next application
}

// Pipelined PCG (Ghysels-Vanroose) on the cluster, pcg_pipe_core's contract.
// bnorm < 0: ||b||^2 and the zero-diagonal flag (zf, per thread) ride on the
// first head's reduction.  xold (global, by node row): the corrector delta
// max|x - xold| / max(1, |xold|) of the head's iterate goes to *delta.
// b: the right-hand side (global, by node row; read in heads only).
template <bool PRE, int RPT>
RF_DEV CpcgOut cpcg_core(CEnv& E, const CRowC (&rc)[RPT], CRow (&R)[RPT], const double2* b, double bnorm, double zf,
                         const double2* xold, double* delta, double2* xout_g) {
    int total = 0, cycles = 0, hlen = 0;  // (caps below 2^31: hist_cap <= 2^20 + 1)
    bool converged = false;
    double rel = INFINITY;
    int status = RAFEM_OK;
    int hb = 0;
    const bool lead = E.rank == 0 && threadIdx.x == 0;
    while (true) {
        // ---- head: r = b - A x, u = M r (x pushed: one exchange)
        const bool with_b = bnorm < 0.0;
        c_xbegin(E);
#pragma unroll
        for (int j = 0; j < RPT; ++j)
            if (rc[j].t < E.nr) {
                c_push(E, rc[j], hb, R[j].x);
                if (xout_g) xout_g[rc[j].gid] = R[j].x;
            }
        c_publish<false>(E, 0.0, 0.0, 0.0, 0.0);
        c_xwait(E);
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        double2 src[RPT], out[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            src[j] = d2(0.0, 0.0);
            if (rc[j].t < E.nr) {
                const double2 y = c_spmv(E, rc[j], c_buf(E, hb));
                const double2 bb = b[rc[j].gid];
                R[j].r = d2(bb.x - y.x, bb.y - y.y);
                src[j] = R[j].r;
                v2 += fma(R[j].r.x, R[j].r.x, R[j].r.y * R[j].r.y);
                if (with_b) v0 += fma(bb.x, bb.x, bb.y * bb.y);
                if (xold) {
                    const double2 xo = xold[rc[j].gid];
                    const double d0 = fabs(R[j].x.x - xo.x) / fmax(1.0, fabs(xo.x));
                    const double d1 = fabs(R[j].x.y - xo.y) / fmax(1.0, fabs(xo.y));
                    v3 = (d0 > v3 || d0 != d0) ? d0 : v3;
                    v3 = (d1 > v3 || d1 != d1) ? d1 : v3;
                }
            }
        }
        if (with_b && threadIdx.x == 0) v1 = zf;
        c_prec<PRE, RPT>(E, rc, src, out);
        c_xbegin(E);
#pragma unroll
        for (int j = 0; j < RPT; ++j)
            if (rc[j].t < E.nr) {
                R[j].u = out[j];
                c_push(E, rc[j], hb ^ 1, R[j].u);
            }
        c_publish<true>(E, v0, v1, v2, v3);
        c_xwait(E);
        double co[4];
        c_gather<true>(E, co);
        if (with_b) {
            if (co[1] > 0.0) {
                status = RAFEM_ERR_INVALID;
                rel = INFINITY;
                break;
            }
            bnorm = sqrt(co[0]);
            if (bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    R[j].x = d2(0.0, 0.0);
                    if (rc[j].t < E.nr && xout_g) xout_g[rc[j].gid] = R[j].x;
                }
                if (delta) *delta = -1.0;
                converged = true;
                rel = 0.0;
                cycles = 1;
                break;
            }
        }
        if (xold && delta) *delta = co[3];
        rel = sqrt(co[2]) / bnorm;
        if (rel <= E.tol) {
            converged = true;
            break;
        }
        if (total >= E.cap) break;
        // ---- w = A u, m = M w, partials of (r.u, w.u, r.r)
        v0 = v1 = v2 = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            src[j] = d2(0.0, 0.0);
            if (rc[j].t < E.nr) {
                const double2 y = c_spmv(E, rc[j], c_buf(E, hb ^ 1));
                R[j].w = y;
                src[j] = y;
                v0 += fma(R[j].r.x, R[j].u.x, R[j].r.y * R[j].u.y);
                v1 += fma(y.x, R[j].u.x, y.y * R[j].u.y);
                v2 += fma(R[j].r.x, R[j].r.x, R[j].r.y * R[j].r.y);
            }
        }
        c_prec<PRE, RPT>(E, rc, src, out);
        c_xbegin(E);
#pragma unroll
        for (int j = 0; j < RPT; ++j)
            if (rc[j].t < E.nr) {
                R[j].q = out[j];  // m of this iterate (kept in q until the first update)
                c_push(E, rc[j], hb, out[j]);  // hb: last read by the x SpMV, before the last exchange
            }
        c_publish<false>(E, v0, v1, v2, 0.0);
        int cur = hb;
        double alpha = 0.0, ig = 0.0, igam = 0.0;
        bool first = true;
        const int hstart = hlen;
        const double thr = (E.tol * bnorm) * (E.tol * bnorm);
        while (true) {
            // own-column part of n = A m_i first: it needs only this CTA's
            // entries of m_i (complete after the publish's bar.sync), so that
            // part of the SpMV overlaps the exchange.  Warp 0 alone folds the
            // CTA partials and forms the scalars while the other warps sum
            // their ghost columns; a named barrier hands the scalars over.
            ++E.sit;
            c_stamp(E, 0);
            const unsigned mcur = c_buf(E, cur);
            double2 n[RPT];
#pragma unroll
            for (int j = 0; j < RPT; ++j)
                n[j] = (rc[j].t < E.nr && !(E.abl & 1)) ? c_spmv_own(E, rc[j], mcur) : d2(0.0, 0.0);
            c_stamp(E, 1);
            c_xwait(E);
            c_stamp(E, 2);
            if (threadIdx.x < 32) {
                c_gather<false>(E, co);
                const double gn = co[0], dn = co[1];
                double beta = 0.0;
                int flag = 0;  // 1: leave for the head (converged estimate / cap), 2: breakdown
                // one division: q = 1 / (gn den) gives alpha = gn^2 q, 1 / gn =
                // den q and 1 / (gn alpha) = den / gn^2 for the next iteration
                double den = dn;
                bool go = false;
                if (first) {
                    if (!(E.abl & 8) && (!(gn > 0.0) || !(dn > 0.0) || !isfinite(gn) || !isfinite(dn)))
                        flag = 2;
                    else
                        go = true;
                } else {
                    const double rr = co[2];
                    if (lead && E.hist && hlen < E.hist_cap) E.hist[hlen] = rr;
                    if ((rr <= thr && !(E.abl & 8)) || total + 1 >= E.cap) {
                        flag = 1;
                    } else {
                        beta = gn * igam;
                        den = fma(-(gn * ig), gn, dn);
                        if (!(E.abl & 8) && (!(gn > 0.0) || !(den > 0.0) || !isfinite(den)))
                            flag = 2;
                        else
                            go = true;
                    }
                }
                if (go) {
                    const double q = 1.0 / (gn * den);
                    alpha = (gn * gn) * q;
                    igam = den * q;
                    ig = (den * igam) * igam;
                }
                if (threadIdx.x == 0) {
                    sts2(E.sc_s, make_double2(alpha, beta));
                    sts2(E.sc_s + 16u, make_double2((double)flag, 0.0));
                }
                __syncwarp();
                asm volatile("bar.arrive 1, %0;" ::"r"((int)blockDim.x) : "memory");
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (rc[j].t < E.nr && !(E.abl & 2)) n[j] = c_spmv_gh(E, rc[j], mcur, n[j]);
            } else {
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (rc[j].t < E.nr && !(E.abl & 2)) n[j] = c_spmv_gh(E, rc[j], mcur, n[j]);
                asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
            }
            const double2 sc01 = lds2(E.sc_s), sc23 = lds2(E.sc_s + 16u);
            const double alpha_i = sc01.x, beta = sc01.y;
            if (!first) {
                ++total;
                ++hlen;
            }
            if (sc23.x != 0.0) {
                if (sc23.x == 2.0) status = RAFEM_ERR_BREAKDOWN;
                break;
            }
            c_stamp(E, 3);
            v0 = v1 = v2 = 0.0;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                src[j] = d2(0.0, 0.0);
                if (rc[j].t < E.nr) {
                    CRow& Q = R[j];
                    const double2 me = lds2(mcur + 16u * rc[j].li);
                    if (first) {
                        Q.z = n[j];
                        Q.q = me;
                        Q.s = Q.w;
                        Q.p = Q.u;
                    } else {
                        Q.z = d2(fma(beta, Q.z.x, n[j].x), fma(beta, Q.z.y, n[j].y));
                        Q.q = d2(fma(beta, Q.q.x, me.x), fma(beta, Q.q.y, me.y));
                        Q.s = d2(fma(beta, Q.s.x, Q.w.x), fma(beta, Q.s.y, Q.w.y));
                        Q.p = d2(fma(beta, Q.p.x, Q.u.x), fma(beta, Q.p.y, Q.u.y));
                    }
                    Q.x = d2(fma(alpha_i, Q.p.x, Q.x.x), fma(alpha_i, Q.p.y, Q.x.y));
                    Q.r = d2(fma(-alpha_i, Q.s.x, Q.r.x), fma(-alpha_i, Q.s.y, Q.r.y));
                    Q.u = d2(fma(-alpha_i, Q.q.x, Q.u.x), fma(-alpha_i, Q.q.y, Q.u.y));
                    Q.w = d2(fma(-alpha_i, Q.z.x, Q.w.x), fma(-alpha_i, Q.z.y, Q.w.y));
                    src[j] = Q.w;
                    v0 += fma(Q.r.x, Q.u.x, Q.r.y * Q.u.y);
                    v1 += fma(Q.w.x, Q.u.x, Q.w.y * Q.u.y);
                    v2 += fma(Q.r.x, Q.r.x, Q.r.y * Q.r.y);
                }
            }
            c_prec<PRE, RPT>(E, rc, src, out);
            c_xbegin(E);
#pragma unroll
            for (int j = 0; j < RPT; ++j)
                if (rc[j].t < E.nr) c_push(E, rc[j], cur ^ 1, out[j]);
            c_stamp(E, 4);
            c_publish<false>(E, v0, v1, v2, 0.0);
            c_stamp(E, 5);
            cur ^= 1;
            first = false;
        }
        // (the loop ends after a wait: every exchange begun has been waited)
        if (E.hist && E.rank == 0) {  // squared estimates of this cycle -> relative residuals
            if (threadIdx.x == 0 && cycles < E.cyc_cap) E.cyc[cycles] = hlen - hstart;
            __syncthreads();
            for (long long h = hstart + threadIdx.x; h < hlen && h < E.hist_cap; h += blockDim.x)
                E.hist[h] = sqrt(E.hist[h]) / bnorm;
        }
        ++cycles;
        if (status != RAFEM_OK) break;
        hb = cur ^ 1;
    }
    return CpcgOut{total, cycles, hlen, rel, converged ? 1 : 0, status};
}

RF_DEV void c_write_result(KResult* res, long long total, long long cycles, long long hlen, double rel,
                           bool converged, int status) {
    res->iterations = total;
    res->restarts = cycles > 0 ? cycles - 1 : 0;
    res->cycles = cycles;
    res->hist_len = hlen;
    res->final_rel = rel;
    res->converged = converged ? 1 : 0;
    res->stagnated = 0;
    res->status = status;
}

// Dynamic shared memory of the engine (same offsets in every CTA, so a
// peer's copy of any array is this CTA's address mapped to the peer):
//   ELL values | 2 gathered-vector buffers | ELL columns |
//   per own row (thread order): M^-1, push targets | block-Jacobi y (local order)
struct CLayout {
    double2 *ev, *mb, *rmv, *yb;
    uint16_t* ec;
    uint4* rdest;
    unsigned char* end;
};
__host__ __device__ inline size_t c_al16(size_t b) { return (b + 15) & ~(size_t)15; }
__host__ __device__ inline size_t c_layout_bytes(int ell_cap, int nloc_cap, int rows_cap, int ndw, int blk,
                                                 int nbuf = 2) {
    return c_al16((size_t)ell_cap * 16) + c_al16((size_t)nbuf * nloc_cap * 16) + c_al16((size_t)ell_cap * 2) +
           c_al16((size_t)rows_cap * 16) + c_al16((size_t)rows_cap * 16 * ndw) + (blk ? c_al16((size_t)rows_cap * 16) : 0);
}
RF_DEV CLayout c_layout(unsigned char* base, const CPlan& P, int blk, int nbuf = 2) {
    CLayout L;
    unsigned char* q = base;
    L.ev = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)P.ell_cap * 16);
    L.mb = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)nbuf * P.nloc_cap * 16);
    L.ec = reinterpret_cast<uint16_t*>(q);
    q += c_al16((size_t)P.ell_cap * 2);
    L.rmv = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)P.rows_cap * 16);
    L.rdest = reinterpret_cast<uint4*>(q);
    q += c_al16((size_t)P.rows_cap * 16 * P.ndw);
    L.yb = reinterpret_cast<double2*>(q);
    if (blk) q += c_al16((size_t)P.rows_cap * 16);
    L.end = q;
    return L;
}

// Per-CTA setup common to the kernels.
template <int RPT>
RF_DEV void c_env(CEnv& E, CRowC (&rc)[RPT], const CPlan& P, const CCta& c, unsigned rank, const CLayout& L,
                  double (*part)[kCMax][4], double (*red)[4], unsigned long long* xbar, double* sc) {
    E.nloc_cap = P.nloc_cap;
    E.C = P.C;
    E.rank = rank;
    E.nr = c.nr;
    E.ndw = P.ndw;
    const int nw = blockDim.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        CRowC& r = rc[j];
        const int wb = (threadIdx.x >> 5) + j * nw;
        r.t = 32 * wb + lane;
        const int4 wv = P.warp[c.wbase + wb];
        r.k0 = wv.x + lane;
        r.w0 = wv.y;
        r.k1 = wv.z + lane;
        r.w1 = wv.w;
        const int2 tr = r.t < c.nr ? __ldg(P.trow + c.lbase + r.t) : make_int2(0, 0);
        r.gid = tr.x;
        r.li = tr.y;
        if (r.t < c.nr)
            for (int w = 0; w < P.ndw; ++w)
                L.rdest[P.ndw * r.t + w] = __ldg(reinterpret_cast<const uint4*>(P.dest) + (size_t)P.ndw * r.gid + w);
    }
    // opaque copies: the compiler would otherwise rematerialise each address
    // from SR_CgaCtaId (an S2R) at its uses instead of keeping the register
    auto opq = [](unsigned v) {
        unsigned r;
        asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
        return r;
    };
    E.mb_s = opq(smem_u32(L.mb));
    E.part_s = opq(smem_u32(part));
    E.xbar_s = opq(smem_u32(xbar));
    E.ev_s = opq(smem_u32(L.ev));
    E.ec_s = opq(smem_u32(L.ec));
    E.rmv_s = opq(smem_u32(L.rmv));
    E.rdest_s = opq(smem_u32(L.rdest));
    E.red_s = opq(smem_u32(red));
    E.sc_s = opq(smem_u32(sc));
    E.yb_s = opq(smem_u32(L.yb));
    E.xk = E.xw = 0;
    E.xbytes = 32u * (unsigned)P.C + 16u * (unsigned)(c.nloc - c.nr);
    E.abl = 0;
    E.sit = -1;
    E.blk = 0;
    E.omega = 1.0;
    E.trace = nullptr;
    E.hist = nullptr;
    E.cyc = nullptr;
    if (threadIdx.x == 0) {
        mbar_init(xbar, 1);
        mbar_init(xbar + 1, 1);
        mbar_fence_init();
    }
}

// Block-Jacobi setup on the staged values: omega from the CTA block's
// Gershgorin bound of D^-1/2 A_bb D^-1/2 (pcg_pipe_core's rule).  Uses yb
// for sqrt(M^-1) in local order.  All threads of the CTA call it.
template <int RPT>
RF_DEV void c_block_setup(CEnv& E, const CRowC (&rc)[RPT], double* red1) {
    double gmax = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
        if (rc[j].t < E.nr) {
            const double2 mv = lds2(E.rmv_s + 16u * rc[j].t);
            sts2(E.yb_s + 16u * rc[j].li, d2(sqrt(mv.x), sqrt(mv.y)));
        }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RPT; ++j)
        if (rc[j].t < E.nr) {
            const double2 si = lds2(E.yb_s + 16u * rc[j].li);
            double gv = 0.0, gt = 0.0;
            for (int l = 0; l < rc[j].w0; ++l) {
                const double2 a = lds2(E.ev_s + 16u * (rc[j].k0 + 32 * l));
                const double2 sj = lds2(E.yb_s + 16u * lds_u16(E.ec_s + 2u * (rc[j].k0 + 32 * l)));
                gv += fabs(a.x) * si.x * sj.x;
                gt += fabs(a.y) * si.y * sj.y;
            }
            gmax = fmax(gmax, fmax(gv, gt));
        }
    gmax = block_max(gmax, red1);
    E.omega = gmax > 1.98 ? 0.98 / (gmax - 1.0) : 1.0;
    __syncthreads();
}

// ---------------------------------------------------------------------------
// standalone solve: rafem_solve / rafem_system_solve on a paper-scale system

template <bool PRE>
__global__ void __launch_bounds__(kCT, 1) cpcg_kernel(CPlan P, const double2* __restrict__ val2, const double* b,
                                                      double* x, const double* minv, const int* flag, double tol,
                                                      long long cap, double* hist, long long hist_cap,
                                                      long long* cyc, long long cyc_cap, KResult* res,
                                                      long long* trace, long long trace_cap, int abl, int blk) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) double part[2][kCMax][4];
    __shared__ __align__(16) double red[32][4];
    __shared__ __align__(8) unsigned long long xbar[2];
    __shared__ __align__(32) double sc[4];
    const unsigned rank = cl_rank();
    const CCta c = P.cta[rank];
    const CLayout L = c_layout(dsm, P, blk);
    for (int k = threadIdx.x; k < c.ell_n; k += blockDim.x) {
        const int s = __ldg(P.esrc + c.ell_base + k);
        L.ev[k] = s >= 0 ? __ldg(val2 + s) : make_double2(0.0, 0.0);
        L.ec[k] = __ldg(P.ecol + c.ell_base + k);
    }
    CEnv E;
    CRowC rc[kRPT];
    c_env<kRPT>(E, rc, P, c, rank, L, part, red, xbar, sc);
    E.tol = tol;
    E.cap = cap;
    E.hist = hist;
    E.hist_cap = hist_cap;
    E.cyc = cyc;
    E.cyc_cap = cyc_cap;
    E.trace = trace;
    E.trace_cap = trace_cap;
    E.abl = abl;
    if (abl & 4) E.xbytes = 32u * (unsigned)P.C;
    CRow R[kRPT];
#pragma unroll
    for (int j = 0; j < kRPT; ++j) {
        const bool act = rc[j].t < c.nr;
        R[j].x = act ? reinterpret_cast<const double2*>(x)[rc[j].gid] : d2(0.0, 0.0);
        if (act) L.rmv[rc[j].t] = PRE ? reinterpret_cast<const double2*>(minv)[rc[j].gid] : d2(1.0, 1.0);
    }
    __syncthreads();
    if (PRE && blk) {
        E.blk = 1;
        c_block_setup<kRPT>(E, rc, &red[0][0]);
    }
    cl_sync();  // every CTA of the cluster runs (barriers initialised) before the first remote store
    if (*flag) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
        if (rank == 0 && threadIdx.x == 0) c_write_result(res, 0, 0, 0, INFINITY, false, RAFEM_ERR_INVALID);
        return;
    }
    const CpcgOut o = cpcg_core<PRE, kRPT>(E, rc, R, reinterpret_cast<const double2*>(b), -1.0, 0.0, nullptr,
                                           nullptr, reinterpret_cast<double2*>(x));
    if (rank == 0 && threadIdx.x == 0)
        c_write_result(res, o.total, o.cycles, o.hlen, o.rel, o.converged != 0, o.status);
    cl_sync();  // no CTA leaves while a peer may still address its shared memory
}

// ---------------------------------------------------------------------------
// GMRES(m) on the cluster — gmres_body's contract (solver.py:381-531: right
// Jacobi, CGS2 Arnoldi, Givens least squares, true-residual restarts,
// stagnation latch, breakdown rules) with the matrix in the CTAs' shared
// memory and the exchanges of the PCG engine.  The Krylov basis does not
// fit beside the matrix: each CTA keeps its rows of V in global memory (L2),
// thread per row, coalesced.  Per inner step: the pushed z_k = M^-1 v_k ->
// w = A z_k -> CGS pass 1 (k+1 dots, a warp per coefficient over the CTA's
// rows) -> exchange -> w -= V h -> pass 2 (k+1 dots + ||w||^2) -> exchange
// -> w -= V c, h_{k+1,k} = sqrt(||w||^2 - ||c||^2) (explicit norm on
// cancellation) -> Givens -> v_{k+1} -> push.  Three exchanges per step and
// no grid barrier.

constexpr int kGM = 30;  // largest restart length of the cluster engine (the reference default)

struct GmScratch {       // per CTA, shared memory (same bits in every CTA)
    double part[2][kCMax][kGM + 2];  // pushed CTA partials (up to m + 2 values)
    double red[kGM + 2];             // this CTA's coefficient sums
    double co[kGM + 2];              // the exchange's cluster sums
    double H[(kGM + 1) * kGM];       // Hessenberg, column-major (m + 1) x m
    double cs[kGM], sn[kGM], gg[kGM + 1], yy[kGM];
    double sc[4];
};

// Send this CTA's nv sums (gs.red) to every CTA (exchange E.xk); warp 0.
RF_DEV void g_send(CEnv& E, GmScratch& gs, int nv) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x, np = (nv + 1) / 2;
        const unsigned par = E.xk & 1;
        for (int j = lane; j < np * E.C; j += 32) {
            const int pr = j % np, dst = j / np;
            const double a = gs.red[2 * pr], b = 2 * pr + 1 < nv ? gs.red[2 * pr + 1] : 0.0;
            st_async2(cl_map_u(smem_u32(&gs.part[par][E.rank][2 * pr]), (unsigned)dst), a, b,
                      cl_map_u(E.xbar_s + 8u * par, (unsigned)dst));
        }
    }
    ++E.xk;
}
// After the wait: cluster sums of the nv values in rank order into gs.co
// (warp 0; the caller's bar.sync publishes them).
RF_DEV void g_sum(const CEnv& E, GmScratch& gs, int nv) {
    const int par = (E.xw - 1) & 1;
    for (int i = threadIdx.x; i < nv; i += 32) {
        double s = 0.0;
        for (int c = 0; c < E.C; ++c) s = add(s, gs.part[par][c][i]);
        gs.co[i] = s;
    }
}
// CTA sums of nv coefficient dots: coefficient i = sum over own rows of
// V_i . w (i < nv - extra) and, with `self`, w . w as the last one; a warp
// per coefficient, lanes striding the rows, fixed butterfly.  ws: own w in
// shared memory (thread order).
RF_DEV void g_dots(const CEnv& E, GmScratch& gs, const double2* Vg, int ld, const double2* ws, int nb, bool self) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = w; i < nb + (self ? 1 : 0); i += nw) {
        const double2* vi = i < nb ? Vg + (size_t)i * ld : ws;
        double acc = 0.0;
        for (int t = lane; t < E.nr; t += 32) {
            const double2 a = i < nb ? __ldcg(vi + t) : vi[t];
            const double2 b = ws[t];
            acc = fma(a.x, b.x, fma(a.y, b.y, acc));
        }
        acc = warp_sum(acc);
        if (lane == 0) gs.red[i] = acc;
    }
}
// acc -= sum_{i < nb} co[i] V_i[t] (SGN = -1; += for SGN = 1)
template <int SGN = -1>
RF_DEV double2 g_axpy_rows(double2 acc, const double2* Vg, int ld, int t, const double* co, int nb) {
    for (int i = 0; i < nb; ++i) {
        const double2 v = __ldcg(Vg + (size_t)i * ld + t);
        const double h = SGN * co[i];
        acc = make_double2(fma(h, v.x, acc.x), fma(h, v.y, acc.y));
    }
    return acc;
}

template <bool PRE>
__global__ void __launch_bounds__(kCT, 1) cgmres_kernel(CPlan P, const double2* __restrict__ val2, const double* b,
                                                        double* x, const double* minv, const int* flag, double tol,
                                                        long long cap, int m, double* hist, long long hist_cap,
                                                        long long* cyc, long long cyc_cap, KResult* res,
                                                        double2* basis) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) double part_unused[2][kCMax][4];
    __shared__ __align__(16) double red4[32][4];
    __shared__ __align__(8) unsigned long long xbar[2];
    __shared__ __align__(32) double sc4[4];
    __shared__ __align__(16) GmScratch gs;
    const unsigned rank = cl_rank();
    const CCta c = P.cta[rank];
    const CLayout L = c_layout(dsm, P, 1, 1);  // one gathered-vector buffer; yb: the own rows of w
    for (int k = threadIdx.x; k < c.ell_n; k += blockDim.x) {
        const int s = __ldg(P.esrc + c.ell_base + k);
        L.ev[k] = s >= 0 ? __ldg(val2 + s) : make_double2(0.0, 0.0);
        L.ec[k] = __ldg(P.ecol + c.ell_base + k);
    }
    CEnv E;
    CRowC rc[1];
    c_env<1>(E, rc, P, c, rank, L, part_unused, red4, xbar, sc4);
    const CRowC& r0 = rc[0];
    const bool act = r0.t < c.nr;
    const int g = r0.gid, t = r0.t;
    double2* ws = L.yb;
    const int ld = P.rows_cap;
    double2* Vg = basis + (size_t)rank * (kGM + 1) * ld;
    const unsigned xv = 16u * (unsigned)(c.nloc - c.nr) + 16u * (unsigned)P.C;  // vector exchange (+ a dummy pair)
    auto xp = [&](int nv) { return 16u * (unsigned)((nv + 1) / 2) * (unsigned)P.C; };
    double2 xr = act ? reinterpret_cast<const double2*>(x)[g] : d2(0.0, 0.0);
    const double2 bb = act ? reinterpret_cast<const double2*>(b)[g] : d2(0.0, 0.0);
    const double2 mv = (PRE && act) ? reinterpret_cast<const double2*>(minv)[g] : d2(1.0, 1.0);
    __syncthreads();
    cl_sync();
    const bool lead = rank == 0 && threadIdx.x == 0;
    if (*flag) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
        if (lead) c_write_result(res, 0, 0, 0, INFINITY, false, RAFEM_ERR_INVALID);
        return;
    }
    // one-value all-reduce (sum) of v over the cluster
    auto allsum1 = [&](double v) -> double {
        double a[1] = {v};
        warp_sum_k<1>(a);
        if ((threadIdx.x & 31) == 0) red4[threadIdx.x >> 5][0] = a[0];
        __syncthreads();
        if (threadIdx.x < 32) {
            double s = threadIdx.x < (int)(blockDim.x >> 5) ? red4[threadIdx.x][0] : 0.0;
            s = warp_sum(s);
            if (threadIdx.x == 0) gs.red[0] = s;
        }
        __syncwarp();
        c_xbegin(E, xp(1));
        g_send(E, gs, 1);
        c_xwait(E);
        if (threadIdx.x < 32) g_sum(E, gs, 1);
        __syncthreads();
        const double r = gs.co[0];
        __syncthreads();
        return r;
    };
    // push v (own row) into buffer 0 of every reader; exchange with a dummy pair
    auto push_vec = [&](double2 v) {
        c_xbegin(E, xv);
        if (act) c_push(E, r0, 0, v);
        if (threadIdx.x == 0) {
            gs.red[0] = 0.0;
            gs.red[1] = 0.0;
        }
        __syncthreads();  // own entries of buffer 0 complete in the CTA
        g_send(E, gs, 2);
    };
    const double bnorm = sqrt(allsum1(act ? fma(bb.x, bb.x, bb.y * bb.y) : 0.0));
    if (bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
        if (act) reinterpret_cast<double2*>(x)[g] = d2(0.0, 0.0);
        if (lead) c_write_result(res, 0, 1, 0, 0.0, true, RAFEM_OK);
        cl_sync();
        return;
    }
    double2 rr = d2(0.0, 0.0);
    auto true_residual = [&]() -> double {  // r = b - A x, ||r|| / ||b|| (solver.py:438-439)
        push_vec(xr);
        c_xwait(E);
        double s = 0.0;
        if (act) {
            const double2 y = c_spmv(E, r0, c_buf(E, 0));
            rr = d2(bb.x - y.x, bb.y - y.y);
            s = fma(rr.x, rr.x, rr.y * rr.y);
        }
        return sqrt(allsum1(s)) / bnorm;
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
        if (rel <= tol) {
            converged = true;
            break;
        }
        if (total >= cap) break;
        const double cycle_start = rel;
        const double beta = rel * bnorm;
        if (threadIdx.x == 0) {
            for (int i = 0; i <= m; ++i) gs.gg[i] = 0.0;
            gs.gg[0] = beta;
        }
        // v_0 = r / beta; push z_0 = M^-1 v_0
        double2 v = d2(rr.x * (1.0 / beta), rr.y * (1.0 / beta));
        if (act) __stcg(Vg + t, v);
        push_vec(d2(mv.x * v.x, mv.y * v.y));
        int used = 0;
        bool broke = false, dead = false;
        const long long hstart = hlen;
        for (int k = 0; k < m; ++k) {
            c_xwait(E);
            // w = A z_k
            double2 w = act ? c_spmv(E, r0, c_buf(E, 0)) : d2(0.0, 0.0);
            if (act) ws[t] = w;
            __syncthreads();
            // CGS pass 1: h_i = v_i . w
            g_dots(E, gs, Vg, ld, ws, k + 1, false);
            __syncthreads();
            c_xbegin(E, xp(k + 1));
            g_send(E, gs, k + 1);
            c_xwait(E);
            if (threadIdx.x < 32) g_sum(E, gs, k + 1);
            __syncthreads();
            if (threadIdx.x == 0)
                for (int i = 0; i <= k; ++i) gs.H[k * (m + 1) + i] = gs.co[i];
            if (act) {
                w = g_axpy_rows(w, Vg, ld, t, gs.co, k + 1);
                ws[t] = w;
            }
            __syncthreads();
            // CGS pass 2: c_i = v_i . w and ||w||^2
            g_dots(E, gs, Vg, ld, ws, k + 1, true);
            __syncthreads();
            c_xbegin(E, xp(k + 2));
            g_send(E, gs, k + 2);
            c_xwait(E);
            if (threadIdx.x < 32) g_sum(E, gs, k + 2);
            __syncthreads();
            if (threadIdx.x == 0)
                for (int i = 0; i <= k; ++i) gs.H[k * (m + 1) + i] = add(gs.H[k * (m + 1) + i], gs.co[i]);
            double cc = 0.0;
            for (int i = 0; i <= k; ++i) cc = fma(gs.co[i], gs.co[i], cc);
            const double ww = gs.co[k + 1];
            double sq = 0.0;
            if (act) {
                w = g_axpy_rows(w, Vg, ld, t, gs.co, k + 1);
                sq = fma(w.x, w.x, w.y * w.y);
            }
            // ||w - V c||^2 = ||w||^2 - ||c||^2; near an invariant subspace the
            // difference cancels: then (same decision everywhere) reduce it
            double hk1;
            if (cc > 1e-8 * ww)
                hk1 = sqrt(allsum1(sq));
            else
                hk1 = sqrt(fmax(ww - cc, 0.0));
            ++total;
            // Givens update of column k (solver.py:478-496), one thread per CTA
            if (threadIdx.x == 0) {
                double* hc = gs.H + k * (m + 1);
                hc[k + 1] = hk1;
                for (int i = 0; i < k; ++i) {
                    const double tt = add(mul(gs.cs[i], hc[i]), mul(gs.sn[i], hc[i + 1]));
                    hc[i + 1] = add(mul(-gs.sn[i], hc[i]), mul(gs.cs[i], hc[i + 1]));
                    hc[i] = tt;
                }
                const double rad = hypot(hc[k], hc[k + 1]);
                double est = 0.0;
                int isdead = 0;
                if (rad == 0.0) {
                    isdead = 1;
                } else {
                    gs.cs[k] = hc[k] / rad;
                    gs.sn[k] = hc[k + 1] / rad;
                    hc[k] = rad;
                    hc[k + 1] = 0.0;
                    gs.gg[k + 1] = mul(-gs.sn[k], gs.gg[k]);
                    gs.gg[k] = mul(gs.cs[k], gs.gg[k]);
                    est = fabs(gs.gg[k + 1]) / bnorm;
                    if (rank == 0 && hlen < hist_cap) hist[hlen] = est;
                }
                gs.sc[0] = isdead;
                gs.sc[1] = est;
            }
            __syncthreads();
            if (gs.sc[0] != 0.0) {  // column added nothing (solver.py:483-487)
                dead = true;
                used = k;
                break;
            }
            used = k + 1;
            const double est = gs.sc[1];
            ++hlen;
            if (hk1 < tiny) {  // breakdown (solver.py:497-499)
                broke = true;
                break;
            }
            if (est <= tol || total >= cap || k + 1 == m) break;
            v = d2(w.x * (1.0 / hk1), w.y * (1.0 / hk1));
            if (act) __stcg(Vg + (size_t)(k + 1) * ld + t, v);
            push_vec(d2(mv.x * v.x, mv.y * v.y));
        }
        if (used > 0) {  // y = R^-1 g ; x += M^-1 (V y)   (solver.py:504-511)
            if (threadIdx.x == 0) {
                for (int i = used - 1; i >= 0; --i) {
                    double d = 0.0;
                    for (int j = i + 1; j < used; ++j) d = add(d, mul(gs.H[j * (m + 1) + i], gs.yy[j]));
                    gs.yy[i] = sub(gs.gg[i], d) / gs.H[i * (m + 1) + i];
                }
            }
            __syncthreads();
            if (act) {
                const double2 u = g_axpy_rows<1>(d2(0.0, 0.0), Vg, ld, t, gs.yy, used);  // V y
                xr = d2(xr.x + mv.x * u.x, xr.y + mv.y * u.y);
            }
            __syncthreads();
        }
        if (lead && cycles < cyc_cap) cyc[cycles] = hlen - hstart;
        ++cycles;
        have_prev = true;
        prev_start = cycle_start;
        if (broke || dead) {  // solver.py:516-524
            rel = true_residual();
            if (rel <= tol)
                converged = true;
            else
                status = RAFEM_ERR_BREAKDOWN;
            break;
        }
    }
    if (act) reinterpret_cast<double2*>(x)[g] = xr;
    if (lead) c_write_result(res, total, cycles, hlen, rel, converged, status);
    if (lead) res->stagnated = (latched && !converged) ? 1 : 0;
    cl_sync();  // no CTA leaves while a peer may still address its shared memory
}

// ---------------------------------------------------------------------------
// The whole adaptive simulation in one cluster (run_simulation fem.py:554-644
// around corrector_step fem.py:463-540, the same control as simulate_dev.cuh).
// Per corrector pass: element scalars (sigma, T-rhs loads) of the CTA's
// element range -> cluster barrier -> every CTA fills its own rows' ELL
// values straight into shared memory from the stored geometry (per-slot
// contributor lists in ascending element order: fill_slot's sums, bit for
// bit) -> ONE all-reduce of the equilibration sums and the PhysicsRange flag
// -> scale, Dirichlet elimination and Jacobi inverse on the own rows in
// place -> the cluster PCG on the staged slice -> corrector delta from its
// final head.  Fields live in global memory (owners write their rows).

struct CSimArgs {
    CPlan P;
    AsmMesh m;
    double* xs;        // 4 x n2 working dof vectors
    double* final_x;   // n2
    double* esig;      // M
    double* eload;     // 4M
    double* rhs;       // n2: the pass's constrained right-hand side (read by the solver heads)
    long long n2;
    rafem_sim_params p;
    double* rec_x;
    double* rec_time;
    double* rec_dt;
    int* rec_iters;
    long long rec_cap;
    SimDevOut* out;
    double* ring;
    int ring_slots;
    volatile long long* prog;
    volatile long long* cons;
    int blk;
    int vx0;
};

// Contribution (e, a, b) of the fused fill: element_core's arithmetic.
RF_DEV double2 c_contrib(const AsmMesh& m, unsigned idx, const double* sig, const double* rk, const double* rrc) {
    const int e = (int)(idx >> 4), a = (int)((idx >> 2) & 3), b = (int)(idx & 3);
    const int rg = __ldg(m.region + e);
    const double vol = __ldg(m.vol + e);
    const double sigma = __ldcg(sig + e);
    const double bab = __ldg(m.base + 10LL * e + sym_index(a, b));
    const double mass = a == b ? mul(vol, 0.1) : mul(vol, 0.05);
    return make_double2(mul(sigma, bab), add(mul(rrc[rg], mass), mul(rk[rg], bab)));
}

template <bool PRE>
__global__ void __launch_bounds__(kCT, 1) csim_kernel(CSimArgs S) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) double part[2][kCMax][4];
    __shared__ __align__(16) double red[32][4];
    __shared__ __align__(8) unsigned long long xbar[2];
    __shared__ __align__(32) double sc[4];
    __shared__ double rk[kCRegions], rrc[kCRegions];
    const CPlan& P = S.P;
    const AsmMesh& m = S.m;
    const rafem_sim_params& p = S.p;
    const unsigned rank = cl_rank();
    const CCta c = P.cta[rank];
    const CLayout L = c_layout(dsm, P, S.blk);
    uint8_t* lkind = L.end;  // kinds of the local nodes: V | T << 2
    for (int k = threadIdx.x; k < c.ell_n; k += blockDim.x) L.ec[k] = __ldg(P.ecol + c.ell_base + k);
    for (int q = threadIdx.x; q < c.nloc; q += blockDim.x) {
        const int g = __ldg(P.lgid + c.lbase + q);
        lkind[q] = (uint8_t)(m.kind[2LL * g] | (m.kind[2LL * g + 1] << 2));
    }
    CEnv E;
    CRowC rc[1];
    c_env<1>(E, rc, P, c, rank, L, part, red, xbar, sc);
    E.tol = p.solver.tolerance;
    E.cap = p.solver.max_total_iters > 0 ? p.solver.max_total_iters : 10LL * S.n2;
    CRowC& r0 = rc[0];
    const bool act = r0.t < c.nr;
    const int g = r0.gid;
    const unsigned xvec = E.xbytes, xpart = 32u * (unsigned)P.C;
    const int M = m.M, e0 = (int)((long long)M * rank / P.C), e1 = (int)((long long)M * (rank + 1) / P.C);
    const long long n2 = S.n2;
    auto X = [&](int i) { return reinterpret_cast<double2*>(S.xs + (long long)i * n2); };
    int iacc = 0, iprev = 1, iit = 2, inew = 3;
    // the row's CSR slots and its diagonal slot
    const int s_beg = act ? __ldg(m.rp + g) : 0, s_end = act ? __ldg(m.rp + g + 1) : 0;
    const int s_diag = act ? (__ldg(m.diag + g) >= 0 ? s_beg + __ldg(m.diag + g) : -1) : -1;
    const uint8_t kvt = act ? lkind[r0.li] : 0;
    const int kV = kvt & 3, kT = kvt >> 2;
    if (act) {  // initial_state (fem.py:170-180)
        X(iacc)[g] = d2(0.0, p.initial_temp);
        X(iprev)[g] = d2(0.0, p.initial_temp);
    }
    __syncthreads();
    cl_sync();

    double t = 0.0, dt_state = p.dt_init, dt_prev = p.dt_init;
    long long step = 0, passes = 0, corr = 0, inner = 0, halv = 0, bad = -1;
    long long asm_ns = 0, sol_ns = 0;
    int status = RAFEM_OK, failed_step = -1;
    double failed_dt = 0.0;
    while (t < p.total_time) {
        if (p.max_steps > 0 && step >= p.max_steps) break;
        const double remaining = p.total_time - t;
        const bool final_step = dt_state >= remaining;
        const double dt = final_step ? remaining : dt_state;
        const double ratio = dt / dt_prev;
        if (act) {  // predictor (fem.py:437-449); the first pass's solver start extrapolates V too
            const double2 xa = X(iacc)[g];
            double2 xe = xa;
            if (step >= 1) {
                const double2 xp = X(iprev)[g];
                xe = d2(add(xa.x, mul(ratio, sub(xa.x, xp.x))), add(xa.y, mul(ratio, sub(xa.y, xp.y))));
            }
            X(iit)[g] = d2(xa.x, xe.y);
            if (S.vx0) X(inew)[g] = xe;
        }
        bool conv = false, abort_run = false;
        int iters = 0;
        for (int it = 1; it <= p.max_corrector_iters; ++it) {
            iters = it;
            ++passes;
            const long long ta = global_ns_c();
            if (S.ring && rank == 0 && threadIdx.x == 0 && it == 1) {
                __threadfence_system();
                *S.prog = step;  // every accepted record is in the ring
                long long spins = 0;
                while (step - *S.cons >= S.ring_slots) {
                    __nanosleep(2000);
                    if (++spins > (1LL << 31)) asm volatile("trap;");
                }
            }
            __syncthreads();
            cl_sync();  // the iterate is complete everywhere (global memory, cluster scope)
            // ---- element scalars of this CTA's element range
            for (int r = threadIdx.x; r < m.nreg && r < kCRegions; r += blockDim.x) {
                rk[r] = m.regtab[r];
                rrc[r] = m.regtab[m.nreg + r] / dt;  // element_core's rcdt
            }
            const double2* xit = X(iit);
            const AsmFields f{S.xs + (long long)iit * n2 + 1, 2, S.xs + (long long)iit * n2, 2,
                              S.xs + (long long)iacc * n2 + 1, 2, dt};
            double badv = 0.0;
            for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
                double sg, l4[4];
                if (element_scalars(e, m, f, &sg, l4)) badv = fmax(badv, (double)(M - e));
                __stcg(S.esig + e, sg);
                __stcg(reinterpret_cast<double2*>(S.eload + 4LL * e), make_double2(l4[0], l4[1]));
                __stcg(reinterpret_cast<double2*>(S.eload + 4LL * e) + 1, make_double2(l4[2], l4[3]));
            }
            __syncthreads();
            cl_sync();  // element scalars visible to every CTA
            // ---- fill the own row's ELL entries in place (contributor lists in
            // ascending element order: fill_slot's sums); T rhs; raw diagonal
            double2 dgv = d2(0.0, 0.0);
            double rt = 0.0;
            if (act) {
                for (int sec = 0; sec < 2; ++sec) {
                    const int k0 = sec ? r0.k1 : r0.k0, wd = sec ? r0.w1 : r0.w0;
                    for (int l = 0; l < wd; ++l) {
                        const int k = k0 + 32 * l;
                        const int s = __ldg(P.esrc + c.ell_base + k);
                        double av = 0.0, at = 0.0;
                        if (s >= 0) {
                            const int q0 = __ldg(m.slot_ptr + s), q1 = __ldg(m.slot_ptr + s + 1);
                            for (int q = q0; q < q1; q += 4) {
                                double2 cv[4];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (q + j < q1) cv[j] = c_contrib(m, (unsigned)__ldg(m.slot_src + q + j), S.esig, rk, rrc);
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (q + j < q1) {
                                        av = add(av, cv[j].x);
                                        at = add(at, cv[j].y);
                                    }
                            }
                            if (s == s_diag) dgv = d2(av, at);
                        }
                        sts2(E.ev_s + 16u * k, d2(av, at));
                    }
                }
                const int p0 = __ldg(m.inc_ptr + g), p1 = __ldg(m.inc_ptr + g + 1);
                for (int q = p0; q < p1; q += 8) {
                    double lv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (q + j < p1) {
                            const unsigned ea = __ldg(m.inc_ea + q + j);
                            lv[j] = __ldcg(S.eload + 4LL * (ea & 0x3fffffffu) + (ea >> 30));
                        }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (q + j < p1) rt = add(rt, lv[j]);
                }
            }
            // equilibration sums (fem.py:390-396) and PhysicsRange, one all-reduce
            double co[4];
            c_xbegin(E, xpart);
            c_publish<true>(E, dgv.x, dgv.y, badv > 0.0 ? 1.0 : 0.0, badv);
            c_xwait(E);
            c_gather<true>(E, co);
            if (co[2] > 0.0) {  // PhysicsRangeError aborts the run (fem.py:274)
                bad = M - (long long)co[3];
                status = RAFEM_ERR_PHYSICS;
                abort_run = true;
                break;
            }
            double scale = 1.0;
            if (co[0] > 0.0 && co[1] > 0.0) scale = ldexp(1.0, (int)rint(log2(co[1] / co[0])));
            // ---- scale + Dirichlet elimination + Jacobi inverse, in place
            // (constrain_node_thread's arithmetic; moved-column sums in storage
            // order: the two ELL sections merged by CSR slot)
            double zf = 0.0;
            if (act) {
                double mV = 0.0, mT = 0.0, dV = 0.0, dT = 0.0;
                int lo = 0, lg = 0;
                const double app = p.applied_voltage, bt = p.boundary_temp;
                for (int n = 0; n < s_end - s_beg; ++n) {
                    const int so = lo < r0.w0 ? __ldg(P.esrc + c.ell_base + r0.k0 + 32 * lo) : 0x7fffffff;
                    const int sg2 = lg < r0.w1 ? __ldg(P.esrc + c.ell_base + r0.k1 + 32 * lg) : 0x7fffffff;
                    const bool own = (unsigned)so < (unsigned)sg2;
                    const int k = own ? r0.k0 + 32 * lo : r0.k1 + 32 * lg;
                    const int s = own ? so : sg2;
                    if (own) ++lo; else ++lg;
                    const uint8_t ck = lkind[lds_u16(E.ec_s + 2u * k)];
                    const int cV = ck & 3, cT = ck >> 2;
                    const double2 v = lds2(E.ev_s + 16u * k);
                    const double vs = mul(v.x, scale);
                    if (!kV && cV) mV = add(mV, mul(vs, dof_value(cV, app, bt)));
                    if (!kT && cT) mT = add(mT, mul(v.y, dof_value(cT, app, bt)));
                    double outV = vs, outT = v.y;
                    const bool diag = s == s_diag;
                    if (kV || cV) outV = (kV && diag) ? 1.0 : 0.0;
                    if (kT || cT) outT = (kT && diag) ? 1.0 : 0.0;
                    sts2(E.ev_s + 16u * k, d2(outV, outT));
                    if (diag) {
                        dV = outV;
                        dT = outT;
                    }
                }
                const double2 b = d2(kV ? dof_value(kV, app, bt) : sub(0.0, mV), kT ? dof_value(kT, app, bt) : sub(rt, mT));
                reinterpret_cast<double2*>(S.rhs)[g] = b;
                if (PRE) {
                    if (s_diag < 0) dV = dT = 0.0;
                    if (dV == 0.0 || dT == 0.0) zf = 1.0;
                    sts2(E.rmv_s + 16u * r0.t, d2(1.0 / dV, 1.0 / dT));
                } else {
                    sts2(E.rmv_s + 16u * r0.t, d2(1.0, 1.0));
                }
            }
            __syncthreads();  // values, rhs and M^-1 of the CTA complete (rhs: own rows only, read by own rows)
            if (PRE && S.blk) {
                E.blk = 1;
                c_block_setup<1>(E, rc, &red[0][0]);
            }
            const long long tb = global_ns_c();
            // ---- solve from the pass's start (the predictor with V extrapolated on a step's first pass)
            CRow R[1];
            const bool x0_new = S.vx0 && it == 1;
            R[0].x = act ? (x0_new ? X(inew)[g] : xit[g]) : d2(0.0, 0.0);
            double delta = -1.0;
            const CpcgOut o = cpcg_core<PRE, 1>(E, rc, R, reinterpret_cast<const double2*>(S.rhs), -1.0, zf, xit,
                                                &delta, X(inew));
            const long long tc = global_ns_c();
            asm_ns += tb - ta;
            sol_ns += tc - tb;
            if (o.status == RAFEM_ERR_INVALID) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
                status = RAFEM_ERR_INVALID;
                abort_run = true;
                break;
            }
            if (o.status == RAFEM_ERR_BREAKDOWN) break;  // SolverError -> step failure (fem.py:511-515)
            inner += o.total;
            if (!o.converged) break;  // fem.py:517-524
            if (!(delta >= 0.0)) {  // b == 0 (x = 0): the delta from the fields
                double dm = 0.0;
                if (act) {
                    const double2 xo = xit[g], xn = d2(0.0, 0.0);
                    const double d0 = fabs(sub(xn.x, xo.x)) / fmax(1.0, fabs(xo.x));
                    const double d1 = fabs(sub(xn.y, xo.y)) / fmax(1.0, fabs(xo.y));
                    dm = (d0 > dm || d0 != d0) ? d0 : dm;
                    dm = (d1 > dm || d1 != d1) ? d1 : dm;
                }
                c_xbegin(E, xpart);
                c_publish<true>(E, 0.0, 0.0, 0.0, dm);
                c_xwait(E);
                c_gather<true>(E, co);
                delta = co[3];
            }
            const int tmp = iit;
            iit = inew;
            inew = tmp;
            if (delta < p.corrector_tol) {
                conv = true;
                break;
            }
        }
        if (abort_run) break;
        corr += iters;
        if (conv) {  // accept (fem.py:603-628)
            const int old_prev = iprev;
            iprev = iacc;
            iacc = iit;
            iit = old_prev;
            dt_prev = dt;
            t = final_step ? p.total_time : t + dt;
            if (S.ring) {
                double* slot = S.ring + (step % S.ring_slots) * (n2 + 4);
                if (act) reinterpret_cast<double2*>(slot + 4)[g] = X(iacc)[g];
                if (rank == 0 && threadIdx.x == 0) {
                    slot[0] = t;
                    slot[1] = dt;
                    slot[2] = (double)iters;
                    slot[3] = 0.0;
                }
            }
            if (step < S.rec_cap) {
                if (S.rec_x && act) reinterpret_cast<double2*>(S.rec_x + step * n2)[g] = X(iacc)[g];
                if (rank == 0 && threadIdx.x == 0) {
                    S.rec_time[step] = t;
                    S.rec_dt[step] = dt;
                    S.rec_iters[step] = iters;
                }
            }
            ++step;
            if (iters <= 5)
                dt_state = fmin(dt * 1.5, p.dt_max);
            else if (iters >= 20)
                dt_state = fmax(dt * 0.75, p.dt_min);
            else
                dt_state = dt;
        } else {
            if (dt <= p.dt_min) {  // StepFailureError (fem.py:629-631)
                status = RAFEM_ERR_STEP_FAILURE;
                failed_step = (int)step;
                failed_dt = dt;
                break;
            }
            dt_state = fmax(dt * 0.5, p.dt_min);
            ++halv;
        }
    }
    if (act) reinterpret_cast<double2*>(S.final_x)[g] = X(iacc)[g];
    __syncthreads();
    cl_sync();  // the last record is complete everywhere; no CTA leaves before its peers
    if (rank == 0 && threadIdx.x == 0) {
        if (S.ring) {
            __threadfence_system();
            *S.prog = step;
        }
        SimDevOut* o = S.out;
        o->accepted = step;
        o->corr = corr;
        o->inner = inner;
        o->halvings = halv;
        o->passes = passes;
        o->t = t;
        o->status = status;
        o->failed_step = failed_step;
        o->failed_dt = failed_dt;
        o->bad = bad;
        o->asm_ns = asm_ns;
        o->solve_ns = sol_ns;
    }
}

// ---------------------------------------------------------------------------
// host: plans

struct ClusterPlan {
    unsigned long long pattern_id = 0;
    const int* rp = nullptr;
    int N = 0, C = 0, nt = 0;
    size_t smem = 0;  // dynamic shared memory of the solve kernel
    size_t smem_blk = 0;  // + the block-Jacobi y buffer
    size_t smem_gm = 0;   // GMRES: one gathered-vector buffer + the own rows of w
    size_t smem_sim = 0;
    void* dev = nullptr;
    CPlan view{};
    bool ok = false;
};

static std::vector<void*>& plans(rafem_ctx* ctx) { return ctx->cluster_plans; }

void cluster_plans_release(rafem_ctx* ctx) {
    auto& v = plans(ctx);
    for (void* q : v) {
        ClusterPlan* p = static_cast<ClusterPlan*>(q);
        if (p->dev) dfree(ctx, p->dev);
        delete p;
    }
    v.clear();
}

static size_t al16(size_t b) { return (b + 15) & ~(size_t)15; }

// Build (or fetch) the plan of a node pattern for C CTAs.  Returns nullptr
// when the pattern does not fit the engine (rows per CTA, shared memory,
// ghost fan-out), with rc = RAFEM_OK; rc != OK on CUDA errors.
static ClusterPlan* cluster_plan(rafem_ctx* ctx, const int* rp_dev, const int* col_dev, const double* coords_dev,
                                 int N, long long S, unsigned long long pattern_id, int C, int& rc) {
    rc = RAFEM_OK;
    auto& v = plans(ctx);
    for (void* q : v) {
        ClusterPlan* p = static_cast<ClusterPlan*>(q);
        if (p->pattern_id == pattern_id && p->rp == rp_dev && p->C == C) return p->ok ? p : nullptr;
    }
    ClusterPlan* P = new ClusterPlan;
    P->pattern_id = pattern_id;
    P->rp = rp_dev;
    P->N = N;
    P->C = C;
    if (v.size() >= 8) {  // bounded cache: drop the oldest plan
        ClusterPlan* old = static_cast<ClusterPlan*>(v.front());
        if (old->dev) dfree(ctx, old->dev);
        delete old;
        v.erase(v.begin());
    }
    v.push_back(P);
    if (N < C || S <= 0 || S > (1LL << 30)) return nullptr;
    std::vector<int> rp(N + 1), col((size_t)S);
    cudaError_t e = cudaMemcpyAsync(rp.data(), rp_dev, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(col.data(), col_dev, sizeof(int) * (size_t)S, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        rc = rafem_fail_cuda(ctx, e, "cluster plan download", __FILE__, __LINE__);
        return nullptr;
    }
    // ---- partition: recursive coordinate bisection of the nodes when the
    // mesh geometry is known (compact blocks: ~3x fewer ghosts than row
    // slabs on box meshes), else contiguous row blocks balanced by slots + rows
    std::vector<int> owner(N, -1);
    auto env_on = [](const char* k, bool dflt) {
        const char* v = getenv(k);
        return v ? v[0] != '0' : dflt;
    };
    // row slabs by default: RCB blocks have ~3x fewer ghosts but their rows'
    // stencils vary within a warp (ELL padding or scattered gathers), which
    // cost more than the halo they save (scripts/cluster_probe2.py)
    const bool use_rcb = env_on("RAFEM_CL_RCB", false), split = env_on("RAFEM_CL_SPLIT", true),
               sort_rows = env_on("RAFEM_CL_SORT", true);
    if (coords_dev && use_rcb) {
        std::vector<double> X((size_t)3 * N);
        e = cudaMemcpyAsync(X.data(), coords_dev, sizeof(double) * 3 * (size_t)N, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            rc = rafem_fail_cuda(ctx, e, "cluster plan coordinates", __FILE__, __LINE__);
            return nullptr;
        }
        std::vector<int> ids(N);
        for (int i = 0; i < N; ++i) ids[i] = i;
        struct Rcb {
            const std::vector<double>& X;
            std::vector<int>& owner;
            void run(std::vector<int>::iterator b, std::vector<int>::iterator e, int parts, int base) {
                if (parts == 1) {
                    for (auto it = b; it != e; ++it) owner[*it] = base;
                    return;
                }
                double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
                for (auto it = b; it != e; ++it)
                    for (int d = 0; d < 3; ++d) {
                        lo[d] = std::min(lo[d], X[3 * (size_t)*it + d]);
                        hi[d] = std::max(hi[d], X[3 * (size_t)*it + d]);
                    }
                int ax = 0;
                for (int d = 1; d < 3; ++d)
                    if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
                std::sort(b, e, [&](int a, int c) {
                    const double xa = X[3 * (size_t)a + ax], xc = X[3 * (size_t)c + ax];
                    return xa < xc || (xa == xc && a < c);
                });
                const int lp = parts / 2;
                const auto m = b + (long long)(e - b) * lp / parts;
                run(b, m, lp, base);
                run(m, e, parts - lp, base + lp);
            }
        } rcb{X, owner};
        rcb.run(ids.begin(), ids.end(), C, 0);
    } else {
        std::vector<int> gp(C + 1);
        auto cut = [&](int wslot) {
            const long long tot = (long long)wslot * rp[N] + N;
            int g = 0;
            gp[0] = 0;
            for (int c = 1; c < C; ++c) {
                const long long want = tot * c / C;
                while (g < N && (long long)wslot * rp[g] + g < want) ++g;
                gp[c] = g;
            }
            gp[C] = N;
            for (int c = 0; c < C; ++c)
                if (gp[c + 1] - gp[c] > kRPT * kCT || gp[c + 1] - gp[c] < 1) return false;
            return true;
        };
        if (!cut(1) && !cut(0)) return nullptr;
        for (int c = 0; c < C; ++c)
            for (int g = gp[c]; g < gp[c + 1]; ++g) owner[g] = c;
    }
    std::vector<std::vector<int>> rows(C);
    for (int g = 0; g < N; ++g) rows[owner[g]].push_back(g);
    for (int c = 0; c < C; ++c)
        if (rows[c].empty() || (int)rows[c].size() > kRPT * kCT) return nullptr;
    std::vector<CCta> ct(C);
    std::vector<int4> warps;
    std::vector<uint16_t> ecol;
    std::vector<int> esrc, lgid;
    std::vector<int2> trow;
    std::vector<unsigned> dest((size_t)N * kCDest, 0xffffffffu);
    std::vector<int> ndest(N, 0);
    int ell_cap = 0, nloc_cap = 0, nt = 32;
    std::vector<int> loc(N, -1);
    for (int c = 0; c < C; ++c) {
        // own rows ordered by (ghost slots, own slots) descending, then id:
        // rows of one warp then share their section widths (little ELL padding)
        std::vector<int>& R = rows[c];
        const int nr = (int)R.size();
        auto n_own = [&](int g) {
            int a = 0;
            for (int s2 = rp[g]; s2 < rp[g + 1]; ++s2) a += owner[col[s2]] == c;
            return a;
        };
        std::vector<std::pair<std::pair<int, int>, int>> key(nr);
        for (int t = 0; t < nr; ++t) {
            const int g = R[t], a = n_own(g), b = rp[g + 1] - rp[g] - a;
            key[t] = {{-b, -a}, g};
        }
        if (sort_rows) {
            std::sort(key.begin(), key.end());
            for (int t = 0; t < nr; ++t) R[t] = key[t].second;
        }
        std::vector<int> gh;
        for (int g : R)
            for (int s2 = rp[g]; s2 < rp[g + 1]; ++s2)
                if (owner[col[s2]] != c) gh.push_back(col[s2]);
        std::sort(gh.begin(), gh.end(), [&](int a, int b) {
            return owner[a] < owner[b] || (owner[a] == owner[b] && a < b);
        });
        gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
        const int nloc = nr + (int)gh.size();
        if (nloc > 65535) return nullptr;
        CCta& cc = ct[c];
        cc.g0 = 0;
        cc.nr = nr;
        cc.nloc = nloc;
        cc.lbase = (int)lgid.size();
        // local (gathered-vector) index: own rows in id order, so a warp's
        // k-th neighbours sit at consecutive slots (conflict-free gathers);
        // threads take the rows in the width-sorted order above
        std::vector<int> Rn = R;
        std::sort(Rn.begin(), Rn.end());
        for (int t = 0; t < nr; ++t) {
            loc[Rn[t]] = t;
            lgid.push_back(Rn[t]);
        }
        for (int t = 0; t < nr; ++t) trow.push_back(make_int2(R[t], loc[R[t]]));
        for (size_t q = 0; q < gh.size(); ++q) trow.push_back(make_int2(-1, -1));
        for (size_t q = 0; q < gh.size(); ++q) {
            const int j = gh[q];
            loc[j] = nr + (int)q;
            lgid.push_back(j);
            if (ndest[j] >= kCDest) return nullptr;
            dest[(size_t)j * kCDest + ndest[j]++] = ((unsigned)c << 16) | (unsigned)(nr + q);
        }
        cc.wbase = (int)warps.size();
        cc.ell_base = (int)esrc.size();
        const int nwarp = (nr + 31) / 32;
        int off = 0;
        // split: own-column slots first (summed before the exchange wait);
        // else every slot in the second section
        auto is_own = [&](int j) { return split && owner[j] == c; };
        for (int w = 0; w < nwarp; ++w) {
            int wo = 0, wg = 0;
            for (int t = 32 * w; t < std::min(nr, 32 * w + 32); ++t) {
                const int g = R[t];
                int a = 0, b = 0;
                for (int s2 = rp[g]; s2 < rp[g + 1]; ++s2) (is_own(col[s2]) ? a : b)++;
                wo = std::max(wo, a);
                wg = std::max(wg, b);
            }
            warps.push_back(make_int4(off, wo, off + 32 * wo, wg));
            for (int sec = 0; sec < 2; ++sec) {
                const int wd = sec ? wg : wo;
                for (int l = 0; l < wd; ++l)
                    for (int ln = 0; ln < 32; ++ln) {
                        const int t = 32 * w + ln;
                        int src = -1, lc = 0;
                        if (t < nr) {  // the l-th slot of this section in storage order
                            const int g = R[t];
                            int k = 0;
                            for (int s2 = rp[g]; s2 < rp[g + 1]; ++s2)
                                if (is_own(col[s2]) == (sec == 0) && k++ == l) {
                                    src = s2;
                                    break;
                                }
                            if (src >= 0) lc = loc[col[src]];
                        }
                        esrc.push_back(src);
                        ecol.push_back((uint16_t)lc);
                    }
            }
            off += 32 * (wo + wg);
        }
        cc.ell_n = off;
        ell_cap = std::max(ell_cap, off);
        nloc_cap = std::max(nloc_cap, nloc);
        nt = std::max(nt, (nwarp + kRPT - 1) / kRPT * 32);
        for (int g : R) loc[g] = -1;
        for (int j : gh) loc[j] = -1;
    }
    // every CTA addresses warp blocks up to kRPT * nt / 32 (idle blocks: width 0)
    {
        std::vector<int4> w2;
        std::vector<CCta> ct2 = ct;
        for (int c = 0; c < C; ++c) {
            ct2[c].wbase = (int)w2.size();
            const int nwarp = (ct[c].nr + 31) / 32;
            for (int w = 0; w < kRPT * nt / 32; ++w)
                w2.push_back(w < nwarp ? warps[ct[c].wbase + w] : make_int4(0, 0, 0, 0));
        }
        warps.swap(w2);
        ct.swap(ct2);
    }
    ell_cap = (ell_cap + 7) & ~7;
    nloc_cap = (nloc_cap + 7) & ~7;
    // push targets: one uint4 per row when no row feeds more than 4 CTAs
    int maxd = 0;
    for (int j = 0; j < N; ++j) maxd = std::max(maxd, ndest[j]);
    const int ndw = maxd <= 4 ? 1 : 2;
    if (ndw == 1) {
        std::vector<unsigned> d1((size_t)N * 4);
        for (int j = 0; j < N; ++j)
            for (int k = 0; k < 4; ++k) d1[(size_t)j * 4 + k] = dest[(size_t)j * kCDest + k];
        dest.swap(d1);
    }
    const int rows_cap = kRPT * nt;
    P->smem = c_layout_bytes(ell_cap, nloc_cap, rows_cap, ndw, 0);
    P->smem_blk = c_layout_bytes(ell_cap, nloc_cap, rows_cap, ndw, 1);
    P->smem_sim = P->smem_blk + al16((size_t)nloc_cap);  // + local node kinds
    P->smem_gm = c_layout_bytes(ell_cap, nloc_cap, rows_cap, ndw, 1, 1);
    if (P->smem > 225 * 1024) return nullptr;
    // upload
    const size_t o_cta = 0, o_w = al16(sizeof(CCta) * C), o_ec = o_w + al16(sizeof(int4) * warps.size());
    const size_t o_es = o_ec + al16(2 * ecol.size()), o_de = o_es + al16(4 * esrc.size());
    const size_t o_lg = o_de + al16(4 * dest.size()), o_tr = o_lg + al16(4 * lgid.size());
    const size_t tot = o_tr + al16(8 * trow.size());
    std::vector<unsigned char> h(tot);
    std::memcpy(h.data() + o_cta, ct.data(), sizeof(CCta) * C);
    std::memcpy(h.data() + o_w, warps.data(), sizeof(int4) * warps.size());
    std::memcpy(h.data() + o_ec, ecol.data(), 2 * ecol.size());
    std::memcpy(h.data() + o_es, esrc.data(), 4 * esrc.size());
    std::memcpy(h.data() + o_de, dest.data(), 4 * dest.size());
    std::memcpy(h.data() + o_lg, lgid.data(), 4 * lgid.size());
    std::memcpy(h.data() + o_tr, trow.data(), 8 * trow.size());
    e = dmalloc(ctx, &P->dev, tot);
    if (e == cudaSuccess) e = cudaMemcpyAsync(P->dev, h.data(), tot, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        rc = rafem_fail_cuda(ctx, e, "cluster plan upload", __FILE__, __LINE__);
        return nullptr;
    }
    unsigned char* d = static_cast<unsigned char*>(P->dev);
    P->view.cta = reinterpret_cast<const CCta*>(d + o_cta);
    P->view.warp = reinterpret_cast<const int4*>(d + o_w);
    P->view.ecol = reinterpret_cast<const uint16_t*>(d + o_ec);
    P->view.esrc = reinterpret_cast<const int*>(d + o_es);
    P->view.dest = reinterpret_cast<const unsigned*>(d + o_de);
    P->view.lgid = reinterpret_cast<const int*>(d + o_lg);
    P->view.trow = reinterpret_cast<const int2*>(d + o_tr);
    P->view.C = C;
    P->view.ell_cap = ell_cap;
    P->view.nloc_cap = nloc_cap;
    P->view.rows_cap = rows_cap;
    P->view.ndw = ndw;
    P->nt = nt;
    P->ok = true;
    return P;
}

static int cluster_size_for(int N) {
    int C = kCMax;
    if (const char* e = getenv("RAFEM_CLUSTER_C")) C = std::max(1, std::min(kCMax, atoi(e)));
    while (C > 1 && N < C * 64) C /= 2;
    return C;
}

static bool cluster_launchable_uncached(rafem_ctx* ctx, const void* fn, int C, int nt, size_t smem);
// The attribute calls and the occupancy query cost tens of microseconds; a
// solve on the plug-in seam is ~100 us, so the answer is cached per
// (kernel, cluster size, threads) and the attribute raised to the largest
// shared memory asked so far.
static bool cluster_launchable(rafem_ctx* ctx, const void* fn, int C, int nt, size_t smem) {
    struct Key {
        const void* fn;
        int C, nt;
        size_t smem;
        bool ok;
    };
    static std::vector<Key> cache;
    for (const Key& k : cache)
        if (k.fn == fn && k.C == C && k.nt == nt && k.smem >= smem && k.ok) return true;
    const bool ok = cluster_launchable_uncached(ctx, fn, C, nt, smem);
    if (ok) cache.push_back({fn, C, nt, smem, ok});
    return ok;
}
static bool cluster_launchable_uncached(rafem_ctx* ctx, const void* fn, int C, int nt, size_t smem) {
    // the attribute never goes down: launches cached earlier may need more
    static std::vector<std::pair<const void*, size_t>> maxset;
    size_t smax = smem;
    for (auto& e : maxset)
        if (e.first == fn) smax = std::max(smax, e.second);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) == cudaSuccess && ncl >= 1;
    cudaGetLastError();
    bool found = false;
    for (auto& e : maxset)
        if (e.first == fn) {
            e.second = smax;
            found = true;
        }
    if (!found) maxset.push_back({fn, smax});
    return ok;
}

static cudaError_t cluster_launch(rafem_ctx* ctx, const void* fn, int C, int nt, size_t smem, void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// GMRES(m <= 30) on a node-paired system that fits one cluster (RAFEM_CLUSTER=0
// disables it).  Same result block and history layout as the grid GMRES.
static int cluster_gmres_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, double* x_dev,
                               const double* minv_dev, const rafem_solver_params& p, KResult* res_dev, int* flag_dev,
                               cudaEvent_t ev_start, cudaEvent_t ev_stop) {
    if (p.restart_m < 1 || p.restart_m > kGM) return RAFEM_ERR_UNSUPPORTED;
    const int N = A.ngroups;
    const int C = cluster_size_for(N);
    int rc = RAFEM_OK;
    ClusterPlan* P = cluster_plan(ctx, A.rp, A.col, A.coords, N, A.slots, A.pattern_id, C, rc);
    if (rc) return rc;
    if (!P) return RAFEM_ERR_UNSUPPORTED;
    const bool pre = p.precondition != RAFEM_PRECOND_NONE;
    const size_t smem = P->smem_gm;
    const void* fn = pre ? (const void*)cgmres_kernel<true> : (const void*)cgmres_kernel<false>;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) {
        cudaGetLastError();
        return RAFEM_ERR_UNSUPPORTED;
    }
    if (smem + fa.sharedSizeBytes > 227 * 1024) return RAFEM_ERR_UNSUPPORTED;
    if (!cluster_launchable(ctx, fn, C, P->nt, smem)) return RAFEM_ERR_UNSUPPORTED;
    const long long n = 2LL * N;
    const long long hist_cap = std::min<long long>(p.max_total_iters > 0 ? p.max_total_iters : 10LL * n, 1LL << 20) + 1;
    if (int r = ensure(ctx, ctx->ws_hist, sizeof(double) * (size_t)hist_cap)) return r;
    if (int r = ensure(ctx, ctx->ws_cyc, sizeof(long long) * (size_t)hist_cap)) return r;
    if (int r = ensure(ctx, ctx->ws_basis, sizeof(double2) * (size_t)C * (kGM + 1) * P->view.rows_cap)) return r;
    CPlan view = P->view;
    const double2* val2 = reinterpret_cast<const double2*>(A.val);
    double tol = p.tolerance;
    long long cap = p.max_total_iters > 0 ? p.max_total_iters : 10LL * n;
    int m = p.restart_m;
    double* hist = static_cast<double*>(ctx->ws_hist.p);
    long long* cyc = static_cast<long long*>(ctx->ws_cyc.p);
    long long hc = hist_cap, cc = hist_cap;
    const double* minv = pre ? minv_dev : nullptr;
    double2* basis = static_cast<double2*>(ctx->ws_basis.p);
    void* args[] = {&view, &val2, &b_dev, &x_dev, &minv, &flag_dev, &tol, &cap, &m, &hist, &hc, &cyc, &cc,
                    &res_dev, &basis};
    if (ev_start) RF_CUDA_TRY(ctx, cudaEventRecord(ev_start, ctx->stream));
    RF_CUDA_TRY(ctx, cluster_launch(ctx, fn, C, P->nt, smem, args));
    if (ev_stop) RF_CUDA_TRY(ctx, cudaEventRecord(ev_stop, ctx->stream));
    ctx->launches++;
    ctx->last_mode = 5;
    ctx->last_ctas = C;
    ctx->last_team = 1;
    ctx->last_precond = pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE;
    return RAFEM_OK;
}

// Eligibility: PCG (Jacobi, block-Jacobi or none) or GMRES(m <= 30) on a
// node-paired system small enough for one cluster's shared memory.
// RAFEM_CLUSTER=0 disables the engine.
int cluster_pcg_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, double* x_dev, const double* minv_dev,
                      const rafem_solver_params& p, KResult* res_dev, int* flag_dev, cudaEvent_t ev_start,
                      cudaEvent_t ev_stop) {
    const char* env = getenv("RAFEM_CLUSTER");
    if (env && env[0] == '0') return RAFEM_ERR_UNSUPPORTED;
    if (A.W != 2 || !A.pattern_id || p.grid_ctas > 0) return RAFEM_ERR_UNSUPPORTED;
    if (p.method != RAFEM_METHOD_PCG) {
        // opt-in (RAFEM_CLUSTER_GMRES=1): measured no faster than the grid
        // GMRES (14.2 vs 14.1 us per inner step on mesh-B; the three
        // exchanges and the basis sweeps through L2 per step are latency
        // chains on 16 SMs, and batching the basis loads spills at the
        // 96-register cap of 576-thread CTAs: 30 us), profiles/r2b_cgmres_probe.txt
        const char* g = getenv("RAFEM_CLUSTER_GMRES");
        if (!(g && g[0] == '1')) return RAFEM_ERR_UNSUPPORTED;
        return cluster_gmres_solve(ctx, A, b_dev, x_dev, minv_dev, p, res_dev, flag_dev, ev_start, ev_stop);
    }
    const int N = A.ngroups;
    const int C = cluster_size_for(N);
    int rc = RAFEM_OK;
    ClusterPlan* P = cluster_plan(ctx, A.rp, A.col, A.coords, N, A.slots, A.pattern_id, C, rc);
    if (rc) return rc;
    if (!P) return RAFEM_ERR_UNSUPPORTED;
    const bool pre = p.precondition != RAFEM_PRECOND_NONE;
    int blk = p.precondition == RAFEM_PRECOND_BLOCK_JACOBI ? 1 : 0;
    const size_t smem = blk ? P->smem_blk : P->smem;
    if (smem > 225 * 1024) return RAFEM_ERR_UNSUPPORTED;
    const void* fn = pre ? (const void*)cpcg_kernel<true> : (const void*)cpcg_kernel<false>;
    if (!cluster_launchable(ctx, fn, C, P->nt, smem)) return RAFEM_ERR_UNSUPPORTED;
    const long long n = 2LL * N;
    const long long hist_cap = std::min<long long>(p.max_total_iters > 0 ? p.max_total_iters : 10LL * n, 1LL << 20) + 1;
    if (int r = ensure(ctx, ctx->ws_hist, sizeof(double) * (size_t)hist_cap)) return r;
    if (int r = ensure(ctx, ctx->ws_cyc, sizeof(long long) * (size_t)hist_cap)) return r;
    CPlan view = P->view;
    const double2* val2 = reinterpret_cast<const double2*>(A.val);
    double tol = p.tolerance;
    long long cap = p.max_total_iters > 0 ? p.max_total_iters : 10LL * n;
    double* hist = static_cast<double*>(ctx->ws_hist.p);
    long long* cyc = static_cast<long long*>(ctx->ws_cyc.p);
    long long hc = hist_cap, cc = hist_cap;
    const double* minv = pre ? minv_dev : nullptr;
    long long* trace = nullptr;
    long long tcap = 0;
    if (ctx->trace_on) {
        if (int r = ensure(ctx, ctx->ws_trace, sizeof(long long) * 8 * 4096)) return r;
        RF_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ws_trace.p, 0, sizeof(long long) * 8 * 4096, ctx->stream));
        trace = static_cast<long long*>(ctx->ws_trace.p);
        tcap = 8 * 4096;
    }
    int abl = 0;
    if (const char* ab = getenv("RAFEM_CL_ABL")) abl = atoi(ab);
    void* args[] = {&view, &val2, &b_dev, &x_dev, &minv, &flag_dev, &tol, &cap, &hist, &hc, &cyc, &cc, &res_dev,
                    &trace, &tcap, &abl, &blk};
    if (ev_start) RF_CUDA_TRY(ctx, cudaEventRecord(ev_start, ctx->stream));
    RF_CUDA_TRY(ctx, cluster_launch(ctx, fn, C, P->nt, smem, args));
    if (ev_stop) RF_CUDA_TRY(ctx, cudaEventRecord(ev_stop, ctx->stream));
    ctx->launches++;
    ctx->last_mode = 5;
    ctx->last_ctas = C;
    ctx->last_team = 1;
    ctx->last_precond = blk ? RAFEM_PRECOND_BLOCK_JACOBI : (pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE);
    return RAFEM_OK;
}

}  // namespace rafem

namespace rafem {

// The whole simulation on one cluster when the mesh fits; opt-in
// (RAFEM_SIM_CLUSTER=1).  Measured on the mesh-B analog (scripts/csim_probe.py,
// profiles/r2b_csim_probe.txt): same trajectory and fields within 2e-7 of
// the 148-CTA fused kernel, block-Jacobi iterations 4,172 vs 4,655, but the
// per-pass assembly on 16 SMs is L2-latency bound (220 us vs 14 us: each
// row's contributor walk is a chain of dependent L2 loads) and the PCG
// loop spills next to the time-loop state, so the fused grid kernel stays
// the default.  RAFEM_ERR_UNSUPPORTED lets simulate_fused take over.
int simulate_cluster(rafem_system* s, const rafem_sim_params* p, SimDevOut* out, double* rec_x_dev,
                     double* rec_time_dev, double* rec_dt_dev, int* rec_iters_dev, long long rec_cap,
                     double* final_x_dev, float* ms, const SimStream* stream) {
    const char* env = getenv("RAFEM_SIM_CLUSTER");
    if (!(env && env[0] == '1')) return RAFEM_ERR_UNSUPPORTED;
    rafem_mesh* mesh = s->mesh;
    rafem_ctx* ctx = mesh->ctx;
    const int N = mesh->N;
    if (N == 0 || mesh->M == 0 || p->solver.method != RAFEM_METHOD_PCG || mesh->nreg > kCRegions)
        return RAFEM_ERR_UNSUPPORTED;
    if (!mesh->slot_lists_tried)
        if (int rc = mesh_slot_lists(mesh)) return rc;
    if (!mesh->slot_ptr) return RAFEM_ERR_UNSUPPORTED;
    const int C = cluster_size_for(N);
    int rc = RAFEM_OK;
    ClusterPlan* P = cluster_plan(ctx, mesh->rp, mesh->col, mesh->nodes, N, mesh->slots, mesh->id, C, rc);
    if (rc) return rc;
    if (!P) return RAFEM_ERR_UNSUPPORTED;
    const bool pre = p->solver.precondition != RAFEM_PRECOND_NONE;
    const int blk = p->solver.precondition == RAFEM_PRECOND_BLOCK_JACOBI ? 1 : 0;
    const size_t smem = P->smem_sim;
    if (smem > 223 * 1024) return RAFEM_ERR_UNSUPPORTED;
    const void* fn = pre ? (const void*)csim_kernel<true> : (const void*)csim_kernel<false>;
    if (!cluster_launchable(ctx, fn, C, P->nt, smem)) return RAFEM_ERR_UNSUPPORTED;
    if (int r = system_escal(s)) return r;
    if (int r = ensure(ctx, ctx->ws_simout, sizeof(SimDevOut))) return r;
    CSimArgs S{};
    S.P = P->view;
    S.m = asm_mesh(mesh);
    S.xs = s->xs;
    S.final_x = final_x_dev;
    S.esig = s->esig;
    S.eload = s->eload;
    S.rhs = s->rhs;
    S.n2 = 2LL * N;
    S.p = *p;
    S.rec_x = rec_x_dev;
    S.rec_time = rec_time_dev;
    S.rec_dt = rec_dt_dev;
    S.rec_iters = rec_iters_dev;
    S.rec_cap = rec_cap;
    S.out = static_cast<SimDevOut*>(ctx->ws_simout.p);
    S.blk = blk;
    {
        const char* nv = getenv("RAFEM_NO_VX0");
        S.vx0 = !(nv && nv[0] == '1');
    }
    if (stream) {
        S.ring = stream->ring;
        S.ring_slots = stream->slots;
        S.prog = stream->prog;
        S.cons = stream->cons;
    }
    void* args[] = {&S};
    RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    RF_CUDA_TRY(ctx, cluster_launch(ctx, fn, C, P->nt, smem, args));
    RF_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->launches++;
    ctx->last_mode = 6;
    ctx->last_ctas = C;
    ctx->last_team = 1;
    ctx->last_precond = blk ? RAFEM_PRECOND_BLOCK_JACOBI : (pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE);
    if (stream && stream->pump) {  // consume records while the kernel runs
        if (int r = stream->pump(stream->user)) return r;
    }
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->ws_simout.p, sizeof(SimDevOut), cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ms) cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1);
    return RAFEM_OK;
}

}  // namespace rafem
