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

constexpr int kCT = 576;     // max node rows (threads) per CTA (launch bound: 112 registers)
constexpr int kCDest = 4;    // max other CTAs one row is a ghost of
constexpr int kCMax = 16;    // max cluster size (non-portable)
constexpr int kCRegions = 16;

struct CCta {
    int g0, nr, nloc, ell_n;
    int ell_base, wbase, lbase, pad;
};

struct CPlan {
    const CCta* cta;
    const int4* warp;        // per warp: own-column section (offset, width), ghost-column section (offset, width)
    const uint16_t* ecol;    // ELL local columns (pads: 0)
    const int* esrc;         // ELL entry -> CSR slot, -1 for pads
    const unsigned* dest;    // N x kCDest: cta << 16 | local index; 0xffffffff none
    const int* lgid;         // per CTA: global node id of every local index
    int C, ell_cap, nloc_cap;
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
RF_DEV unsigned cl_map(const void* local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
RF_DEV void st_cluster2(unsigned addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
// 16 bytes into a peer's shared memory, completing 16 transaction bytes on
// the peer's mbarrier (data and signal in one message, no fence)
RF_DEV void st_async2(unsigned addr, double a, double b, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(a), "d"(b), "r"(rbar)
                 : "memory");
}
RF_DEV void mbar_wait_cluster(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "XW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra XW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Shared state of one CTA of the engine.
struct CEnv {
    double2* ev;        // ELL values
    const uint16_t* ec; // ELL local columns
    double2* mb;        // 2 x nloc_cap gathered-vector buffers
    int nloc_cap;
    double (*part)[kCMax][4];  // [2][C][4] pushed CTA partials
    double (*red)[4];          // [32][4] warp partials
    int C;
    unsigned rank;
    int t, nr;          // this thread's local row (active when t < nr)
    int k0, width;      // own-column ELL section: this thread's first entry, slot positions
    int k1, width1;     // ghost-column section
    const uint4* rdest; // per own row: the CTAs (cta << 16 | ghost index) it is pushed to
    double2* rb;        // per own row: right-hand side (heads only)
    const double2* rmv; // per own row: Jacobi inverse diagonal
    // exchanges: every CTA pushes its vector entries into the ghost slots of
    // its readers and its 4 CTA partials into every CTA, each message
    // completing transaction bytes on the receiver's mbarrier xbar[k & 1]
    unsigned long long* xbar;  // 2 mbarriers
    unsigned xk, xw;           // exchanges begun / waited
    unsigned xbytes;           // bytes a CTA receives per exchange
    // PCG contract
    double tol;
    long long cap;
    double* hist;
    long long hist_cap;
    long long* cyc;
    long long cyc_cap;
    long long* trace;   // optional per-iteration clock64 stamps (rank 0, thread 0), 8 per iteration
    long long trace_cap;
};

RF_DEV void c_stamp(const CEnv& E, long long it, int k) {
    if (E.trace && E.rank == 0 && threadIdx.x == 0 && it * 8 + k < E.trace_cap) E.trace[it * 8 + k] = clock64();
}

// Partial row sum over one ELL section (left to right over its positions).
RF_DEV void c_spmv_sec(const double2* __restrict__ ev, const uint16_t* __restrict__ ec, int width,
                       const double2* src, double& av, double& at) {
    int l = 0;
#pragma unroll 1
    for (; l + 4 <= width; l += 4) {
        int c[4];
        double2 a[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c[j] = ec[(l + j) * 32];
            a[j] = ev[(l + j) * 32];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = src[c[j]];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            av = fma(a[j].x, v[j].x, av);
            at = fma(a[j].y, v[j].y, at);
        }
    }
#pragma unroll 1
    for (; l < width; ++l) {
        const double2 a = ev[l * 32];
        const double2 v = src[ec[l * 32]];
        av = fma(a.x, v.x, av);
        at = fma(a.y, v.y, at);
    }
}
// Own-column part of row t of A src (needs only this CTA's entries of src).
RF_DEV double2 c_spmv_own(const CEnv& E, const double2* src) {
    double av = 0.0, at = 0.0;
    c_spmv_sec(E.ev + E.k0, E.ec + E.k0, E.width, src, av, at);
    return make_double2(av, at);
}
// + the ghost-column part (needs the pushed ghost entries).
RF_DEV double2 c_spmv_gh(const CEnv& E, const double2* src, double2 acc) {
    c_spmv_sec(E.ev + E.k1, E.ec + E.k1, E.width1, src, acc.x, acc.y);
    return acc;
}
RF_DEV double2 c_spmv(const CEnv& E, const double2* src) { return c_spmv_gh(E, src, c_spmv_own(E, src)); }

// Exchange k (= E.xk) begins: thread 0 arms the CTA's mbarrier with the
// bytes it will receive (peers' messages may already have landed: the
// transaction count then runs negative until this arrive).
RF_DEV void c_xbegin(const CEnv& E) {
    if (threadIdx.x == 0) mbar_expect_tx(E.xbar + (E.xk & 1), E.xbytes);
}

// Own row's entry of buffer `buf`: local store + a push into every CTA that
// holds the row as a ghost (exchange E.xk).
RF_DEV void c_push(const CEnv& E, int buf, double2 v) {
    double2* b = E.mb + (size_t)buf * E.nloc_cap;
    b[E.t] = v;
    const unsigned long long* bar = E.xbar + (E.xk & 1);
    const uint4 dq = E.rdest[E.t];
    const unsigned qs[4] = {dq.x, dq.y, dq.z, dq.w};
#pragma unroll
    for (int d = 0; d < kCDest; ++d) {
        const unsigned q = qs[d];
        if (q != 0xffffffffu) st_async2(cl_map(b + (q & 0xffffu), q >> 16), v.x, v.y, cl_map(bar, q >> 16));
    }
}

// CTA partials (v0..v2 summed, v3 max) of exchange E.xk into part[xk & 1][rank]
// of every CTA; closes the CTA's side of the exchange.  The bar.sync also
// publishes the own entries of the pushed vector inside the CTA.
RF_DEV void c_publish(CEnv& E, double v0, double v1, double v2, double v3) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    v2 = warp_sum(v2);
    v3 = warp_max(v3);
    if (lane == 0) {
        E.red[w][0] = v0;
        E.red[w][1] = v1;
        E.red[w][2] = v2;
        E.red[w][3] = v3;
    }
    __syncthreads();
    if (w == 0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (lane < nw) {
            s0 = E.red[lane][0];
            s1 = E.red[lane][1];
            s2 = E.red[lane][2];
            s3 = E.red[lane][3];
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        s3 = warp_max(s3);
        if (lane < E.C) {
            const unsigned a = cl_map(&E.part[E.xk & 1][E.rank][0], (unsigned)lane);
            const unsigned rb = cl_map(E.xbar + (E.xk & 1), (unsigned)lane);
            st_async2(a, s0, s1, rb);
            st_async2(a + 16, s2, s3, rb);
        }
    }
    ++E.xk;
}

// Wait for the oldest outstanding exchange (its ghosts and partials are then
// visible to every thread of the CTA).
RF_DEV void c_xwait(CEnv& E) {
    const unsigned k = E.xw++;
    mbar_wait_cluster(E.xbar + (k & 1), (k >> 1) & 1u);
}

// After the wait: combine the C partials of the last waited exchange in rank
// order (same bits in every warp of every CTA).
RF_DEV void c_gather(const CEnv& E, double (&co)[4]) {
    const int lane = threadIdx.x & 31;
    const int par = (E.xw - 1) & 1;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (lane < E.C) {
        const double2 a = *reinterpret_cast<const double2*>(&E.part[par][lane][0]);
        const double2 b = *reinterpret_cast<const double2*>(&E.part[par][lane][2]);
        s0 = a.x;
        s1 = a.y;
        s2 = b.x;
        s3 = b.y;
    }
    co[0] = warp_sum(s0);
    co[1] = warp_sum(s1);
    co[2] = warp_sum(s2);
    co[3] = warp_max(s3);
}

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

RF_DEV double2 d2(double a, double b) { return make_double2(a, b); }

// Pipelined PCG (Ghysels-Vanroose) on the cluster, pcg_pipe_core's contract.
// bnorm < 0: ||b||^2 and the zero-diagonal flag (zf, per thread) ride on the
// first head's reduction.  xold (own row, when `delta`): the corrector delta
// max|x - xold| / max(1, |xold|) of the head's iterate goes to *delta.
template <bool PRE>
RF_DEV CpcgOut cpcg_core(CEnv& E, CRow& R, double bnorm, double zf, const double2* xold, double* delta,
                         double2* xout_g) {
    const bool act = E.t < E.nr;
    long long total = 0, cycles = 0, hlen = 0;
    bool converged = false;
    double rel = INFINITY;
    int status = RAFEM_OK;
    int hb = 0;
    const bool lead = E.rank == 0 && threadIdx.x == 0;
    while (true) {
        // ---- head: r = b - A x, u = M r (x pushed, one full barrier)
        const bool with_b = bnorm < 0.0;
        c_xbegin(E);
        if (act) {
            c_push(E, hb, R.x);
            if (xout_g) xout_g[E.t] = R.x;
        }
        c_publish(E, 0.0, 0.0, 0.0, 0.0);
        c_xwait(E);
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        if (act) {
            const double2 y = c_spmv(E, E.mb + (size_t)hb * E.nloc_cap);
            const double2 bb = E.rb[E.t], mv = E.rmv[E.t];
            R.r = d2(bb.x - y.x, bb.y - y.y);
            R.u = PRE ? d2(mv.x * R.r.x, mv.y * R.r.y) : R.r;
            v2 = fma(R.r.x, R.r.x, R.r.y * R.r.y);
            if (with_b) {
                v0 = fma(bb.x, bb.x, bb.y * bb.y);
                v1 = zf;
            }
            if (xold) {
                const double2 xo = *xold;
                const double d0 = fabs(R.x.x - xo.x) / fmax(1.0, fabs(xo.x));
                const double d1 = fabs(R.x.y - xo.y) / fmax(1.0, fabs(xo.y));
                v3 = (d0 > v3 || d0 != d0) ? d0 : v3;
                v3 = (d1 > v3 || d1 != d1) ? d1 : v3;
            }
        }
        c_xbegin(E);
        if (act) c_push(E, hb ^ 1, R.u);
        c_publish(E, v0, v1, v2, v3);
        c_xwait(E);
        double co[4];
        c_gather(E, co);
        if (with_b) {
            if (co[1] > 0.0) {
                status = RAFEM_ERR_INVALID;
                rel = INFINITY;
                break;
            }
            bnorm = sqrt(co[0]);
            if (bnorm == 0.0) {  // zero data: zero solution (solver.py:422-425)
                R.x = d2(0.0, 0.0);
                if (act && xout_g) xout_g[E.t] = R.x;
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
        if (act) {
            const double2 y = c_spmv(E, E.mb + (size_t)(hb ^ 1) * E.nloc_cap);
            R.w = y;
            const double2 mv = E.rmv[E.t];
            const double2 m = PRE ? d2(mv.x * y.x, mv.y * y.y) : y;
            R.q = m;  // m of this iterate (kept in q until the first update)
            v0 = fma(R.r.x, R.u.x, R.r.y * R.u.y);
            v1 = fma(y.x, R.u.x, y.y * R.u.y);
            v2 = fma(R.r.x, R.r.x, R.r.y * R.r.y);
        }
        c_xbegin(E);
        if (act) c_push(E, hb, R.q);  // hb: last read by the x SpMV, before the last exchange
        c_publish(E, v0, v1, v2, 0.0);
        int cur = hb;
        double alpha = 0.0, ig = 0.0, igam = 0.0, dnm = 0.0;
        bool first = true;
        const long long hstart = hlen;
        const double thr = (E.tol * bnorm) * (E.tol * bnorm);
        while (true) {
            // own-column part of n = A m_i first: it needs only this CTA's
            // entries of m_i (complete after the publish's bar.sync), so the
            // bandwidth-bound half of the SpMV overlaps the cluster barrier
            c_stamp(E, total, 0);
            const double2* mcur = E.mb + (size_t)cur * E.nloc_cap;
            double2 n = act ? c_spmv_own(E, mcur) : d2(0.0, 0.0);
            c_stamp(E, total, 1);
            c_xwait(E);
            c_stamp(E, total, 2);
            if (act) n = c_spmv_gh(E, mcur, n);  // ghost part: loads in flight during the gather
            c_gather(E, co);
            const double gn = co[0], dn = co[1];
            double beta = 0.0;
            if (first) {
                if (!(gn > 0.0) || !(dn > 0.0) || !isfinite(gn) || !isfinite(dn)) {
                    status = RAFEM_ERR_BREAKDOWN;
                    break;
                }
                alpha = gn / dn;
            } else {
                ++total;
                const double rr = co[2];
                if (lead && E.hist && hlen < E.hist_cap) E.hist[hlen] = rr;
                ++hlen;
                if (rr <= thr || total >= E.cap) break;
                beta = gn * igam;
                const double den = fma(-(gn * ig), gn, dn);
                if (!(gn > 0.0) || !(den > 0.0) || !isfinite(den)) {
                    status = RAFEM_ERR_BREAKDOWN;
                    break;
                }
                alpha = gn / den;
                dnm = den;
            }
            c_stamp(E, total, 3);
            v0 = v1 = v2 = 0.0;
            if (act) {
                const double2 me = mcur[E.t];
                if (first) {
                    R.z = n;
                    R.q = me;
                    R.s = R.w;
                    R.p = R.u;
                } else {
                    R.z = d2(fma(beta, R.z.x, n.x), fma(beta, R.z.y, n.y));
                    R.q = d2(fma(beta, R.q.x, me.x), fma(beta, R.q.y, me.y));
                    R.s = d2(fma(beta, R.s.x, R.w.x), fma(beta, R.s.y, R.w.y));
                    R.p = d2(fma(beta, R.p.x, R.u.x), fma(beta, R.p.y, R.u.y));
                }
                R.x = d2(fma(alpha, R.p.x, R.x.x), fma(alpha, R.p.y, R.x.y));
                R.r = d2(fma(-alpha, R.s.x, R.r.x), fma(-alpha, R.s.y, R.r.y));
                R.u = d2(fma(-alpha, R.q.x, R.u.x), fma(-alpha, R.q.y, R.u.y));
                R.w = d2(fma(-alpha, R.z.x, R.w.x), fma(-alpha, R.z.y, R.w.y));
                v0 = fma(R.r.x, R.u.x, R.r.y * R.u.y);
                v1 = fma(R.w.x, R.u.x, R.w.y * R.u.y);
                v2 = fma(R.r.x, R.r.x, R.r.y * R.r.y);
            }
            c_xbegin(E);
            if (act) {
                const double2 mv = E.rmv[E.t];
                c_push(E, cur ^ 1, PRE ? d2(mv.x * R.w.x, mv.y * R.w.y) : R.w);
            }
            c_stamp(E, total, 4);
            c_publish(E, v0, v1, v2, 0.0);
            c_stamp(E, total, 5);
            // 1 / gn and 1 / (gn alpha) = den / gn^2 for the next iteration
            igam = 1.0 / gn;
            ig = (first ? dn : dnm) * igam * igam;
            cur ^= 1;
            first = false;
        }
        // (the loop ends after a wait: every arrive is matched)
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

// Per-thread setup common to the kernels: the row, its warp's ELL slice and
// its push destinations.
// Dynamic shared memory of the engine (same offsets in every CTA, so a
// peer's copy of any array is this CTA's address mapped to the peer):
//   ELL values | 2 gathered-vector buffers | ELL columns | per own row: b, M^-1, push targets
struct CLayout {
    double2 *ev, *mb, *rb, *rmv;
    uint16_t* ec;
    uint4* rdest;
    unsigned char* end;
};
__host__ __device__ inline size_t c_al16(size_t b) { return (b + 15) & ~(size_t)15; }
__host__ __device__ inline size_t c_layout_bytes(int ell_cap, int nloc_cap, int nt) {
    return c_al16((size_t)ell_cap * 16) + c_al16((size_t)2 * nloc_cap * 16) + c_al16((size_t)ell_cap * 2) +
           3 * c_al16((size_t)nt * 16);
}
RF_DEV CLayout c_layout(unsigned char* base, const CPlan& P) {
    CLayout L;
    unsigned char* q = base;
    L.ev = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)P.ell_cap * 16);
    L.mb = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)2 * P.nloc_cap * 16);
    L.ec = reinterpret_cast<uint16_t*>(q);
    q += c_al16((size_t)P.ell_cap * 2);
    L.rb = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)blockDim.x * 16);
    L.rmv = reinterpret_cast<double2*>(q);
    q += c_al16((size_t)blockDim.x * 16);
    L.rdest = reinterpret_cast<uint4*>(q);
    q += c_al16((size_t)blockDim.x * 16);
    L.end = q;
    return L;
}

RF_DEV void c_env(CEnv& E, const CPlan& P, const CCta& c, unsigned rank, const CLayout& L,
                  double (*part)[kCMax][4], double (*red)[4], unsigned long long* xbar) {
    E.ev = L.ev;
    E.ec = L.ec;
    E.mb = L.mb;
    E.rb = L.rb;
    E.rmv = L.rmv;
    E.rdest = L.rdest;
    E.nloc_cap = P.nloc_cap;
    E.part = part;
    E.red = red;
    E.C = P.C;
    E.rank = rank;
    E.t = threadIdx.x;
    E.nr = c.nr;
    const int4 wv = P.warp[c.wbase + (threadIdx.x >> 5)];
    E.k0 = wv.x + (threadIdx.x & 31);
    E.width = wv.y;
    E.k1 = wv.z + (threadIdx.x & 31);
    E.width1 = wv.w;
    {
        uint4* rd = const_cast<uint4*>(E.rdest);
        for (int t = threadIdx.x; t < c.nr; t += blockDim.x)
            rd[t] = __ldg(reinterpret_cast<const uint4*>(P.dest) + (c.g0 + t));
    }
    E.xbar = xbar;
    E.xk = E.xw = 0;
    E.xbytes = 16u * (unsigned)(c.nloc - c.nr) + 32u * (unsigned)P.C;
    if (threadIdx.x == 0) {
        mbar_init(xbar, 1);
        mbar_init(xbar + 1, 1);
        mbar_fence_init();
    }
}

// ---------------------------------------------------------------------------
// standalone solve: rafem_solve / rafem_system_solve on a paper-scale system

template <bool PRE>
__global__ void __launch_bounds__(kCT, 1) cpcg_kernel(CPlan P, const double2* __restrict__ val2, const double* b,
                                                      double* x, const double* minv, const int* flag, double tol,
                                                      long long cap, double* hist, long long hist_cap,
                                                      long long* cyc, long long cyc_cap, KResult* res,
                                                      long long* trace, long long trace_cap) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) double part[2][kCMax][4];
    __shared__ __align__(16) double red[32][4];
    __shared__ __align__(8) unsigned long long xbar[2];
    const unsigned rank = cl_rank();
    const CCta c = P.cta[rank];
    const CLayout L = c_layout(dsm, P);
    for (int k = threadIdx.x; k < c.ell_n; k += blockDim.x) {
        const int s = __ldg(P.esrc + c.ell_base + k);
        L.ev[k] = s >= 0 ? __ldg(val2 + s) : make_double2(0.0, 0.0);
        L.ec[k] = __ldg(P.ecol + c.ell_base + k);
    }
    CEnv E;
    c_env(E, P, c, rank, L, part, red, xbar);
    E.tol = tol;
    E.cap = cap;
    E.hist = hist;
    E.hist_cap = hist_cap;
    E.cyc = cyc;
    E.cyc_cap = cyc_cap;
    E.trace = trace;
    E.trace_cap = trace_cap;
    CRow R;
    const int g = c.g0 + E.t;
    const bool act = E.t < E.nr;
    R.x = act ? reinterpret_cast<const double2*>(x)[g] : d2(0.0, 0.0);
    if (act) {
        L.rb[E.t] = reinterpret_cast<const double2*>(b)[g];
        L.rmv[E.t] = PRE ? reinterpret_cast<const double2*>(minv)[g] : d2(1.0, 1.0);
    }
    __syncthreads();
    cl_sync();  // every CTA of the cluster runs (barriers initialised) before the first remote store
    if (*flag) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
        if (rank == 0 && threadIdx.x == 0) c_write_result(res, 0, 0, 0, INFINITY, false, RAFEM_ERR_INVALID);
        return;
    }
    const CpcgOut o = cpcg_core<PRE>(E, R, -1.0, 0.0, nullptr, nullptr, reinterpret_cast<double2*>(x) + c.g0);
    if (rank == 0 && threadIdx.x == 0)
        c_write_result(res, o.total, o.cycles, o.hlen, o.rel, o.converged != 0, o.status);
    cl_sync();  // no CTA leaves while a peer may still address its shared memory
}

// ---------------------------------------------------------------------------
// host: plans

struct ClusterPlan {
    unsigned long long pattern_id = 0;
    const int* rp = nullptr;
    int N = 0, C = 0, nt = 0;
    size_t smem = 0;  // dynamic shared memory of the solve kernel
    size_t smem_sim = 0;
    void* dev = nullptr;
    CPlan view{};
    std::vector<int> gpart;  // host copy (C + 1)
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
static ClusterPlan* cluster_plan(rafem_ctx* ctx, const int* rp_dev, const int* col_dev, int N, long long S,
                                 unsigned long long pattern_id, int C, int& rc) {
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
    // row blocks balanced by slots + rows, at most kCT rows each (else
    // balanced by rows: a thread per row sets the floor)
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
            if (gp[c + 1] - gp[c] > kCT || gp[c + 1] - gp[c] < 1) return false;
        return true;
    };
    if (!cut(1) && !cut(0)) return nullptr;
    std::vector<int> owner(N);
    for (int c = 0; c < C; ++c)
        for (int g = gp[c]; g < gp[c + 1]; ++g) owner[g] = c;
    std::vector<CCta> ct(C);
    std::vector<int4> warps;
    std::vector<uint16_t> ecol;
    std::vector<int> esrc, lgid;
    std::vector<unsigned> dest((size_t)N * kCDest, 0xffffffffu);
    std::vector<int> ndest(N, 0);
    int ell_cap = 0, nloc_cap = 0, nt = 32;
    std::vector<int> loc(N, -1);
    for (int c = 0; c < C; ++c) {
        const int g0 = gp[c], g1 = gp[c + 1], nr = g1 - g0;
        std::vector<int> gh;
        for (int g = g0; g < g1; ++g)
            for (int s = rp[g]; s < rp[g + 1]; ++s)
                if (col[s] < g0 || col[s] >= g1) gh.push_back(col[s]);
        std::sort(gh.begin(), gh.end());
        gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
        const int nloc = nr + (int)gh.size();
        if (nloc > 65535) return nullptr;
        CCta& cc = ct[c];
        cc.g0 = g0;
        cc.nr = nr;
        cc.nloc = nloc;
        cc.lbase = (int)lgid.size();
        for (int g = g0; g < g1; ++g) {
            loc[g] = g - g0;
            lgid.push_back(g);
        }
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
        auto is_own = [&](int j) { return j >= g0 && j < g1; };
        for (int w = 0; w < nwarp; ++w) {
            int wo = 0, wg = 0;
            for (int t = 32 * w; t < std::min(nr, 32 * w + 32); ++t) {
                int a = 0, b = 0;
                for (int s = rp[g0 + t]; s < rp[g0 + t + 1]; ++s) (is_own(col[s]) ? a : b)++;
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
                            int k = 0;
                            for (int s2 = rp[g0 + t]; s2 < rp[g0 + t + 1]; ++s2)
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
        nt = std::max(nt, nwarp * 32);
        for (int g = g0; g < g1; ++g) loc[g] = -1;
        for (int j : gh) loc[j] = -1;
    }
    // every CTA addresses warp entries up to nt / 32 (idle warps: width 0)
    {
        std::vector<int4> w2;
        std::vector<CCta> ct2 = ct;
        for (int c = 0; c < C; ++c) {
            ct2[c].wbase = (int)w2.size();
            const int nwarp = (ct[c].nr + 31) / 32;
            for (int w = 0; w < nt / 32; ++w) w2.push_back(w < nwarp ? warps[ct[c].wbase + w] : make_int4(0, 0, 0, 0));
        }
        warps.swap(w2);
        ct.swap(ct2);
    }
    ell_cap = (ell_cap + 7) & ~7;
    nloc_cap = (nloc_cap + 7) & ~7;
    P->smem = c_layout_bytes(ell_cap, nloc_cap, nt);
    P->smem_sim = P->smem + al16((size_t)nloc_cap) + al16((size_t)nt * 24);
    if (P->smem > 224 * 1024) return nullptr;
    // upload
    const size_t o_cta = 0, o_w = al16(sizeof(CCta) * C), o_ec = o_w + al16(sizeof(int4) * warps.size());
    const size_t o_es = o_ec + al16(2 * ecol.size()), o_de = o_es + al16(4 * esrc.size());
    const size_t o_lg = o_de + al16(4 * dest.size()), tot = o_lg + al16(4 * lgid.size());
    std::vector<unsigned char> h(tot);
    std::memcpy(h.data() + o_cta, ct.data(), sizeof(CCta) * C);
    std::memcpy(h.data() + o_w, warps.data(), sizeof(int4) * warps.size());
    std::memcpy(h.data() + o_ec, ecol.data(), 2 * ecol.size());
    std::memcpy(h.data() + o_es, esrc.data(), 4 * esrc.size());
    std::memcpy(h.data() + o_de, dest.data(), 4 * dest.size());
    std::memcpy(h.data() + o_lg, lgid.data(), 4 * lgid.size());
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
    P->view.C = C;
    P->view.ell_cap = ell_cap;
    P->view.nloc_cap = nloc_cap;
    P->nt = nt;
    P->gpart = gp;
    P->ok = true;
    return P;
}

static int cluster_size_for(int N) {
    int C = kCMax;
    if (const char* e = getenv("RAFEM_CLUSTER_C")) C = std::max(1, std::min(kCMax, atoi(e)));
    while (C > 1 && N < C * 64) C /= 2;
    return C;
}

static bool cluster_launchable(rafem_ctx* ctx, const void* fn, int C, int nt, size_t smem) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
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

// Eligibility: PCG with point Jacobi (or none) on a node-paired system small
// enough for one cluster's shared memory.  RAFEM_CLUSTER=0 disables it,
// RAFEM_CLUSTER=1 also takes block-Jacobi requests (applied as point Jacobi).
int cluster_pcg_solve(rafem_ctx* ctx, const MatView& A, const double* b_dev, double* x_dev, const double* minv_dev,
                      const rafem_solver_params& p, KResult* res_dev, int* flag_dev, cudaEvent_t ev_start,
                      cudaEvent_t ev_stop) {
    const char* env = getenv("RAFEM_CLUSTER");
    if (env && env[0] == '0') return RAFEM_ERR_UNSUPPORTED;
    const bool force = env && env[0] == '1';
    if (p.method != RAFEM_METHOD_PCG || A.W != 2 || !A.pattern_id || p.grid_ctas > 0) return RAFEM_ERR_UNSUPPORTED;
    if (p.precondition == RAFEM_PRECOND_BLOCK_JACOBI && !force) return RAFEM_ERR_UNSUPPORTED;
    const int N = A.ngroups;
    const int C = cluster_size_for(N);
    int rc = RAFEM_OK;
    ClusterPlan* P = cluster_plan(ctx, A.rp, A.col, N, A.slots, A.pattern_id, C, rc);
    if (rc) return rc;
    if (!P) return RAFEM_ERR_UNSUPPORTED;
    const bool pre = p.precondition != RAFEM_PRECOND_NONE;
    const void* fn = pre ? (const void*)cpcg_kernel<true> : (const void*)cpcg_kernel<false>;
    if (!cluster_launchable(ctx, fn, C, P->nt, P->smem)) return RAFEM_ERR_UNSUPPORTED;
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
    void* args[] = {&view, &val2, &b_dev, &x_dev, &minv, &flag_dev, &tol, &cap, &hist, &hc, &cyc, &cc, &res_dev,
                    &trace, &tcap};
    if (ev_start) RF_CUDA_TRY(ctx, cudaEventRecord(ev_start, ctx->stream));
    RF_CUDA_TRY(ctx, cluster_launch(ctx, fn, C, P->nt, P->smem, args));
    if (ev_stop) RF_CUDA_TRY(ctx, cudaEventRecord(ev_stop, ctx->stream));
    ctx->launches++;
    ctx->last_mode = 5;
    ctx->last_ctas = C;
    ctx->last_team = 1;
    ctx->last_precond = pre ? RAFEM_PRECOND_JACOBI : RAFEM_PRECOND_NONE;
    return RAFEM_OK;
}

}  // namespace rafem
