// simulate_dev.cuh — the whole adaptive RAFEM simulation in ONE persistent
// cooperative kernel (included by krylov.cu; uses its solver internals).
//
// Reference: run_simulation (fem.py:554-644) around corrector_step
// (fem.py:463-540), assemble_global (fem.py:325-430) and the Krylov solve.
// Every CTA owns a contiguous block of node rows (the solver partition) and
// a contiguous block of elements.  Per corrector pass:
//   barrier (first pass of a step) -> element phase (own elements: sigma,
//   16 (V,T) contributions, T loads, scattered to their slot-list
//   positions; diagonal sums) -> ONE reduction of the equilibration sums
//   and the PhysicsRange flag -> the row block's contributions and loads
//   by two TMA bulk copies, fill sums into the CTA's shared-memory matrix
//   slice -> equilibration scale + Dirichlet elimination + Jacobi inverse
//   diagonal on own rows -> pipelined PCG on the smem slice (||b||^2 and
//   the zero-diagonal flag ride on its head reduction) -> max-reduce the
//   corrector delta.
// The time-step control (predictor, acceptance, dt growth / shrink /
// halving, StepFailure) is scalar logic every CTA evaluates on identical,
// deterministically reduced values, so all CTAs take the same branches and
// the host launches once per simulation.
#pragma once

namespace rafem {

struct SimArgs {
    KArgs k;  // solver workspace: partition, vectors, minv, partials, flags, team, tol, cap
    AsmMesh m;
    double2* contrib;  // M x 16
    double* load;      // M x 4
    double* rhs;       // 2N
    double* diag_raw;  // 2N
    double* xs;        // 4 x n2: working dof vectors
    double* final_x;   // n2: last accepted state
    long long n2;
    rafem_sim_params p;
    double* rec_x;  // device records (rec_cap x n2) or null
    double* rec_time;
    double* rec_dt;
    int* rec_iters;
    long long rec_cap;
    SimDevOut* out;
    // streamed records (rafem_simulate_stream): ring of ring_slots slots of
    // (time, dt, iters, pad, 2N dofs); prog / cons live in mapped host memory
    double* ring;
    int ring_slots;
    volatile long long* prog;  // accepted records complete in the ring (kernel writes)
    volatile long long* cons;  // records the host has consumed (host writes)
    long long* ptrace;         // optional per-pass phase stamps (globaltimer ns), 8 per pass
    long long ptrace_cap;
    int stage_fill;            // contributor lists, incidences and dof kinds staged in smem
    int vx0;                   // pipelined PCG: first pass of a step starts from V extrapolated in time
    // Galerkin solver start (pipelined PCG path): ring of the last gal_k
    // increments between successive pass solutions (gal_k x n2) and the
    // last solution (n2); gal_k == 0 disables it
    double* gal_d;
    double* gal_xl;
    int gal_k;
    int gal_dbg;  // cost study: 1 skip products, 2 skip dots, 4 skip gather, 8 skip Cholesky,
                  // 16 only on a step's first pass
};

constexpr int kGalMax = 16;  // largest Galerkin window
#ifndef GAL_NQ
#define GAL_NQ 3  // Galerkin products: sources per sweep (r2e sweep: 6x4 21.98 ms, 3x7 20.93, 5x5 22.05, 2x14 23.27 per run;
#endif
#ifndef GAL_SL
#define GAL_SL 7  // Galerkin products: slots per lane in flight (3x7 is the one without spills in the lean kernel)
#endif

// Galerkin start of a pass's solve (the native loop's own choice of x0; the
// plug-in seam keeps the reference's x0): with D the nv most recent
// increments between successive pass solutions, x0 += D c where
// (D^T A D) c = D^T (b - A x0) with this pass's A — the A-norm-closest
// point of x0 + span(D) to the solution, so the Krylov solve starts
// without the components the last passes already resolved.  Everything is
// on the CTA's own rows and its shared-memory matrix slice: 1 + nv slice
// products (x0 and the d_j, gathered from L2), nv (nv + 3) / 2 dots in one
// reduction, a scaled pivot-thresholded Gauss-Jordan solve of the nv x nv system on
// every CTA (identical bits everywhere: the reduction is fixed-order), the
// update of x0 and a barrier.  CPU study (scripts/galerkin_x0_probe.py,
// the 900 s mesh-B run, block-Jacobi PCG): 4,655 -> 2,997 (nv = 8) and
// 2,223 (nv = 12) iterations with the same trajectory.
// scr: shared memory for (2 nv + 1) x 2 nr doubles; gco: >= nv (nv + 3) / 2.
template <class Mode, class R>
RF_DEV void galerkin_start(const KArgs& a, const R& rows, Sync<Mode>& sy, const double* b,
                                            const double* xsrc, double* x, const double* D, long long n2, int K,
                                            int head, int nv, double* scr, double* P, double* gco,
                                            int skip = 0) {
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1], lo = 2 * g0, nd = 2 * (g1 - g0);
    double* sR = scr;                    // r0 = b - A x0 (own dofs)
    double* sD = scr + nd;               // d_j (own dofs), j < nv
    double* sAD = sD + (size_t)nv * nd;  // A d_j
    // ring rows, most recent first (the modulo once per start, not per use)
    __shared__ const double* sdrow[kGalMax];
    if (tid < nv) sdrow[tid] = D + (size_t)((head - 1 - tid + 2 * K) % K) * n2;
    __syncthreads();
    auto dvec = [&](int j) { return sdrow[j]; };
    // RAFEM trace on: phase clocks of the last start (CTA 0) at trace[8 * 4000 + k]
#define GAL_STAMP(k) \
    if (a.trace && cta == 0 && tid == 0 && 8 * 4000 + (k) < a.trace_cap) a.trace[8 * 4000 + (k)] = clock64()
    GAL_STAMP(0);
    const long long gal_t0 = clock64();
    // the d_j rows (own dofs) stream into shared memory while the products run
    if (!(nd & 1)) {
        const int h = nd >> 1;
        for (int j = 0; j < nv; ++j)
            for (int e2 = tid; e2 < h; e2 += blockDim.x) cp_async16(sD + (size_t)j * nd + 2 * e2, dvec(j) + lo + 2 * e2);
    } else {
        for (int j = 0; j < nv; ++j)
            for (int e = tid; e < nd; e += blockDim.x) cp_async8(sD + (size_t)j * nd + e, dvec(j) + lo + e);
    }
    // products of the slice with x0 and the d_j, six sources per sweep (a
    // team of lanes per row; a lane's slots and all their gathers issued
    // before the first accumulation, so a sweep is one L2 round trip)
    constexpr int NQ = GAL_NQ, SL = GAL_SL;  // sources per sweep, slots per lane in flight
    for (int q0 = -1; q0 < ((skip & 1) ? -1 : nv); q0 += NQ) {
        const int nq = min(NQ, nv - q0);
        const double2* src[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = q0 + q;
            src[q] = reinterpret_cast<const double2*>(j < 0 ? xsrc : (j < nv ? dvec(j) : xsrc));
        }
        // its own team width: the largest with every row in one round (the
        // solver's SpMV team is sized for two rows per thread group)
        int team = 1;
        while (team < 8 && (g1 - g0) * team * 2 <= (int)blockDim.x) team *= 2;
        const int tl = tid & (team - 1), nteams = blockDim.x / team;
        for (int gb = g0; gb < g1; gb += nteams) {
            const int g = gb + tid / team;
            double acc[2 * NQ];
#pragma unroll
            for (int k = 0; k < 2 * NQ; ++k) acc[k] = 0.0;
            if (g < g1) {
                const int s0 = rows.start(g), s1 = rows.start(g + 1);
                for (int sb = s0 + tl; sb < s1; sb += SL * team) {
                    int c[SL];
                    double2 v[SL], xv[SL][NQ];
#pragma unroll
                    for (int u = 0; u < SL; ++u) {
                        const int sl = sb + u * team;
                        c[u] = sl < s1 ? rows.column(sl) : -1;
                        v[u] = sl < s1 ? rows.value2(sl) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < SL; ++u)
#pragma unroll
                        for (int q = 0; q < NQ; ++q)
                            if (c[u] >= 0 && q < nq) xv[u][q] = __ldca(src[q] + c[u]);
#pragma unroll
                    for (int u = 0; u < SL; ++u)
#pragma unroll
                        for (int q = 0; q < NQ; ++q)
                            if (c[u] >= 0 && q < nq) {
                                acc[2 * q] = fma(v[u].x, xv[u][q].x, acc[2 * q]);
                                acc[2 * q + 1] = fma(v[u].y, xv[u][q].y, acc[2 * q + 1]);
                            }
                }
            }
            for (int o = team >> 1; o > 0; o >>= 1)
#pragma unroll
                for (int k = 0; k < 2 * NQ; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
            if (g < g1 && tl == 0) {
                const int e = 2 * g - lo;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int j = q0 + q;
                    if (q >= nq) continue;
                    if (j < 0) {
                        sR[e] = sub(b[2 * g], acc[0]);
                        sR[e + 1] = sub(b[2 * g + 1], acc[1]);
                    } else {
                        sAD[(size_t)j * nd + e] = acc[2 * q];
                        sAD[(size_t)j * nd + e + 1] = acc[2 * q + 1];
                    }
                }
            }
        }
    }
    GAL_STAMP(1);
    cp_async_wait_all();
    __syncthreads();
    GAL_STAMP(2);
    // coefficient c: g_i (c < nv), then M_ij (i <= j) row by row; four
    // lanes each over quarters of the own dofs (two interleaved partial sums
    // per lane), then ((q0 + q1) + (q2 + q3))
    const int nvals = nv + nv * (nv + 1) / 2;
    const int nq = ((nd >> 1) + 3) >> 2;  // dof pairs per quarter
    for (int c0 = 0; c0 < ((skip & 2) ? 0 : nvals); c0 += blockDim.x >> 2) {
        const int c = c0 + (tid >> 2), qd = tid & 3;
        int i = 0, j;
        const double* u;
        const int cc = c < nvals ? c : nvals - 1;  // the quad's shuffles need every lane
        if (cc < nv) {
            i = cc;
            u = sR;
        } else {
            int q = cc - nv;
            while (q >= nv - i) {
                q -= nv - i;
                ++i;
            }
            j = i + q;
            u = sAD + (size_t)j * nd;
        }
        // (shared-space loads: the scratch pointer arrives as a generic one)
        const unsigned dis = smem_u32(sD + (size_t)i * nd), us = smem_u32(u);
        double a0 = 0.0, a1 = 0.0;
        const int e0 = 2 * qd * nq, e1 = min(nd & ~1, e0 + 2 * nq);
        for (int e = e0; e < e1; e += 2) {
            double d0, d1, u0, u1;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(d0), "=d"(d1) : "r"(dis + 8u * e));
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(u0), "=d"(u1) : "r"(us + 8u * e));
            a0 = fma(d0, u0, a0);
            a1 = fma(d1, u1, a1);
        }
        if (qd == 3 && (nd & 1)) {
            double d0, u0;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(d0) : "r"(dis + 8u * (nd - 1)));
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(u0) : "r"(us + 8u * (nd - 1)));
            a0 = fma(d0, u0, a0);
        }
        double sq = a0 + a1;
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        if (qd == 0 && c < nvals) P[(long long)c * G + cta] = sq;
    }
    GAL_STAMP(3);
    if (a.trace && tid == 0 && 8 * 4002 + cta < a.trace_cap) a.trace[8 * 4002 + cta] = clock64() - gal_t0;
    sy.barrier();
    GAL_STAMP(4);
    // two-level gather: CTA c folds coefficient c (c, c + G, ...) over the G
    // partials in CTA order, a barrier, every CTA reads the nvals totals
    double* T = P + (long long)nvals * G;
    for (int c = cta; c < ((skip & 4) ? 0 : nvals); c += G)
        if (warp == 0) {
            const double s = reduce_partials_warp(P + (long long)c * G, G);
            if (lane == 0) T[c] = s;
        }
    GAL_STAMP(5);
    sy.barrier();
    GAL_STAMP(6);
    for (int c = tid; c < nvals; c += blockDim.x) gco[c] = __ldcg(T + c);
    __syncthreads();
    GAL_STAMP(7);
    // the scaled system with a pivot threshold (dependent directions drop
    // out), solved by Gauss-Jordan with the whole CTA: thread = entry (i, k)
    // of the augmented matrix [S M S | S g], one barrier per pivot, the
    // pivots being Cholesky's Schur complements; a pivot <= 1e-10 is
    // skipped and its coefficient is 0, as a dropped Cholesky column gives.
    // (On warp 0 alone the elimination's registers spilled next to the
    // solver state: 8 us per start.)
    __shared__ double Ms[kGalMax][kGalMax + 1];
    __shared__ double cf[kGalMax], sc[kGalMax];
    if (!(skip & 8)) {
        auto Mij = [&](int i, int j) {  // M packed after g in gco: row i holds j = i..nv-1
            if (i > j) {
                const int t = i;
                i = j;
                j = t;
            }
            return gco[nv + i * nv - (i * (i - 1)) / 2 + (j - i)];
        };
        if (tid < nv) {
            const double m = Mij(tid, tid);
            sc[tid] = m > 0.0 ? rsqrt(m) : 0.0;
        }
        __syncthreads();
        const int w = nv + 1, ne = nv * w, bd = blockDim.x;
        const int i0 = tid < ne ? tid / w : -1, k0 = tid < ne ? tid - i0 * w : -1;
        const int i1 = tid + bd < ne ? (tid + bd) / w : -1, k1 = tid + bd < ne ? tid + bd - i1 * w : -1;
        if (i0 >= 0) Ms[i0][k0] = k0 < nv ? Mij(i0, k0) * sc[i0] * sc[k0] : gco[i0] * sc[i0];
        if (i1 >= 0) Ms[i1][k1] = k1 < nv ? Mij(i1, k1) * sc[i1] * sc[k1] : gco[i1] * sc[i1];
        __syncthreads();
        unsigned ac = 0;
        for (int j = 0; j < nv; ++j) {
            const double d = Ms[j][j];
            if (sc[j] > 0.0 && d > 1e-10) {  // the same decision in every thread
                ac |= 1u << j;
                const double r = 1.0 / d;
                if (i0 >= 0 && i0 != j && k0 > j) Ms[i0][k0] = fma(-Ms[i0][j] * r, Ms[j][k0], Ms[i0][k0]);
                if (i1 >= 0 && i1 != j && k1 > j) Ms[i1][k1] = fma(-Ms[i1][j] * r, Ms[j][k1], Ms[i1][k1]);
            }
            __syncthreads();
        }
        if (tid < nv) cf[tid] = (ac >> tid & 1u) ? Ms[tid][nv] / Ms[tid][tid] * sc[tid] : 0.0;
    }
    __syncthreads();
    GAL_STAMP(8);
    // x0 += D c on the own rows and, exactly, r0 -= (A D) c: the solver's first
    // head takes r from sR (no product, so no barrier for the new x here)
    for (int e = tid; e < nd; e += blockDim.x) {
        double v = xsrc[lo + e], rr = sR[e];
        for (int j = 0; j < nv; ++j) {
            v = fma(cf[j], sD[(size_t)j * nd + e], v);
            rr = fma(-cf[j], sAD[(size_t)j * nd + e], rr);
        }
        x[lo + e] = v;
        sR[e] = rr;
    }
    __syncthreads();
    GAL_STAMP(9);
#undef GAL_STAMP
}

// Max over CTAs of one nonnegative value (exact, order independent).
template <class Mode>
RF_DEV double reduce_max1(Sync<Mode>& sy, double v, double* P, double* red) {
    __shared__ double res;
    v = block_max(v, red);
    if (threadIdx.x == 0) P[blockIdx.x] = v;
    sy.barrier();
    if (threadIdx.x < 32) {
        const double m = reduce_max_partials_warp(P, (int)gridDim.x);
        if (threadIdx.x == 0) res = m;
    }
    __syncthreads();
    return res;
}

RF_DEV long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Fill phase with stage_fill == 2: every contribution and load of the CTA's
// rows copied into shared memory by cp.async (no registers held across the
// round trip: one round trip for the whole fill), then the same left-to-
// right sums per slot and per row from shared memory (bit-identical to the
// register-chunked fill).  Out of line: a once-per-pass phase that should
// not share a register allocation with the PCG loop.
__device__ __noinline__ void fill_staged_cp(int nsrc, int ninc, int ns, int nr, int g0, double2* cst, double* lst,
                                            const int* ssrc, const unsigned* iea, const int* sptr, const int* iptr,
                                            double2* sv2, double* srt, const int* sdg, const int* srp,
                                            const double2* contrib, const double* load, double* diag_raw,
                                            double* dv, int sp0, int ip0, unsigned long long* fbar,
                                            unsigned fpar) {
    const int tid = threadIdx.x;
    if (sp0 >= 0) {
        // slot-major element outputs: the block's contributions and loads are
        // two contiguous ranges, streamed in by two TMA bulk copies (the loads
        // from the 16-byte aligned element at or before ip0; an odd last
        // element is read by thread 0)
        const int a0 = ip0 & ~1, tot = (ip0 - a0) + ninc, nb = tot & ~1;
        double* lraw = lst - (ip0 - a0);
        if (tid == 0) {
            fence_proxy_async_all();  // generic accesses (earlier sums, other CTAs' stores) before the async copies
            const unsigned cb = 16u * (unsigned)nsrc, lb = 8u * (unsigned)nb;
            mbar_expect_tx(fbar, cb + lb);
            if (cb) tma_load_1d(cst, contrib + sp0, cb, fbar);
            if (lb) tma_load_1d(lraw, load + a0, lb, fbar);
            if (tot & 1) lraw[nb] = __ldcg(load + a0 + nb);
        }
        mbar_wait(fbar, fpar);
    } else {
        for (int k = tid; k < nsrc; k += blockDim.x) cp_async16(cst + k, contrib + ssrc[k]);
        for (int k = tid; k < ninc; k += blockDim.x) {
            const unsigned ea = iea[k];
            cp_async8(lst + k, load + 4LL * (ea & 0x3fffffffu) + (ea >> 30));
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // slots and rows (T rhs) as one work list over the CTA; each sum runs
    // left to right in list order, four loads in flight ahead of the adds
    for (int w = tid; w < ns + nr; w += blockDim.x) {
        if (w < ns) {
            double av = 0.0, at = 0.0;
            int k = sptr[w];
            const int k1 = sptr[w + 1];
            for (; k + 4 <= k1; k += 4) {
                const double2 c0 = cst[k], c1 = cst[k + 1], c2 = cst[k + 2], c3 = cst[k + 3];
                av = add(add(add(add(av, c0.x), c1.x), c2.x), c3.x);
                at = add(add(add(add(at, c0.y), c1.y), c2.y), c3.y);
            }
            for (; k < k1; ++k) {
                const double2 c = cst[k];
                av = add(av, c.x);
                at = add(at, c.y);
            }
            sv2[w] = make_double2(av, at);
        } else {
            const int r = w - ns;
            double racc = 0.0;
            int k = iptr[r];
            const int k1 = iptr[r + 1];
            for (; k + 4 <= k1; k += 4) {
                const double l0 = lst[k], l1 = lst[k + 1], l2 = lst[k + 2], l3 = lst[k + 3];
                racc = add(add(add(add(racc, l0), l1), l2), l3);
            }
            for (; k < k1; ++k) racc = add(racc, lst[k]);
            srt[r] = racc;
        }
    }
    __syncthreads();
    double d0 = dv[0], d1 = dv[1];
    for (int r = tid; r < nr; r += blockDim.x) {
        const long long i = g0 + r;
        const double2 dvv = sdg[r] >= 0 ? sv2[srp[r] + sdg[r]] : make_double2(0.0, 0.0);
        diag_raw[2 * i] = dvv.x;
        diag_raw[2 * i + 1] = dvv.y;
        d0 = add(d0, dvv.x);
        d1 = add(d1, dvv.y);
    }
    dv[0] = d0;
    dv[1] = d1;
}

// LEAN: the paper-scale instantiation (pipelined PCG, cp.async-staged fill)
// with every other path compiled out: a smaller kernel whose PCG loop does
// not share instruction-cache space and register allocation with code it
// never runs (the generic instantiation picks its paths at run time).
template <bool PRE, int NT, bool LEAN>
__global__ void __launch_bounds__(NT, 1) simulate_kernel(SimArgs S) {
    extern __shared__ __align__(16) double sval[];
    __shared__ double red[32 * 8];
    __shared__ double co[8];
    __shared__ double gco[LEAN ? kGalMax + kGalMax * (kGalMax + 1) / 2 : 1];
    __shared__ FillScratch ws[LEAN ? 1 : NT / 32];
    __shared__ int zflag;
    const KArgs& a = S.k;
    const rafem_sim_params& p = S.p;
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int g0 = a.gpart[cta], g1 = a.gpart[cta + 1];
    const int lo = 2 * g0, hi = 2 * g1;
    const long long n2 = S.n2;
    const int M = S.m.M;
    const int e0 = (int)((long long)M * cta / G), e1 = (int)((long long)M * (cta + 1) / G);

    // the pattern slice (columns, row starts) is constant: stage it once
    const int s0 = __ldg(a.A.rp + g0), ns = __ldg(a.A.rp + g1) - s0;
    int* scol = reinterpret_cast<int*>(sval + 2LL * ns);
    int* srp = scol + ((ns + 3) & ~3);
    for (int g = g0 + tid; g <= g1; g += blockDim.x) srp[g - g0] = __ldg(a.A.rp + g) - s0;
    for (int s = tid; s < ns; s += blockDim.x) scol[s] = __ldg(a.A.col + s0 + s);
    // the assembly's constant index data for this CTA's rows, staged once so
    // a pass's fill and constraint steps do no dependent index loads:
    // [slot list offsets | contributor list | incidence offsets | incidences |
    //  diagonal offsets | column kinds per slot | dof kinds per row]
    const int nr = g1 - g0;
    int* sptr = srp + nr + 1;
    int nsrc = 0, ninc = 0;
    int *ssrc = nullptr, *iptr = nullptr, *sdg = nullptr;
    unsigned* iea = nullptr;
    uint8_t *ckd = nullptr, *rkd = nullptr;
    double* srt = nullptr;  // T rhs of the own rows between the fill and the constraints
    double2* cst = nullptr;  // stage_fill 2: the pass's slot contributions, list order
    double* lst = nullptr;   //               and the rows' element loads, incidence order
    int sp0 = -1, ip0 = -1;  // slot-major contributions: the block's list offsets
    __shared__ __align__(8) unsigned long long fbar;  // TMA fill copies
    unsigned fpar = 0;
    if (tid == 0) {
        mbar_init(&fbar, 1);
        mbar_fence_init();
    }
    if (LEAN || S.stage_fill) {
        sp0 = __ldg(S.m.slot_ptr + s0);
        ip0 = __ldg(S.m.inc_ptr + g0);
        nsrc = __ldg(S.m.slot_ptr + s0 + ns) - sp0;
        ninc = __ldg(S.m.inc_ptr + g1) - ip0;
        ssrc = sptr + ns + 1;
        iptr = ssrc + nsrc;
        iea = reinterpret_cast<unsigned*>(iptr + nr + 1);
        sdg = reinterpret_cast<int*>(iea + ninc);
        ckd = reinterpret_cast<uint8_t*>(sdg + nr);
        rkd = ckd + ns;
        srt = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(rkd + 2 * nr) + 7) & ~uintptr_t(7));
        if (LEAN || S.stage_fill == 2) {
            cst = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(srt + nr) + 15) & ~uintptr_t(15));
            lst = reinterpret_cast<double*>(cst + nsrc) + (ip0 & 1);  // TMA: 16-byte aligned at element ip0 & ~1
        }
        for (int k = tid; k <= ns; k += blockDim.x) sptr[k] = __ldg(S.m.slot_ptr + s0 + k) - sp0;
        for (int k = tid; k < nsrc; k += blockDim.x) ssrc[k] = __ldg(S.m.slot_src + sp0 + k);
        for (int r = tid; r <= nr; r += blockDim.x) iptr[r] = __ldg(S.m.inc_ptr + g0 + r) - ip0;
        for (int k = tid; k < ninc; k += blockDim.x) iea[k] = __ldg(S.m.inc_ea + ip0 + k);
        for (int r = tid; r < nr; r += blockDim.x) {
            sdg[r] = __ldg(S.m.diag + g0 + r);
            rkd[2 * r] = S.m.kind[2LL * (g0 + r)];
            rkd[2 * r + 1] = S.m.kind[2LL * (g0 + r) + 1];
        }
        for (int k = tid; k < ns; k += blockDim.x) {
            const int j = __ldg(a.A.col + s0 + k);
            ckd[k] = (uint8_t)(S.m.kind[2LL * j] | (S.m.kind[2LL * j + 1] << 2));
        }
    }
    if (tid == 0) zflag = 0;
    __syncthreads();
    const Rows<2, true, false> rows{srp, scol, sval, g0};
    double2* sv2 = reinterpret_cast<double2*>(sval);

    Sync<GridMode> sy{a};
    int par = 0;
    const long long pstride = 8LL * G;
    auto P = [&]() { return a.partial + par * pstride; };
    int iacc = 0, iprev = 1, iit = 2, inew = 3;
    const bool smaj = S.m.cpos != nullptr && (LEAN || S.stage_fill == 2);
    auto X = [&](int i) { return S.xs + (long long)i * n2; };

    for (int e = lo + tid; e < hi; e += blockDim.x) {  // initial_state (fem.py:170-180)
        const double v0 = (e & 1) ? p.initial_temp : 0.0;
        X(iacc)[e] = v0;
        X(iprev)[e] = v0;
    }

    double t = 0.0, dt_state = p.dt_init, dt_prev = p.dt_init;
    long long step = 0, passes = 0, corr = 0, inner = 0, halv = 0, bad = -1;
    int gal_n = 0, gal_head = 0;  // Galerkin ring: valid increments, next slot
    bool gal_last = false;        // gal_xl holds the previous pass's solution
    long long asm_ns = 0, sol_ns = 0;
    int status = RAFEM_OK, failed_step = -1;
    double failed_dt = 0.0;

    while (t < p.total_time) {
        if (p.max_steps > 0 && step >= p.max_steps) break;
        const double remaining = p.total_time - t;
        const bool final_step = dt_state >= remaining;
        const double dt = final_step ? remaining : dt_state;
        const double ratio = dt / dt_prev;
        // predictor (fem.py:437-449): T extrapolated in time, V carried over.
        // With vx0 the first pass's SOLVER starts from both extrapolated
        // (X(inew), complete everywhere after the pass's first barrier); the
        // iterate the pass assembles from and measures its delta against is
        // still the reference predictor in X(iit).  Same systems, same
        // trajectory, ~30 % fewer PCG iterations on the first passes
        // (scripts/x0_extrap_probe.py).
        const bool vx0 = S.vx0 != 0;
        for (int e = lo + tid; e < hi; e += blockDim.x) {
            const double xa = X(iacc)[e];
            const double xe = step >= 1 ? add(xa, mul(ratio, sub(xa, X(iprev)[e]))) : xa;
            X(iit)[e] = (e & 1) ? xe : xa;
            if (vx0) X(inew)[e] = xe;
        }
        bool conv = false, abort_run = false;
        int iters = 0;
        for (int it = 1; it <= p.max_corrector_iters; ++it) {
            iters = it;
            ++passes;
            const long long ta = global_ns();
            // phase stamps: recomputed from `passes` at each use, so no extra
            // register stays live across the PCG loop
#define SIM_STAMP(k, v)                                                                     \
    do {                                                                                    \
        if (S.ptrace && cta == 0 && tid == 0 && passes * 8 <= S.ptrace_cap)                 \
            S.ptrace[(passes - 1) * 8 + (k)] = (v);                                         \
    } while (0)
            SIM_STAMP(0, ta);
            // the predicted iterate is complete everywhere; a later pass's
            // iterate was completed before the previous pass's delta reduction
            if (it == 1) sy.barrier();
            SIM_STAMP(1, global_ns());
            if (S.ring && cta == 0 && tid == 0 && it == 1) {
                __threadfence_system();
                *S.prog = step;  // every accepted record is in the ring
                // this step's record goes to slot step % slots: one thread waits
                // until the host has consumed that slot; the element-phase
                // reduction below holds every other CTA back until it returns,
                // so no other CTA ever polls host memory
                long long spins = 0;
                while (step - *S.cons >= S.ring_slots) {
                    __nanosleep(2000);
                    if (++spins > (1LL << 31)) asm volatile("trap;");
                }
            }
            // ---- element phase (own elements)
            const AsmFields f{X(iit) + 1, 2, X(iit), 2, X(iacc) + 1, 2, dt};
            double badv = 0.0;
            if (smaj) {
                // the equilibration sums come from the elements' diagonal
                // contributions and ride, with the PhysicsRange count, on the
                // reduction that also orders the contributions before the fill
                double ev[3] = {0.0, 0.0, 0.0};
                for (int e = e0 + tid; e < e1; e += blockDim.x)
                    if (element_tet_slot_major(e, S.m, f, S.contrib, S.load, ev)) badv = fmax(badv, (double)(M - e));
                ev[2] = badv > 0.0 ? 1.0 : 0.0;
                sy.template reduce<3>(ev, 3, P(), co, red);
                par ^= 1;
            } else {
                for (int e = e0 + tid; e < e1; e += blockDim.x)
                    if (element_tet(e, S.m, f, S.contrib, S.load)) badv = fmax(badv, (double)(M - e));
                sy.barrier();  // a row's fill gathers contributions of other CTAs' elements
            }
            SIM_STAMP(2, global_ns());
            // ---- fill own rows into the shared-memory slice
            // diagonal sums and the PhysicsRange count in ONE reduction; the
            // offending element is located only on the (aborting) bad path
            double dv[3] = {0.0, 0.0, badv > 0.0 ? 1.0 : 0.0};
            if (LEAN || S.stage_fill == 2) {
                fill_staged_cp(nsrc, ninc, ns, nr, g0, cst, lst, ssrc, iea, sptr, iptr, sv2, srt, sdg, srp, S.contrib,
                               S.load, S.diag_raw, dv, smaj ? sp0 : -1, ip0, &fbar, fpar);
                if (smaj) fpar ^= 1u;
            } else if (LEAN) {
            } else if (S.stage_fill) {
                // thread per slot over its staged contributor list (every gather of
                // a chunk in flight), then thread per row for the T rhs and diagonal
                for (int sl = tid; sl < ns; sl += blockDim.x) {
                    const int k0 = sptr[sl], k1 = sptr[sl + 1];
                    double av = 0.0, at = 0.0;
                    for (int k = k0; k < k1; k += 8) {
                        double2 c[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (k + q < k1) c[q] = __ldcg(S.contrib + ssrc[k + q]);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (k + q < k1) {
                                av = add(av, c[q].x);
                                at = add(at, c[q].y);
                            }
                    }
                    sv2[sl] = make_double2(av, at);
                }
                __syncthreads();
                for (int r = tid; r < nr; r += blockDim.x) {
                    const int p0 = iptr[r], p1 = iptr[r + 1];
                    double racc = 0.0;
                    for (int pp = p0; pp < p1; pp += 8) {
                        double l[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (pp + q < p1) {
                                const unsigned ea = iea[pp + q];
                                l[q] = __ldcg(S.load + 4LL * (ea & 0x3fffffffu) + (ea >> 30));
                            }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (pp + q < p1) racc = add(racc, l[q]);
                    }
                    const long long i = g0 + r;
                    srt[r] = racc;
                    const double2 dvv = sdg[r] >= 0 ? sv2[srp[r] + sdg[r]] : make_double2(0.0, 0.0);
                    S.diag_raw[2 * i] = dvv.x;
                    S.diag_raw[2 * i + 1] = dvv.y;
                    dv[0] = add(dv[0], dvv.x);  // same rows, same order as the loop below
                    dv[1] = add(dv[1], dvv.y);
                }
            } else if (NT == 256 && S.m.slot_src) {
                // thread per slot over its contributor list, then thread per row
                // (at 256 threads the kernel has the registers for the wide batches)
                for (int sl = tid; sl < ns; sl += blockDim.x) sv2[sl] = fill_slot(s0 + sl, S.m, S.contrib);
                __syncthreads();
                for (int i = g0 + tid; i < g1; i += blockDim.x)
                    fill_node_rhs(i, S.m, S.load, sv2 + srp[i - g0], S.rhs, S.diag_raw);
            } else {
                for (int i = g0 + warp; i < g1; i += nwarps)
                    fill_node_warp(i, S.m, S.contrib, S.load, sv2 + srp[i - g0], S.rhs, S.diag_raw, ws[warp]);
            }
            __syncthreads();
            if (!LEAN && !S.stage_fill)
                for (int i = g0 + tid; i < g1; i += blockDim.x) {
                    dv[0] = add(dv[0], S.diag_raw[2LL * i]);
                    dv[1] = add(dv[1], S.diag_raw[2LL * i + 1]);
                }
            if (!smaj) {
                sy.template reduce<3>(dv, 3, P(), co, red);
                par ^= 1;
            }
            if (co[2] > 0.0) {  // PhysicsRangeError aborts the run (fem.py:274)
                const double badmax = reduce_max1(sy, badv, P(), red);
                par ^= 1;
                bad = M - (long long)badmax;
                status = RAFEM_ERR_PHYSICS;
                abort_run = true;
                break;
            }
            SIM_STAMP(3, global_ns());
            double scale = 1.0;  // fem.py:390-396
            if (co[0] > 0.0 && co[1] > 0.0) scale = ldexp(1.0, (int)rint(log2(co[1] / co[0])));
            // ---- scale + Dirichlet + Jacobi on own rows; x0 = iterate (its
            // loads issued ahead of the constraint loop)
            const int ec = lo + tid;
            const double xc = ec < hi ? X(iit)[ec] : 0.0;
            if (LEAN || S.stage_fill)
                for (int r = tid; r < nr; r += blockDim.x)
                    constrain_node_thread(g0 + r, scale, p.applied_voltage, p.boundary_temp, sv2 + srp[r], S.rhs,
                                          PRE ? const_cast<double*>(a.minv) : nullptr, &zflag, scol + srp[r],
                                          ckd + srp[r], srp[r + 1] - srp[r], sdg[r], rkd[2 * r], rkd[2 * r + 1],
                                          srt[r]);
            else
                for (int i = g0 + warp; i < g1; i += nwarps) {
                    const int r = i - g0;
                    constrain_node_warp(i, S.m, scale, 1, p.applied_voltage, p.boundary_temp, sv2 + srp[r], S.rhs,
                                        PRE ? const_cast<double*>(a.minv) : nullptr, &zflag, scol + srp[r]);
                }
            const bool x0_new = vx0 && it == 1;  // X(inew) already holds the first pass's start
            if (!x0_new) {
                if (ec < hi) X(inew)[ec] = xc;
                for (int e = ec + blockDim.x; e < hi; e += blockDim.x) X(inew)[e] = X(iit)[e];
            }
            __syncthreads();
            PcgOut o{0, 0.0, 1, RAFEM_OK};
            double hdelta = -1.0;  // delta from the pipelined PCG's final head (< 0: not computed)
            long long tb;
            if (LEAN || a.pipe) {
                // ||b|| and the zero-diagonal flag ride on the PCG head's reduction
                tb = global_ns();
                SIM_STAMP(4, tb);
                KArgs kk = a;
                kk.b = S.rhs;
                kk.x = X(inew);
                kk.res = nullptr;
                bool gal = false;
                if constexpr (LEAN) {
                    if (S.gal_k > 0 && gal_n > 0 && cst && (it == 1 || !(S.gal_dbg & 16))) {
                        // (X(inew) holds the start on every CTA's own rows; the
                        // constraints' writes of the rhs are visible after the bar.sync)
                        KArgs kg = kk;  // the start's phase clocks (trace on) past the per-pass stamps
                        kg.trace = S.ptrace;
                        kg.trace_cap = S.ptrace ? (int)S.ptrace_cap : 0;
                        galerkin_start<GridMode>(kg, rows, sy, S.rhs, x0_new ? X(inew) : X(iit), X(inew), S.gal_d,
                                                 n2, S.gal_k, gal_head, gal_n, reinterpret_cast<double*>(cst),
                                                 a.partial + 16LL * G, gco, S.gal_dbg);
                        gal = true;
                    }
                }
                o = pcg_pipe_core<PRE, GridMode>(kk, rows, sy, -1.0, co, red, par, &zflag,
                                                 x0_new ? X(inew) : X(iit), X(iit), &hdelta,
                                                 gal ? reinterpret_cast<const double*>(cst) - 2LL * a.gpart[cta] : nullptr);
                if (S.gal_k > 0 && o.status == RAFEM_OK && o.converged) {
                    // the ring: d = x_new - (previous pass's solution), own rows
                    double* dn = S.gal_d + (size_t)gal_head * n2;
                    for (int e = lo + tid; e < hi; e += blockDim.x) {
                        const double xn = X(inew)[e];
                        if (gal_last) dn[e] = sub(xn, S.gal_xl[e]);
                        S.gal_xl[e] = xn;
                    }
                    if (gal_last) {
                        gal_head = (gal_head + 1) % S.gal_k;
                        gal_n = gal_n < S.gal_k ? gal_n + 1 : S.gal_k;
                    }
                    gal_last = true;
                }
                if (o.status == RAFEM_ERR_INVALID) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
                    status = RAFEM_ERR_INVALID;
                    abort_run = true;
                    break;
                }
            } else {
                double bv[2] = {0.0, 0.0};
                for (int e = lo + tid; e < hi; e += blockDim.x) bv[0] = add(bv[0], mul(S.rhs[e], S.rhs[e]));
                if (tid == 0) bv[1] = (double)zflag;
                sy.template reduce<2>(bv, 2, P(), co, red);
                par ^= 1;
                if (co[1] > 0.0) {  // ValueError: zero diagonal under Jacobi (solver.py:416-417)
                    status = RAFEM_ERR_INVALID;
                    abort_run = true;
                    break;
                }
                tb = global_ns();
                SIM_STAMP(4, tb);
                const double bnorm = sqrt(co[0]);
                if (bnorm == 0.0) {
                    for (int e = lo + tid; e < hi; e += blockDim.x) X(inew)[e] = 0.0;
                } else {
                    KArgs kk = a;
                    kk.b = S.rhs;
                    kk.x = X(inew);
                    kk.res = nullptr;
                    o = pcg_core<2, PRE, GridMode>(kk, rows, sy, bnorm, co, red, par);
                }
            }
            const long long tc = global_ns();
            SIM_STAMP(5, tc);
            SIM_STAMP(7, o.total);
            asm_ns += tb - ta;
            sol_ns += tc - tb;
            if (o.status == RAFEM_ERR_BREAKDOWN) break;  // SolverError -> step failure (fem.py:511-515)
            inner += o.total;
            if (!o.converged) break;  // fem.py:517-524
            // ---- corrector delta (fem.py:527-528): from the PCG's final head
            // (the converged iterate) when it computed one
            double delta = hdelta;
            if (!(delta >= 0.0)) {
                double dmax = 0.0;
                for (int e = lo + tid; e < hi; e += blockDim.x) {
                    const double xo = X(iit)[e];
                    const double d = fabs(sub(X(inew)[e], xo)) / fmax(1.0, fabs(xo));
                    dmax = (d > dmax || d != d) ? d : dmax;
                }
                delta = reduce_max1(sy, dmax, P(), red);
                par ^= 1;
            }
            SIM_STAMP(6, global_ns());
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
            if (S.ring) {  // stream: the slot was freed before this step's first barrier
                double* slot = S.ring + (step % S.ring_slots) * (n2 + 4);
                for (int e = lo + tid; e < hi; e += blockDim.x) slot[4 + e] = X(iacc)[e];
                if (cta == 0 && tid == 0) {
                    slot[0] = t;
                    slot[1] = dt;
                    slot[2] = (double)iters;
                    slot[3] = 0.0;
                }
            }
            if (step < S.rec_cap) {
                if (S.rec_x)
                    for (int e = lo + tid; e < hi; e += blockDim.x) S.rec_x[step * n2 + e] = X(iacc)[e];
                if (cta == 0 && tid == 0) {
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
#undef SIM_STAMP
    for (int e = lo + tid; e < hi; e += blockDim.x) S.final_x[e] = X(iacc)[e];
    if (S.ring) {
        sy.barrier();  // the last record is complete everywhere
        if (cta == 0 && tid == 0) {
            __threadfence_system();
            *S.prog = step;
        }
    }
    if (cta == 0 && tid == 0) {
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

}  // namespace rafem
