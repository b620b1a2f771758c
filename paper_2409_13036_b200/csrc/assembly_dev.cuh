// assembly_dev.cuh — per-element and per-node-row assembly steps as device
// functions, shared by the standalone assembly kernels (assembly.cu) and
// the fused device-resident simulation kernel (simulate.cu).
//
// Arithmetic follows the reference expression by expression (fem.py:247-430)
// with every operation rounded separately (no FMA contraction):
//   sigma  = sigma0 * (1 + alpha * (Tbar - Tref))            fem.py:273
//   K_sig  = sigma * (vol * grad_a.grad_b)                    fem.py:280-282
//   T blk  = (rho_c/dt) * (vol * (1+d_ab)/20) + k * base       fem.py:283-284, 317
//   load_a = sum_b (rho_c/dt) M_ab T_prev,b + sigma|gradV|^2 vol / 4   fem.py:286-288, 319-321
// and the per-slot sums run over the node's incident elements in ascending
// element order, which is the reference's duplicate-summation order.
#pragma once

#include "../../include/rafem_b200.h"
#include "common.cuh"

namespace rafem {

struct AsmMesh {
    const int* tets;      // M x 4
    const int* region;    // M
    const double* regtab; // 5 x nreg: k, rho_c, sigma0, alpha, t_ref
    int nreg;
    const double* base;   // M x 10 packed symmetric vol*grad.grad
    const double* grad;   // M x 12
    const double* vol;    // M
    const int* rp;        // N + 1 node pattern
    const int* col;       // slots
    const int* diag;      // N diagonal offsets
    const int* inc_ptr;   // N + 1
    const unsigned* inc_ea;   // tet | local << 30, ascending tet per node
    const unsigned* inc_slot; // 4 x uint8 row offsets
    const uint8_t* kind;  // 2N dof kinds
    const int* slot_ptr;  // S + 1: per-slot contributor lists (null: warp fill)
    const int* slot_src;  // 16 M: contrib index 16 e + 4 a + b, ascending e per slot
    const int* cpos;      // 16 M: slot-list position of contribution 16 e + 4 a + b (null: tet-major)
    const int* lpos;      // 4 M: incidence-list position of load 4 e + a
    int N, M;
    int own_end, below_end;  // rafem_mesh::own_end / below_end (N, N: natural order)
};

// nodal fields with strides (host inputs are contiguous N-arrays; the device
// loop reads the interleaved dof vectors directly)
struct AsmFields {
    const double* t;
    int ts;
    const double* v;
    int vs;
    const double* tp;
    int ps;
    double dt;
};

RF_DEV int sym_index(int a, int b) {
    // packed upper triangle of a symmetric 4x4: (0,0)(0,1)(0,2)(0,3)(1,1)(1,2)(1,3)(2,2)(2,3)(3,3)
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
    return a * 4 - (a * (a - 1)) / 2 + (b - a);
}

// Element e: 16 (V, T) block contributions in (a, b) row-major order and the
// four T-rhs loads, from the element's packed base (10), gradients (12) and
// volume wherever they are staged.  Returns true when sigma(Tbar) <= 0
// (PhysicsRangeError).
RF_DEV bool element_core(int e, const AsmMesh& m, const AsmFields& f, const double* b10, const double* g12,
                         double vol, double2* out16, double* out4) {
    int nd[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) nd[a] = __ldg(m.tets + 4 * e + a);
    const int rg = __ldg(m.region + e);
    const double kk = m.regtab[rg];
    const double rcdt = m.regtab[m.nreg + rg] / f.dt;
    const double sigma0 = m.regtab[2 * m.nreg + rg], alpha = m.regtab[3 * m.nreg + rg];
    const double tref = m.regtab[4 * m.nreg + rg];
    double tv[4], vv[4], tp[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        tv[a] = __ldcg(f.t + (long long)f.ts * nd[a]);
        vv[a] = __ldcg(f.v + (long long)f.vs * nd[a]);
        tp[a] = __ldcg(f.tp + (long long)f.ps * nd[a]);
    }
    double tsum = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) tsum = add(tsum, tv[a]);
    const double tbar = tsum / 4.0;
    const double sigma = mul(sigma0, add(1.0, mul(alpha, sub(tbar, tref))));
    const double mdia = mul(vol, 0.1), moff = mul(vol, 0.05);  // vol (1 + d_ab) / 20
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double bab = b10[sym_index(a, b)];
            const double mass = a == b ? mdia : moff;
            out16[4 * a + b] = make_double2(mul(sigma, bab), add(mul(rcdt, mass), mul(kk, bab)));
        }
    double gv[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int d = 0; d < 3; ++d) gv[d] = add(gv[d], mul(vv[a], g12[3 * a + d]));
    const double gg = add(add(mul(gv[0], gv[0]), mul(gv[2], gv[2])), mul(gv[1], gv[1]));
    const double fj = mul(mul(sigma, gg), vol) / 4.0;
    const double mo = mul(rcdt, moff), md = mul(rcdt, mdia);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double t[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) t[b] = mul(a == b ? md : mo, tp[b]);
        out4[a] = add(add(add(t[0], t[2]), add(t[1], t[3])), fj);
    }
    return sigma <= 0.0;  // fem.py:274
}

// The same, reading the geometry and writing the outputs in global memory.
RF_DEV bool element_tet(int e, const AsmMesh& m, const AsmFields& f, double2* contrib, double* load) {
    double b10[10], g12[12];
#pragma unroll
    for (int k = 0; k < 10; ++k) b10[k] = __ldg(m.base + 10LL * e + k);
#pragma unroll
    for (int k = 0; k < 12; ++k) g12[k] = __ldg(m.grad + 12LL * e + k);
    return element_core(e, m, f, b10, g12, __ldg(m.vol + e), contrib + 16LL * e, load + 4LL * e);
}

// The same with the outputs scattered to their positions in the per-slot
// contributor lists and per-node incidence lists (m.cpos, m.lpos), so a
// row block's contributions and loads are contiguous, already in summation
// order, for the fill that follows.  ds[0], ds[1] accumulate the element's
// diagonal V and T contributions (the equilibration sums, fem.py:390-396).
RF_DEV bool element_tet_slot_major(int e, const AsmMesh& m, const AsmFields& f, double2* contrib, double* load,
                                   double* ds) {
    double b10[10], g12[12];
#pragma unroll
    for (int k = 0; k < 10; ++k) b10[k] = __ldg(m.base + 10LL * e + k);
#pragma unroll
    for (int k = 0; k < 12; ++k) g12[k] = __ldg(m.grad + 12LL * e + k);
    const int4* cp = reinterpret_cast<const int4*>(m.cpos + 16LL * e);
    int4 q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = __ldg(cp + k);
    const int4 lp = __ldg(reinterpret_cast<const int4*>(m.lpos + 4LL * e));
    double2 o16[16];
    double o4[4];
    const bool bad = element_core(e, m, f, b10, g12, __ldg(m.vol + e), o16, o4);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        contrib[q[k].x] = o16[4 * k];
        contrib[q[k].y] = o16[4 * k + 1];
        contrib[q[k].z] = o16[4 * k + 2];
        contrib[q[k].w] = o16[4 * k + 3];
    }
    load[lp.x] = o4[0];
    load[lp.y] = o4[1];
    load[lp.z] = o4[2];
    load[lp.w] = o4[3];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        ds[0] = add(ds[0], o16[5 * a].x);
        ds[1] = add(ds[1], o16[5 * a].y);
    }
    return bad;
}

// Per-warp staging for one node row's incident elements.
struct FillScratch {
    double2 c[32][4];
    unsigned off[32];
    double ld[32];
};

// Node row i, one warp: lane l accumulates slot l.  The warp loads up to 32
// incidence records and their element contributions in parallel, stages
// them in shared memory, then every lane walks the incidences in ascending
// element order adding the contributions that land on its column.
// Writes raw (unscaled, unconstrained) slot values to out[l], the T rhs and
// the raw diagonal (V, T).
RF_DEV void fill_node_warp(int i, const AsmMesh& m, const double2* contrib, const double* load,
                           double2* out, double* rhs, double* diag_raw, FillScratch& ws) {
    const int lane = threadIdx.x & 31;
    const int deg = __ldg(m.rp + i + 1) - __ldg(m.rp + i);
    const int p0 = __ldg(m.inc_ptr + i), ninc = __ldg(m.inc_ptr + i + 1) - p0;
    const int dslot = __ldg(m.diag + i);
    for (int cb = 0; cb < deg; cb += 32) {
        const int l = cb + lane;
        double accV = 0.0, accT = 0.0, racc = 0.0;
        for (int pc = 0; pc < ninc; pc += 32) {
            const int p = pc + lane;
            if (p < ninc) {
                const unsigned ea = __ldg(m.inc_ea + p0 + p);
                const unsigned e = ea & 0x3fffffffu, a = ea >> 30;
                ws.off[lane] = __ldg(m.inc_slot + p0 + p);
#pragma unroll
                for (int b = 0; b < 4; ++b) ws.c[lane][b] = __ldcg(contrib + 16LL * e + 4 * a + b);
                ws.ld[lane] = __ldcg(load + 4LL * e + a);
            }
            __syncwarp();
            const int nq = min(32, ninc - pc);
            for (int q = 0; q < nq; ++q) {
                const unsigned offs = ws.off[q];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if ((int)((offs >> (8 * b)) & 255u) == l) {
                        const double2 c = ws.c[q][b];
                        accV = add(accV, c.x);
                        accT = add(accT, c.y);
                    }
                }
                racc = add(racc, ws.ld[q]);
            }
            __syncwarp();
        }
        if (l < deg) {
            out[l] = make_double2(accV, accT);
            if (l == dslot) {
                diag_raw[2LL * i] = accV;
                diag_raw[2LL * i + 1] = accT;
            }
        }
        if (cb == 0 && lane == 0) {
            rhs[2LL * i] = 0.0;
            rhs[2LL * i + 1] = racc;
        }
    }
    if (dslot < 0 && lane == 0) {
        diag_raw[2LL * i] = 0.0;
        diag_raw[2LL * i + 1] = 0.0;
    }
}

// Per-element scalars of the fused fill (element_scalars_kernel): sigma(Tbar)
// and the four T-rhs loads, with element_core's arithmetic operation for
// operation (the same bits).  Returns true when sigma <= 0.
RF_DEV bool element_scalars(int e, const AsmMesh& m, const AsmFields& f, double* sig, double* load4) {
    int nd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nd[k] = __ldg(m.tets + 4 * e + k);
    const int rg = __ldg(m.region + e);
    const double rcdt = m.regtab[m.nreg + rg] / f.dt;
    const double sigma0 = m.regtab[2 * m.nreg + rg], alpha = m.regtab[3 * m.nreg + rg];
    const double tref = m.regtab[4 * m.nreg + rg];
    double g[12];
    const double2* gp = reinterpret_cast<const double2*>(m.grad + 12LL * e);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 q = __ldg(gp + k);
        g[2 * k] = q.x;
        g[2 * k + 1] = q.y;
    }
    const double vol = __ldg(m.vol + e);
    double tv[4], vv[4], tp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        tv[k] = __ldcg(f.t + (long long)f.ts * nd[k]);
        vv[k] = __ldcg(f.v + (long long)f.vs * nd[k]);
        tp[k] = __ldcg(f.tp + (long long)f.ps * nd[k]);
    }
    double tsum = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) tsum = add(tsum, tv[k]);
    const double tbar = tsum / 4.0;
    const double sigma = mul(sigma0, add(1.0, mul(alpha, sub(tbar, tref))));
    const double mdia = mul(vol, 0.1), moff = mul(vol, 0.05);
    double gv[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) gv[d] = add(gv[d], mul(vv[k], g[3 * k + d]));
    const double gg = add(add(mul(gv[0], gv[0]), mul(gv[2], gv[2])), mul(gv[1], gv[1]));
    const double fj = mul(mul(sigma, gg), vol) / 4.0;
    const double mo = mul(rcdt, moff), md = mul(rcdt, mdia);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double t[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) t[b] = mul(a == b ? md : mo, tp[b]);
        load4[a] = add(add(add(t[0], t[2]), add(t[1], t[3])), fj);
    }
    *sig = sigma;
    return sigma <= 0.0;  // fem.py:274
}

// Row a of element e: the four (V, T) contributions (a, b = 0..3) from the
// stored base row, the volume, the region's k and rho_c / dt and the
// element's sigma (element_core's arithmetic, the same bits).
RF_DEV void element_row(int e, int a, const AsmMesh& m, double dt, const double* sig, double2* out4) {
    const int rg = __ldg(m.region + e);
    const double kk = m.regtab[rg];
    const double rcdt = m.regtab[m.nreg + rg] / dt;
    const double vol = __ldg(m.vol + e);
    const double sigma = __ldcg(sig + e);
    const double mdia = mul(vol, 0.1), moff = mul(vol, 0.05);
    const double* b10 = m.base + 10LL * e;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        const double bab = __ldg(b10 + lo * 4 - (lo * (lo - 1)) / 2 + (hi - lo));
        const double mass = a == b ? mdia : moff;
        out4[b] = make_double2(mul(sigma, bab), add(mul(rcdt, mass), mul(kk, bab)));
    }
}

// Node row i, one warp, element phase fused into the fill: lane p computes
// row a of its incident element p (ascending element order) in registers
// from the element's stored geometry and its sigma (element_scalars), stages
// the four contributions, their row offsets and the load in shared memory,
// and every lane (slot l) then walks the incidences in order adding what
// lands on its column — fill_node_warp's summation with the contributions
// computed instead of read back from HBM (bit-identical).
RF_DEV void fill_node_fused(int i, const AsmMesh& m, double dt, const double* sig, const double* load4,
                            double2* out, double* rhs, double* diag_raw, FillScratch& ws) {
    const int lane = threadIdx.x & 31;
    const int deg = __ldg(m.rp + i + 1) - __ldg(m.rp + i);
    const int p0 = __ldg(m.inc_ptr + i), ninc = __ldg(m.inc_ptr + i + 1) - p0;
    const int dslot = __ldg(m.diag + i);
    // one pass over the incidences when the row fits a warp (box meshes);
    // longer rows recompute per 32-slot chunk
    for (int cb = 0; cb < deg; cb += 32) {
        const int l = cb + lane;
        double accV = 0.0, accT = 0.0, racc = 0.0;
        for (int pc = 0; pc < ninc; pc += 32) {
            const int p = pc + lane;
            if (p < ninc) {
                const unsigned ea = __ldg(m.inc_ea + p0 + p);
                const int e = (int)(ea & 0x3fffffffu), a = (int)(ea >> 30);
                ws.off[lane] = __ldg(m.inc_slot + p0 + p);
                element_row(e, a, m, dt, sig, ws.c[lane]);
                ws.ld[lane] = __ldcg(load4 + 4LL * e + a);
            }
            __syncwarp();
            // a tet holds column l at most once: one SIMD byte compare finds
            // which of its four row offsets (if any) is this lane's slot
            const int nq = min(32, ninc - pc);
            const unsigned lrep = (unsigned)l * 0x01010101u;
            for (int q = 0; q < nq; ++q) {
                const unsigned hit = __vcmpeq4(ws.off[q], lrep);
                if (hit) {
                    const double2 c = ws.c[q][(__ffs(hit) - 1) >> 3];
                    accV = add(accV, c.x);
                    accT = add(accT, c.y);
                }
                if (lane == 0) racc = add(racc, ws.ld[q]);
            }
            __syncwarp();
        }
        if (l < deg) {
            out[l] = make_double2(accV, accT);
            if (l == dslot) {
                diag_raw[2LL * i] = accV;
                diag_raw[2LL * i + 1] = accT;
            }
        }
        if (cb == 0 && lane == 0) {
            rhs[2LL * i] = 0.0;
            rhs[2LL * i + 1] = racc;
        }
    }
    if (dslot < 0 && lane == 0) {
        diag_raw[2LL * i] = 0.0;
        diag_raw[2LL * i + 1] = 0.0;
    }
}

// The same with 16 lanes per row, two rows per warp (rows of at most 16
// slots and 32 incident elements, e.g. Kuhn boxes: 15 and 24): twice the
// rows in flight per warp and half the accumulation instructions per row.
// A lane's (up to) two incidences issue all their loads before either is
// computed; the region's k and rho_c / dt come from a per-block table (rk,
// rrc; the same IEEE quotient).  Same per-contribution arithmetic and order.
struct RowLoads {
    double bab[4], vol, sigma, ld;
    int rg;
};
RF_DEV void row_loads(unsigned ea, const AsmMesh& m, const double* sig, const double* load4, RowLoads& r) {
    const int e = (int)(ea & 0x3fffffffu), a = (int)(ea >> 30);
    r.rg = __ldg(m.region + e);
    r.vol = __ldg(m.vol + e);
    r.sigma = __ldcg(sig + e);
    r.ld = __ldcg(load4 + 4LL * e + a);
    const double* b10 = m.base + 10LL * e;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        r.bab[b] = __ldg(b10 + lo * 4 - (lo * (lo - 1)) / 2 + (hi - lo));
    }
}
RF_DEV void row_contrib(unsigned ea, const RowLoads& r, const double* rk, const double* rrc, double2* out4) {
    const int a = (int)(ea >> 30);
    const double kk = rk[r.rg], rcdt = rrc[r.rg];
    const double mdia = mul(r.vol, 0.1), moff = mul(r.vol, 0.05);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const double mass = a == b ? mdia : moff;
        out4[b] = make_double2(mul(r.sigma, r.bab[b]), add(mul(rcdt, mass), mul(kk, r.bab[b])));
    }
}
RF_DEV void fill_node_fused_half(int i, const AsmMesh& m, const double* rk, const double* rrc, const double* sig,
                                 const double* load4, double2* val2, double* rhs, double* diag_raw, FillScratch& ws) {
    const int lane = threadIdx.x & 31, hl = lane & 15;
    const unsigned hmask = 0xffffu << (lane & 16);
    const int r0 = __ldg(m.rp + i), deg = __ldg(m.rp + i + 1) - r0;
    const int p0 = __ldg(m.inc_ptr + i), ninc = __ldg(m.inc_ptr + i + 1) - p0;
    const int dslot = __ldg(m.diag + i);
    const bool ha = hl < ninc, hb = hl + 16 < ninc;
    unsigned ea = 0, eb = 0;
    if (ha) {
        ea = __ldg(m.inc_ea + p0 + hl);
        ws.off[hl] = __ldg(m.inc_slot + p0 + hl);
    }
    if (hb) {
        eb = __ldg(m.inc_ea + p0 + hl + 16);
        ws.off[hl + 16] = __ldg(m.inc_slot + p0 + hl + 16);
    }
    RowLoads la, lb;
    if (ha) row_loads(ea, m, sig, load4, la);
    if (hb) row_loads(eb, m, sig, load4, lb);
    if (ha) {
        row_contrib(ea, la, rk, rrc, ws.c[hl]);
        ws.ld[hl] = la.ld;
    }
    if (hb) {
        row_contrib(eb, lb, rk, rrc, ws.c[hl + 16]);
        ws.ld[hl + 16] = lb.ld;
    }
    __syncwarp(hmask);
    // branch-free walk: every lane reads the (q, b) entry its column would
    // take and adds it only on a hit (an add of the untaken value would
    // change nothing but the bits of -0.0; the select keeps them exact)
    double accV = 0.0, accT = 0.0, racc = 0.0;
    const unsigned lrep = (unsigned)hl * 0x01010101u;
#pragma unroll 4
    for (int q = 0; q < ninc; ++q) {
        const unsigned hit = __vcmpeq4(ws.off[q], lrep);
        const double2 c = ws.c[q][(__ffs(hit | 0x80000000u) - 1) >> 3];
        const double av = add(accV, c.x), at = add(accT, c.y);
        accV = hit ? av : accV;
        accT = hit ? at : accT;
        racc = add(racc, ws.ld[q]);  // (used by lane 0 only)
    }
    if (hl < deg) {
        val2[r0 + hl] = make_double2(accV, accT);
        if (hl == dslot) {
            diag_raw[2LL * i] = accV;
            diag_raw[2LL * i + 1] = accT;
        }
    }
    if (hl == 0) {
        rhs[2LL * i] = 0.0;
        rhs[2LL * i + 1] = racc;
        if (dslot < 0) {
            diag_raw[2LL * i] = 0.0;
            diag_raw[2LL * i + 1] = 0.0;
        }
    }
}

// Slot s: sum of its contributions in ascending element order (the
// reference's duplicate-summation order, fem.py:381-387 + sparse.py:180-190),
// every load of the list issued before the first add.  Same bits as
// fill_node_warp, one thread per slot.
RF_DEV double2 fill_slot(int s, const AsmMesh& m, const double2* __restrict__ contrib) {
    const int k0 = __ldg(m.slot_ptr + s), k1 = __ldg(m.slot_ptr + s + 1);
    double av = 0.0, at = 0.0;
    for (int k = k0; k < k1; k += 8) {
        double2 c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (k + j < k1) c[j] = __ldcg(contrib + __ldg(m.slot_src + k + j));
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (k + j < k1) {
                av = add(av, c[j].x);
                at = add(at, c[j].y);
            }
    }
    return make_double2(av, at);
}

// Node i after its slots are filled: T rhs = sum of the incident element
// loads in ascending element order (fem.py:388), V rhs 0, raw diagonal.
RF_DEV void fill_node_rhs(int i, const AsmMesh& m, const double* __restrict__ load, const double2* row,
                          double* rhs, double* diag_raw) {
    const int p0 = __ldg(m.inc_ptr + i), p1 = __ldg(m.inc_ptr + i + 1);
    double racc = 0.0;
    for (int p = p0; p < p1; p += 8) {
        double l[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (p + j < p1) {
                const unsigned ea = __ldg(m.inc_ea + p + j);
                l[j] = __ldcg(load + 4LL * (ea & 0x3fffffffu) + (ea >> 30));
            }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (p + j < p1) racc = add(racc, l[j]);
    }
    rhs[2LL * i] = 0.0;
    rhs[2LL * i + 1] = racc;
    const int d = __ldg(m.diag + i);
    const double2 dv = d >= 0 ? row[d] : make_double2(0.0, 0.0);
    diag_raw[2LL * i] = dv.x;
    diag_raw[2LL * i + 1] = dv.y;
}

RF_DEV double dof_value(int kind, double applied, double btemp) {
    return kind == RAFEM_DOF_APPLIED_VOLTAGE ? applied : (kind == RAFEM_DOF_BOUNDARY_TEMP ? btemp : 0.0);
}

// Node row i, one thread, everything staged in shared memory (the fused
// simulation's slice): the same per-slot arithmetic as constrain_node_warp
// and the moved-column sums in the same storage order, so the row is
// bit-identical; the rows of a CTA run side by side instead of a warp
// walking them one after another.
RF_DEV void constrain_node_thread(int i, double scale, double applied, double btemp, double2* vals, double* rhs,
                                  double* minv, int* zero_diag, const int* cols, const uint8_t* ckind, int deg,
                                  int dslot, int kV, int kT, double rt) {
    double mV = 0.0, mT = 0.0, dV = 0.0, dT = 0.0;
    for (int l = 0; l < deg; ++l) {
        const int j = cols[l];
        const int cV = ckind[l] & 3, cT = ckind[l] >> 2;
        const double2 v = vals[l];
        const double vs = mul(v.x, scale);
        if (!kV && cV) mV = add(mV, mul(vs, dof_value(cV, applied, btemp)));
        if (!kT && cT) mT = add(mT, mul(v.y, dof_value(cT, applied, btemp)));
        double outV = vs, outT = v.y;
        if (kV || cV) outV = (kV && j == i) ? 1.0 : 0.0;
        if (kT || cT) outT = (kT && j == i) ? 1.0 : 0.0;
        vals[l] = make_double2(outV, outT);
        if (l == dslot) {
            dV = outV;
            dT = outT;
        }
    }
    rhs[2LL * i] = kV ? dof_value(kV, applied, btemp) : sub(0.0, mV);
    rhs[2LL * i + 1] = kT ? dof_value(kT, applied, btemp) : sub(rt, mT);
    if (minv) {
        if (dslot < 0) dV = dT = 0.0;
        if (dV == 0.0 || dT == 0.0) atomicOr(zero_diag, 1);
        minv[2LL * i] = 1.0 / dV;
        minv[2LL * i + 1] = 1.0 / dT;
    }
}

// Node row i, one warp: voltage-row scaling and symmetric Dirichlet
// elimination keeping the explicit zeros (fem.py:398-428), in place on the
// row's slots; optional Jacobi inverse diagonal of the final row.
// Staged variant: the row's length, diagonal offset, its own dof kinds and
// its columns' kinds (ckind[l] = kind(2 col) | kind(2 col + 1) << 2) come
// from shared memory; null ckind reads them from the mesh.
RF_DEV void constrain_node_warp(int i, const AsmMesh& m, double scale, int apply, double applied, double btemp,
                                double2* vals, double* rhs, double* minv, int* zero_diag,
                                const int* cols = nullptr, const uint8_t* ckind = nullptr, int sdeg = 0,
                                int sdslot = -1, int skV = 0, int skT = 0, const double* srt = nullptr) {
    const int lane = threadIdx.x & 31;
    int deg, kV, kT, dslot;
    if (ckind) {
        deg = sdeg;
        dslot = sdslot;
        kV = apply ? skV : 0;
        kT = apply ? skT : 0;
    } else {
        const int s0 = __ldg(m.rp + i);
        deg = __ldg(m.rp + i + 1) - s0;
        if (!cols) cols = m.col + s0;
        kV = apply ? m.kind[2LL * i] : 0;
        kT = apply ? m.kind[2LL * i + 1] : 0;
        dslot = __ldg(m.diag + i);
    }
    double mV = 0.0, mT = 0.0;  // moved-column sums in storage order (fem.py:419-424)
    double dV = 0.0, dT = 0.0;
    for (int cb = 0; cb < deg; cb += 32) {
        const int l = cb + lane;
        double termV = 0.0, termT = 0.0;
        int movV = 0, movT = 0;
        if (l < deg) {
            const int j = cols[l];
            int cV = 0, cT = 0;
            if (apply) {
                if (ckind) {
                    cV = ckind[l] & 3;
                    cT = ckind[l] >> 2;
                } else {
                    cV = m.kind[2LL * j];
                    cT = m.kind[2LL * j + 1];
                }
            }
            const double2 v = vals[l];
            const double vs = mul(v.x, scale);
            if (!kV && cV) {
                movV = 1;
                termV = mul(vs, dof_value(cV, applied, btemp));
            }
            if (!kT && cT) {
                movT = 1;
                termT = mul(v.y, dof_value(cT, applied, btemp));
            }
            double outV = vs, outT = v.y;
            if (kV || cV) outV = (kV && j == i) ? 1.0 : 0.0;
            if (kT || cT) outT = (kT && j == i) ? 1.0 : 0.0;
            vals[l] = make_double2(outV, outT);
            if (l == dslot) {
                dV = outV;
                dT = outT;
            }
        }
        // moved-column terms in global column order (= storage order except
        // on shard meshes, whose below-owner ghosts are stored after the
        // owned columns: those lanes go first); most rows have none
        const unsigned bv = __ballot_sync(0xffffffffu, movV), bt = __ballot_sync(0xffffffffu, movT);
        if (bv | bt) {
            const int jc = l < deg ? cols[l] : 0x7fffffff;
            const unsigned gb = __ballot_sync(0xffffffffu, jc >= m.own_end && jc < m.below_end);
            const unsigned groups[3] = {gb, ~gb & __ballot_sync(0xffffffffu, jc < m.own_end), 0xffffffffu};
            unsigned done = 0;
#pragma unroll
            for (int gi = 0; gi < 3; ++gi) {
                unsigned gv = bv & groups[gi] & ~done, gt = bt & groups[gi] & ~done;
                done |= groups[gi];
                while (gv) {
                    const int t = __ffs(gv) - 1;
                    gv &= gv - 1;
                    mV = add(mV, __shfl_sync(0xffffffffu, termV, t));
                }
                while (gt) {
                    const int t = __ffs(gt) - 1;
                    gt &= gt - 1;
                    mT = add(mT, __shfl_sync(0xffffffffu, termT, t));
                }
            }
        }
    }
    if (minv && dslot >= 0) {
        const int src = dslot & 31;
        dV = __shfl_sync(0xffffffffu, dV, src);
        dT = __shfl_sync(0xffffffffu, dT, src);
    }
    if (lane == 0) {
        double rv = 0.0;  // V rhs is zero before constraints (fem.py:388, 400)
        double rt = srt ? *srt : rhs[2LL * i + 1];  // srt: the fill's T rhs staged in smem
        if (apply) {
            rv = kV ? dof_value(kV, applied, btemp) : sub(rv, mV);
            rt = kT ? dof_value(kT, applied, btemp) : sub(rt, mT);
        }
        rhs[2LL * i] = rv;
        rhs[2LL * i + 1] = rt;
        if (minv) {  // solver.py:413-418 on the final stored diagonal
            if (dslot < 0) dV = dT = 0.0;
            if (dV == 0.0 || dT == 0.0) atomicOr(zero_diag, 1);
            minv[2LL * i] = 1.0 / dV;
            minv[2LL * i + 1] = 1.0 / dT;
        }
    }
}


// Node row i, 16 lanes (rows of at most 16 slots, two rows per warp): the
// same per-slot arithmetic and moved-column order as constrain_node_warp
// (global column order on shard meshes), bit-identical rows with half the
// instructions per row.
RF_DEV void constrain_node_half(int i, const AsmMesh& m, double scale, int apply, double applied, double btemp,
                                double2* vals, double* rhs) {
    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16;
    const unsigned hmask = 0xffffu << hb;
    const int s0 = __ldg(m.rp + i), deg = __ldg(m.rp + i + 1) - s0;
    const int kV = apply ? m.kind[2LL * i] : 0, kT = apply ? m.kind[2LL * i + 1] : 0;
    double termV = 0.0, termT = 0.0;
    int movV = 0, movT = 0, jc = 0x7fffffff;
    if (hl < deg) {
        const int j = __ldg(m.col + s0 + hl);
        jc = j;
        const int cV = apply ? m.kind[2LL * j] : 0, cT = apply ? m.kind[2LL * j + 1] : 0;
        const double2 v = vals[s0 + hl];
        const double vs = mul(v.x, scale);
        if (!kV && cV) {
            movV = 1;
            termV = mul(vs, dof_value(cV, applied, btemp));
        }
        if (!kT && cT) {
            movT = 1;
            termT = mul(v.y, dof_value(cT, applied, btemp));
        }
        double outV = vs, outT = v.y;
        if (kV || cV) outV = (kV && j == i) ? 1.0 : 0.0;
        if (kT || cT) outT = (kT && j == i) ? 1.0 : 0.0;
        vals[s0 + hl] = make_double2(outV, outT);
    }
    double mV = 0.0, mT = 0.0;
    const unsigned bv = (__ballot_sync(hmask, movV) >> hb) & 0xffffu;
    const unsigned bt = (__ballot_sync(hmask, movT) >> hb) & 0xffffu;
    if (bv | bt) {
        const unsigned gb = (__ballot_sync(hmask, jc >= m.own_end && jc < m.below_end) >> hb) & 0xffffu;
        const unsigned ob = (__ballot_sync(hmask, jc < m.own_end) >> hb) & 0xffffu;
        const unsigned groups[3] = {gb, ~gb & ob, 0xffffu};
        unsigned done = 0;
#pragma unroll
        for (int gi = 0; gi < 3; ++gi) {
            unsigned gv = bv & groups[gi] & ~done, gt = bt & groups[gi] & ~done;
            done |= groups[gi];
            while (gv) {
                const int t = __ffs(gv) - 1;
                gv &= gv - 1;
                mV = add(mV, __shfl_sync(hmask, termV, t + hb));
            }
            while (gt) {
                const int t = __ffs(gt) - 1;
                gt &= gt - 1;
                mT = add(mT, __shfl_sync(hmask, termT, t + hb));
            }
        }
    }
    if (hl == 0) {
        double rv = 0.0, rt = rhs[2LL * i + 1];
        if (apply) {
            rv = kV ? dof_value(kV, applied, btemp) : sub(rv, mV);
            rt = kT ? dof_value(kT, applied, btemp) : sub(rt, mT);
        }
        rhs[2LL * i] = rv;
        rhs[2LL * i + 1] = rt;
    }
}

}  // namespace rafem
