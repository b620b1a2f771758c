// assembly.cu — device-resident global assembly of the RAFEM corrector-pass
// system (reference: fem.py:212-430).
//
// Symbolic phase (once per mesh, all on device):
//   node -> incident-tet lists in ascending tet order, the node adjacency
//   pattern (sorted columns), the diagonal slot of each row, and for every
//   (node, incident tet) pair the four row offsets of the tet's nodes.
//   The dof CSR of the reference is this node pattern expanded: row 2i has
//   columns 2j, row 2i+1 has columns 2j+1 (fem.py:310-316), so V and T
//   share one int32 column array and one double2 (V, T) value per slot.
// Geometry (once per mesh): P1 gradients, volumes, vol * grad_a . grad_b.
// Numeric fill (every pass):
//   1. element kernel: sigma(T iterate), PhysicsRangeError check, T-rhs
//      element loads (rho_c/dt M T_prev + Joule share).
//   2. slot fill, one team of lanes per node row: lane l owns slot l and
//      walks the node's incident tets in ascending element order, adding
//      the contributions that land on its column.  That is exactly the
//      order the reference's stable lexsort + sequential bincount sums
//      duplicates in (sparse.py:180-190 over fem.py:381-383), with no
//      atomics, so every pass is bit-stable.
//   3. equilibration scale from deterministic diagonal sums (fem.py:390-400).
//   4. scale + symmetric Dirichlet elimination per row (fem.py:402-428).
#include "assembly_dev.cuh"
#include "common.cuh"
#include "internal.hpp"

#include <cstdlib>

#include <algorithm>
#include <vector>

namespace rafem {

constexpr int kMaxDeg = 255;  // row offsets are packed as uint8

// ---------------------------------------------------------------------------
// scan (exclusive, out[n] = total) — used by the symbolic phase only

__global__ void scan_block_kernel(const int* in, int* out, int n, int* block_sums) {
    __shared__ int s[1024];
    const int base = blockIdx.x * 1024;
    const int t = threadIdx.x;  // 256 threads x 4 elements
    int v[4];
    int local = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int i = base + t * 4 + k;
        v[k] = (i < n) ? in[i] : 0;
        local += v[k];
    }
    s[t] = local;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        int add_ = (t >= off) ? s[t - off] : 0;
        __syncthreads();
        s[t] += add_;
        __syncthreads();
    }
    int run = (t > 0) ? s[t - 1] : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int i = base + t * 4 + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (t == 255) block_sums[blockIdx.x] = s[255];
}

__global__ void scan_add_kernel(int* out, int n, const int* block_offsets) {
    const int i = blockIdx.x * 1024 + threadIdx.x * 4;
    const int off = block_offsets[blockIdx.x];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i + k < n) out[i + k] += off;
}

int scan_ints(rafem_ctx* ctx, const int* in, int* out, int n) {
    // out has n + 1 entries; out[n] = total
    const int blocks = (n + 1023) / 1024;
    int* sums = nullptr;
    int* offs = nullptr;
    // context-cached blocks (stream order makes the immediate dfree safe):
    // the driver's stream-ordered pool trims itself at synchronisations and
    // was measured stalling mesh setup for 0.1-0.4 s now and then
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&sums, sizeof(int) * (blocks + 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&offs, sizeof(int) * (blocks + 1)));
    if (blocks > 0) {
        scan_block_kernel<<<blocks, 256, 0, ctx->stream>>>(in, out, n, sums);
        ctx->launches++;
        if (blocks > 1) {
            if (int rc = scan_ints(ctx, sums, offs, blocks)) return rc;
            scan_add_kernel<<<blocks, 256, 0, ctx->stream>>>(out, n, offs);
            ctx->launches++;
            RF_CUDA_TRY(ctx, cudaMemcpyAsync(out + n, offs + blocks, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            RF_CUDA_TRY(ctx, cudaMemcpyAsync(out + n, sums, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
        }
    } else {
        RF_CUDA_TRY(ctx, cudaMemsetAsync(out, 0, sizeof(int), ctx->stream));
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    dfree(ctx, sums);
    dfree(ctx, offs);
    return RAFEM_OK;
}

// ---------------------------------------------------------------------------
// symbolic kernels

__global__ void inc_count_kernel(const int* tets, int M, int* cnt) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
#pragma unroll
    for (int a = 0; a < 4; ++a) atomicAdd(cnt + tets[4 * e + a], 1);
}

__global__ void inc_fill_kernel(const int* tets, int M, int* cursor, unsigned* inc_ea) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int p = atomicAdd(cursor + tets[4 * e + a], 1);
        inc_ea[p] = (unsigned)e | ((unsigned)a << 30);
    }
}

// Sort each node's incidence list by element (the atomic fill above is
// unordered); insertion sort, lists are short (<= 24 on Kuhn boxes).
__global__ void inc_sort_kernel(const int* inc_ptr, int N, unsigned* inc_ea, int* maxinc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int p0 = inc_ptr[i], p1 = inc_ptr[i + 1];
    for (int p = p0 + 1; p < p1; ++p) {
        const unsigned v = inc_ea[p];
        const unsigned key = v & 0x3fffffffu;
        int q = p - 1;
        while (q >= p0 && (inc_ea[q] & 0x3fffffffu) > key) {
            inc_ea[q + 1] = inc_ea[q];
            --q;
        }
        inc_ea[q + 1] = v;
    }
    atomicMax(maxinc, p1 - p0);
}

// Sorted, de-duplicated neighbour list of node i (including i) into buf;
// returns its length, or -1 if it exceeds cap.
RF_DEV int node_neighbours(int i, const int* inc_ptr, const unsigned* inc_ea, const int* tets,
                           int* buf, int cap) {
    int len = 0;
    for (int p = inc_ptr[i]; p < inc_ptr[i + 1]; ++p) {
        const int e = (int)(inc_ea[p] & 0x3fffffffu);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = tets[4 * e + b];
            int q = len - 1;
            while (q >= 0 && buf[q] > j) --q;
            if (q >= 0 && buf[q] == j) continue;
            if (len >= cap) return -1;
            for (int r = len - 1; r > q; --r) buf[r + 1] = buf[r];
            buf[q + 1] = j;
            ++len;
        }
    }
    return len;
}

__global__ void adj_count_kernel(const int* inc_ptr, const unsigned* inc_ea, const int* tets, int N,
                                 int* deg, int* maxdeg, int* overflow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int buf[kMaxDeg + 1];
    const int len = node_neighbours(i, inc_ptr, inc_ea, tets, buf, kMaxDeg);
    if (len < 0) {
        atomicOr(overflow, 1);
        deg[i] = 0;
        return;
    }
    deg[i] = len;
    atomicMax(maxdeg, len);
}

__global__ void adj_fill_kernel(const int* inc_ptr, const unsigned* inc_ea, const int* tets, int N,
                                const int* rp, int* col, int* diag, unsigned* inc_slot) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int buf[kMaxDeg + 1];
    const int len = node_neighbours(i, inc_ptr, inc_ea, tets, buf, kMaxDeg);
    const int s0 = rp[i];
    int d = -1;
    for (int l = 0; l < len; ++l) {
        col[s0 + l] = buf[l];
        if (buf[l] == i) d = l;
    }
    diag[i] = d;
    for (int p = inc_ptr[i]; p < inc_ptr[i + 1]; ++p) {
        const int e = (int)(inc_ea[p] & 0x3fffffffu);
        unsigned packed = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = tets[4 * e + b];
            int lo = 0, hi = len - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (buf[mid] < j)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            packed |= (unsigned)lo << (8 * b);
        }
        inc_slot[p] = packed;
    }
}

// Per-slot contributor lists: thread per node row walks its incidences in
// ascending element order; slot l of the row receives 16 e + 4 a + b for
// every (element e, local row node a, local column node b) landing on it.
__global__ void slot_count_kernel(const int* inc_ptr, const unsigned* inc_slot, const int* rp, int N, int* cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int c[kMaxDeg];
    const int deg = rp[i + 1] - rp[i];
    for (int l = 0; l < deg; ++l) c[l] = 0;
    for (int p = inc_ptr[i]; p < inc_ptr[i + 1]; ++p) {
        const unsigned pk = inc_slot[p];
#pragma unroll
        for (int b = 0; b < 4; ++b) c[(pk >> (8 * b)) & 255u] += 1;
    }
    for (int l = 0; l < deg; ++l) cnt[rp[i] + l] = c[l];
}

__global__ void slot_fill_kernel(const int* inc_ptr, const unsigned* inc_ea, const unsigned* inc_slot,
                                 const int* rp, int N, const int* slot_ptr, int* slot_src) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int cur[kMaxDeg];
    const int s0 = rp[i], deg = rp[i + 1] - s0;
    for (int l = 0; l < deg; ++l) cur[l] = slot_ptr[s0 + l];
    for (int p = inc_ptr[i]; p < inc_ptr[i + 1]; ++p) {
        const unsigned ea = inc_ea[p], pk = inc_slot[p];
        const int e = (int)(ea & 0x3fffffffu), a = (int)(ea >> 30);
#pragma unroll
        for (int b = 0; b < 4; ++b) slot_src[cur[(pk >> (8 * b)) & 255u]++] = 16 * e + 4 * a + b;
    }
}

// ---------------------------------------------------------------------------
// geometry (fem.py:229-244): edges e_k = p_k - p_0, det, inverse by
// cofactors (column j of E^-1 is the cross product of the other two edges
// over det), grad_0 = -(grad_1 + grad_2 + grad_3).


__global__ void geometry_kernel(const double* nodes, const int* tets, int M, double* base,
                                double* grad, double* vol_out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
    double p[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int nd = tets[4 * e + a];
#pragma unroll
        for (int d = 0; d < 3; ++d) p[a][d] = nodes[3 * nd + d];
    }
    double E[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) E[k][d] = sub(p[k + 1][d], p[0][d]);
    // cofactor columns c_j: c_0 = e2 x e3, c_1 = e3 x e1, c_2 = e1 x e2
    double c[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double* u = E[(j + 1) % 3];
        const double* v = E[(j + 2) % 3];
        c[j][0] = u[1] * v[2] - u[2] * v[1];
        c[j][1] = u[2] * v[0] - u[0] * v[2];
        c[j][2] = u[0] * v[1] - u[1] * v[0];
    }
    const double det = E[0][0] * c[0][0] + E[0][1] * c[0][1] + E[0][2] * c[0][2];
    const double vol = det / 6.0;
    const double inv = 1.0 / det;
    double g[4][3];
#pragma unroll
    for (int a = 1; a < 4; ++a)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[a][d] = c[a - 1][d] * inv;
#pragma unroll
    for (int d = 0; d < 3; ++d) g[0][d] = -(add(add(g[1][d], g[2][d]), g[3][d]));
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int d = 0; d < 3; ++d) grad[12LL * e + 3 * a + d] = g[a][d];
    vol_out[e] = vol;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b) {
            const double dot = add(add(mul(g[a][0], g[b][0]), mul(g[a][2], g[b][2])), mul(g[a][1], g[b][1]));
            base[10LL * e + sym_index(a, b)] = mul(vol, dot);
        }
}

// base = vol * grad_a . grad_b from given gradients and volumes, the dot in
// np.einsum("mid,mjd->mij")'s order ((d0 + d2) + d1; geometry_kernel's too)
__global__ void base_from_grad_kernel(const double* grad, const double* vol_in, int M, double* base) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
    double g[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[a][d] = grad[12LL * e + 3 * a + d];
    const double vol = vol_in[e];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b) {
            const double dot = add(add(mul(g[a][0], g[b][0]), mul(g[a][2], g[b][2])), mul(g[a][1], g[b][1]));
            base[10LL * e + sym_index(a, b)] = mul(vol, dot);
        }
}

int mesh_set_geometry(rafem_mesh* m, const double* grad, const double* vol) {
    rafem_ctx* ctx = m->ctx;
    const int M = m->M;
    if (M <= 0) return RAFEM_OK;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(m->grad, grad, sizeof(double) * 12 * (size_t)M, cudaMemcpyHostToDevice,
                                     ctx->stream));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(m->vol, vol, sizeof(double) * (size_t)M, cudaMemcpyHostToDevice, ctx->stream));
    base_from_grad_kernel<<<(M + 127) / 128, 128, 0, ctx->stream>>>(m->grad, m->vol, M, m->base);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

// ---------------------------------------------------------------------------
// numeric fill (device functions in assembly_dev.cuh)

// 1. per element: sigma, the 16 (V, T) block contributions, T-rhs loads
// 1. element kernel: a block of kElemBlock tets stages its geometry (base,
//    gradients, volume: contiguous per block) through shared memory with
//    coalesced loads, computes one tet per thread, and writes the block's
//    contributions and loads back coalesced (each thread's 256 B of
//    contributions would otherwise be 16 scattered 16-B stores).
constexpr int kElemBlock = 64;
__global__ void __launch_bounds__(kElemBlock) element_kernel(AsmMesh m, AsmFields f, double2* contrib, double* load,
                                                             unsigned long long* bad) {
    __shared__ double sgeo[kElemBlock * 23];
    __shared__ double2 sout[kElemBlock * 16];
    __shared__ double sload[kElemBlock * 4];
    const long long e0 = (long long)blockIdx.x * kElemBlock;
    const int nb = (int)min((long long)kElemBlock, (long long)m.M - e0);
    for (int k = threadIdx.x; k < nb * 10; k += kElemBlock) sgeo[k] = __ldg(m.base + 10 * e0 + k);
    for (int k = threadIdx.x; k < nb * 12; k += kElemBlock) sgeo[kElemBlock * 10 + k] = __ldg(m.grad + 12 * e0 + k);
    for (int k = threadIdx.x; k < nb; k += kElemBlock) sgeo[kElemBlock * 22 + k] = __ldg(m.vol + e0 + k);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nb) {
        const int e = (int)(e0 + t);
        if (element_core(e, m, f, sgeo + 10 * t, sgeo + kElemBlock * 10 + 12 * t, sgeo[kElemBlock * 22 + t],
                         sout + 16 * t, sload + 4 * t))
            atomicMin(bad, (unsigned long long)e);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nb * 16; k += kElemBlock) __stcg(contrib + 16 * e0 + k, sout[k]);
    for (int k = threadIdx.x; k < nb * 4; k += kElemBlock) __stcg(load + 4 * e0 + k, sload[k]);
}

// 2. slot fill: one thread per slot over its contributor list, then one
//    thread per node row for the T rhs and the raw diagonal
__global__ void __launch_bounds__(256) fill_slots_kernel(AsmMesh m, const double2* contrib, double2* val2, int S) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < S) val2[s] = fill_slot(s, m, contrib);
}
__global__ void __launch_bounds__(256) fill_rows_kernel(AsmMesh m, const double* load, const double2* val2,
                                                        double* rhs, double* diag_raw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m.N) fill_node_rhs(i, m, load, val2 + __ldg(m.rp + i), rhs, diag_raw);
}

// 2'. slot fill, one warp per node row (no contributor lists)
__global__ void __launch_bounds__(256) fill_kernel(AsmMesh m, const double2* contrib, const double* load,
                                                   double2* val2, double* rhs, double* diag_raw) {
    __shared__ FillScratch ws[8];
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= m.N) return;  // whole warps exit together
    fill_node_warp(i, m, contrib, load, val2 + __ldg(m.rp + i), rhs, diag_raw, ws[threadIdx.x >> 5]);
}

// 1+2 fused: one warp per node row computes its incident elements' rows and
//    sums them in place (no per-element intermediate in HBM: 288 B per tet
//    written and read back by the two-kernel path)
__global__ void __launch_bounds__(256) element_scalars_kernel(AsmMesh m, AsmFields f, double* sig, double* load4,
                                                             unsigned long long* bad) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m.M) return;
    double s, l4[4];
    if (element_scalars(e, m, f, &s, l4)) atomicMin(bad, (unsigned long long)e);
    __stcg(sig + e, s);
    __stcg(reinterpret_cast<double2*>(load4 + 4LL * e), make_double2(l4[0], l4[1]));
    __stcg(reinterpret_cast<double2*>(load4 + 4LL * e) + 1, make_double2(l4[2], l4[3]));
}
constexpr int kFillRegions = 64;  // region table of the half-warp fill in shared memory
__global__ void __launch_bounds__(256) fused_fill_half_kernel(AsmMesh m, double dt, const double* sig,
                                                              const double* load4, double2* val2, double* rhs,
                                                              double* diag_raw) {
    __shared__ FillScratch ws[16];
    __shared__ double rk[kFillRegions], rrc[kFillRegions];
    for (int r = threadIdx.x; r < m.nreg; r += blockDim.x) {
        rk[r] = m.regtab[r];
        rrc[r] = m.regtab[m.nreg + r] / dt;  // element_core's rcdt
    }
    __syncthreads();
    const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4);
    if (i >= m.N) return;  // whole half-warps exit together
    fill_node_fused_half(i, m, rk, rrc, sig, load4, val2, rhs, diag_raw, ws[threadIdx.x >> 4]);
}
// The same half-warp fill as a persistent grid-stride loop with a software
// pipeline across rows: while row i's element data are fetched and summed,
// the incidence records of row i + s and the row / incidence pointers of
// row i + 2s are already in flight, so each row exposes one dependent
// round trip (the element data) instead of three.  Per row the arithmetic
// and the walk are fill_node_fused_half's, so the values are bitwise equal.
struct FillMeta {
    int r0, deg, p0, ninc, dslot;
};
RF_DEV FillMeta fill_meta(const AsmMesh& m, int i) {
    FillMeta t{0, 0, 0, 0, -1};
    if (i < m.N) {
        t.r0 = __ldg(m.rp + i);
        t.deg = __ldg(m.rp + i + 1);  // end; made a count on use
        t.p0 = __ldg(m.inc_ptr + i);
        t.ninc = __ldg(m.inc_ptr + i + 1);
        t.dslot = __ldg(m.diag + i);
    }
    return t;
}
__global__ void __launch_bounds__(256) fused_fill_half_pipe_kernel(AsmMesh m, double dt, const double* sig,
                                                                   const double* load4, double2* val2, double* rhs,
                                                                   double* diag_raw) {
    __shared__ FillScratch wsa[16];
    __shared__ double rk[kFillRegions], rrc[kFillRegions];
    for (int r = threadIdx.x; r < m.nreg; r += blockDim.x) {
        rk[r] = m.regtab[r];
        rrc[r] = m.regtab[m.nreg + r] / dt;  // element_core's rcdt
    }
    __syncthreads();
    FillScratch& ws = wsa[threadIdx.x >> 4];
    const int lane = threadIdx.x & 31, hl = lane & 15;
    const unsigned hmask = 0xffffu << (lane & 16);
    const int s = (int)(((long long)gridDim.x * blockDim.x) >> 4);
    int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4);
    // pipeline fill: meta of i and i + s, incidence records of i
    FillMeta cur = fill_meta(m, i);
    FillMeta nxt = fill_meta(m, i + s);
    auto inc_load = [&](const FillMeta& t, unsigned& ea, unsigned& eb, unsigned& oa, unsigned& ob) {
        const int n = t.ninc - t.p0;
        ea = eb = oa = ob = 0;
        if (hl < n) {
            ea = __ldg(m.inc_ea + t.p0 + hl);
            oa = __ldg(m.inc_slot + t.p0 + hl);
        }
        if (hl + 16 < n) {
            eb = __ldg(m.inc_ea + t.p0 + hl + 16);
            ob = __ldg(m.inc_slot + t.p0 + hl + 16);
        }
    };
    unsigned ea, eb, oa, ob;
    inc_load(cur, ea, eb, oa, ob);
    for (; i < m.N; i += s) {
        // in flight while this row is processed
        const FillMeta nn = fill_meta(m, i + 2 * s);
        unsigned ean, ebn, oan, obn;
        inc_load(nxt, ean, ebn, oan, obn);
        const int r0 = cur.r0, deg = cur.deg - cur.r0, ninc = cur.ninc - cur.p0, dslot = cur.dslot;
        const bool ha = hl < ninc, hb = hl + 16 < ninc;
        __syncwarp(hmask);  // the previous row's walk is done with ws
        if (ha) ws.off[hl] = oa;
        if (hb) ws.off[hl + 16] = ob;
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
        cur = nxt;
        nxt = nn;
        ea = ean;
        eb = ebn;
        oa = oan;
        ob = obn;
    }
}
__global__ void __launch_bounds__(256) fused_fill_kernel(AsmMesh m, double dt, const double* sig, const double* load4,
                                                         double2* val2, double* rhs, double* diag_raw) {
    __shared__ FillScratch ws[8];
    const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= m.N) return;  // whole warps exit together
    fill_node_fused(i, m, dt, sig, load4, val2 + __ldg(m.rp + i), rhs, diag_raw, ws[threadIdx.x >> 5]);
}

// 3. scale = 2^round(log2(sum diag_T / sum diag_V)) (fem.py:390-396) from
//    the raw diagonal sums:
// 3'. the same sums over n rows in two deterministic stages (G CTAs over
//     contiguous chunks, then one CTA over the G partials in order), for
//     large meshes where one CTA walking every row costs milliseconds
__global__ void __launch_bounds__(256) diag_partial_kernel(const double* diag_raw, int n, int chunk, double* part) {
    __shared__ double red[64];
    const int r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
    double v[2] = {0.0, 0.0};
    for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        v[0] = add(v[0], diag_raw[2LL * i]);
        v[1] = add(v[1], diag_raw[2LL * i + 1]);
    }
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = v[0];
        part[2 * blockIdx.x + 1] = v[1];
    }
}
__global__ void diag_finish_kernel(const double* part, int G, int equilibrate, double* sums, double* scale_out) {
    if (threadIdx.x != 0) return;
    double a = 0.0, b = 0.0;
    for (int c = 0; c < G; ++c) {
        a = add(a, part[2 * c]);
        b = add(b, part[2 * c + 1]);
    }
    if (sums) {
        sums[0] = a;
        sums[1] = b;
    }
    if (scale_out) {
        double scale = 1.0;
        if (equilibrate && a > 0.0 && b > 0.0) scale = ldexp(1.0, (int)rint(log2(b / a)));
        *scale_out = scale;
    }
}

int diag_sums_launch(rafem_ctx* ctx, const double* diag_raw, int n, int equilibrate, double* sums_dev,
                     double* scale_dev) {
    const int chunk = 8192;
    const int G = std::max(1, (n + chunk - 1) / chunk);
    if (int rc = ensure(ctx, ctx->ws_diag, sizeof(double) * 2 * (size_t)G)) return rc;
    double* part = static_cast<double*>(ctx->ws_diag.p);
    if (n > 0) {
        diag_partial_kernel<<<G, 256, 0, ctx->stream>>>(diag_raw, n, chunk, part);
    } else {
        RF_CUDA_TRY(ctx, cudaMemsetAsync(part, 0, sizeof(double) * 2, ctx->stream));
    }
    diag_finish_kernel<<<1, 32, 0, ctx->stream>>>(part, G, equilibrate, sums_dev, scale_dev);
    ctx->launches += 2;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

// 4. voltage-row scaling and symmetric Dirichlet elimination, one warp per node row
__global__ void __launch_bounds__(256) constrain_kernel(AsmMesh m, const double* scale_p, int apply, double applied,
                                                        double btemp, double2* val2, double* rhs) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= m.N) return;
    constrain_node_warp(i, m, *scale_p, apply, applied, btemp, val2 + __ldg(m.rp + i), rhs, nullptr, nullptr);
}

__global__ void __launch_bounds__(256) constrain_half_kernel(AsmMesh m, const double* scale_p, int apply,
                                                             double applied, double btemp, double2* val2,
                                                             double* rhs) {
    const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4);
    if (i >= m.N) return;  // whole half-warps exit together
    constrain_node_half(i, m, *scale_p, apply, applied, btemp, val2, rhs);
}

// dof-order values for CsrMatrix.vals: row 2i then row 2i+1 per node.
__global__ void expand_kernel(const int* rp, int N, const double* val2, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int s0 = rp[i], deg = rp[i + 1] - s0;
    for (int l = 0; l < deg; ++l) {
        const double2 v = reinterpret_cast<const double2*>(val2)[s0 + l];
        out[2LL * s0 + l] = v.x;
        out[2LL * s0 + deg + l] = v.y;
    }
}

// predictor (fem.py:437-449) on interleaved dof vectors: V carries over,
// T + (dt/dt_prev)(T - T_prev) once history exists.
// fem.py:437-449: T extrapolated in time, V carried over.  x_start (may be
// null): the first pass's solver start, with V extrapolated like T.
__global__ void predictor_kernel(double* x_it, const double* x_acc, const double* x_prev, int N,
                                 int step, double ratio, double* x_start) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double t = x_acc[2LL * i + 1];
    const double tp = step >= 1 ? add(t, mul(ratio, sub(t, x_prev[2LL * i + 1]))) : t;
    x_it[2LL * i] = x_acc[2LL * i];
    x_it[2LL * i + 1] = tp;
    if (x_start) {
        const double v = x_acc[2LL * i];
        x_start[2LL * i] = step >= 1 ? add(v, mul(ratio, sub(v, x_prev[2LL * i]))) : v;
        x_start[2LL * i + 1] = tp;
    }
}

__global__ void fill_state_kernel(double* x, int N, double t0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    x[2LL * i] = 0.0;
    x[2LL * i + 1] = t0;
}

// ---------------------------------------------------------------------------
// host side

int mesh_symbolic(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    const int N = m->N, M = m->M;
    cudaStream_t st = ctx->stream;
    int* cnt = nullptr;
    int* cursor = nullptr;
    int* flags = nullptr;  // [0] maxinc, [1] maxdeg, [2] overflow
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&cnt, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&cursor, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&flags, sizeof(int) * 4));
    RF_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * (N + 1), st));
    RF_CUDA_TRY(ctx, cudaMemsetAsync(flags, 0, sizeof(int) * 4, st));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->inc_ptr, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->inc_ea, sizeof(unsigned) * 4 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->inc_slot, sizeof(unsigned) * 4 * (size_t)std::max(M, 1)));
    const int tb = 256;
    if (M > 0) {
        inc_count_kernel<<<(M + tb - 1) / tb, tb, 0, st>>>(m->tets, M, cnt);
        ctx->launches++;
    }
    if (int rc = scan_ints(ctx, cnt, m->inc_ptr, N)) return rc;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(cursor, m->inc_ptr, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
    if (M > 0) {
        inc_fill_kernel<<<(M + tb - 1) / tb, tb, 0, st>>>(m->tets, M, cursor, m->inc_ea);
        ctx->launches++;
    }
    if (N > 0) {
        inc_sort_kernel<<<(N + tb - 1) / tb, tb, 0, st>>>(m->inc_ptr, N, m->inc_ea, flags + 0);
        adj_count_kernel<<<(N + 127) / 128, 128, 0, st>>>(m->inc_ptr, m->inc_ea, m->tets, N, cnt, flags + 1, flags + 2);
        ctx->launches += 2;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    int hflags[4] = {0, 0, 0, 0};
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(hflags, flags, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    if (hflags[2]) {
        dfree(ctx, cnt);
        dfree(ctx, cursor);
        dfree(ctx, flags);
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "a node has more than 255 neighbours; pattern too dense for the packed slot map");
    }
    m->maxinc = hflags[0];
    m->maxdeg = hflags[1];
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->rp, sizeof(int) * (N + 1)));
    if (int rc = scan_ints(ctx, cnt, m->rp, N)) return rc;
    int slots = 0;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&slots, m->rp + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    m->slots = slots;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->col, sizeof(int) * ((size_t)std::max(slots, 1) + 8)));  // +8: 16-B TMA tail
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->diag, sizeof(int) * (size_t)std::max(N, 1)));
    if (N > 0) {
        adj_fill_kernel<<<(N + 127) / 128, 128, 0, st>>>(m->inc_ptr, m->inc_ea, m->tets, N, m->rp, m->col, m->diag, m->inc_slot);
        ctx->launches++;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, cnt);
    dfree(ctx, cursor);
    dfree(ctx, flags);
    return RAFEM_OK;
}

// Per-slot contributor lists for the thread-per-slot fill; built on first
// use (the fused simulation kernel fills warp-per-row and never needs them).
// Returns without lists when 16 M does not fit an int.
int mesh_slot_lists(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    cudaStream_t st = ctx->stream;
    m->slot_lists_tried = true;
    const int N = m->N, M = m->M;
    const long long slots = m->slots;
    if (N <= 0 || slots <= 0 || 16LL * M >= (1LL << 31) || m->maxdeg > kMaxDeg) return RAFEM_OK;
    int* scnt = nullptr;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&scnt, sizeof(int) * (size_t)slots));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->slot_ptr, sizeof(int) * ((size_t)slots + 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->slot_src, sizeof(int) * 16 * (size_t)M));
    slot_count_kernel<<<(N + 127) / 128, 128, 0, st>>>(m->inc_ptr, m->inc_slot, m->rp, N, scnt);
    ctx->launches++;
    if (int rc = scan_ints(ctx, scnt, m->slot_ptr, (int)slots)) return rc;
    slot_fill_kernel<<<(N + 127) / 128, 128, 0, st>>>(m->inc_ptr, m->inc_ea, m->inc_slot, m->rp, N, m->slot_ptr,
                                                      m->slot_src);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, scnt);
    return RAFEM_OK;
}

__global__ void slot_pos_kernel(const int* slot_src, long long n, int* cpos) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        cpos[slot_src[k]] = (int)k;
}
__global__ void load_pos_kernel(const unsigned* inc_ea, long long n, int* lpos) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const unsigned ea = inc_ea[p];
        lpos[4LL * (ea & 0x3fffffffu) + (ea >> 30)] = (int)p;
    }
}

// Inverse maps of the contributor and incidence lists: where the element
// phase of the fused simulation stores each contribution and load so that
// every row block reads its own as one contiguous range.
int mesh_slot_positions(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    if (m->contrib_pos || !m->slot_src) return RAFEM_OK;
    const long long M = m->M;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->contrib_pos, sizeof(int) * 16 * (size_t)M));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->load_pos, sizeof(int) * 4 * (size_t)M));
    const int blocks = (int)std::min<long long>((16 * M + 255) / 256, 4LL * ctx->sm_count * 8);
    slot_pos_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(m->slot_src, 16 * M, m->contrib_pos);
    load_pos_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(m->inc_ea, 4 * M, m->load_pos);
    ctx->launches += 2;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

// Stencil classes.  A row's signature is its length and its column offsets
// (col - row), sorted like the columns; rows with the same signature share
// a class, and the SpMV kernels then compute columns instead of streaming
// them (4 of the 20 bytes per slot).  64-bit FNV-1a hashes on the device,
// classes assigned on the host, every row verified against its class on
// the device (a hash collision disables the classes).
__global__ void row_sig_kernel(const int* rp, const int* col, int N, unsigned long long* sig) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    unsigned long long h = 1469598103934665603ULL;
    const int s0 = rp[i], s1 = rp[i + 1];
    h = (h ^ (unsigned long long)(s1 - s0)) * 1099511628211ULL;
    for (int s = s0; s < s1; ++s) h = (h ^ (unsigned long long)(unsigned)(col[s] - i)) * 1099511628211ULL;
    sig[i] = h;
}
__global__ void cls_verify_kernel(const int* rp, const int* col, int N, const uint8_t* cls, const int* off,
                                  const int* deg, int* bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int c = cls[i], s0 = rp[i], d = rp[i + 1] - s0;
    bool ok = d == deg[c];
    for (int k = 0; ok && k < d; ++k) ok = col[s0 + k] - i == off[c * kClsWidth + k];
    if (!ok) atomicOr(bad, 1);
}

int mesh_stencil_classes(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    cudaStream_t st = ctx->stream;
    m->cls_tried = true;
    const int N = m->N;
    if (N <= 0 || m->maxdeg > kClsWidth) return RAFEM_OK;
    unsigned long long* dsig = nullptr;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&dsig, sizeof(unsigned long long) * N));
    row_sig_kernel<<<(N + 255) / 256, 256, 0, st>>>(m->rp, m->col, N, dsig);
    ctx->launches++;
    std::vector<unsigned long long> sig(N);
    std::vector<int> rp(N + 1);
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(sig.data(), dsig, sizeof(unsigned long long) * N, cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(rp.data(), m->rp, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, dsig);
    std::vector<uint8_t> cls(N);
    std::vector<unsigned long long> keys;
    std::vector<int> rep;
    for (int i = 0; i < N; ++i) {
        int c = -1;
        for (size_t k = 0; k < keys.size(); ++k)
            if (keys[k] == sig[i]) {
                c = (int)k;
                break;
            }
        if (c < 0) {
            if ((int)keys.size() >= kMaxClasses) return RAFEM_OK;  // unstructured: explicit columns
            c = (int)keys.size();
            keys.push_back(sig[i]);
            rep.push_back(i);
        }
        cls[i] = (uint8_t)c;
    }
    const int ncls = (int)keys.size();
    std::vector<int> off((size_t)ncls * kClsWidth, 0), deg(ncls);
    {  // every class representative's columns in one pinned staging area, one synchronisation
        int* pc = static_cast<int*>(pinned(ctx, sizeof(int) * (size_t)std::max(ncls, 1) * kClsWidth));
        if (!pc) return rafem_fail(ctx, RAFEM_ERR_CUDA, "pinned staging allocation failed");
        for (int c = 0; c < ncls; ++c) {
            const int i = rep[c], d = rp[i + 1] - rp[i];
            deg[c] = d;
            if (d > 0)
                RF_CUDA_TRY(ctx, cudaMemcpyAsync(pc + (size_t)c * kClsWidth, m->col + rp[i], sizeof(int) * d,
                                                 cudaMemcpyDeviceToHost, st));
        }
        RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
        for (int c = 0; c < ncls; ++c)
            for (int k = 0; k < deg[c]; ++k) off[(size_t)c * kClsWidth + k] = pc[(size_t)c * kClsWidth + k] - rep[c];
    }
    uint8_t* dcls = nullptr;
    int* doff = nullptr;
    int* ddeg = nullptr;
    int* dbad = nullptr;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&dcls, N));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&doff, sizeof(int) * off.size()));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&ddeg, sizeof(int) * ncls + sizeof(int)));
    dbad = ddeg + ncls;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(dcls, cls.data(), N, cudaMemcpyHostToDevice, st));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(doff, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice, st));
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(ddeg, deg.data(), sizeof(int) * ncls, cudaMemcpyHostToDevice, st));
    RF_CUDA_TRY(ctx, cudaMemsetAsync(dbad, 0, sizeof(int), st));
    cls_verify_kernel<<<(N + 255) / 256, 256, 0, st>>>(m->rp, m->col, N, dcls, doff, ddeg, dbad);
    ctx->launches++;
    int hbad = 0;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    dfree(ctx, ddeg);
    if (hbad) {  // hash collision: keep explicit columns
        dfree(ctx, dcls);
        dfree(ctx, doff);
        return RAFEM_OK;
    }
    m->cls = dcls;
    m->cls_off = doff;
    m->ncls = ncls;
    return RAFEM_OK;
}

int mesh_geometry(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    const int M = m->M;
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->base, sizeof(double) * 10 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->grad, sizeof(double) * 12 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&m->vol, sizeof(double) * (size_t)std::max(M, 1)));
    if (M > 0) {
        geometry_kernel<<<(M + 127) / 128, 128, 0, ctx->stream>>>(m->nodes, m->tets, M, m->base, m->grad, m->vol);
        ctx->launches++;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int system_contrib(rafem_system* s) {
    if (s->contrib) return RAFEM_OK;
    rafem_ctx* ctx = s->mesh->ctx;
    const size_t M = std::max(s->mesh->M, 1);
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&s->contrib, sizeof(double) * 32 * M));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&s->load, sizeof(double) * 4 * M));
    return RAFEM_OK;
}

int system_escal(rafem_system* s) {
    if (s->esig) return RAFEM_OK;
    rafem_ctx* ctx = s->mesh->ctx;
    const size_t M = std::max(s->mesh->M, 1);
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&s->esig, sizeof(double) * M));
    RF_CUDA_TRY(ctx, dmalloc(ctx, (void**)&s->eload, sizeof(double) * 4 * M));
    return RAFEM_OK;
}

AsmMesh asm_mesh(const rafem_mesh* m) {
    AsmMesh a;
    a.tets = m->tets;
    a.region = m->region;
    a.regtab = m->regtab;
    a.nreg = m->nreg;
    a.base = m->base;
    a.grad = m->grad;
    a.vol = m->vol;
    a.rp = m->rp;
    a.col = m->col;
    a.diag = m->diag;
    a.inc_ptr = m->inc_ptr;
    a.inc_ea = m->inc_ea;
    a.inc_slot = m->inc_slot;
    a.kind = m->kind;
    a.slot_ptr = m->slot_ptr;
    a.slot_src = m->slot_src;
    a.cpos = m->contrib_pos;
    a.lpos = m->load_pos;
    a.N = m->N;
    a.M = m->M;
    a.own_end = m->own_end >= 0 ? m->own_end : m->N;
    a.below_end = m->below_end >= 0 ? m->below_end : m->N;
    return a;
}

// element + fill kernels: raw (unscaled, unconstrained) values, rhs and the
// per-row diagonal entries in s->diagpart
int assemble_fill_launch(rafem_system* s, const double* t_it, int ts, const double* v_it, int vs,
                         const double* t_prev, int ps, double dt, long long* bad_dev) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    cudaStream_t st = ctx->stream;
    const int N = m->N, M = m->M;
    const char* wf = getenv("RAFEM_WARP_FILL");
    const bool warp_fill = wf && wf[0] == '1';
    // fused element + fill (default; RAFEM_FUSED_FILL=0: element kernel +
    // contributor-list fill through the per-element intermediate)
    const char* ff = getenv("RAFEM_FUSED_FILL");
    const bool fused = !(ff && ff[0] == '0') && !warp_fill;
    if (!fused && !warp_fill && !m->slot_lists_tried)
        if (int rc = mesh_slot_lists(m)) return rc;
    const AsmMesh am = asm_mesh(m);
    const AsmFields f{t_it, ts, v_it, vs, t_prev, ps, dt};
    double2* contrib = reinterpret_cast<double2*>(s->contrib);
    double2* val2 = reinterpret_cast<double2*>(s->val2);
    RF_CUDA_TRY(ctx, cudaMemsetAsync(bad_dev, 0xff, sizeof(long long), st));
    if (fused) {
        if (int rc = system_escal(s)) return rc;
        if (M > 0) {
            element_scalars_kernel<<<(M + 255) / 256, 256, 0, st>>>(am, f, s->esig, s->eload,
                                                                    reinterpret_cast<unsigned long long*>(bad_dev));
            ctx->launches++;
        }
        if (N > 0) {
            const char* hf = getenv("RAFEM_HALF_FILL");
            const char* fp = getenv("RAFEM_FILL_PIPE");
            if (m->maxdeg <= 16 && m->maxinc <= 32 && m->nreg <= kFillRegions && !(hf && hf[0] == '0') &&
                !(fp && fp[0] == '0')) {
                // persistent: the blocks that fit at once (whole waves), or fewer for small meshes
                static int occ = 0;
                if (!occ) {
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_fill_half_pipe_kernel, 256, 0);
                    occ = std::max(occ, 1);
                }
                const long long need = ((long long)N * 16 + 255) / 256;
                const long long blocks = std::min<long long>(need, (long long)occ * ctx->sm_count);
                fused_fill_half_pipe_kernel<<<(unsigned)blocks, 256, 0, st>>>(am, dt, s->esig, s->eload, val2,
                                                                              s->rhs, s->diagpart);
            } else if (m->maxdeg <= 16 && m->maxinc <= 32 && m->nreg <= kFillRegions && !(hf && hf[0] == '0')) {
                const long long blocks = ((long long)N * 16 + 255) / 256;
                fused_fill_half_kernel<<<(unsigned)blocks, 256, 0, st>>>(am, dt, s->esig, s->eload, val2, s->rhs,
                                                                         s->diagpart);
            } else {
                const long long blocks = ((long long)N * 32 + 255) / 256;
                fused_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(am, dt, s->esig, s->eload, val2, s->rhs,
                                                                    s->diagpart);
            }
            ctx->launches++;
        }
        RF_CUDA_TRY(ctx, cudaGetLastError());
        return RAFEM_OK;
    }
    if (int rc = system_contrib(s)) return rc;
    contrib = reinterpret_cast<double2*>(s->contrib);
    if (M > 0) {
        element_kernel<<<(M + kElemBlock - 1) / kElemBlock, kElemBlock, 0, st>>>(am, f, contrib, s->load,
                                                        reinterpret_cast<unsigned long long*>(bad_dev));
        ctx->launches++;
    }
    if (N > 0) {
        if (am.slot_src && !warp_fill) {
            const int S = (int)m->slots;
            fill_slots_kernel<<<(S + 255) / 256, 256, 0, st>>>(am, contrib, val2, S);
            fill_rows_kernel<<<(N + 255) / 256, 256, 0, st>>>(am, s->load, val2, s->rhs, s->diagpart);
            ctx->launches += 2;
        } else {
            const int blocks = (int)(((long long)N * 32 + 255) / 256);
            fill_kernel<<<blocks, 256, 0, st>>>(am, contrib, s->load, val2, s->rhs, s->diagpart);
            ctx->launches++;
        }
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

// V-row scaling + Dirichlet elimination (fem.py:394-428) of the filled rows:
// 16 lanes per row when rows have at most 16 slots (RAFEM_HALF_FILL=0: a warp)
static int constrain_launch(rafem_system* s, const rafem_assemble_params& p, const double* scale_dev) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    const char* hf = getenv("RAFEM_HALF_FILL");
    if (m->maxdeg <= 16 && !(hf && hf[0] == '0')) {
        const int blocks = (int)(((long long)m->N * 16 + 255) / 256);
        constrain_half_kernel<<<blocks, 256, 0, ctx->stream>>>(asm_mesh(m), scale_dev, p.apply_constraints,
                                                               p.applied_voltage, p.boundary_temp,
                                                               reinterpret_cast<double2*>(s->val2), s->rhs);
    } else {
        const int blocks = (int)(((long long)m->N * 32 + 255) / 256);
        constrain_kernel<<<blocks, 256, 0, ctx->stream>>>(asm_mesh(m), scale_dev, p.apply_constraints,
                                                          p.applied_voltage, p.boundary_temp,
                                                          reinterpret_cast<double2*>(s->val2), s->rhs);
    }
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

// equilibration by a given (already reduced) scale + Dirichlet elimination
int assemble_constrain_launch(rafem_system* s, const rafem_assemble_params& p, double scale) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    double* scale_dev = reinterpret_cast<double*>(s->status) + 104;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(scale_dev, &scale, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (m->N > 0) {
        if (int rc = constrain_launch(s, p, scale_dev)) return rc;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int assemble_launch(rafem_system* s, const double* t_it, int ts, const double* v_it, int vs,
                    const double* t_prev, int ps, const rafem_assemble_params& p,
                    double* scale_dev, long long* bad_dev) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    cudaStream_t st = ctx->stream;
    const int N = m->N;
    if (int rc = assemble_fill_launch(s, t_it, ts, v_it, vs, t_prev, ps, p.dt, bad_dev)) return rc;
    if (N > 0) {
        const int blocks = (int)(((long long)N * 32 + 255) / 256);
        if (int rc = diag_sums_launch(ctx, s->diagpart, N, p.equilibrate, nullptr, scale_dev)) return rc;
        (void)blocks;
        (void)st;
        if (int rc = constrain_launch(s, p, scale_dev)) return rc;
    } else {
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(scale_dev, &s->scale, sizeof(double), cudaMemcpyHostToDevice, st));
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int expand_dof_vals(rafem_system* s, double* out_dev) {
    rafem_mesh* m = s->mesh;
    rafem_ctx* ctx = m->ctx;
    if (m->N > 0) {
        expand_kernel<<<(m->N + 255) / 256, 256, 0, ctx->stream>>>(m->rp, m->N, s->val2, out_dev);
        ctx->launches++;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int predictor_launch(rafem_ctx* ctx, double* x_it, const double* x_acc, const double* x_prev, int N,
                     int step, double ratio, double* x_start) {
    predictor_kernel<<<(N + 255) / 256, 256, 0, ctx->stream>>>(x_it, x_acc, x_prev, N, step, ratio, x_start);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

int fill_initial(rafem_ctx* ctx, double* x, int N, double t0) {
    fill_state_kernel<<<(N + 255) / 256, 256, 0, ctx->stream>>>(x, N, t0);
    ctx->launches++;
    RF_CUDA_TRY(ctx, cudaGetLastError());
    return RAFEM_OK;
}

}  // namespace rafem
