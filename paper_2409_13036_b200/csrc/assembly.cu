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
#include "common.cuh"
#include "internal.hpp"

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
    RF_CUDA_TRY(ctx, cudaMallocAsync(&sums, sizeof(int) * (blocks + 1), ctx->stream));
    RF_CUDA_TRY(ctx, cudaMallocAsync(&offs, sizeof(int) * (blocks + 1), ctx->stream));
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
    RF_CUDA_TRY(ctx, cudaFreeAsync(sums, ctx->stream));
    RF_CUDA_TRY(ctx, cudaFreeAsync(offs, ctx->stream));
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

// ---------------------------------------------------------------------------
// geometry (fem.py:229-244): edges e_k = p_k - p_0, det, inverse by
// cofactors (column j of E^-1 is the cross product of the other two edges
// over det), grad_0 = -(grad_1 + grad_2 + grad_3).

RF_DEV int sym_index(int a, int b) {
    // packed upper triangle of a symmetric 4x4: (0,0)(0,1)(0,2)(0,3)(1,1)(1,2)(1,3)(2,2)(2,3)(3,3)
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
    return a * 4 - (a * (a - 1)) / 2 + (b - a);
}

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

// ---------------------------------------------------------------------------
// numeric fill

struct Regions {
    const double* tab;  // 5 x nreg: k, rho_c, sigma0, alpha, t_ref
    int nreg;
};

// 1. per element: sigma(Tbar) (fem.py:272-278), Joule load (fem.py:286-288),
//    T-rhs load rho_c/dt M T_prev + f_joule (fem.py:317-321).
__global__ void element_kernel(const int* tets, const int* region, Regions R, const double* grad,
                               const double* volv, int M, const double* t_it, int ts,
                               const double* v_it, int vs, const double* t_prev, int ps, double dt,
                               double* sigma_out, double* load_out, unsigned long long* bad) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
    int nd[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) nd[a] = tets[4 * e + a];
    const int rg = region[e];
    const double sigma0 = R.tab[2 * R.nreg + rg], alpha = R.tab[3 * R.nreg + rg];
    const double tref = R.tab[4 * R.nreg + rg];
    const double rcdt = R.tab[1 * R.nreg + rg] / dt;
    double tsum = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) tsum = add(tsum, t_it[(long long)ts * nd[a]]);
    const double tbar = tsum / 4.0;
    const double sigma = mul(sigma0, add(1.0, mul(alpha, sub(tbar, tref))));
    if (sigma <= 0.0) atomicMin(bad, (unsigned long long)e);  // fem.py:274
    sigma_out[e] = sigma;
    const double vol = volv[e];
    double gv[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double va = v_it[(long long)vs * nd[a]];
#pragma unroll
        for (int d = 0; d < 3; ++d) gv[d] = add(gv[d], mul(va, grad[12LL * e + 3 * a + d]));
    }
    const double gg = add(add(mul(gv[0], gv[0]), mul(gv[2], gv[2])), mul(gv[1], gv[1]));
    const double fj = mul(mul(sigma, gg), vol) / 4.0;
    double tp[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) tp[b] = t_prev[(long long)ps * nd[b]];
    const double moff = mul(rcdt, mul(vol, 0.05));  // rho_c/dt * vol/20
    const double mdia = mul(rcdt, mul(vol, 0.1));   // rho_c/dt * vol/10
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double t[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) t[b] = mul(a == b ? mdia : moff, tp[b]);
        const double mt = add(add(t[0], t[2]), add(t[1], t[3]));
        load_out[4LL * e + a] = add(mt, fj);
    }
}

// 2. slot fill, TEAM lanes per node row.
template <int TEAM>
__global__ void fill_kernel(const int* rp, const int* inc_ptr, const unsigned* inc_ea,
                            const unsigned* inc_slot, const int* region, Regions R,
                            const double* base, const double* volv, const double* sigma,
                            const double* load, int N, double dt, double* val2, double* rhs,
                            double* diag_raw, const int* diag) {
    const int team = (blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
    const int lane = threadIdx.x % TEAM;
    if (team >= N) return;
    const int i = team;
    const int s0 = rp[i], deg = rp[i + 1] - s0;
    const int p0 = inc_ptr[i], p1 = inc_ptr[i + 1];
    const int dslot = diag[i];
    for (int cb = 0; cb < deg; cb += TEAM) {
        const int l = cb + lane;
        double accV = 0.0, accT = 0.0;
        for (int p = p0; p < p1; ++p) {
            const unsigned offs = __ldg(inc_slot + p);
            int b = -1;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
                if ((int)((offs >> (8 * bb)) & 255u) == l) b = bb;
            if (b >= 0) {
                const unsigned ea = __ldg(inc_ea + p);
                const int e = (int)(ea & 0x3fffffffu), a = (int)(ea >> 30);
                const double bab = __ldg(base + 10LL * e + sym_index(a, b));
                accV = add(accV, mul(__ldg(sigma + e), bab));
                const int rg = __ldg(region + e);
                const double kk = R.tab[rg];
                const double rcdt = R.tab[R.nreg + rg] / dt;
                const double mass = mul(__ldg(volv + e), a == b ? 0.1 : 0.05);
                accT = add(accT, add(mul(rcdt, mass), mul(kk, bab)));
            }
        }
        if (l < deg) {
            reinterpret_cast<double2*>(val2)[s0 + l] = make_double2(accV, accT);
            if (l == dslot) {
                diag_raw[2LL * i] = accV;
                diag_raw[2LL * i + 1] = accT;
            }
        }
    }
    if (dslot < 0 && lane == 0) {
        diag_raw[2LL * i] = 0.0;
        diag_raw[2LL * i + 1] = 0.0;
    }
    if (lane == 0) {  // T rhs: sum of element loads in ascending element order
        double r = 0.0;
        for (int p = p0; p < p1; ++p) {
            const unsigned ea = __ldg(inc_ea + p);
            r = add(r, __ldg(load + 4LL * (ea & 0x3fffffffu) + (ea >> 30)));
        }
        rhs[2LL * i] = 0.0;
        rhs[2LL * i + 1] = r;
    }
}

// 3. scale = 2^round(log2(sum diag_T / sum diag_V)) from a fixed-order
//    reduction (one CTA, so the bits never depend on the grid).
__global__ void __launch_bounds__(1024) equil_kernel(const double* diag_raw, int N, int equilibrate,
                                                     double* scale_out) {
    __shared__ double red[32 * 2];
    double v[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        v[0] = add(v[0], diag_raw[2LL * i]);
        v[1] = add(v[1], diag_raw[2LL * i + 1]);
    }
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        double scale = 1.0;
        if (equilibrate && v[0] > 0.0 && v[1] > 0.0) scale = ldexp(1.0, (int)rint(log2(v[1] / v[0])));
        *scale_out = scale;
    }
}

RF_DEV double dof_value(int kind, double applied, double btemp) {
    return kind == RAFEM_DOF_APPLIED_VOLTAGE ? applied : (kind == RAFEM_DOF_BOUNDARY_TEMP ? btemp : 0.0);
}

// 4. voltage-row scaling and symmetric Dirichlet elimination, keeping the
//    explicit zeros so the pattern is step-invariant (fem.py:398-428).
template <int TEAM>
__global__ void constrain_kernel(const int* rp, const int* col, const uint8_t* kind, int N,
                                 const double* scale_p, int apply, double applied, double btemp,
                                 double* val2, double* rhs) {
    const int team = (blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
    const int lane = threadIdx.x % TEAM;
    const unsigned mask = (TEAM == 32) ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
    if (team >= N) return;  // whole teams exit together (N teams, TEAM | 32)
    const int i = team;
    const double scale = *scale_p;
    const int s0 = rp[i], deg = rp[i + 1] - s0;
    const int kV = apply ? kind[2LL * i] : 0, kT = apply ? kind[2LL * i + 1] : 0;
    double mV = 0.0, mT = 0.0;  // moved-column sums, storage order (fem.py:419-424)
    for (int cb = 0; cb < deg; cb += TEAM) {
        const int l = cb + lane;
        double termV = 0.0, termT = 0.0;
        int movV = 0, movT = 0;
        if (l < deg) {
            const int j = col[s0 + l];
            const int cV = apply ? kind[2LL * j] : 0, cT = apply ? kind[2LL * j + 1] : 0;
            double2 v = reinterpret_cast<double2*>(val2)[s0 + l];
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
            reinterpret_cast<double2*>(val2)[s0 + l] = make_double2(outV, outT);
        }
        for (int t = 0; t < TEAM; ++t) {
            const double tv = __shfl_sync(mask, termV, t, TEAM);
            const double tt = __shfl_sync(mask, termT, t, TEAM);
            const int fv = __shfl_sync(mask, movV, t, TEAM);
            const int ft = __shfl_sync(mask, movT, t, TEAM);
            if (fv) mV = add(mV, tv);
            if (ft) mT = add(mT, tt);
        }
    }
    if (lane == 0) {
        double rv = 0.0;  // V rhs is zero before constraints (fem.py:388, 400)
        double rt = rhs[2LL * i + 1];
        if (apply) {
            rv = kV ? dof_value(kV, applied, btemp) : sub(rv, mV);
            rt = kT ? dof_value(kT, applied, btemp) : sub(rt, mT);
        }
        rhs[2LL * i] = rv;
        rhs[2LL * i + 1] = rt;
    }
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
__global__ void predictor_kernel(double* x_it, const double* x_acc, const double* x_prev, int N,
                                 int step, double ratio) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double t = x_acc[2LL * i + 1];
    x_it[2LL * i] = x_acc[2LL * i];
    x_it[2LL * i + 1] = step >= 1 ? add(t, mul(ratio, sub(t, x_prev[2LL * i + 1]))) : t;
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
    RF_CUDA_TRY(ctx, cudaMalloc(&cnt, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&cursor, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&flags, sizeof(int) * 4));
    RF_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * (N + 1), st));
    RF_CUDA_TRY(ctx, cudaMemsetAsync(flags, 0, sizeof(int) * 4, st));
    RF_CUDA_TRY(ctx, cudaMalloc(&m->inc_ptr, sizeof(int) * (N + 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&m->inc_ea, sizeof(unsigned) * 4 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&m->inc_slot, sizeof(unsigned) * 4 * (size_t)std::max(M, 1)));
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
        cudaFree(cnt);
        cudaFree(cursor);
        cudaFree(flags);
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "a node has more than 255 neighbours; pattern too dense for the packed slot map");
    }
    m->maxinc = hflags[0];
    m->maxdeg = hflags[1];
    RF_CUDA_TRY(ctx, cudaMalloc(&m->rp, sizeof(int) * (N + 1)));
    if (int rc = scan_ints(ctx, cnt, m->rp, N)) return rc;
    int slots = 0;
    RF_CUDA_TRY(ctx, cudaMemcpyAsync(&slots, m->rp + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    m->slots = slots;
    RF_CUDA_TRY(ctx, cudaMalloc(&m->col, sizeof(int) * ((size_t)std::max(slots, 1) + 8)));  // +8: 16-B TMA tail
    RF_CUDA_TRY(ctx, cudaMalloc(&m->diag, sizeof(int) * (size_t)std::max(N, 1)));
    if (N > 0) {
        adj_fill_kernel<<<(N + 127) / 128, 128, 0, st>>>(m->inc_ptr, m->inc_ea, m->tets, N, m->rp, m->col, m->diag, m->inc_slot);
        ctx->launches++;
    }
    RF_CUDA_TRY(ctx, cudaGetLastError());
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(st));
    cudaFree(cnt);
    cudaFree(cursor);
    cudaFree(flags);
    return RAFEM_OK;
}

int mesh_geometry(rafem_mesh* m) {
    rafem_ctx* ctx = m->ctx;
    const int M = m->M;
    RF_CUDA_TRY(ctx, cudaMalloc(&m->base, sizeof(double) * 10 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&m->grad, sizeof(double) * 12 * (size_t)std::max(M, 1)));
    RF_CUDA_TRY(ctx, cudaMalloc(&m->vol, sizeof(double) * (size_t)std::max(M, 1)));
    if (M > 0) {
        geometry_kernel<<<(M + 127) / 128, 128, 0, ctx->stream>>>(m->nodes, m->tets, M, m->base, m->grad, m->vol);
        ctx->launches++;
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
    const int N = m->N, M = m->M;
    const Regions R{m->regtab, m->nreg};
    RF_CUDA_TRY(ctx, cudaMemsetAsync(bad_dev, 0xff, sizeof(long long), st));
    if (M > 0) {
        element_kernel<<<(M + 127) / 128, 128, 0, st>>>(m->tets, m->region, R, m->grad, m->vol, M, t_it, ts,
                                                        v_it, vs, t_prev, ps, p.dt, s->sigma, s->load,
                                                        reinterpret_cast<unsigned long long*>(bad_dev));
        ctx->launches++;
    }
    if (N > 0) {
        const int team = m->maxdeg <= 16 ? 16 : 32;
        const long long threads = (long long)N * team;
        const int blocks = (int)((threads + 255) / 256);
        if (team == 16) {
            fill_kernel<16><<<blocks, 256, 0, st>>>(m->rp, m->inc_ptr, m->inc_ea, m->inc_slot, m->region, R, m->base,
                                                    m->vol, s->sigma, s->load, N, p.dt, s->val2, s->rhs, s->diagpart, m->diag);
        } else {
            fill_kernel<32><<<blocks, 256, 0, st>>>(m->rp, m->inc_ptr, m->inc_ea, m->inc_slot, m->region, R, m->base,
                                                    m->vol, s->sigma, s->load, N, p.dt, s->val2, s->rhs, s->diagpart, m->diag);
        }
        equil_kernel<<<1, 1024, 0, st>>>(s->diagpart, N, p.equilibrate, scale_dev);
        if (team == 16) {
            constrain_kernel<16><<<blocks, 256, 0, st>>>(m->rp, m->col, m->kind, N, scale_dev, p.apply_constraints,
                                                         p.applied_voltage, p.boundary_temp, s->val2, s->rhs);
        } else {
            constrain_kernel<32><<<blocks, 256, 0, st>>>(m->rp, m->col, m->kind, N, scale_dev, p.apply_constraints,
                                                         p.applied_voltage, p.boundary_temp, s->val2, s->rhs);
        }
        ctx->launches += 3;
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
                     int step, double ratio) {
    predictor_kernel<<<(N + 255) / 256, 256, 0, ctx->stream>>>(x_it, x_acc, x_prev, N, step, ratio);
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
