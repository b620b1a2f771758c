// boxmesh.cu — generate_box_mesh (mesh.py:306-375) on the device, plus the
// per-step field comparison behind psnr_series (metrics.py:47-166).
//
// The box generator writes nodes, tets and Dirichlet dof kinds straight
// into a rafem_mesh and runs the symbolic phase on them, so the 16M-64M
// dof configurations never mesh or validate on the host (SURVEY.md
// §8(f)3).  Output is bit-identical to the host generator:
//   * coordinates follow numpy.linspace: x_i = i * ((stop - start) / (n - 1))
//     + start, each op rounded once, last point = stop exactly;
//   * node id (i * ny + j) * nz + k; six Kuhn tets per cell in cell-major,
//     lexicographic axis-order order, negative-parity tets with local
//     vertices 1 and 2 swapped (the orientation fix of mesh.py:115-120);
//   * outer-surface nodes get the boundary-temperature kind on their T dof,
//     electrode columns (passed in, chosen on the host by the same nearest-
//     coordinate rule) the applied / zero voltage kind on their V dof.
#include "common.cuh"
#include "internal.hpp"

#include <algorithm>
#include <cstdio>
#include <vector>

namespace rafem {

__constant__ int kKuhnOrder[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int kKuhnOdd[6] = {0, 1, 1, 0, 0, 1};

RF_DEV double linspace_at(double a, double b, int n, int i) {
    if (i == n - 1) return b;
    const double step = (b - a) / (double)(n - 1);
    return add(mul((double)i, step), a);
}

__global__ void box_nodes_kernel(int nx, int ny, int nz, double x0, double x1, double y0, double y1, double z0,
                                 double z1, double* nodes, uint8_t* kind) {
    const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long N = (long long)nx * ny * nz;
    if (id >= N) return;
    const int k = (int)(id % nz);
    const int j = (int)((id / nz) % ny);
    const int i = (int)(id / ((long long)ny * nz));
    nodes[3 * id] = linspace_at(x0, x1, nx, i);
    nodes[3 * id + 1] = linspace_at(y0, y1, ny, j);
    nodes[3 * id + 2] = linspace_at(z0, z1, nz, k);
    const bool surf = i == 0 || i == nx - 1 || j == 0 || j == ny - 1 || k == 0 || k == nz - 1;
    kind[2 * id] = RAFEM_DOF_FREE;
    kind[2 * id + 1] = surf ? RAFEM_DOF_BOUNDARY_TEMP : RAFEM_DOF_FREE;
}

__global__ void box_tets_kernel(int nx, int ny, int nz, int* tets, int* region) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long cells = (long long)(nx - 1) * (ny - 1) * (nz - 1);
    if (c >= cells) return;
    const int k = (int)(c % (nz - 1));
    const int j = (int)((c / (nz - 1)) % (ny - 1));
    const int i = (int)(c / ((long long)(ny - 1) * (nz - 1)));
    const int corner = (i * ny + j) * nz + k;
    const int step[3] = {ny * nz, nz, 1};
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        int off[4];
        off[0] = 0;
#pragma unroll
        for (int v = 0; v < 3; ++v) off[v + 1] = off[v] + step[kKuhnOrder[t][v]];
        if (kKuhnOdd[t]) {
            const int s = off[1];
            off[1] = off[2];
            off[2] = s;
        }
        int4 tv = make_int4(corner + off[0], corner + off[1], corner + off[2], corner + off[3]);
        reinterpret_cast<int4*>(tets)[c * 6 + t] = tv;
        region[c * 6 + t] = 0;
    }
}

__global__ void set_kind_kernel(const long long* ids, int n, uint8_t* kind, int dof, uint8_t value) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) kind[2 * ids[i] + dof] = value;
}

// per (step, field): sum of squared differences and max |ref|; grid (G, steps)
__global__ void __launch_bounds__(256) field_diff_kernel(const double* ref, const double* test, long long n,
                                                         long long stride, double* part) {
    __shared__ double red[64];
    const long long base = (long long)blockIdx.y * stride;
    double v[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = ref[base + i];
        const double d = sub(r, test[base + i]);
        v[0] = add(v[0], mul(d, d));
        v[1] = fmax(v[1], fabs(r));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v[0] = warp_sum(v[0]);
    v[1] = warp_max(v[1]);
    if (lane == 0) {
        red[wid] = v[0];
        red[32 + wid] = v[1];
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        double s = lane < nw ? red[lane] : 0.0, m = lane < nw ? red[32 + lane] : 0.0;
        s = warp_sum(s);
        m = warp_max(m);
        if (lane == 0) {
            part[2 * ((long long)blockIdx.y * gridDim.x + blockIdx.x)] = s;
            part[2 * ((long long)blockIdx.y * gridDim.x + blockIdx.x) + 1] = m;
        }
    }
}

__global__ void field_diff_finish(const double* part, int G, int steps, double* sq, double* mx) {
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= steps) return;
    const int lane = threadIdx.x & 31;
    double a = 0.0, m = 0.0;
    for (int c = lane; c < G; c += 32) {
        a = add(a, part[2 * ((long long)s * G + c)]);
        m = fmax(m, part[2 * ((long long)s * G + c) + 1]);
    }
    a = warp_sum(a);
    m = warp_max(m);
    if (lane == 0) {
        sq[s] = a;
        mx[s] = m;
    }
}

}  // namespace rafem

using namespace rafem;

extern "C" {

int rafem_mesh_create_box(rafem_ctx* ctx, int32_t nx, int32_t ny, int32_t nz, const double* extent,
                          const int64_t* electrode_pos, int64_t n_pos, const int64_t* electrode_neg, int64_t n_neg,
                          double k, double rho_c, double sigma0, double alpha, double t_ref, rafem_mesh** out) {
    if (!ctx || !out || !extent) return RAFEM_ERR_INVALID;
    *out = nullptr;
    if (nx < 2 || ny < 2 || nz < 2) return rafem_fail(ctx, RAFEM_ERR_INVALID, "generate_box_mesh requires nx, ny, nz >= 2");
    for (int a = 0; a < 3; ++a)
        if (!(extent[2 * a] < extent[2 * a + 1]))
            return rafem_fail(ctx, RAFEM_ERR_INVALID, "extent bounds must be strictly increasing per axis");
    const long long N = (long long)nx * ny * nz;
    const long long M = 6LL * (nx - 1) * (ny - 1) * (nz - 1);
    if (N >= (1LL << 30) || M >= (1LL << 30))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "mesh too large for 30-bit element ids");
    for (int64_t i = 0; i < n_pos; ++i)
        if (electrode_pos[i] < 0 || electrode_pos[i] >= N) return rafem_fail(ctx, RAFEM_ERR_INVALID, "electrode node out of range");
    for (int64_t i = 0; i < n_neg; ++i)
        if (electrode_neg[i] < 0 || electrode_neg[i] >= N) return rafem_fail(ctx, RAFEM_ERR_INVALID, "electrode node out of range");
    rafem_mesh* m = new rafem_mesh();
    static unsigned long long next_id = 1ULL << 40;
    m->ctx = ctx;
    m->id = next_id++;
    m->N = (int)N;
    m->M = (int)M;
    m->nreg = 1;
    cudaStream_t st = ctx->stream;
    cudaError_t e;
    long long* dids = nullptr;
#define RF_MS(x) do { e = (x); if (e != cudaSuccess) { cudaFree(dids); rafem_mesh_destroy(m); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    RF_MS(dmalloc(ctx, (void**)&m->nodes, sizeof(double) * 3 * N));
    RF_MS(dmalloc(ctx, (void**)&m->tets, sizeof(int) * 4 * M));
    RF_MS(dmalloc(ctx, (void**)&m->region, sizeof(int) * M));
    RF_MS(dmalloc(ctx, (void**)&m->regtab, sizeof(double) * 5));
    RF_MS(dmalloc(ctx, (void**)&m->kind, 2 * N));
    const double tab[5] = {k, rho_c, sigma0, alpha, t_ref};
    RF_MS(cudaMemcpyAsync(m->regtab, tab, sizeof(tab), cudaMemcpyHostToDevice, st));
    box_nodes_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(nx, ny, nz, extent[0], extent[1], extent[2],
                                                                  extent[3], extent[4], extent[5], m->nodes, m->kind);
    const long long cells = M / 6;
    box_tets_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, st>>>(nx, ny, nz, m->tets, m->region);
    ctx->launches += 2;
    const int64_t nids = n_pos + n_neg;
    if (nids > 0) {
        RF_MS(cudaMalloc(&dids, sizeof(long long) * nids));
        if (n_pos) RF_MS(cudaMemcpyAsync(dids, electrode_pos, sizeof(long long) * n_pos, cudaMemcpyHostToDevice, st));
        if (n_neg)
            RF_MS(cudaMemcpyAsync(dids + n_pos, electrode_neg, sizeof(long long) * n_neg, cudaMemcpyHostToDevice, st));
        // fem.py:403-413 order: positive electrode, then negative (distinct V dofs)
        if (n_pos) set_kind_kernel<<<(unsigned)((n_pos + 255) / 256), 256, 0, st>>>(dids, (int)n_pos, m->kind, 0, RAFEM_DOF_APPLIED_VOLTAGE);
        if (n_neg) set_kind_kernel<<<(unsigned)((n_neg + 255) / 256), 256, 0, st>>>(dids + n_pos, (int)n_neg, m->kind, 0, RAFEM_DOF_ZERO);
        ctx->launches += 2;
    }
    RF_MS(cudaGetLastError());
#undef RF_MS
    if (int rc = mesh_symbolic(m)) {
        cudaFree(dids);
        rafem_mesh_destroy(m);
        return rc;
    }
    if (int rc = mesh_geometry(m)) {
        cudaFree(dids);
        rafem_mesh_destroy(m);
        return rc;
    }
    cudaError_t se = cudaStreamSynchronize(st);
    cudaFree(dids);
    if (se != cudaSuccess) {
        rafem_mesh_destroy(m);
        return rafem_fail_cuda(ctx, se, "box mesh setup", __FILE__, __LINE__);
    }
    *out = m;
    return RAFEM_OK;
}

int rafem_mesh_download(rafem_mesh* m, double* nodes, int32_t* tets, uint8_t* dof_kind) {
    if (!m) return RAFEM_ERR_INVALID;
    rafem_ctx* ctx = m->ctx;
    if (nodes) RF_CUDA_TRY(ctx, cudaMemcpyAsync(nodes, m->nodes, sizeof(double) * 3 * m->N, cudaMemcpyDeviceToHost, ctx->stream));
    if (tets) RF_CUDA_TRY(ctx, cudaMemcpyAsync(tets, m->tets, sizeof(int) * 4 * (size_t)m->M, cudaMemcpyDeviceToHost, ctx->stream));
    if (dof_kind) RF_CUDA_TRY(ctx, cudaMemcpyAsync(dof_kind, m->kind, 2 * (size_t)m->N, cudaMemcpyDeviceToHost, ctx->stream));
    RF_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return RAFEM_OK;
}

int64_t rafem_mesh_counts(const rafem_mesh* m, int64_t* n_tets) {
    if (!m) return -1;
    if (n_tets) *n_tets = m->M;
    return m->N;
}

int rafem_field_compare(rafem_ctx* ctx, int64_t n, int64_t steps, const double* ref, const double* test,
                        int32_t on_device, double* sq_err, double* max_abs_ref) {
    if (!ctx || n < 1 || steps < 0 || !sq_err || !max_abs_ref) return RAFEM_ERR_INVALID;
    if (steps == 0) return RAFEM_OK;
    cudaStream_t st = ctx->stream;
    const double* dr = ref;
    const double* dt = test;
    double* buf = nullptr;
    const size_t bytes = sizeof(double) * (size_t)n * steps;
    if (!on_device) {
        RF_CUDA_TRY(ctx, cudaMalloc(&buf, 2 * bytes));
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(buf, ref, bytes, cudaMemcpyHostToDevice, st));
        RF_CUDA_TRY(ctx, cudaMemcpyAsync(buf + (size_t)n * steps, test, bytes, cudaMemcpyHostToDevice, st));
        dr = buf;
        dt = buf + (size_t)n * steps;
    }
    const int G = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 2LL * ctx->sm_count));
    if (steps > 65535) {
        cudaFree(buf);
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "field_compare: at most 65535 steps per call");
    }
    double* part = nullptr;
    double* outs = nullptr;
    RF_CUDA_TRY(ctx, cudaMalloc(&part, sizeof(double) * 2 * G * steps));
    RF_CUDA_TRY(ctx, cudaMalloc(&outs, sizeof(double) * 2 * steps));
    field_diff_kernel<<<dim3(G, (unsigned)steps), 256, 0, st>>>(dr, dt, n, n, part);
    field_diff_finish<<<(unsigned)((steps + 7) / 8), 256, 0, st>>>(part, G, (int)steps, outs, outs + steps);
    ctx->launches += 2;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(sq_err, outs, sizeof(double) * steps, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(max_abs_ref, outs + steps, sizeof(double) * steps, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(part);
    cudaFree(outs);
    cudaFree(buf);
    if (e != cudaSuccess) return rafem_fail_cuda(ctx, e, "field_compare", __FILE__, __LINE__);
    return RAFEM_OK;
}

}  // extern "C"
