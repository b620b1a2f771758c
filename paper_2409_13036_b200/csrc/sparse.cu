// sparse.cu — device coo_to_csr (reference: sparse.py:164-197).
//
// The reference stably lexsorts triplets by (row, col) and sums each run
// of equal coordinates first-to-last with a sequential bincount, so every
// output value is ((0 + v_a) + v_b) + ... over the duplicates in input
// order.  Here: rows are bucketed with a count/scan, each row's entries are
// sorted on the 64-bit key (col << 32 | input position) — which is the
// stable order — and each run is summed left to right from 0.0.  The
// result is bit-identical to the reference for any input.
#include "common.cuh"
#include "internal.hpp"

#include <algorithm>
#include <vector>

namespace rafem {

constexpr int kShortRow = 64;
constexpr int kLongRowMax = 4096;

__global__ void coo_count_kernel(const long long* rows, long long nnz, int* cnt) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k < nnz) atomicAdd(cnt + rows[k], 1);
}

__global__ void coo_scatter_kernel(const long long* rows, const long long* cols, long long nnz,
                                   int* cursor, unsigned long long* keys) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int p = atomicAdd(cursor + rows[k], 1);
    keys[p] = ((unsigned long long)cols[k] << 32) | (unsigned long long)k;
}

__global__ void row_sort_short_kernel(const int* rp, int nrows, unsigned long long* keys, int* maxlen) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int p0 = rp[r], p1 = rp[r + 1];
    atomicMax(maxlen, p1 - p0);
    if (p1 - p0 > kShortRow) return;
    for (int p = p0 + 1; p < p1; ++p) {
        const unsigned long long v = keys[p];
        int q = p - 1;
        while (q >= p0 && keys[q] > v) {
            keys[q + 1] = keys[q];
            --q;
        }
        keys[q + 1] = v;
    }
}

// one CTA per long row: bitonic sort in shared memory
__global__ void row_sort_long_kernel(const int* rp, unsigned long long* keys) {
    __shared__ unsigned long long s[kLongRowMax];
    const int r = blockIdx.x;
    const int p0 = rp[r], len = rp[r + 1] - p0;
    if (len <= kShortRow) return;
    int np2 = 1;
    while (np2 < len) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += blockDim.x) s[i] = (i < len) ? keys[p0 + i] : ~0ULL;
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long a = s[i], b = s[ixj];
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) keys[p0 + i] = s[i];
}

__global__ void run_count_kernel(const int* rp, int nrows, const unsigned long long* keys, int* ucnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    int u = 0;
    long long last = -1;
    for (int p = rp[r]; p < rp[r + 1]; ++p) {
        const long long c = (long long)(keys[p] >> 32);
        if (c != last) {
            ++u;
            last = c;
        }
    }
    ucnt[r] = u;
}

__global__ void run_sum_kernel(const int* rp, int nrows, const unsigned long long* keys,
                               const double* vals, const int* orp, long long* out_col,
                               double* out_val) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    int o = orp[r] - 1;
    long long last = -1;
    double acc = 0.0;
    for (int p = rp[r]; p < rp[r + 1]; ++p) {
        const unsigned long long k = keys[p];
        const long long c = (long long)(k >> 32);
        if (c != last) {
            if (o >= orp[r]) out_val[o] = acc;
            ++o;
            out_col[o] = c;
            acc = 0.0;
            last = c;
        }
        acc = add(acc, vals[k & 0xffffffffULL]);
    }
    if (o >= orp[r]) out_val[o] = acc;
}

// exclusive scan helper shared with assembly.cu (defined there)
int scan_ints(rafem_ctx* ctx, const int* in, int* out, int n);

int coo_to_csr_device(rafem_ctx* ctx, long long nrows, long long ncols, long long nnz,
                      const int64_t* rows, const int64_t* cols, const double* vals,
                      int64_t* row_ptr_out, int64_t* col_idx_out, double* vals_out,
                      int64_t* nnz_out) {
    (void)ncols;
    if (nrows < 0 || nnz < 0) return rafem_fail(ctx, RAFEM_ERR_INVALID, "negative size");
    if (nrows >= (1LL << 31) - 1 || nnz >= (1LL << 31) - 1 || ncols >= (1LL << 31))
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "coo_to_csr: sizes must fit in int32");
    cudaStream_t st = ctx->stream;
    const int nr = (int)nrows;
    if (nnz == 0) {
        for (long long i = 0; i <= nrows; ++i) row_ptr_out[i] = 0;
        *nnz_out = 0;
        return RAFEM_OK;
    }
    long long *drows = nullptr, *dcols = nullptr, *dcol_out = nullptr;
    double *dvals = nullptr, *dval_out = nullptr;
    int *cnt = nullptr, *rp = nullptr, *cursor = nullptr, *ucnt = nullptr, *orp = nullptr, *maxlen = nullptr;
    unsigned long long* keys = nullptr;
    auto cleanup = [&]() {
        cudaFree(drows); cudaFree(dcols); cudaFree(dcol_out); cudaFree(dvals); cudaFree(dval_out);
        cudaFree(cnt); cudaFree(rp); cudaFree(cursor); cudaFree(ucnt); cudaFree(orp); cudaFree(maxlen);
        cudaFree(keys);
    };
    cudaError_t e = cudaSuccess;
#define RF_STEP(x) do { e = (x); if (e != cudaSuccess) { cleanup(); return rafem_fail_cuda(ctx, e, #x, __FILE__, __LINE__); } } while (0)
    RF_STEP(cudaMalloc(&drows, 8 * nnz));
    RF_STEP(cudaMalloc(&dcols, 8 * nnz));
    RF_STEP(cudaMalloc(&dvals, 8 * nnz));
    RF_STEP(cudaMalloc(&keys, 8 * nnz));
    RF_STEP(cudaMalloc(&dcol_out, 8 * nnz));
    RF_STEP(cudaMalloc(&dval_out, 8 * nnz));
    RF_STEP(cudaMalloc(&cnt, sizeof(int) * (nr + 1)));
    RF_STEP(cudaMalloc(&rp, sizeof(int) * (nr + 1)));
    RF_STEP(cudaMalloc(&cursor, sizeof(int) * (nr + 1)));
    RF_STEP(cudaMalloc(&ucnt, sizeof(int) * (nr + 1)));
    RF_STEP(cudaMalloc(&orp, sizeof(int) * (nr + 1)));
    RF_STEP(cudaMalloc(&maxlen, sizeof(int)));
    RF_STEP(cudaMemcpyAsync(drows, rows, 8 * nnz, cudaMemcpyHostToDevice, st));
    RF_STEP(cudaMemcpyAsync(dcols, cols, 8 * nnz, cudaMemcpyHostToDevice, st));
    RF_STEP(cudaMemcpyAsync(dvals, vals, 8 * nnz, cudaMemcpyHostToDevice, st));
    RF_STEP(cudaMemsetAsync(cnt, 0, sizeof(int) * (nr + 1), st));
    RF_STEP(cudaMemsetAsync(maxlen, 0, sizeof(int), st));
    const int tb = 256;
    const long long nb = (nnz + tb - 1) / tb;
    coo_count_kernel<<<(unsigned)nb, tb, 0, st>>>(drows, nnz, cnt);
    ctx->launches++;
    if (int rc = scan_ints(ctx, cnt, rp, nr)) { cleanup(); return rc; }
    RF_STEP(cudaMemcpyAsync(cursor, rp, sizeof(int) * nr, cudaMemcpyDeviceToDevice, st));
    coo_scatter_kernel<<<(unsigned)nb, tb, 0, st>>>(drows, dcols, nnz, cursor, keys);
    ctx->launches++;
    if (nr > 0) {
        row_sort_short_kernel<<<(nr + tb - 1) / tb, tb, 0, st>>>(rp, nr, keys, maxlen);
        ctx->launches++;
    }
    int hmax = 0;
    RF_STEP(cudaMemcpyAsync(&hmax, maxlen, sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_STEP(cudaStreamSynchronize(st));
    if (hmax > kLongRowMax) {
        cleanup();
        return rafem_fail(ctx, RAFEM_ERR_UNSUPPORTED, "coo_to_csr: a row holds more than 4096 triplets");
    }
    if (hmax > kShortRow) {
        row_sort_long_kernel<<<nr, 512, 0, st>>>(rp, keys);
        ctx->launches++;
    }
    run_count_kernel<<<(nr + tb - 1) / tb, tb, 0, st>>>(rp, nr, keys, ucnt);
    ctx->launches++;
    if (int rc = scan_ints(ctx, ucnt, orp, nr)) { cleanup(); return rc; }
    run_sum_kernel<<<(nr + tb - 1) / tb, tb, 0, st>>>(rp, nr, keys, dvals, orp, dcol_out, dval_out);
    ctx->launches++;
    RF_STEP(cudaGetLastError());
    std::vector<int> hrp(nr + 1);
    RF_STEP(cudaMemcpyAsync(hrp.data(), orp, sizeof(int) * (nr + 1), cudaMemcpyDeviceToHost, st));
    RF_STEP(cudaStreamSynchronize(st));
    const long long nout = hrp[nr];
    for (int i = 0; i <= nr; ++i) row_ptr_out[i] = hrp[i];
    RF_STEP(cudaMemcpyAsync(col_idx_out, dcol_out, 8 * nout, cudaMemcpyDeviceToHost, st));
    RF_STEP(cudaMemcpyAsync(vals_out, dval_out, 8 * nout, cudaMemcpyDeviceToHost, st));
    RF_STEP(cudaStreamSynchronize(st));
#undef RF_STEP
    *nnz_out = nout;
    cleanup();
    return RAFEM_OK;
}

}  // namespace rafem
