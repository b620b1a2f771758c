// microbench_bsum.cu — cost of the per-iteration CTA reduction of three
// dot-product partials (256 threads) on the B200: the two-level
// shuffle tree (block_sum<3>) vs a transposed form (threads store to
// shared memory, three warps each sum one value), and of a CTA barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_bsum microbench_bsum.cu
#include <cstdio>

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int NV>
__device__ void block_sum(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) red[i * 32 + wid] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = (lane < nw) ? red[i * 32 + lane] : 0.0;
        v[i] = warp_sum(s);
    }
}

template <int MODE>
__global__ void bench(int iters, double* out, long long* cyc) {
    __shared__ double red[3 * 32];
    __shared__ double tv[3][256];
    double acc = threadIdx.x * 1e-9;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double v[3] = {acc, acc * 2, acc * 3};
        if (MODE == 0) {
            block_sum<3>(v, red);
            if (threadIdx.x == 0) out[it & 1023] = v[0] + v[1] + v[2];
        } else if (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 3; ++j) tv[j][threadIdx.x] = v[j];
            __syncthreads();
            if (warp < 3) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) s = add(s, tv[warp][lane * 8 + k]);
                s = warp_sum(s);
                if (lane == 0) out[(it & 1023) * 3 + warp] = s;
            }
        } else if (MODE == 2) {
            __syncthreads();
        } else {
            // one warp-level tree only, partials of all 8 warps written out
#pragma unroll
            for (int j = 0; j < 3; ++j) v[j] = warp_sum(v[j]);
            if (lane == 0)
#pragma unroll
                for (int j = 0; j < 3; ++j) out[(it & 1023) * 24 + j * 8 + warp] = v[j];
        }
        acc = add(acc, 1e-12);
        if (MODE != 0) __syncthreads();  // the iteration's next CTA barrier (present in every mode)
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int MODE>
void run(const char* name, double* out, long long* cyc) {
    const int iters = 10000;
    bench<MODE><<<148, 256>>>(iters, out, cyc);
    bench<MODE><<<148, 256>>>(iters, out, cyc);
    long long c = 0;
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %8.1f cycles  %.3f us per iteration\n", name, (double)c / iters, (double)c / iters / 1965.0);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 24 * 8 * 148);
    cudaMalloc(&cyc, 148 * 8);
    run<0>("block_sum<3> (2 shuffle trees, 2 bars)", out, cyc);
    run<1>("transposed (1 bar + 1 tree) + bar", out, cyc);
    run<2>("bar.sync only", out, cyc);
    run<3>("warp trees only + bar", out, cyc);
    return 0;
}
