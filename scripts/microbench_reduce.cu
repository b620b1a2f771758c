// microbench_reduce.cu — grid-wide deterministic 3-value all-reduce variants
// over one CTA per SM (148 x 512 threads), the per-iteration floor of the
// single-reduction PCG.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_reduce microbench_reduce.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
typedef unsigned long long u64;

__device__ __forceinline__ void st_rel(u64* p, u64 v) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ u64 ld_rel(const u64* p) { u64 v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }

__device__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ void block_sum3(double* v, double* red) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = 0; i < 3; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0) for (int i = 0; i < 3; ++i) red[i * 32 + wid] = v[i];
    __syncthreads();
    for (int i = 0; i < 3; ++i) v[i] = warp_sum(lane < nw ? red[i * 32 + lane] : 0.0);
}

struct Buf {
    double* partial;   // 2 x 3 x G
    u64* ll;           // 2 x G x 8 (all-poll) / 2 x 8 (result slot)
    unsigned* counter; // monotonically increasing
};

// MODE 0: cg grid sync + gather.  1: LL all-poll.  2: last arriver + LL result.
// 3: custom counter barrier + gather.
template <int MODE>
__global__ void bench(int iters, Buf b, double* out) {
    __shared__ double red[96];
    __shared__ double co[3];
    const int G = gridDim.x, lane = threadIdx.x & 31;
    double acc = threadIdx.x * 1e-12;
    for (int it = 0; it < iters; ++it) {
        double v[3] = {acc, 2 * acc, 3 * acc};
        block_sum3(v, red);
        const int par = it & 1;
        const unsigned flag = (unsigned)it + 1;
        if (MODE == 0 || MODE == 3) {
            double* P = b.partial + par * 3 * G;
            if (threadIdx.x == 0) for (int j = 0; j < 3; ++j) P[j * G + blockIdx.x] = v[j];
            if (MODE == 0) {
                cg::this_grid().sync();
            } else {
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    atomicAdd(b.counter, 1u);
                    const unsigned target = (unsigned)(it + 1) * G;
                    while (ld_acq(b.counter) < target) {}
                    __threadfence();
                }
                __syncthreads();
            }
            if (threadIdx.x < 96) {
                int w = threadIdx.x >> 5;
                double s = 0;
                for (int c = lane; c < G; c += 32) s += __ldcg(P + w * G + c);
                s = warp_sum(s);
                if (lane == 0) co[w] = s;
            }
            __syncthreads();
        } else if (MODE == 1) {
            u64* slot = b.ll + ((size_t)par * G + blockIdx.x) * 8;
            if (threadIdx.x == 0) {
                __threadfence();
                for (int j = 0; j < 3; ++j) {
                    u64 bits = (u64)__double_as_longlong(v[j]);
                    st_rel(slot + 2 * j, ((u64)flag << 32) | (bits & 0xffffffffu));
                    st_rel(slot + 2 * j + 1, ((u64)flag << 32) | (bits >> 32));
                }
            }
            if (threadIdx.x < 32) {
                double s[3] = {0, 0, 0};
                for (int c = lane; c < G; c += 32) {
                    const u64* sl = b.ll + ((size_t)par * G + c) * 8;
                    u64 w[6];
                    bool ok;
                    do {
                        ok = true;
                        for (int k = 0; k < 6; ++k) { w[k] = ld_rel(sl + k); ok = ok && (unsigned)(w[k] >> 32) == flag; }
                    } while (!ok);
                    for (int j = 0; j < 3; ++j) s[j] += __longlong_as_double((long long)((w[2 * j] & 0xffffffffu) | (w[2 * j + 1] << 32)));
                }
                for (int j = 0; j < 3; ++j) s[j] = warp_sum(s[j]);
                if (lane == 0) for (int j = 0; j < 3; ++j) co[j] = s[j];
                __threadfence();
            }
            __syncthreads();
        } else {  // MODE 2: last arriver reduces, publishes LL result; others poll one 64-B slot
            double* P = b.partial + par * 3 * G;
            u64* res = b.ll + par * 8;
            __shared__ int last;
            if (threadIdx.x == 0) {
                for (int j = 0; j < 3; ++j) P[j * G + blockIdx.x] = v[j];
                __threadfence();
                const unsigned old = atomicAdd(b.counter, 1u);
                last = (old == (unsigned)(it + 1) * G - 1);
                if (last) __threadfence();
            }
            __syncthreads();
            if (last) {
                if (threadIdx.x < 96) {
                    int w = threadIdx.x >> 5;
                    double s = 0;
                    for (int c = lane; c < G; c += 32) s += __ldcg(P + w * G + c);
                    s = warp_sum(s);
                    if (lane == 0) {
                        u64 bits = (u64)__double_as_longlong(s);
                        st_rel(res + 2 * w, ((u64)flag << 32) | (bits & 0xffffffffu));
                        st_rel(res + 2 * w + 1, ((u64)flag << 32) | (bits >> 32));
                        co[w] = s;
                    }
                }
            } else if (threadIdx.x < 6) {
                u64 w;
                do { w = ld_rel(res + threadIdx.x); } while ((unsigned)(w >> 32) != flag);
                // reassemble in lane pairs
                unsigned lo = (unsigned)w;
                unsigned other = __shfl_xor_sync(0x3fu, lo, 1);
                if ((threadIdx.x & 1) == 0) co[threadIdx.x >> 1] = __longlong_as_double((long long)(((u64)other << 32) | lo));
            }
            if (threadIdx.x == 0) __threadfence();
            __syncthreads();
        }
        acc += co[0] * 1e-30 + co[2] * 1e-31;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

template <int MODE>
float run(int G, int iters, Buf b, double* out) {
    cudaMemset(b.counter, 0, 4);
    cudaMemset(b.ll, 0, 1 << 16);
    void* args[] = {&iters, &b, &out};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel((void*)bench<MODE>, G, 512, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(err)); return -1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3f / iters;
}

int main() {
    Buf b;
    double* out;
    cudaMalloc(&b.partial, 1 << 16);
    cudaMalloc(&b.ll, 1 << 16);
    cudaMalloc(&b.counter, 64);
    cudaMalloc(&out, 1 << 16);
    const int iters = 4000;
    for (int G : {16, 74, 148}) {
        run<0>(G, 100, b, out);
        printf("G=%3d  cg-sync+gather %.3f us | LL all-poll %.3f us | last-arriver+LL %.3f us | counter+gather %.3f us\n", G,
               run<0>(G, iters, b, out), run<1>(G, iters, b, out), run<2>(G, iters, b, out), run<3>(G, iters, b, out));
    }
    return 0;
}
