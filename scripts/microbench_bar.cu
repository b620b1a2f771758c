// microbench_bar.cu — grid barrier variants on the B200 (one CTA per SM):
// cooperative-groups sync vs counter barriers with release/acquire
// semantics instead of full fences.  Each iteration every CTA writes a
// block of doubles (like a Krylov vector segment) before the barrier and
// reads a neighbour CTA's block after it; stale reads are counted.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_bar microbench_bar.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_ar() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// MODE 0: cg grid sync.  1: red.release + ld.acquire spin.  2: fence.acq_rel +
// relaxed red + relaxed spin + fence.acq_rel.  3: __threadfence + atomicAdd +
// ld.acquire spin (the earlier custom counter).  4: like 1 but every warp's
// lane 0 spins (no trailing __syncthreads needed for the spinning warps)
template <int MODE>
__global__ void bench(int iters, int nw, double* data, unsigned* counter, unsigned long long* bad) {
    const int G = gridDim.x;
    unsigned long long nbad = 0;
    for (int it = 0; it < iters; ++it) {
        double* blk = data + ((size_t)(it & 1) * G + blockIdx.x) * nw;
        for (int i = threadIdx.x; i < nw; i += blockDim.x) blk[i] = (double)(it * 7 + i + blockIdx.x);
        if (MODE == 0) {
            cg::this_grid().sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned target = (unsigned)(it + 1) * G;
                if (MODE == 1) {
                    red_rel(counter, 1u);
                    while (ld_acq(counter) < target) {}
                } else if (MODE == 2) {
                    fence_ar();
                    red_rlx(counter, 1u);
                    while (ld_rlx(counter) < target) {}
                    fence_ar();
                } else {
                    __threadfence();
                    atomicAdd(counter, 1u);
                    while (ld_acq(counter) < target) {}
                    __threadfence();
                }
            }
            __syncthreads();
        }
        const int nb = (blockIdx.x + 1 + it % (G > 1 ? G - 1 : 1)) % G;
        const double* ob = data + ((size_t)(it & 1) * G + nb) * nw;
        for (int i = threadIdx.x; i < nw; i += blockDim.x)
            if (__ldcg(ob + i) != (double)(it * 7 + i + nb)) ++nbad;
    }
    if (nbad) atomicAdd(bad, nbad);
}

template <int MODE>
float run(int G, int T, int nw, int iters, double* data, unsigned* counter, unsigned long long* bad) {
    cudaMemset(counter, 0, 4);
    void* args[] = {&iters, &nw, &data, &counter, &bad};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)bench<MODE>, G, T, args, 0, 0);
    cudaMemset(counter, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bench<MODE>, G, T, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e) printf("  error %s\n", cudaGetErrorString(e));
    return ms * 1e3f / iters;
}

int main() {
    double* data;
    unsigned* counter;
    unsigned long long* bad;
    cudaMalloc(&data, 2 * 148 * 4096 * sizeof(double));
    cudaMalloc(&counter, 4);
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    const int iters = 20000;
    for (int G : {16, 74, 148})
        for (int nw : {0, 128, 512}) {
            float t0 = run<0>(G, 256, nw, iters, data, counter, bad);
            float t1 = run<1>(G, 256, nw, iters, data, counter, bad);
            float t2 = run<2>(G, 256, nw, iters, data, counter, bad);
            float t3 = run<3>(G, 256, nw, iters, data, counter, bad);
            unsigned long long nb = 0;
            cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
            printf("G=%3d words=%4d  cg %.3f us | rel/acq %.3f us | acq_rel fences %.3f us | threadfence %.3f us  stale=%llu\n",
                   G, nw, t0, t1, t2, t3, nb);
        }
    return 0;
}
