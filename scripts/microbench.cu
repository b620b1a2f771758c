// microbench.cu — barrier / reduction round-trip costs on the B200 that set
// the per-iteration floor of the persistent Krylov kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__device__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ double block_sum(double v, double* red) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    return warp_sum(lane < nw ? red[lane] : 0.0);
}

template <int MODE>  // 0 grid sync only, 1 grid round (publish+sync+gather), 2 cluster sync, 3 cluster round, 4 cluster DSMEM round
__global__ void bench(int iters, double* partial, double* out) {
    __shared__ double red[32];
    __shared__ double co;
    __shared__ double inbox[32];
    double acc = threadIdx.x * 1e-9;
    const int G = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            cg::this_grid().sync();
        } else if (MODE == 2) {
            cg::this_cluster().sync();
        } else if (MODE == 1 || MODE == 3) {
            double s = block_sum(acc, red);
            double* P = partial + (it & 1) * G;
            if (threadIdx.x == 0) P[blockIdx.x] = s;
            if (MODE == 1) cg::this_grid().sync(); else cg::this_cluster().sync();
            if (threadIdx.x < 32) {
                double t = 0;
                for (int c = threadIdx.x; c < G; c += 32) t += __ldcg(P + c);
                t = warp_sum(t);
                if (threadIdx.x == 0) co = t;
            }
            __syncthreads();
            acc += co * 1e-30;
        } else {  // MODE 4: every CTA writes its partial into all CTAs' inbox via DSMEM
            cg::cluster_group cl = cg::this_cluster();
            double s = block_sum(acc, red);
            double* box = inbox + (it & 1) * 16;
            if (threadIdx.x < G) {
                double* remote = cl.map_shared_rank(box, threadIdx.x);
                remote[blockIdx.x] = s;
            }
            cl.sync();
            if (threadIdx.x < 32) {
                double t = threadIdx.x < G ? box[threadIdx.x] : 0.0;
                t = warp_sum(t);
                if (threadIdx.x == 0) co = t;
            }
            __syncthreads();
            acc += co * 1e-30;
        }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// dependent L2 load chain: ns per load
__global__ void chase(const int* next, int steps, int* out) {
    int p = 0;
    for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
    *out = p;
}

template <int MODE>
float run_grid(int G, int threads, int iters, double* partial, double* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void* args[] = {&iters, &partial, &out};
    cudaLaunchCooperativeKernel((void*)bench<MODE>, G, threads, args, 0, 0);  // warm
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bench<MODE>, G, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (cudaGetLastError() != cudaSuccess) return -1;
    return ms * 1e3f / iters;
}

template <int MODE>
float run_cluster(int C, int threads, int iters, double* partial, double* out) {
    cudaFuncSetAttribute((void*)bench<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, bench<MODE>, iters, partial, out);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, bench<MODE>, iters, partial, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("  error %s\n", cudaGetErrorString(e));
        return -1;
    }
    return ms * 1e3f / iters;
}

int main() {
    double *partial, *out;
    cudaMalloc(&partial, 1 << 20);
    cudaMalloc(&out, 1 << 20);
    const int iters = 4000;
    for (int threads : {256, 512}) {
        for (int G : {1, 8, 16, 33, 74, 148}) {
            printf("grid    G=%3d thr=%d  sync %.3f us   reduce-round %.3f us\n", G, threads,
                   run_grid<0>(G, threads, iters, partial, out), run_grid<1>(G, threads, iters, partial, out));
        }
        for (int C : {2, 4, 8, 16}) {
            printf("cluster C=%3d thr=%d  sync %.3f us   reduce-round %.3f us   dsmem-round %.3f us\n", C, threads,
                   run_cluster<2>(C, threads, iters, partial, out), run_cluster<3>(C, threads, iters, partial, out),
                   run_cluster<4>(C, threads, iters, partial, out));
        }
    }
    // L2 latency: random permutation chase over 8 MB
    const int n = 1 << 21;
    std::vector<int> h(n);
    for (int i = 0; i < n; ++i) h[i] = i;
    unsigned s = 12345;
    for (int i = n - 1; i > 0; --i) {
        s = s * 1103515245u + 12345u;
        int j = s % (i + 1);
        std::swap(h[i], h[j]);
    }
    std::vector<int> nxt(n);
    for (int i = 0; i < n; ++i) nxt[h[i]] = h[(i + 1) % n];
    int *dn, *dout;
    cudaMalloc(&dn, n * 4);
    cudaMalloc(&dout, 4);
    cudaMemcpy(dn, nxt.data(), n * 4, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(dn, 100000, dout);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    chase<<<1, 1>>>(dn, 100000, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("L2 dependent load latency: %.1f ns\n", ms * 1e6 / 100000);
    return 0;
}
