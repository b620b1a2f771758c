// microbench_cl.cu — latency constants behind the cluster-resident PCG
// (cluster.cu): FP64 chains, 64-bit butterflies, smem chases, division, and
// the DSMEM exchange primitives (st.async + mbarrier, barrier.cluster).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mbcl scripts/microbench_cl.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_async2(unsigned addr, double a, double b, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(a), "d"(b), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned par) {
    asm volatile(
        "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra "
        "W_%=;\n}" ::"r"(smem_u32(b)),
        "r"(par)
        : "memory");
}

__global__ void chains(int n, double seed, double* out, long long* cyc) {
    __shared__ double2 sm[1024];
    __shared__ int nxt[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        sm[i] = make_double2(seed + i, seed - i);
        nxt[i] = (i * 37 + 11) & 1023;
    }
    __syncthreads();
    double a = seed, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = a + c;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i)
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    long long t3 = clock64();
    int k = threadIdx.x;
    double2 acc = make_double2(0, 0);
    for (int i = 0; i < n; ++i) {
        k = nxt[k];
        acc.x += sm[k].x;
    }
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) a = 1.0 / a + 1e-300;
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) a = (a + 1.0) / (a + 2.0);
    long long t6 = clock64();
    for (int i = 0; i < n; ++i) {
        k = nxt[k];
        acc.x += sm[k].y;  // LDS then dependent LDS.128 address
        acc.y = sm[(k + (int)acc.x) & 1023].x;
    }
    long long t7 = clock64();
    out[threadIdx.x] = a + acc.x + acc.y + k;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
        cyc[4] = t5 - t4;
        cyc[5] = t6 - t5;
        cyc[6] = t7 - t6;
    }
}

// MODE 0: barrier.cluster (release/acquire) rounds; 1: relaxed barrier.cluster;
// 2: all-to-all st.async exchange (32 B per CTA pair) + mbarrier wait;
// 3: same + __syncthreads + warp reduce (the engine's publish);
// 4: ping-pong st.async between rank 0 and 1 (others idle)
// halo variants (every thread sends 16 B to each of its two neighbour CTAs,
// then the partials all-to-all):
// 5: st.async everything; 6: st.shared::cluster + barrier.cluster release/acquire;
// 7: st.shared::cluster + fence.*.sync_restrict + relaxed barrier.cluster;
// 8: halo packed locally + one cp.async.bulk per neighbour, partials st.async
template <int MODE>
__global__ void xbench(int iters, double* out, long long* cyc) {
    __shared__ __align__(16) double2 halo[2][2][544];
    __shared__ __align__(16) double2 sendb[2][288];
    __shared__ __align__(16) double part[2][16][4];
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ double red[32];
    const unsigned rank = cl_rank(), C = gridDim.x;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cl_sync();
    double acc = threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            cl_sync();
        } else if (MODE == 1) {
            cl_sync_relaxed();
        } else if (MODE == 2 || MODE == 3) {
            const int p = it & 1;
            if (threadIdx.x == 0) mbar_expect(&bar[p], 32u * C);
            double v = acc;
            if (MODE == 3) {
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
                __syncthreads();
                if (threadIdx.x < 32) {
                    v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                }
            }
            if (threadIdx.x < C) {
                const unsigned a = cl_map(&part[p][rank][0], threadIdx.x), rb = cl_map(&bar[p], threadIdx.x);
                st_async2(a, v, 1.0, rb);
                st_async2(a + 16, 2.0, 3.0, rb);
            }
            mbar_wait(&bar[p], (it >> 1) & 1);
            if (threadIdx.x < 32) {
                double s = threadIdx.x < C ? part[p][threadIdx.x][0] : 0.0;
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                acc += s * 1e-30;
            }
        } else if (MODE >= 5) {
            const int p = it & 1;
            const unsigned nb[2] = {(rank + 1) % C, (rank + C - 1) % C};
            const unsigned hbytes = MODE == 8 ? 2u * 16u * (blockDim.x < 288 ? blockDim.x : 288) : 2u * 16u * blockDim.x;
            if (MODE == 5 || MODE == 8) {
                if (threadIdx.x == 0) mbar_expect(&bar[p], 32u * C + hbytes);
            }
            const double2 v = make_double2(acc, acc + 1.0);
            if (MODE == 5) {
                for (int d = 0; d < 2; ++d)
                    st_async2(cl_map(&halo[p][d][threadIdx.x], nb[d]), v.x, v.y, cl_map(&bar[p], nb[d]));
            } else if (MODE == 7) {
                sendb[p][threadIdx.x % 288] = v;  // pull model: own smem, peers read it after the barrier
            } else if (MODE == 6) {
                for (int d = 0; d < 2; ++d) {
                    const unsigned a = cl_map(&halo[p][d][threadIdx.x], nb[d]);
                    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
                }
            } else {
                sendb[p][threadIdx.x % 288] = v;
            }
            double r = acc;
            for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
            __syncthreads();
            if (MODE == 8 && threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                for (int d = 0; d < 2; ++d)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            cl_map(&halo[p][d][0], nb[d])),
                        "r"(smem_u32(&sendb[p][0])), "r"(16u * (blockDim.x < 288 ? blockDim.x : 288)), "r"(cl_map(&bar[p], nb[d]))
                        : "memory");
            }
            if (threadIdx.x < 32) {
                r = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
                for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
                if (threadIdx.x < C) {
                    const unsigned a = cl_map(&part[p][rank][0], threadIdx.x);
                    if (MODE == 7) {
                        // pull model: partials stay local too
                    }
                    if (MODE == 5 || MODE == 8) {
                        const unsigned rb = cl_map(&bar[p], threadIdx.x);
                        st_async2(a, r, 1.0, rb);
                        st_async2(a + 16, 2.0, 3.0, rb);
                    } else {
                        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(r), "d"(1.0) : "memory");
                        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a + 16), "d"(2.0), "d"(3.0) : "memory");
                    }
                }
            }
            if (MODE == 5 || MODE == 8) {
                mbar_wait(&bar[p], (it >> 1) & 1);
            } else if (MODE == 6) {
                cl_sync();
            } else {
                asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
                asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
                asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
                asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
                for (int d = 0; d < 2; ++d) {  // pull the two neighbours' values
                    double2 h;
                    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(h.x), "=d"(h.y)
                                 : "r"(cl_map(&sendb[p][threadIdx.x % 288], nb[d])) : "memory");
                    halo[p][d][threadIdx.x] = h;
                }
                __syncthreads();
            }
            if (threadIdx.x < 32) {
                double s = threadIdx.x < C ? part[p][threadIdx.x][0] : 0.0;
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                acc += s * 1e-30 + halo[p][0][threadIdx.x].x * 1e-30;
            }
        } else {
            const int p = it & 1;
            if (rank < 2) {
                if (threadIdx.x == 0) mbar_expect(&bar[p], 16);
                if (threadIdx.x == 0 && ((it & 1) == (int)rank)) {
                    const unsigned a = cl_map(&part[p][0][0], rank ^ 1), rb = cl_map(&bar[p], rank ^ 1);
                    st_async2(a, acc, 1.0, rb);
                }
                if (threadIdx.x == 0 && ((it & 1) != (int)rank)) {
                    // receiver for this round
                }
                // both wait: the sender's barrier gets the reply in the next round
                if ((it & 1) != (int)rank) mbar_wait(&bar[p], (it >> 1) & 1);
                else {
                    // sender: its own barrier expects the peer's reply next round; complete this phase locally
                    if (threadIdx.x == 0) asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(16));
                    mbar_wait(&bar[p], (it >> 1) & 1);
                }
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    cl_sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && rank == 0) cyc[MODE] = t1 - t0;
}

template <int MODE>
static void run(int C, int nt, int iters, double* out, long long* cyc) {
    cudaFuncSetAttribute(xbench<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(nt);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, xbench<MODE>, iters, out, cyc);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMallocManaged(&cyc, 64 * sizeof(long long));
    const int n = 4096;
    chains<<<1, 32>>>(n, 1.5, out, cyc);
    cudaDeviceSynchronize();
    printf("per-op latency (clk): dfma %.1f  dadd %.1f  warp_sum(5 x shfl64+dadd) %.1f  lds chase %.1f  "
           "rcp-div %.1f  div %.1f  lds->lds.128 %.1f\n",
           cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n, cyc[4] / (double)n,
           cyc[5] / (double)n, cyc[6] / (double)n);
    const int iters = 2000;
    for (int C : {2, 8, 16}) {
        for (int nt : {128, 544}) {
            for (int k = 0; k < 8; ++k) cyc[k] = 0;
            run<0>(C, nt, iters, out, cyc);
            run<1>(C, nt, iters, out, cyc);
            run<2>(C, nt, iters, out, cyc);
            run<3>(C, nt, iters, out, cyc);
            run<5>(C, nt, iters, out, cyc);
            run<6>(C, nt, iters, out, cyc);
            run<7>(C, nt, iters, out, cyc);
            run<8>(C, nt, iters, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            printf("   halo+partials: st.async %.0f  st.cluster+bar.cluster %.0f  st.cluster+sync_restrict+relaxed %.0f  "
                   "bulk %.0f\n", cyc[5] / (double)iters, cyc[6] / (double)iters, cyc[7] / (double)iters,
                   cyc[8] / (double)iters);
            printf("C=%2d nt=%3d: barrier.cluster %.0f clk  relaxed %.0f  st.async all-to-all %.0f  +publish %.0f  (%s)\n",
                   C, nt, cyc[0] / (double)iters, cyc[1] / (double)iters, cyc[2] / (double)iters,
                   cyc[3] / (double)iters, cudaGetErrorString(e));
        }
    }
    return 0;
}
