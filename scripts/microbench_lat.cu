// microbench_lat.cu — dependent-latency of the fp64 / shared-memory
// operations on the pipelined PCG's per-iteration critical path (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_lat microbench_lat.cu
#include <cstdio>

template <int OP>
__global__ void chain(int n, double seed, double* out, long long* cyc) {
    __shared__ double sm[1024];
    __shared__ int si[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        sm[i] = 1.0 + i * 1e-9;
        si[i] = (i * 7 + 1) & 1023;
    }
    __syncthreads();
    double a = seed + threadIdx.x * 1e-12, b = 1.0000001;
    int k = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) a = __dadd_rn(a, b);                 // DADD
        else if (OP == 1) a = __fma_rn(a, b, 1e-9);       // DFMA
        else if (OP == 2) a = b / a;                       // IEEE fp64 division
        else if (OP == 3) a = __drcp_rn(a);                // IEEE reciprocal
        else if (OP == 4) { k = si[k]; }                   // dependent smem int load
        else if (OP == 5) a = __dadd_rn(sm[(int)a & 1023], 1.0);  // smem double load + add
        else if (OP == 6) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));  // shfl double + add
        else if (OP == 7) a = sqrt(a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[threadIdx.x] = a + k;
}

template <int OP>
void run(const char* name) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8 * 8);
    const int n = 4096;
    chain<OP><<<1, 256>>>(n, 1.5, out, cyc);
    chain<OP><<<1, 256>>>(n, 1.5, out, cyc);
    long long c;
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %7.1f cycles per dependent op (256 threads)\n", name, (double)c / n);
}

int main() {
    run<0>("DADD");
    run<1>("DFMA");
    run<2>("fp64 division b / a");
    run<3>("__drcp_rn");
    run<4>("smem int load (pointer chase)");
    run<5>("smem double load + DADD");
    run<6>("shfl.xor double + DADD");
    run<7>("fp64 sqrt");
    return 0;
}
