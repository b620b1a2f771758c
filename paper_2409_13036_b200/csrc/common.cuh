// common.cuh — shared device helpers for librafem_b200 (sm_100a).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

#define RF_DEV __device__ __forceinline__

namespace rafem {

// Exact IEEE-754 ops.  FMA contraction would change the rounding of the
// reference's numpy expressions (each numpy op rounds separately), so
// every accumulation that must be bit-stable spells its ops explicitly.
RF_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
RF_DEV double add(double a, double b) { return __dadd_rn(a, b); }
RF_DEV double sub(double a, double b) { return __dsub_rn(a, b); }

constexpr int kWarp = 32;

// Streaming (evict-first) loads for matrix data that is read once per
// sweep, so the gathered vector keeps its place in L2.
RF_DEV double ld_stream(const double* p) { return __ldcs(p); }
RF_DEV double2 ld_stream(const double2* p) { return __ldcs(p); }
RF_DEV int ld_stream(const int* p) { return __ldcs(p); }

// Deterministic warp sum: fixed xor-butterfly, so every lane ends with
// the same bits and the result depends only on the lane values.
RF_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
RF_DEV double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide deterministic sum of NV values per thread.  Result valid in
// all threads.  `red` must hold NV * 32 doubles of shared memory.
template <int NV>
RF_DEV void block_sum(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();  // protect `red` from a previous use
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) red[i * 32 + wid] = v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = (lane < nw) ? red[i * 32 + lane] : 0.0;
        v[i] = warp_sum(s);
    }
}

RF_DEV double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = (lane < nw) ? red[lane] : 0.0;
    return warp_max(s);
}

// ---- per-thread asynchronous global -> shared copies (cp.async) ----------
RF_DEV void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
RF_DEV void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
RF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- TMA 1-D bulk copies (cp.async.bulk) completing on an mbarrier -------
RF_DEV unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
RF_DEV void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
RF_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
RF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
RF_DEV void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
RF_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
RF_DEV void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Same, with an L2 cache-policy hint (e.g. evict_first for data read once).
RF_DEV void tma_load_1d_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                             unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// bulk L2 prefetch of [src, src + bytes) (16-byte aligned and sized)
RF_DEV void prefetch_l2_bulk(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
RF_DEV unsigned long long l2_policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
RF_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Sum of partial[0..G) (one per CTA) in a fixed order, by one warp.
// Every CTA that calls this sees identical bits.
// Each lane's loads are issued as one batch before its adds (the adds keep
// the ascending order, so the sum is the same bits as a plain strided loop):
// one L2 round trip per 256 partials instead of one per 32.
RF_DEV double reduce_partials_warp(const double* partial, int G) {
    const int lane = threadIdx.x & 31;
    constexpr int B = 8;
    double s = 0.0;
    for (int c0 = 0; c0 < G; c0 += 32 * B) {
        double v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int c = c0 + lane + 32 * j;
            v[j] = c < G ? __ldcg(partial + c) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < B; ++j)
            if (c0 + lane + 32 * j < G) s = add(s, v[j]);
    }
    return warp_sum(s);
}

// Max of partial[0..G) by one warp, loads batched the same way.
RF_DEV double reduce_max_partials_warp(const double* partial, int G) {
    const int lane = threadIdx.x & 31;
    constexpr int B = 8;
    double m = 0.0;
    for (int c0 = 0; c0 < G; c0 += 32 * B) {
        double v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int c = c0 + lane + 32 * j;
            v[j] = c < G ? __ldcg(partial + c) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < B; ++j) m = fmax(m, v[j]);
    }
    return warp_max(m);
}

}  // namespace rafem

// Host-side error plumbing shared by the .cu translation units.
#define RF_CUDA_TRY(ctx, expr)                                                   \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) return rafem_fail_cuda((ctx), _e, #expr, __FILE__, __LINE__); \
    } while (0)
