// mma2_probe.cu -- pair-wide (cta_group::2, M = 256) tcgen05.mma dispatch rate at N = 64 / 128 / 256,
// SS and TS forms: the shapes of the attention kernel's QK^T (N = 64) and P V (N = 128) MMAs.
// One 2-CTA cluster per SM pair, the leader CTA's thread issues kIters MMAs back to back.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2509_13523_b200/csrc
//   tools/mma2_probe.cu -o tools/_mma2_probe
#include <cstdio>

#include "tc_ptx.cuh"

using namespace swf::tc;

constexpr int kIters = 8192;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc));
}

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_probe2(unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    csync();
    fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1 && cta_rank() == 0 && (threadIdx.x & 31) == 0) {
        const uint64_t a = desc_kmajor(smem_u32(sm), 128), b = desc_kmajor(smem_u32(sm + 32768), 128);
        const uint32_t idesc = idesc_bf16(256, N);
        const unsigned long long m0 = clock64();
#pragma unroll 16
        for (int i = 0; i < kIters; ++i) {
            if constexpr (TS)
                mma2_ts(tmem + 256, tmem, b, idesc);
            else
                mma2(tmem + 256, a, b, idesc);
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        mbar_wait(smem_u32(&bar), 0);
        cyc[blockIdx.x / 2] = clock64() - m0;
    }
    fence_before();
    csync();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// issue cost seen by the issuing thread: per iteration 4 pair MMAs (N = 128) then C commits
// (multicast to both CTAs); the pipe is drained between iterations so every MMA issues into an empty
// queue; reports cycles from the first MMA issue to the return of the last commit instruction
template <int C>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_issue(unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar[i]), 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    csync();
    fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1 && cta_rank() == 0 && (threadIdx.x & 31) == 0) {
        const uint64_t a = desc_kmajor(smem_u32(sm), 128), b = desc_kmajor(smem_u32(sm + 32768), 128);
        const uint32_t idesc = idesc_bf16(256, 128);
        unsigned long long tot = 0;
        for (int it = 0; it < 64; ++it) {
            const unsigned long long t0 = clock64();
#pragma unroll
            for (int k = 0; k < 4; ++k) mma2(tmem + 256, a + 2 * k, b + 2 * k, idesc);
#pragma unroll
            for (int c = 0; c < C; ++c)
                asm volatile(
                    "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
                        smem_u32(&bar[c]))
                    : "memory");
            const unsigned long long t1 = clock64();
            tot += t1 - t0;
            for (int c = 0; c < C; ++c) mbar_wait(smem_u32(&bar[c]), it & 1);  // drain
            if (C == 0) {
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&bar[3]))
                             : "memory");
                mbar_wait(smem_u32(&bar[3]), it & 1);
            }
        }
        cyc[blockIdx.x / 2] = tot / 64;
    }
    fence_before();
    csync();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
template <int C>
void run_issue() {
    unsigned long long* d;
    cudaMalloc(&d, 74 * 8);
    auto k = k_issue<C>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    k<<<148, 128, 65536 + 1024>>>(d);
    cudaDeviceSynchronize();
    unsigned long long h[74];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("issue: 4 MMAs (N=128) + %d commits: %llu cycles seen by the issuing thread  %s\n", C, h[0],
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int N, bool TS>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 74 * 8);
    auto k = k_probe2<N, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 128, 65536 + 1024>>>(d);
        cudaDeviceSynchronize();
    }
    unsigned long long h[74];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double c = double(h[0]) / kIters;
    const double macs = 256.0 * N * 16;  // per pair per MMA
    printf("%-10s N=%3d: %.1f cyc/MMA per pair, %.0f MAC/cyc/SM (peak 4096)  %s\n", name, N, c, macs / c / 2,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<64, false>("SS 2CTA");
    run<128, false>("SS 2CTA");
    run<256, false>("SS 2CTA");
    run<64, true>("TS 2CTA");
    run<128, true>("TS 2CTA");
    run_issue<0>();
    run_issue<1>();
    run_issue<3>();
    return 0;
}
