// issue_probe.cu -- does a warp issuing tcgen05.mma steal issue slots from other warps on its SM
// sub-partition? Warp 1 issues N=128 MMAs back to back; warps 4-11 run an FMA/MUFU loop (like the
// attention softmax); report each FMA warp's cycles (SMSP = warp % 4).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2509_13523_b200/csrc
//   tools/issue_probe.cu -o tools/_issue_probe
#include <cstdio>

#include "tc_ptx.cuh"

using namespace swf::tc;

template <int MODE>  // 0: no MMAs, 1: MMA warp 1 (per-MMA asm), 2: MMA warp 1 (8-MMA asm blocks)
                     // +3: the compute warps also read TMEM (tcgen05.ld x32) every 16 FMA/MUFU pairs
__global__ void __launch_bounds__(384, 1) k_probe(unsigned long long* cyc, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tslot;
    constexpr int MM = MODE % 3;
    constexpr bool LD = MODE >= 3;
    if (warp == 1 && MM > 0) {
        const uint64_t a = desc_kmajor(smem_u32(sm), 128), b = desc_kmajor(smem_u32(sm + 32768), 128);
        const uint32_t idesc = idesc_bf16(128, 128);
        int it = 0;
        while (!stop) {
            if (MM == 1) {
#pragma unroll 1
                for (int k = 0; k < 8; ++k) {
                    asm volatile(
                        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 256),
                        "l"(a + uint64_t(2 * k)), "l"(b + uint64_t(2 * k)), "r"(idesc), "r"(1));
                }
            } else {
                asm volatile(
                    "{\n.reg .pred e;\n.reg .b64 x, y;\nelect.sync _|e, 0xffffffff;\n"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n"
                    "add.s64 x, %1, 2; add.s64 y, %2, 2;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 4; add.s64 y, %2, 4;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 6; add.s64 y, %2, 6;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 8; add.s64 y, %2, 8;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 10; add.s64 y, %2, 10;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 12; add.s64 y, %2, 12;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "add.s64 x, %1, 14; add.s64 y, %2, 14;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, 1;\n"
                    "}\n" ::"r"(tmem + 256),
                    "l"(a), "l"(b), "r"(idesc));
            }
            ++it;
        }
        if ((threadIdx.x & 31) == 0) cyc[gridDim.x * 8 + blockIdx.x] = it;
    } else if (warp >= 4) {
        const unsigned long long t0 = clock64();
        float x = threadIdx.x * 1e-3f, y = 1.f;
#pragma unroll 1
        for (int i = 0; i < 20000; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                x = fmaf(x, 0.999f, 0.001f);
                y += ex2(x);
            }
            if (LD) {
                uint32_t r[32];
                ld32(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) & 1) * 32, r);
                wait_ld_dep(r);
                x += __uint_as_float(r[0] & 1);
            }
        }
        if (y == 1.2345f) sink[0] = y;
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 8 + warp - 4] = clock64() - t0;
    }
    if (warp >= 4) {
        asm volatile("bar.sync 1, 256;" ::: "memory");  // all FMA warps done
        if (threadIdx.x == 128) stop = 1;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        tmem_free(tmem, 512);
    }
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 9 * 8);
    cudaMalloc(&sink, 4);
    void (*k[6])(unsigned long long*, float*) = {k_probe<0>, k_probe<1>, k_probe<2>,
                                                 k_probe<3>, k_probe<4>, k_probe<5>};
    for (int m = 0; m < 6; ++m) {
        cudaFuncSetAttribute(k[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        k[m]<<<148, 384, 65536>>>(d, sink);
        cudaDeviceSynchronize();
        unsigned long long h[148 * 9];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("mode %d (%s): FMA warp cycles by warp 4..11:", m,
               m % 3 == 0 ? "no MMA" : m % 3 == 1 ? "MMA per asm" : "8-MMA asm blocks");
        for (int w = 0; w < 8; ++w) printf(" %llu", h[w]);
        printf("  | err=%s\n", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
