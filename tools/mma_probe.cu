// mma_probe.cu -- microbenchmark of the tcgen05 shapes the attention kernel issues (1 CTA per SM):
// MMA dispatch rate for SS / TS forms at N = 128 / 256, tcgen05.ld read bandwidth alone and
// concurrently with MMAs. Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   -I paper_2509_13523_b200/csrc tools/mma_probe.cu -o tools/_mma_probe -lcuda
#include <cstdio>

#include "tc_ptx.cuh"

using namespace swf::tc;

constexpr int kIters = 8192;

// mode: 0 SS N128, 1 TS N128, 2 SS N256, 3 SS N128 + 4 warps tcgen05.ld, 4 tcgen05.ld only (4 warps),
//       5 tcgen05.ld only (8 warps), 6 SS N128 + 8 warps ld, 7 TS N256, 8 SS N64, 9 TS N64,
//       10 SS N128 + 4 warps st.shared stream, 11 TS N128 + 4 warps st.shared stream,
//       12-15 round-robin over 2 / 4 accumulators, 16 no accumulate
template <int mode>
__global__ void __launch_bounds__(384, 1) k_probe(unsigned long long* cyc, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tslot;
    const bool do_mma = mode != 4 && mode != 5;
    const int ld_warps = (mode == 3 || mode == 4) ? 4 : (mode == 5 || mode == 6) ? 8 : 0;
    if (warp == 1 && do_mma) {
        if ((threadIdx.x & 31) == 0) {
            const uint64_t a = desc_kmajor(smem_u32(sm), 128), b = desc_kmajor(smem_u32(sm + 32768), 128);
            const uint32_t idesc128 = idesc_bf16(128, 128), idesc256 = idesc_bf16(128, 256),
                           idesc64 = idesc_bf16(128, 64);
            const unsigned long long m0 = clock64();
#pragma unroll 16
            for (int i = 0; i < kIters; ++i) {
                if constexpr (mode == 1 || mode == 11)
                    mma_ts(tmem + 256, tmem, b, idesc128, 1);
                else if constexpr (mode == 2)
                    mma_ss(tmem + 256, a, b, idesc256, 1);
                else if constexpr (mode == 7)
                    mma_ts(tmem + 256, tmem, b, idesc256, 1);
                else if constexpr (mode == 8)
                    mma_ss(tmem + 256, a, b, idesc64, 1);
                else if constexpr (mode == 9)
                    mma_ts(tmem + 256, tmem, b, idesc64, 1);
                else if constexpr (mode == 12)
                    mma_ss(tmem + 256 + (i & 1) * 128, a, b, idesc128, 1);
                else if constexpr (mode == 13)
                    mma_ss(tmem + (i & 3) * 128, a, b, idesc128, 1);
                else if constexpr (mode == 14)
                    mma_ts(tmem + 256 + (i & 1) * 128, tmem, b, idesc128, 1);
                else if constexpr (mode == 15)
                    mma_ss(tmem + (i & 1) * 256, a, b, idesc256, 1);
                else if constexpr (mode == 16)
                    mma_ss(tmem + 256, a, b, idesc128, 0);
                else
                    mma_ss(tmem + 384, a, b, idesc128, 1);
            }
            commit(smem_u32(&bar));
            mbar_wait(smem_u32(&bar), 0);
            cyc[148 + blockIdx.x] = clock64() - m0;
        }
    } else if (warp >= 4 && warp - 4 < ld_warps) {
        const uint32_t lane_off = uint32_t(((warp - 4) & 3) * 32) << 16;
        const uint32_t col = uint32_t(((warp - 4) >> 2) * 128);
        float acc = 0.f;
        const int n = kIters / 8;
        const unsigned long long l0 = clock64();
        for (int i = 0; i < n; ++i) {
            uint32_t r[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) ld32(tmem + lane_off + col + uint32_t(c * 32), r + 32 * c);
#pragma unroll
            for (int c = 0; c < 4; ++c) wait_ld_dep(r + 32 * c);
#pragma unroll
            for (int k = 0; k < 128; ++k) acc += __uint_as_float(r[k]);
        }
        if (acc == 1.2345f) sink[0] = acc;
        if (threadIdx.x == 128) cyc[blockIdx.x] = clock64() - l0;
    } else if (warp >= 4 && warp < 8 && (mode == 10 || mode == 11)) {
        // shared-memory write stream into the upper 32 KB (what TMA fills compete with)
        uint4* dst = reinterpret_cast<uint4*>(sm + 32768 + 16384);
        const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (int i = 0; i < kIters * 2; ++i) dst[(threadIdx.x - 128 + i * 128) & 1023] = v;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        tmem_free(tmem, 512);
    }
}

int main() {
    unsigned long long* d_cyc;
    float* d_sink;
    cudaMalloc(&d_cyc, 2 * 148 * sizeof(unsigned long long));
    cudaMalloc(&d_sink, 4);
    void (*kern[17])(unsigned long long*, float*) = {k_probe<0>,  k_probe<1>,  k_probe<2>,  k_probe<3>,  k_probe<4>,
                                                     k_probe<5>,  k_probe<6>,  k_probe<7>,  k_probe<8>,  k_probe<9>,
                                                     k_probe<10>, k_probe<11>, k_probe<12>, k_probe<13>, k_probe<14>,
                                                     k_probe<15>, k_probe<16>};
    for (auto k : kern) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const char* names[] = {"SS M128 N128 K16", "TS M128 N128 K16", "SS M128 N256 K16", "SS N128 + 4w ld",
                           "ld only 4 warps", "ld only 8 warps", "SS N128 + 8w ld", "TS M128 N256 K16",
                           "SS M128 N64 K16", "TS M128 N64 K16", "SS N128 + STS", "TS N128 + STS",
                           "SS N128 2 accums", "SS N128 4 accums", "TS N128 2 accums", "SS N256 2 accums",
                           "SS N128 no-acc"};
    for (int mode = 0; mode < 17; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kern[mode]<<<148, 384, 65536 + 1024>>>(d_cyc, d_sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long h[296];
            cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
            const int nmma = (mode != 4 && mode != 5) ? kIters : 0;
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += double(h[(nmma ? 148 : 0) + i]) / 148;
            const int nn = (mode == 2 || mode == 7 || mode == 15) ? 256 : (mode == 8 || mode == 9) ? 64 : 128;
            const double macs = double(nmma) * 128 * nn * 16;
            const int ldw = (mode == 3 || mode == 4) ? 4 : (mode == 5 || mode == 6) ? 8 : 0;
            const double ldbytes = double(ldw) * (kIters / 8) * 32 * 128 * 4;
            printf("%-20s rep%d: %.3f ms, %.0f cyc/CTA, %.0f MAC/cyc/SM, %.1f cyc/MMA, TMEM ld %.1f B/cyc/SM%s\n",
                   names[mode], rep, ms, avg, macs / avg, nmma ? avg / nmma : 0.0, ldbytes / avg,
                   cudaGetLastError() == cudaSuccess ? "" : " (error)");
        }
    }
    return 0;
}
