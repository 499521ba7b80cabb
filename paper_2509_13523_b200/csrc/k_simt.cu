// k_simt.cu -- FP32 validation mode: SIMT fp32 GEMM (all epilogues) and windowed attention.
// These exist so the GPU path can be checked against the oracle at <= 1e-4 (north_star);
// the throughput path is the BF16 tcgen05 path (k_gemm_tc.cu, k_attn.cu).
#include "epilogue.cuh"

namespace swf {

namespace {

constexpr int BM = 128, BN = 128, BK = 16;

template <int MODE>
__global__ void __launch_bounds__(256) k_gemm_f32(const float* __restrict__ A, const float* __restrict__ B, i64 M,
                                                  int N, int K, EpiParams ep) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const i64 m0 = i64(blockIdx.x) * BM;
    const int n0 = blockIdx.y * BN;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int idx = tid * 2 + q;  // 512 float4 per operand tile
            const int row = idx >> 2, c4 = idx & 3;
            float4 av = make_float4(0.f, 0.f, 0.f, 0.f), bv = av;
            if (m0 + row < M) av = *reinterpret_cast<const float4*>(A + (m0 + row) * K + k0 + c4 * 4);
            if (n0 + row < N) bv = *reinterpret_cast<const float4*>(B + i64(n0 + row) * K + k0 + c4 * 4);
            As[c4 * 4 + 0][row] = av.x;
            As[c4 * 4 + 1][row] = av.y;
            As[c4 * 4 + 2][row] = av.z;
            As[c4 * 4 + 3][row] = av.w;
            Bs[c4 * 4 + 0][row] = bv.x;
            Bs[c4 * 4 + 1][row] = bv.y;
            Bs[c4 * 4 + 2][row] = bv.z;
            Bs[c4 * 4 + 3][row] = bv.w;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[kk][ty * 8 + i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx * 8 + j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    const int nc = n0 + tx * 8;
    if (nc >= N) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const i64 m = m0 + ty * 8 + i;
        if constexpr (MODE == EPI_SWIGLU) {
            // interleave G = 4: columns [8t, 8t+4) gate, [8t+4, 8t+8) up of ffn units [4t, 4t+4)
            epi_swiglu<float, 4>(ep, m, nc / 2, &acc[i][0], &acc[i][4]);
        } else {
            epi_apply<MODE, float, 8>(ep, m, nc, acc[i]);
        }
    }
}

// One warp per query row: logits row, max-subtracted softmax normalised by the sum, then
// O = sum_j p_j v_j -- the reference's per-row order (swin.hpp:176-186).
__global__ void k_attn_f32(AttnParams p) {
    extern __shared__ float sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int s = p.s, d = p.d;
    float* prow = sm + warp * (s + d);
    float* qrow = prow + s;
    const int tok = blockIdx.x * nw + warp;
    const int head = blockIdx.y, lw = blockIdx.z;
    if (tok >= s) return;
    const i64 base = (i64(lw) * p.heads + head) * s;
    const float* Q = reinterpret_cast<const float*>(p.q) + base * d;
    const float* Kp = reinterpret_cast<const float*>(p.k) + base * d;
    const float* Vp = reinterpret_cast<const float*>(p.v) + base * d;
    for (int e = lane; e < d; e += 32) qrow[e] = Q[i64(tok) * d + e];
    __syncwarp();
    const int gw = p.lay.loc2glob[lw];
    const bool masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;  // window.hpp:60
    const int split = (p.w - p.lay.g.shift) * p.w;  // seam groups are [0,split) and [split,s)
    const int gq = tok < split ? 0 : 1;
    float mx = -INFINITY;
    for (int j = lane; j < s; j += 32) {
        const float* kr = Kp + i64(j) * d;
        float acc = 0.f;
        for (int e = 0; e < d; ++e) acc = fmaf(qrow[e], kr[e], acc);
        float l = acc * p.scale;
        if (masked && ((j < split ? 0 : 1) != gq)) l = -INFINITY;
        prow[j] = l;
        mx = fmaxf(mx, l);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < s; j += 32) {
        const float e = expf(prow[j] - mx);
        prow[j] = e;
        sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    for (int j = lane; j < s; j += 32) prow[j] = prow[j] / sum;
    __syncwarp();
    float* O = reinterpret_cast<float*>(p.o) + (i64(lw) * s + tok) * p.ldo + head * d;
    for (int e = lane; e < d; e += 32) {
        float acc = 0.f;
        for (int j = 0; j < s; ++j) acc = fmaf(Vp[i64(j) * d + e], prow[j], acc);
        O[e] = acc;
    }
}

}  // namespace

void gemm_f32(const float* A, const float* B, i64 M, int N, int K, int mode, const EpiParams& ep, cudaStream_t st) {
    if (K % BK != 0) throw CudaError("gemm_f32: K must be a multiple of 16");
    dim3 grid(unsigned((M + BM - 1) / BM), unsigned((N + BN - 1) / BN));
    switch (mode) {
        case EPI_ENCODE: k_gemm_f32<EPI_ENCODE><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        case EPI_QKV: k_gemm_f32<EPI_QKV><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        case EPI_RESID: k_gemm_f32<EPI_RESID><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        case EPI_SWIGLU: k_gemm_f32<EPI_SWIGLU><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        case EPI_DOWN: k_gemm_f32<EPI_DOWN><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        case EPI_DECODE: k_gemm_f32<EPI_DECODE><<<grid, 256, 0, st>>>(A, B, M, N, K, ep); break;
        default: throw CudaError("gemm_f32: bad epilogue mode");
    }
    SWF_LAUNCH_CHECK();
}

void attention_f32(const AttnParams& p, cudaStream_t st) {
    const int nw = 4;
    const size_t smem = size_t(nw) * (p.s + p.d) * sizeof(float);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        SWF_CUDA(cudaFuncSetAttribute(k_attn_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        configured = smem;
    }
    dim3 grid(unsigned((p.s + nw - 1) / nw), unsigned(p.heads), unsigned(p.nloc));
    k_attn_f32<<<grid, nw * 32, smem, st>>>(p);
    SWF_LAUNCH_CHECK();
}

}  // namespace swf
