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

// Windowed attention (swin.hpp:160-187) on 64-query tiles: 256 threads, K / V tiles of 64 keys
// staged in shared memory (row pitch d+1). Pass 1 computes each row's max m and sum l of
// exp(s - m) (online over key tiles); pass 2 accumulates O = sum_j (exp(s_j - m) / l) v_j in
// ascending key order, the reference's normalise-then-multiply order. Each thread owns a 4 x 4 block
// of the 64 x 64 score tile (rows ty*4+u, keys tx*4+v; a row group is one half-warp) and a
// 4 x ceil(d/16) block of the output tile (columns tx + 16*w). d <= 128.
constexpr int AT = 64, ADW = 8;

__device__ __forceinline__ float hw_max(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float hw_sum(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ void load_tile(float* dst, const float* src, int r0, int s, int d) {
    const int ld = d + 1;
    for (int idx = threadIdx.x; idx < AT * d; idx += blockDim.x) {
        const int r = idx / d, e = idx - (idx / d) * d;
        dst[r * ld + e] = r0 + r < s ? src[i64(r0 + r) * d + e] : 0.f;
    }
}

__global__ void __launch_bounds__(256) k_attn_f32(AttnParams p) {
    extern __shared__ float smf[];
    const int d = p.d, ld = d + 1, s = p.s;
    float *Qs = smf, *Ks = Qs + AT * ld, *Ps = Ks + AT * ld;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int head = blockIdx.y, lw = blockIdx.z, i0 = blockIdx.x * AT;
    const i64 base = (i64(lw) * p.heads + head) * s;
    const float* Q = reinterpret_cast<const float*>(p.q) + base * d;
    const float* Kp = reinterpret_cast<const float*>(p.k) + base * d;
    const float* Vp = reinterpret_cast<const float*>(p.v) + base * d;
    const int gw = p.lay.loc2glob[lw];
    const bool masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;  // window.hpp:60
    const int split = (p.w - p.lay.g.shift) * p.w;  // seam groups are [0,split) and [split,s)
    int gq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gq[u] = i0 + ty * 4 + u < split ? 0 : 1;
    load_tile(Qs, Q, i0, s, d);
    float mr[4], lr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) mr[u] = -INFINITY, lr[u] = 0.f;
    float o[4][ADW] = {};
    for (int pass = 0; pass < 2; ++pass)
        for (int j0 = 0; j0 < s; j0 += AT) {
            __syncthreads();
            load_tile(Ks, Kp, j0, s, d);
            __syncthreads();
            float acc[4][4] = {};
            for (int e = 0; e < d; ++e) {
                float a[4], b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = Qs[(ty * 4 + u) * ld + e], b[u] = Ks[(tx * 4 + u) * ld + e];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
            }
            float x[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int j = j0 + tx * 4 + v;
                    const bool ok = j < s && (!masked || (j < split ? 0 : 1) == gq[u]);
                    x[u][v] = ok ? acc[u][v] * p.scale : -INFINITY;
                }
            if (pass == 0) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float mn = fmaxf(mr[u], hw_max(fmaxf(fmaxf(x[u][0], x[u][1]), fmaxf(x[u][2], x[u][3]))));
                    float sum = 0.f;
#pragma unroll
                    for (int v = 0; v < 4; ++v) sum += x[u][v] == -INFINITY ? 0.f : expf(x[u][v] - mn);
                    sum = hw_sum(sum);
                    lr[u] = (mr[u] == -INFINITY ? 0.f : lr[u] * expf(mr[u] - mn)) + sum;
                    mr[u] = mn;
                }
                continue;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    Ps[(ty * 4 + u) * (AT + 1) + tx * 4 + v] =
                        x[u][v] == -INFINITY ? 0.f : expf(x[u][v] - mr[u]) / lr[u];
            __syncthreads();
            load_tile(Ks, Vp, j0, s, d);  // V tile over the K buffer
            __syncthreads();
            for (int c = 0; c < AT; ++c) {
                float vr[ADW];
#pragma unroll
                for (int w = 0; w < ADW; ++w) vr[w] = tx + 16 * w < d ? Ks[c * ld + tx + 16 * w] : 0.f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float pp = Ps[(ty * 4 + u) * (AT + 1) + c];
#pragma unroll
                    for (int w = 0; w < ADW; ++w) o[u][w] = fmaf(pp, vr[w], o[u][w]);
                }
            }
        }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty * 4 + u;
        if (i >= s) continue;
        float* O = reinterpret_cast<float*>(p.o) + (i64(lw) * s + i) * p.ldo + head * d;
#pragma unroll
        for (int w = 0; w < ADW; ++w)
            if (tx + 16 * w < d) O[tx + 16 * w] = o[u][w];
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

// The SIMT GEMM's epilogue applied to a product computed elsewhere (the tensor cores): C is the plain
// [M][ldc] fp32 product A . W^T with the same column layout (interleave G = 4 for SWIGLU).
template <int MODE>
__global__ void k_epi_rows(const float* __restrict__ Cm, int ldc, i64 M, int N, EpiParams ep) {
    const int nch = (N + 7) / 8;
    for (i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x; t < M * nch; t += i64(gridDim.x) * blockDim.x) {
        const i64 m = t / nch;
        const int nc = int(t - m * nch) * 8;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = nc + j < N ? Cm[m * ldc + nc + j] : 0.f;
        if constexpr (MODE == EPI_SWIGLU)
            epi_swiglu<float, 4>(ep, m, nc / 2, &v[0], &v[4]);
        else
            epi_apply<MODE, float, 8>(ep, m, nc, v);
    }
}
void epi_rows_f32(const float* Cm, int ldc, i64 M, int N, int mode, const EpiParams& ep, cudaStream_t st) {
    const i64 work = M * ((N + 7) / 8);
    const unsigned grid = unsigned(std::min<i64>((work + 255) / 256, 148 * 16));
    switch (mode) {
        case EPI_ENCODE: k_epi_rows<EPI_ENCODE><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        case EPI_QKV: k_epi_rows<EPI_QKV><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        case EPI_RESID: k_epi_rows<EPI_RESID><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        case EPI_SWIGLU: k_epi_rows<EPI_SWIGLU><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        case EPI_DOWN: k_epi_rows<EPI_DOWN><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        case EPI_DECODE: k_epi_rows<EPI_DECODE><<<grid, 256, 0, st>>>(Cm, ldc, M, N, ep); break;
        default: throw CudaError("epi_rows_f32: bad epilogue mode");
    }
    SWF_LAUNCH_CHECK();
}

void attention_f32(const AttnParams& p, cudaStream_t st) {
    if (p.d > 16 * ADW) throw CudaError("attention (FP32 mode): head dim must be <= 128");
    const size_t smem = (2 * size_t(AT) * (p.d + 1) + AT * (AT + 1)) * sizeof(float);
    dim3 grid(unsigned((p.s + AT - 1) / AT), unsigned(p.heads), unsigned(p.nloc));
    k_attn_f32<<<grid, 256, smem, st>>>(p);
    SWF_LAUNCH_CHECK();
}

void preload_simt_kernels() {
    cudaFuncAttributes a;
    const void* k[] = {(const void*)k_gemm_f32<EPI_ENCODE>, (const void*)k_gemm_f32<EPI_QKV>,
                       (const void*)k_gemm_f32<EPI_RESID>, (const void*)k_gemm_f32<EPI_SWIGLU>,
                       (const void*)k_gemm_f32<EPI_DOWN>, (const void*)k_gemm_f32<EPI_DECODE>,
                       (const void*)k_attn_f32, (const void*)k_epi_rows<EPI_ENCODE>, (const void*)k_epi_rows<EPI_QKV>,
                       (const void*)k_epi_rows<EPI_RESID>, (const void*)k_epi_rows<EPI_SWIGLU>,
                       (const void*)k_epi_rows<EPI_DOWN>, (const void*)k_epi_rows<EPI_DECODE>};
    for (const void* f : k) SWF_CUDA(cudaFuncGetAttributes(&a, f));
    int dev = 0, mx = 0;
    SWF_CUDA(cudaGetDevice(&dev));
    SWF_CUDA(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    SWF_CUDA(cudaFuncSetAttribute(k_attn_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
}

}  // namespace swf
