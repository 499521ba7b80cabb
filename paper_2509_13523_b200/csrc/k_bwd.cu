// k_bwd.cu -- backward of the denoiser forward (swin.hpp:370-467), FP32 validation mode.
//
// The reference backward (block_window_backward, head_attention_bwd, swiglu_bwd,
// prenorm_modulate_bwd, prenorm_plain_bwd) restated as device kernels over the rank's local tokens:
//   * every weight gradient (accum_outer, swin.hpp:64-68) and input gradient (linear_cols_t,
//     :57-62) is one strided FP32 GEMM, C[i][j] (+)= sum_k A(i,k) B(k,j), so the reference's
//     column-major weight layout is used as is;
//   * the RMS-norm / AdaLN backward is split into a per-token pass (the input gradient, one warp per
//     token) and a per-channel pass (gain / AdaLN gradients summed over tokens in a fixed order:
//     results are deterministic, no atomics);
//   * attention backward recomputes P from q, k and the stored row statistics: a query-major pass
//     (dQ, and D_i = dO_i . O_i) and a key-major pass (dK, dV), then the inverse RoPE rotation.
// With swf_set_backward_precision(BF16) the linears' GEMMs run on the tensor cores instead
// (gemm_strided_tc: bf16 operands, fp32 accumulation).
#include <algorithm>
#include <vector>

#include "kernels.cuh"

namespace swf {

namespace {


// C[i][j] = beta * C[i][j] + sum_k A(i,k) B(k,j); A(i,k) = A[i*sai + k*sak], B(k,j) = B[k*sbk + j*sbj],
// C row stride ldc. 256 threads, 128 x 128 tile, 8 x 8 per thread (rows ty*4 + {0..3, 64..67},
// columns tx*4 + {0..3, 64..67}: two float4 shared-memory reads per operand per k), k slices of 8
// double-buffered in shared memory; each operand is loaded along its contiguous dimension.
constexpr int GB = 128, GK = 8;
__global__ void __launch_bounds__(256) k_gemm_strided(int M, int N, int K, const float* __restrict__ A, i64 sai,
                                                      i64 sak, const float* __restrict__ B, i64 sbk, i64 sbj,
                                                      float* __restrict__ C, i64 ldc, float beta) {
    __shared__ __align__(16) float As[2][GK][GB + 4], Bs[2][GK][GB + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int i0 = blockIdx.y * GB, j0 = blockIdx.x * GB;
    const bool a_k_fast = sak == 1, b_k_fast = sbk == 1;
    float ra[4], rb[4];  // this thread's 4 elements of each operand's next k slice
    auto fetch = [&](int k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = tid + 256 * u;  // 1024 elements = 128 rows x 8 k
            const int r = a_k_fast ? t / GK : t % GB, k = a_k_fast ? t % GK : t / GB;
            const int gi = i0 + r, gk = k0 + k;
            ra[u] = (gi < M && gk < K) ? A[gi * sai + gk * sak] : 0.f;
            const int c = b_k_fast ? t / GK : t % GB, kk = b_k_fast ? t % GK : t / GB;
            const int gj = j0 + c, gk2 = k0 + kk;
            rb[u] = (gj < N && gk2 < K) ? B[gk2 * sbk + gj * sbj] : 0.f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = tid + 256 * u;
            const int r = a_k_fast ? t / GK : t % GB, k = a_k_fast ? t % GK : t / GB;
            As[buf][k][r] = ra[u];
            const int c = b_k_fast ? t / GK : t % GB, kk = b_k_fast ? t % GK : t / GB;
            Bs[buf][kk][c] = rb[u];
        }
    };
    float acc[8][8] = {};
    fetch(0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += GK) {
        const bool more = k0 + GK < K;
        if (more) fetch(k0 + GK);  // global loads in flight during this slice's FMAs
#pragma unroll
        for (int k = 0; k < GK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
        }
        if (more) {
            stash(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int gi = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + u - 4);
        if (gi >= M) continue;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int gj = j0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + v - 4);
            if (gj >= N) continue;
            float* c = C + gi * ldc + gj;
            *c = beta == 0.f ? acc[u][v] : beta * *c + acc[u][v];
        }
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// per-token pass of prenorm_modulate_bwd / prenorm_plain_bwd (swin.hpp:86-107, 125-136):
// du = dxm .* gate .* (1 + a) .* g ; dx += du / r - x (x . du) / (h r^3); r = rms(x) written out.
// a / gate may be null (plain RMS norm).
__global__ void k_norm_bwd_rows(const float* __restrict__ X, int ldx, const float* __restrict__ dXM, int lddxm,
                                i64 M, int h, const float* __restrict__ g, const float* __restrict__ a,
                                const float* __restrict__ gate, float* __restrict__ dX, int lddx,
                                float* __restrict__ rms) {
    const i64 j = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= M) return;
    const float* x = X + j * ldx;
    const float* dxm = dXM + j * lddxm;
    float ss = 0.f, xdu = 0.f;
#pragma unroll 4
    for (int i = lane; i < h; i += 32) {
        ss = fmaf(x[i], x[i], ss);
        const float du = dxm[i] * (gate ? gate[i] : 1.f) * (a ? 1.f + a[i] : 1.f) * g[i];
        xdu = fmaf(x[i], du, xdu);
    }
    ss = warp_sum(ss);
    xdu = warp_sum(xdu);
    const float r = sqrtf(ss / float(h) + 1e-8f);
    const float c = xdu / (float(h) * r * r * r);
    float* dx = dX + j * lddx;
#pragma unroll 4
    for (int i = lane; i < h; i += 32) {
        const float du = dxm[i] * (gate ? gate[i] : 1.f) * (a ? 1.f + a[i] : 1.f) * g[i];
        dx[i] += du / r - x[i] * c;
    }
    if (lane == 0) rms[j] = r;
}

// per-channel pass: dg[i] += sum_j dxm gate (1+a) u ; da[i] += sum_j dxm gate g u ; db[i] += sum_j dxm gate ;
// dgate[i] += sum_j dxm (g u (1+a) + b), u = x / r. One thread per (channel, token slice): slice sl of
// S sums its tokens in order into part[sl][4][h]; k_norm_bwd_cols_sum adds the slices in order (a fixed
// order for given M, h: deterministic, no atomics).
__global__ void k_norm_bwd_cols(const float* __restrict__ X, int ldx, const float* __restrict__ dXM, int lddxm,
                                const float* __restrict__ rms, i64 M, int h, const float* __restrict__ g,
                                const float* __restrict__ a, const float* __restrict__ b,
                                const float* __restrict__ gate, int S, float* __restrict__ part) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int sl = blockIdx.y;
    if (i >= h) return;
    const float gi = g[i], ai = a ? a[i] : 0.f, bi = b ? b[i] : 0.f, qi = gate ? gate[i] : 1.f;
    float sg = 0.f, sa = 0.f, sb = 0.f, sq = 0.f;
    const i64 j1 = M * (sl + 1) / S;
    auto acc = [&](float xv, float r, float dxm) {
        const float u = xv / r;
        const float gu = gi * u;
        sa = fmaf(dxm * qi, gu, sa);
        sb = fmaf(dxm, qi, sb);
        sq = fmaf(dxm, gu * (1.f + ai) + bi, sq);
        sg = fmaf(dxm * qi * (1.f + ai), u, sg);
    };
    i64 j = M * sl / S;
    for (; j + 4 <= j1; j += 4) {  // 4 tokens' loads in flight, accumulated in token order
        float xv[4], r[4], dv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            xv[e] = X[(j + e) * ldx + i];
            r[e] = rms[j + e];
            dv[e] = dXM[(j + e) * lddxm + i];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) acc(xv[e], r[e], dv[e]);
    }
    for (; j < j1; ++j) acc(X[j * ldx + i], rms[j], dXM[j * lddxm + i]);
    float* pt = part + size_t(sl) * 4 * h;
    pt[i] = sg;
    pt[h + i] = sa;
    pt[2 * h + i] = sb;
    pt[3 * h + i] = sq;
}
__global__ void k_norm_bwd_cols_sum(const float* __restrict__ part, int S, int h, float* __restrict__ dg,
                                    float* __restrict__ da, float* __restrict__ db, float* __restrict__ dgate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h) return;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int sl = 0; sl < S; ++sl)
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] += part[(size_t(sl) * 4 + q) * h + i];
    dg[i] += s[0];
    if (da) da[i] += s[1];
    if (db) db[i] += s[2];
    if (dgate) dgate[i] += s[3];
}

// column sums (bias gradients): out[i] += sum_j X[j][i]. One thread per (column, token slice) into
// part[sl][n], then the slices added in order (deterministic; one thread per column over all M rows
// had left 1-12 blocks for 148 SMs: 6.9 ms per call at 240x480)
__global__ void k_colsum(const float* __restrict__ X, int ldx, i64 M, int n, int S, float* __restrict__ part) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int sl = blockIdx.y;
    if (i >= n) return;
    float s = 0.f;
    const i64 j1 = M * (sl + 1) / S;
    i64 j = M * sl / S;
    for (; j + 4 <= j1; j += 4) {  // 4 loads in flight, summed in token order
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = X[(j + e) * ldx + i];
#pragma unroll
        for (int e = 0; e < 4; ++e) s += v[e];
    }
    for (; j < j1; ++j) s += X[j * ldx + i];
    part[size_t(sl) * n + i] = s;
}
__global__ void k_colsum_sum(const float* __restrict__ part, int S, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float s = 0.f;
    for (int sl = 0; sl < S; ++sl) s += part[size_t(sl) * n + i];
    out[i] += s;
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.f + expf(-x)); }
__device__ __forceinline__ float silu_grad_f(float x) {  // model.hpp:248-252
    const float s = 1.f / (1.f + expf(-x));
    return s * (1.f + x * (1.f - s));
}

// SwiGLU backward elementwise (swin.hpp:236-252) from the interleaved gate/up pre-activations
// (G-unit groups [gate G | up G]): act = silu(gp) up ; dG = dS up silu'(gp) ; dU = dS silu(gp).
__global__ void k_swiglu_bwd(const float* __restrict__ gu, int ldgu, const float* __restrict__ dS, int ldds,
                             i64 M, int f, int G, float* __restrict__ act, float* __restrict__ dG,
                             float* __restrict__ dU) {
    const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= M * f) return;
    const i64 j = t / f;
    const int o = int(t - j * f);
    const int col = (o / G) * 2 * G + (o % G);
    const float gp = gu[j * ldgu + col], up = gu[j * ldgu + col + G];
    const float sg = silu_f(gp);
    act[t] = sg * up;
    if (dS) {
        const float ds = dS[j * ldds + o];
        dG[t] = ds * up * silu_grad_f(gp);
        dU[t] = ds * sg;
    }
}

// The same, 4 consecutive units per thread (G % 4 == 0, f % 4 == 0, 16-byte rows): 16-byte accesses and
// the group / row arithmetic once per 4 units, rows strided over grid.y (was 64-bit div / mod per unit)
__global__ void k_swiglu_bwd4(const float* __restrict__ gu, int ldgu, const float* __restrict__ dS, int ldds,
                              i64 M, int f, int G, float* __restrict__ act, float* __restrict__ dG,
                              float* __restrict__ dU) {
    const int o = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (o >= f) return;
    const int col = (o / G) * 2 * G + (o % G);
    for (i64 j = blockIdx.y; j < M; j += gridDim.y) {
        const float4 gp = *reinterpret_cast<const float4*>(gu + j * ldgu + col);
        const float4 up = *reinterpret_cast<const float4*>(gu + j * ldgu + col + G);
        const float g[4] = {gp.x, gp.y, gp.z, gp.w}, u[4] = {up.x, up.y, up.z, up.w};
        float a[4], dg[4], du[4], ds[4] = {0.f, 0.f, 0.f, 0.f};
        if (dS) {
            const float4 d4 = *reinterpret_cast<const float4*>(dS + j * ldds + o);
            ds[0] = d4.x, ds[1] = d4.y, ds[2] = d4.z, ds[3] = d4.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float sg = silu_f(g[e]);
            a[e] = sg * u[e];
            dg[e] = ds[e] * u[e] * silu_grad_f(g[e]);
            du[e] = ds[e] * sg;
        }
        const i64 t = j * f + o;
        *reinterpret_cast<float4*>(act + t) = make_float4(a[0], a[1], a[2], a[3]);
        if (dS) {
            *reinterpret_cast<float4*>(dG + t) = make_float4(dg[0], dg[1], dg[2], dg[3]);
            *reinterpret_cast<float4*>(dU + t) = make_float4(du[0], du[1], du[2], du[3]);
        }
    }
}

// rows of src (layout A order) gathered into layout B order: dst[i] = src[A.pix_to_loc(B.loc_to_pix(i))]
__global__ void k_relayout(const float* __restrict__ src, LayMap A, LayMap B, i64 M, int h, float* __restrict__ dst) {
    const i64 i = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= M) return;
    int rk;
    const i64 j = A.pix_to_loc(B.loc_to_pix(i), &rk);
    for (int e = lane; e < h; e += 32) dst[i * h + e] = src[j * h + e];
}

// window parallelism: push row i of layout A (this rank's rows) to its owner under layout B,
// dst[rank] = that rank's landing buffer (CUDA-IPC mapped), one warp per row
__global__ void k_relayout_push(const float* __restrict__ src, LayMap A, LayMap B, i64 M, int h,
                                float* const* __restrict__ dst) {
    const i64 i = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= M) return;
    int rk;
    const i64 j = B.pix_to_loc(A.loc_to_pix(i), &rk);
    float* d = dst[rk] + j * h;
    for (int e = lane; e < h; e += 32) d[e] = src[i * h + e];
}

// ---- attention backward (head_attention_bwd, swin.hpp:189-226), planes [nloc][heads][s][d],
// O / dO rows [lw*s + tok][ldo] (head-concatenated), one thread per query (pass 1) or key (pass 2).
struct AttnBwd {
    const float *q, *k, *v, *o, *dO;
    float *dq, *dk, *dv;  // planes
    float *m, *l, *D;     // [nloc][heads][s] row statistics
    int ldo, nloc, heads, s, d, w;
    float scale;
    LayMap lay;
};
__device__ __forceinline__ void seam(const AttnBwd& p, int lw, int& split, bool& masked) {
    const int gw = p.lay.loc2glob[lw];
    masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;  // window.hpp:60
    split = (p.w - p.lay.g.shift) * p.w;
}
// Tiled flash-style backward (FP32 SIMT): 64-token tiles staged in shared memory with a padded row
// pitch d+1, 256 threads, each owning a 4 x 4 block of the 64 x 64 score tile (rows ty*4+u, columns
// tx*4+v; the 16 threads of a row group are one half-warp, so row reductions are shuffles) and a
// 4 x ceil(d/16) block of the 64 x d output tile (columns tx + 16*w). d <= 128.
constexpr int AT = 64, ADW = 8;  // tile, output columns per thread (d / 16)

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
// rows [r0, r0+64) of a plane ([s][d], row pitch d) or of O / dO ([token][ldo] at column off) into smem
__device__ __forceinline__ void load_tile(float* dst, const float* src, i64 pitch, int r0, int s, int d) {
    const int ld = d + 1;
    for (int idx = threadIdx.x; idx < AT * d; idx += blockDim.x) {
        const int r = idx / d, e = idx - (idx / d) * d;
        dst[r * ld + e] = r0 + r < s ? src[i64(r0 + r) * pitch + e] : 0.f;
    }
}

// pass 1 (query tiles): row statistics m, l (online over key tiles), D = dO . O, and dQ
__global__ void __launch_bounds__(256) k_attn_bwd_q(AttnBwd p) {
    extern __shared__ float smf[];
    const int d = p.d, ld = d + 1, s = p.s;
    float *Qs = smf, *dOs = Qs + AT * ld, *Ks = dOs + AT * ld, *Vs = Ks + AT * ld, *Ss = Vs + AT * ld;
    float* Dr = Ss + AT * (AT + 1);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4, warp = tid >> 5, lane = tid & 31;
    const int head = blockIdx.y, lw = blockIdx.z, i0 = blockIdx.x * AT;
    const i64 base = (i64(lw) * p.heads + head) * s;
    int split;
    bool masked;
    seam(p, lw, split, masked);
    load_tile(Qs, p.q + base * d, d, i0, s, d);
    load_tile(dOs, p.dO + i64(lw) * s * p.ldo + head * d, p.ldo, i0, s, d);
    __syncthreads();
    for (int r = warp; r < AT; r += 8) {  // D_i = dO_i . O_i
        float acc = 0.f;
        if (i0 + r < s) {
            const float* o = p.o + (i64(lw) * s + i0 + r) * p.ldo + head * d;
            for (int e = lane; e < d; e += 32) acc = fmaf(dOs[r * ld + e], o[e], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) Dr[r] = acc;
    }
    int gq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gq[u] = i0 + ty * 4 + u < split ? 0 : 1;
    float mr[4], lr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) mr[u] = -INFINITY, lr[u] = 0.f;
    __syncthreads();
    for (int j0 = 0; j0 < s; j0 += AT) {  // statistics
        load_tile(Ks, p.k + base * d, d, j0, s, d);
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
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float x[4], tm = -INFINITY;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int j = j0 + tx * 4 + v;
                const bool ok = j < s && (!masked || (j < split ? 0 : 1) == gq[u]);
                x[v] = ok ? acc[u][v] * p.scale : -INFINITY;
                tm = fmaxf(tm, x[v]);
            }
            const float mn = fmaxf(mr[u], hw_max(tm));
            float sum = 0.f;
#pragma unroll
            for (int v = 0; v < 4; ++v) sum += x[v] == -INFINITY ? 0.f : expf(x[v] - mn);
            sum = hw_sum(sum);
            lr[u] = (mr[u] == -INFINITY ? 0.f : lr[u] * expf(mr[u] - mn)) + sum;
            mr[u] = mn;
        }
        __syncthreads();
    }
    float dq[4][ADW] = {};
    for (int j0 = 0; j0 < s; j0 += AT) {  // dQ = sum_j dS_ij k_j
        load_tile(Ks, p.k + base * d, d, j0, s, d);
        load_tile(Vs, p.v + base * d, d, j0, s, d);
        __syncthreads();
        float acc[4][4] = {}, dp[4][4] = {};
        for (int e = 0; e < d; ++e) {
            float a[4], b[4], g[4], h[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = Qs[(ty * 4 + u) * ld + e], g[u] = dOs[(ty * 4 + u) * ld + e];
                b[u] = Ks[(tx * 4 + u) * ld + e], h[u] = Vs[(tx * 4 + u) * ld + e];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]), dp[u][v] = fmaf(g[u], h[v], dp[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int r = ty * 4 + u, j = j0 + tx * 4 + v;
                const bool ok = j < s && (!masked || (j < split ? 0 : 1) == gq[u]);
                const float pij = ok ? expf(acc[u][v] * p.scale - mr[u]) / lr[u] : 0.f;
                Ss[r * (AT + 1) + tx * 4 + v] = pij * (dp[u][v] - Dr[r]) * p.scale;
            }
        __syncthreads();
        for (int c = 0; c < AT; ++c) {
            float kr[ADW];
#pragma unroll
            for (int w = 0; w < ADW; ++w) kr[w] = tx + 16 * w < d ? Ks[c * ld + tx + 16 * w] : 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float ds = Ss[(ty * 4 + u) * (AT + 1) + c];
#pragma unroll
                for (int w = 0; w < ADW; ++w) dq[u][w] = fmaf(ds, kr[w], dq[u][w]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty * 4 + u;
        if (i >= s) continue;
#pragma unroll
        for (int w = 0; w < ADW; ++w)
            if (tx + 16 * w < d) p.dq[(base + i) * d + tx + 16 * w] = dq[u][w];
        if (tx == 0) {
            p.m[base + i] = mr[u];
            p.l[base + i] = lr[u];
            p.D[base + i] = Dr[ty * 4 + u];
        }
    }
}

// pass 2 (key tiles): dV = sum_i P_ij dO_i, dK = sum_i dS_ij q_i
__global__ void __launch_bounds__(256) k_attn_bwd_kv(AttnBwd p) {
    extern __shared__ float smf[];
    const int d = p.d, ld = d + 1, s = p.s;
    float *Ks = smf, *Vs = Ks + AT * ld, *Qs = Vs + AT * ld, *dOs = Qs + AT * ld, *Ps = dOs + AT * ld;
    float *dSs = Ps + AT * (AT + 1), *Mq = dSs + AT * (AT + 1), *Lq = Mq + AT, *Dq = Lq + AT;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int head = blockIdx.y, lw = blockIdx.z, j0 = blockIdx.x * AT;
    const i64 base = (i64(lw) * p.heads + head) * s;
    int split;
    bool masked;
    seam(p, lw, split, masked);
    load_tile(Ks, p.k + base * d, d, j0, s, d);
    load_tile(Vs, p.v + base * d, d, j0, s, d);
    int gk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gk[u] = j0 + ty * 4 + u < split ? 0 : 1;
    float dk[4][ADW] = {}, dv[4][ADW] = {};
    for (int i0 = 0; i0 < s; i0 += AT) {
        load_tile(Qs, p.q + base * d, d, i0, s, d);
        load_tile(dOs, p.dO + i64(lw) * s * p.ldo + head * d, p.ldo, i0, s, d);
        for (int r = tid; r < AT; r += blockDim.x) {
            const bool in = i0 + r < s;
            Mq[r] = in ? p.m[base + i0 + r] : 0.f;
            Lq[r] = in ? p.l[base + i0 + r] : 1.f;
            Dq[r] = in ? p.D[base + i0 + r] : 0.f;
        }
        __syncthreads();
        float acc[4][4] = {}, dp[4][4] = {};  // rows: keys ty*4+u, columns: queries tx*4+v
        for (int e = 0; e < d; ++e) {
            float a[4], b[4], g[4], h[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = Ks[(ty * 4 + u) * ld + e], g[u] = Vs[(ty * 4 + u) * ld + e];
                b[u] = Qs[(tx * 4 + u) * ld + e], h[u] = dOs[(tx * 4 + u) * ld + e];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]), dp[u][v] = fmaf(g[u], h[v], dp[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int c = tx * 4 + v, i = i0 + c;
                const bool ok = i < s && j0 + ty * 4 + u < s && (!masked || (i < split ? 0 : 1) == gk[u]);
                const float pij = ok ? expf(acc[u][v] * p.scale - Mq[c]) / Lq[c] : 0.f;
                Ps[(ty * 4 + u) * (AT + 1) + c] = pij;
                dSs[(ty * 4 + u) * (AT + 1) + c] = pij * (dp[u][v] - Dq[c]) * p.scale;
            }
        __syncthreads();
        for (int c = 0; c < AT; ++c) {
            float qr[ADW], gr[ADW];
#pragma unroll
            for (int w = 0; w < ADW; ++w) {
                const bool in = tx + 16 * w < d;
                qr[w] = in ? Qs[c * ld + tx + 16 * w] : 0.f;
                gr[w] = in ? dOs[c * ld + tx + 16 * w] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float pp = Ps[(ty * 4 + u) * (AT + 1) + c], ds = dSs[(ty * 4 + u) * (AT + 1) + c];
#pragma unroll
                for (int w = 0; w < ADW; ++w) dv[u][w] = fmaf(pp, gr[w], dv[u][w]), dk[u][w] = fmaf(ds, qr[w], dk[u][w]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int j = j0 + ty * 4 + u;
        if (j >= s) continue;
#pragma unroll
        for (int w = 0; w < ADW; ++w)
            if (tx + 16 * w < d) {
                p.dk[(base + j) * d + tx + 16 * w] = dk[u][w];
                p.dv[(base + j) * d + tx + 16 * w] = dv[u][w];
            }
    }
}
// dQ, dK, dV planes -> dqkv token rows [lw*s + tok][3h] (rows [q; k; v], head-major), with the
// inverse RoPE rotation (rope_rotate(..., inverse=true)) on dQ and dK.
__global__ void k_attn_bwd_pack(const float* __restrict__ dq, const float* __restrict__ dk,
                                const float* __restrict__ dv, EpiParams ep, int nloc, float* __restrict__ dqkv) {
    const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;  // (token, pair) over all heads
    const int h = ep.h, d = ep.d, s = ep.cur.g.w * ep.cur.g.w;
    const i64 M = i64(nloc) * s;
    if (t >= M * (h / 2)) return;
    const i64 m = t / (h / 2);
    const int pr = int(t - m * (h / 2));
    const int head = (2 * pr) / d, dd = (2 * pr) % d;
    int gw, tok, lw;
    ep.cur.loc_to_wtok(m, gw, tok, lw);
    const int wy = gw / ep.cur.g.nx, wx = gw - (gw / ep.cur.g.nx) * ep.cur.g.nx, w = ep.cur.g.w;
    const int prow = wy * w + ep.cur.g.shift + tok / w, pcol = wx * w + ep.cur.g.shift + tok % w;
    const i64 src = ((i64(lw) * ep.heads + head) * s + tok) * d + dd;
    float* row = dqkv + m * 3 * h;
    const int q4 = d >> 2, j = dd >> 1;
    const float2 cs = j < q4 ? ep.rope_row[j * ep.rope_nrow + prow] : ep.rope_col[(j - q4) * ep.rope_ncol + pcol];
    for (int which = 0; which < 2; ++which) {  // rotate by -angle
        const float* P = which == 0 ? dq : dk;
        const float x = P[src], y = P[src + 1];
        row[which * h + head * d + dd] = cs.x * x + cs.y * y;
        row[which * h + head * d + dd + 1] = -cs.y * x + cs.x * y;
    }
    row[2 * h + head * d + dd] = dv[src];
    row[2 * h + head * d + dd + 1] = dv[src + 1];
}

// time embedding / AdaLN tails (model.hpp:261-269, swin.hpp:28-41, 458-465), one thread per output:
// gW_ada[k][o] += d6[o] emb[k] (W_ada 6h x td column-major), gb_ada += d6, d_emb[k] += W_ada(:,k) . d6
__global__ void k_ada_bwd(const float* __restrict__ d6, const float* __restrict__ emb, const float* __restrict__ Wa,
                          int n6, int td, float* __restrict__ gWa, float* __restrict__ gba, float* __restrict__ demb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n6 * td) {
        const int k = t / n6, o = t % n6;
        gWa[t] += d6[o] * emb[k];
    }
    if (t < n6) gba[t] += d6[t];
    if (t < td) {
        float s = 0.f;
        for (int o = 0; o < n6; ++o) s = fmaf(Wa[i64(t) * n6 + o], d6[o], s);
        demb[t] += s;
    }
}
// embed = silu(lin), lin = W_time feat + b_time: gW_time[k][o] += dlin[o] feat[k], gb_time += dlin
__global__ void k_time_bwd(const float* __restrict__ demb, const float* __restrict__ feat,
                           const float* __restrict__ Wt, const float* __restrict__ bt, int td, float* __restrict__ gWt,
                           float* __restrict__ gbt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= td * td) return;
    const int k = t / td, o = t % td;
    float lin = bt[o];
    for (int kk = 0; kk < td; ++kk) lin = fmaf(Wt[i64(kk) * td + o], feat[kk], lin);
    const float dl = demb[o] * silu_grad_f(lin);
    gWt[t] += dl * feat[k];
    if (k == 0) gbt[o] += dl;
}


// ---- diffusion training loss (diffusion.hpp:57-67, 111-133, 168-192)
// x_t = c x0 + s z (interpolate), v = c z - s x0 (velocity_target)
__global__ void k_train_prep(const float* __restrict__ x0, const float* __restrict__ z, i64 n, float cs, float sn,
                             float* __restrict__ xt, float* __restrict__ v) {
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += i64(gridDim.x) * blockDim.x) {
        const float a = x0[e], b = z[e];
        xt[e] = cs * a + sn * b;
        v[e] = cs * b - sn * a;
    }
}

// err = sd f - v; loss terms alpha(row) kappa(c) err^2 summed per block in double (fixed grid, fixed
// order: deterministic); dS = sd * 2 alpha kappa err / N (weighted_sq_loss_grad scaled by sigma_d).
__global__ void __launch_bounds__(256) k_train_loss(const float* __restrict__ f, const float* __restrict__ v,
                                                    LayMap lay, i64 M, int C, const float* __restrict__ kappa,
                                                    const float* __restrict__ alpha_row, float sd, float g_scale,
                                                    float* __restrict__ dS, double* __restrict__ part) {
    __shared__ double red[256];
    double acc = 0.0;
    const i64 total = M * C;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e / C;
        const int ch = int(e - i * C);
        const float alpha = alpha_row[lay.loc_to_pix(i) / lay.g.W];
        const float err = sd * f[e] - v[e];
        const float ak = alpha * kappa[ch];
        acc += double(ak) * double(err) * double(err);
        dS[e] = sd * (g_scale * ak * err);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_axpy(const float* __restrict__ x, i64 n, float a, float* __restrict__ y) {
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += i64(gridDim.x) * blockDim.x)
        y[e] += a * x[e];
}

}  // namespace

void gemm_strided_f32(int M, int N, int K, const float* A, i64 sai, i64 sak, const float* B, i64 sbk, i64 sbj,
                      float* C, i64 ldc, float beta, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    dim3 grid(unsigned((N + GB - 1) / GB), unsigned((M + GB - 1) / GB));
    k_gemm_strided<<<grid, 256, 0, st>>>(M, N, K, A, sai, sak, B, sbk, sbj, C, ldc, beta);
    SWF_LAUNCH_CHECK();
}
__global__ void k_to_bf16(const float* __restrict__ x, i64 n, __nv_bfloat16* __restrict__ y) {
    const i64 n4 = n >> 2;
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += i64(gridDim.x) * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        reinterpret_cast<uint2*>(y)[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    }
    for (i64 i = 4 * n4 + i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}
void to_bf16(const float* x, i64 n, __nv_bfloat16* y, cudaStream_t st) {
    if (n <= 0) return;
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) throw CudaError("to_bf16: source must be 16-byte aligned");
    const i64 blocks = std::min<i64>((n / 4 + 255) / 256 + 1, 148 * 16);
    k_to_bf16<<<unsigned(blocks), 256, 0, st>>>(x, n, y);
    SWF_LAUNCH_CHECK();
}
__global__ void k_to_f32(const __nv_bfloat16* __restrict__ x, i64 n, float* __restrict__ y) {
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
        y[i] = __bfloat162float(x[i]);
}
void to_f32(const __nv_bfloat16* x, i64 n, float* y, cudaStream_t st) {
    if (n <= 0) return;
    k_to_f32<<<unsigned(std::min<i64>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(x, n, y);
    SWF_LAUNCH_CHECK();
}
// V planes [planes][s][d] fp32 -> V^T planes [planes][d][s] bf16 (the tensor-core attention's P V
// operand), 32 x 32 tiles through shared memory
__global__ void k_vt_bf16(const float* __restrict__ v, int s, int d, __nv_bfloat16* __restrict__ vt) {
    __shared__ float t[32][33];
    const i64 pl = blockIdx.z;
    const int s0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    const float* src = v + pl * s * d;
    __nv_bfloat16* dst = vt + pl * s * d;
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
        t[r][threadIdx.x] = (s0 + r < s && d0 + int(threadIdx.x) < d) ? src[i64(s0 + r) * d + d0 + threadIdx.x] : 0.f;
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
        if (d0 + r < d && s0 + int(threadIdx.x) < s)
            dst[i64(d0 + r) * s + s0 + threadIdx.x] = __float2bfloat16_rn(t[threadIdx.x][r]);
}
void vt_bf16(const float* v, i64 planes, int s, int d, __nv_bfloat16* vt, cudaStream_t st) {
    dim3 grid(unsigned((s + 31) / 32), unsigned((d + 31) / 32), unsigned(planes));
    k_vt_bf16<<<grid, dim3(32, 8), 0, st>>>(v, s, d, vt);
    SWF_LAUNCH_CHECK();
}
// gemm_strided_f32's product on the tensor cores: the FP32 operands are rounded to bf16 copies in ta /
// tb (same layout) and multiplied by one tcgen05 GEMM with FP32 accumulation. The backward's linears
// take this path when it runs in BF16 (swf_set_backward_precision): data gradients with both operands
// K-major, weight gradients (K = tokens) with both MN-major, straight from the row-major activations.
// rows x cols of a row-major fp32 matrix (pitch ld) into bf16 rows of pitch ldo (ldo >= cols; the
// pad columns are zeroed)
__global__ void k_to_bf16_2d(const float* __restrict__ x, i64 rows, int cols, i64 ld, __nv_bfloat16* __restrict__ y,
                             int ldo) {
    const i64 n = rows * ldo;
    for (i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += i64(gridDim.x) * blockDim.x) {
        const i64 r = t / ldo;
        const int c = int(t - r * ldo);
        y[t] = __float2bfloat16_rn(c < cols ? x[r * ld + c] : 0.f);
    }
}
void gemm_strided_tc(int M, int N, int K, const float* A, i64 sai, i64 sak, const float* B, i64 sbk, i64 sbj, float* C,
                     i64 ldc, float beta, __nv_bfloat16* ta, __nv_bfloat16* tb, int* sched, cudaStream_t st) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    const bool a_mn = sai == 1 && sak != 1, b_mn = sbj == 1 && sbk != 1;
    const i64 lda = a_mn ? sak : sai, ldb = b_mn ? sbk : sbj;
    // the bf16 copies keep the layout; pitches rounded up to 8 elements (16-byte TMA rows)
    auto conv = [&](const float* x, i64 rows, int cols, i64 ld, __nv_bfloat16* y) -> i64 {
        const i64 ldo = (ld % 8 == 0) ? ld : (cols + 7) / 8 * 8;
        if (ldo == ld) {
            to_bf16(x, rows * ld, y, st);
        } else {
            const i64 n = rows * ldo;
            k_to_bf16_2d<<<unsigned(std::min<i64>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(x, rows, cols, ld, y,
                                                                                              int(ldo));
            SWF_LAUNCH_CHECK();
        }
        return ldo;
    };
    const i64 pa = a_mn ? conv(A, K, M, lda, ta) : conv(A, M, K, lda, ta);
    const i64 pb = b_mn ? conv(B, K, N, ldb, tb) : conv(B, N, K, ldb, tb);
    gemm_bf16_general(ta, a_mn, pa, tb, b_mn, pb, M, N, K, C, ldc, beta != 0.f, sched, st);
}
void norm_bwd(const float* X, int ldx, const float* dXM, int lddxm, i64 M, int h, const float* g, const float* a,
              const float* b, const float* gate, float* dX, int lddx, float* rms, float* dg, float* da, float* db,
              float* dgate, float* part, cudaStream_t st) {
    k_norm_bwd_rows<<<unsigned((M + 7) / 8), 256, 0, st>>>(X, ldx, dXM, lddxm, M, h, g, a, gate, dX, lddx, rms);
    SWF_LAUNCH_CHECK();
    const int cb = (h + 127) / 128;  // channel blocks; token slices fill ~4 waves, >= 64 tokens each
    const int S = int(std::max<i64>(1, std::min<i64>({i64(kNormSlices), (M + 63) / 64, i64(148 * 4 / cb + 1)})));
    k_norm_bwd_cols<<<dim3(unsigned(cb), unsigned(S)), 128, 0, st>>>(X, ldx, dXM, lddxm, rms, M, h, g, a, b, gate, S,
                                                                     part);
    SWF_LAUNCH_CHECK();
    k_norm_bwd_cols_sum<<<unsigned(cb), 128, 0, st>>>(part, S, h, dg, da, db, dgate);
    SWF_LAUNCH_CHECK();
}
void colsum_f32(const float* X, int ldx, i64 M, int n, float* out, float* part, cudaStream_t st) {
    const int cb = (n + 127) / 128;
    const int S = int(std::max<i64>(1, std::min<i64>({i64(kNormSlices), (M + 63) / 64, i64(148 * 4 / cb + 1)})));
    k_colsum<<<dim3(unsigned(cb), unsigned(S)), 128, 0, st>>>(X, ldx, M, n, S, part);
    SWF_LAUNCH_CHECK();
    k_colsum_sum<<<unsigned(cb), 128, 0, st>>>(part, S, n, out);
    SWF_LAUNCH_CHECK();
}
void swiglu_bwd(const float* gu, int ldgu, const float* dS, int ldds, i64 M, int f, int G, float* act, float* dG,
                float* dU, cudaStream_t st) {
    const i64 n = M * f;
    const bool v4 = G % 4 == 0 && f % 4 == 0 && ldgu % 4 == 0 && ldds % 4 == 0 &&
                    ((reinterpret_cast<uintptr_t>(gu) | reinterpret_cast<uintptr_t>(dS) |
                      reinterpret_cast<uintptr_t>(act) | reinterpret_cast<uintptr_t>(dG) |
                      reinterpret_cast<uintptr_t>(dU)) & 15) == 0;
    if (v4) {
        const dim3 grid(unsigned((f / 4 + 255) / 256), unsigned(std::min<i64>(M, 2048)));
        k_swiglu_bwd4<<<grid, 256, 0, st>>>(gu, ldgu, dS, ldds, M, f, G, act, dG, dU);
    } else {
        k_swiglu_bwd<<<unsigned((n + 255) / 256), 256, 0, st>>>(gu, ldgu, dS, ldds, M, f, G, act, dG, dU);
    }
    SWF_LAUNCH_CHECK();
}
void relayout_rows(const float* src, const LayMap& A, const LayMap& B, i64 M, int h, float* dst, cudaStream_t st) {
    k_relayout<<<unsigned((M + 7) / 8), 256, 0, st>>>(src, A, B, M, h, dst);
    SWF_LAUNCH_CHECK();
}
void relayout_push(const float* src, const LayMap& A, const LayMap& B, i64 M, int h, float* const* dst,
                   cudaStream_t st) {
    k_relayout_push<<<unsigned((M + 7) / 8), 256, 0, st>>>(src, A, B, M, h, dst);
    SWF_LAUNCH_CHECK();
}
void attention_bwd_f32(const float* q, const float* k, const float* v, const float* o, const float* dO, int ldo,
                       float* dq, float* dk, float* dv, float* stats, int nloc, int heads, int s, int d, int w,
                       const LayMap& lay, const EpiParams& ep, float* dqkv, cudaStream_t st) {
    AttnBwd p;
    p.q = q;
    p.k = k;
    p.v = v;
    p.o = o;
    p.dO = dO;
    p.dq = dq;
    p.dk = dk;
    p.dv = dv;
    const i64 nst = i64(nloc) * heads * s;
    p.m = stats;
    p.l = stats + nst;
    p.D = stats + 2 * nst;
    p.ldo = ldo;
    p.nloc = nloc;
    p.heads = heads;
    p.s = s;
    p.d = d;
    p.w = w;
    p.scale = 1.0f / sqrtf(float(d));
    p.lay = lay;
    if (d > 16 * ADW) throw CudaError("attention backward: head dim must be <= 128");
    dim3 grid(unsigned((s + AT - 1) / AT), unsigned(heads), unsigned(nloc));
    const size_t ld = size_t(d) + 1;
    const size_t smq = (4 * AT * ld + AT * (AT + 1) + AT) * sizeof(float);
    const size_t smkv = (4 * AT * ld + 2 * AT * (AT + 1) + 3 * AT) * sizeof(float);
    k_attn_bwd_q<<<grid, 256, smq, st>>>(p);
    SWF_LAUNCH_CHECK();
    k_attn_bwd_kv<<<grid, 256, smkv, st>>>(p);
    SWF_LAUNCH_CHECK();
    EpiParams e = ep;
    e.cur = lay;
    const i64 n = i64(nloc) * s * (ep.h / 2);
    k_attn_bwd_pack<<<unsigned((n + 255) / 256), 256, 0, st>>>(dq, dk, dv, e, nloc, dqkv);
    SWF_LAUNCH_CHECK();
}
// ---- attention backward on the tensor cores (BF16 training mode), one (window, head) plane at a time
// (head_attention_bwd, swin.hpp:189-226): P = 2^(S log2e / sqrt(d) - lse) in the epilogue of S = Q K^T
// (lse = the forward kernel's per-row log2-sum-exp, seam mask as key ranges), dV = P^T dO, dS =
// P (dP - D) / sqrt(d) in the epilogue of dP = dO V^T, dQ = dS K, dK = dS^T Q -- five tcgen05 GEMMs
// (K-major or MN-major operands, no transposes); the s x s plane exists only as bf16 P and dS.
// D_i = dO_i . O_i for every row of every plane ([nloc][heads][s]), one warp per row.
__global__ void k_attn_bwd_D(const float* __restrict__ O, const float* __restrict__ dO, int ldo, int heads, int s,
                             int d, i64 rows, float* __restrict__ D) {
    const i64 t = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= rows) return;
    const i64 lh = t / s;
    const int i = int(t - lh * s);
    const i64 lw = lh / heads;
    const int hh = int(lh - lw * heads);
    const i64 off = (lw * s + i) * ldo + i64(hh) * d;
    float dd = 0.f;
    for (int e = lane; e < d; e += 32) dd = fmaf(O[off + e], dO[off + e], dd);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
    if (lane == 0) D[t] = dd;
}
size_t attention_bwd_tc_scratch(int s, int heads) {  // bytes: P / dS bf16 of a window's heads, zero K-tail rows
    const size_t sp = size_t((s + 7) / 8 * 8), spad = size_t((s + 63) / 64 * 64);
    return size_t(heads) * spad * sp * (2 + 2) + 1024;
}
void attention_bwd_tc(const float* q, const float* k, const float* v, const float* o, const float* dO, int ldo,
                      float* dq, float* dk, float* dv, int nloc, int heads, int s, int d, int w, const LayMap& lay,
                      const EpiParams& ep, float* dqkv, __nv_bfloat16* qkv16, __nv_bfloat16* dO16,
                      const float* lse, float* Dbuf, const AttnBwdStreams& ws, cudaStream_t st) {
    const i64 M = i64(nloc) * s, hd = i64(heads) * d;
    const int sp = (s + 7) / 8 * 8;
    to_bf16(q, M * hd, qkv16, st);  // q, k, v planes [nloc][heads][s][d]
    to_bf16(k, M * hd, qkv16 + M * hd, st);
    to_bf16(v, M * hd, qkv16 + 2 * M * hd, st);
    to_bf16(dO, M * ldo, dO16, st);
    const float scale = 1.0f / sqrtf(float(d));
    if (s % 8 != 0) throw CudaError("attention backward (tensor cores): s must be a multiple of 8");
    const i64 rows = i64(nloc) * heads * s;
    k_attn_bwd_D<<<unsigned((rows + 7) / 8), 256, 0, st>>>(o, dO, ldo, heads, s, d, rows, Dbuf);
    SWF_LAUNCH_CHECK();
    // host copy of the window ids (seam windows), one small read per call
    std::vector<int> gw(static_cast<size_t>(nloc));
    SWF_CUDA(cudaMemcpyAsync(gw.data(), lay.loc2glob, size_t(nloc) * 4, cudaMemcpyDeviceToHost, st));
    SWF_CUDA(cudaStreamSynchronize(st));
    const int split = (w - lay.g.shift) * w;
    // one window's heads per launch (plane-batched GEMMs: a plane's d-wide products are only 15 tiles),
    // windows round-robin over the worker streams, each with its own scratch and tile counter. The P / dS
    // planes of a window sit spad (s rounded up to 64) rows apart with zero pad rows, so the K tails of
    // the MN-major products (P^T dO, dS^T Q) read zeros on the P / dS side; the K-major ones stay
    // inside the maps' inner extent.
    const int spad = (s + 63) / 64 * 64;
    const i64 pst = i64(spad) * sp;  // elements per P / dS plane
    SWF_CUDA(cudaEventRecord(ws.ev[0], st));
    for (int i = 0; i < ws.n; ++i) SWF_CUDA(cudaStreamWaitEvent(ws.st[i], ws.ev[0], 0));
    for (int lw = 0; lw < nloc; ++lw) {
        const int masked = lay.g.shift > 0 && gw[size_t(lw)] / lay.g.nx == lay.g.ny - 1;
        const int wi = lw % ws.n;
        cudaStream_t ss = ws.st[wi];
        int* sched = ws.sched[wi];
        __nv_bfloat16* P = static_cast<__nv_bfloat16*>(ws.scratch[wi]);
        __nv_bfloat16* dS = P + size_t(heads) * pst;
        const i64 prow = i64(lw) * heads * s;  // rows of head 0 of this window in lse / D / the q, k, v planes
        const i64 pl = prow * d;
        const __nv_bfloat16 *q16 = qkv16 + pl, *k16 = qkv16 + M * hd + pl, *v16 = qkv16 + 2 * M * hd + pl;
        const __nv_bfloat16* dOw = dO16 + i64(lw) * s * ldo;  // head hh at column hh d
        const i64 prows = i64(heads) * s;                      // q / k / v plane rows of the window
        // P from S = Q K^T
        gemm_bf16_attn_rows(EPI_SMAX, q16, d, k16, d, s, d, P, sp, lse + prow, nullptr, split, masked,
                            scale * 1.4426950408889634f, sched, ss, heads, s, 0, s, pst);
        // dV = P^T dO: A = P MN-major (K = queries: spad rows per plane), B = dO MN-major (head columns)
        gemm_bf16_batched(P, true, sp, i64(heads) * spad, s, dOw, true, ldo, s, i64(heads) * d, s, d, s, dv + pl, d,
                          heads, 0, spad, d, 0, i64(s) * d, sched, ss);
        // dS from dP = dO V^T
        gemm_bf16_attn_rows(EPI_DSM, dOw, ldo, v16, d, s, d, dS, sp, Dbuf + prow, P, split, masked, scale, sched, ss,
                            heads, 0, d, s, pst);
        // dQ = dS K: A = dS K-major (inner = keys, s), B = K MN-major (K = keys: the next plane's rows meet
        // dS's zero-filled columns)
        gemm_bf16_batched(dS, false, sp, (i64(heads) - 1) * spad + s, s, k16, true, d, prows, d, s, d, s, dq + pl, d,
                          heads, 0, spad, 0, s, i64(s) * d, sched, ss);
        // dK = dS^T Q: A = dS MN-major (K = queries: zero pad rows), B = Q MN-major
        gemm_bf16_batched(dS, true, sp, i64(heads) * spad, s, q16, true, d, prows, d, s, d, s, dk + pl, d, heads, 0,
                          spad, 0, s, i64(s) * d, sched, ss);
    }
    for (int i = 0; i < ws.n; ++i) {
        SWF_CUDA(cudaEventRecord(ws.ev[1 + i], ws.st[i]));
        SWF_CUDA(cudaStreamWaitEvent(st, ws.ev[1 + i], 0));
    }
    EpiParams e = ep;
    e.cur = lay;
    const i64 n = i64(nloc) * s * (ep.h / 2);
    k_attn_bwd_pack<<<unsigned((n + 255) / 256), 256, 0, st>>>(dq, dk, dv, e, nloc, dqkv);
    SWF_LAUNCH_CHECK();
}
void ada_bwd(const float* d6, const float* emb, const float* Wa, int n6, int td, float* gWa, float* gba, float* demb,
             cudaStream_t st) {
    const int n = n6 * td;
    k_ada_bwd<<<unsigned((n + 255) / 256), 256, 0, st>>>(d6, emb, Wa, n6, td, gWa, gba, demb);
    SWF_LAUNCH_CHECK();
}
void time_bwd(const float* demb, const float* feat, const float* Wt, const float* bt, int td, float* gWt, float* gbt,
              cudaStream_t st) {
    k_time_bwd<<<unsigned((td * td + 255) / 256), 256, 0, st>>>(demb, feat, Wt, bt, td, gWt, gbt);
    SWF_LAUNCH_CHECK();
}


void train_prep(const float* x0, const float* z, i64 n, float cs, float sn, float* xt, float* v, cudaStream_t st) {
    k_train_prep<<<unsigned(std::min<i64>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(x0, z, n, cs, sn, xt, v);
    SWF_LAUNCH_CHECK();
}
void train_loss(const float* f, const float* v, const LayMap& lay, i64 M, int C, const float* kappa,
                const float* alpha_row, float sd, float g_scale, float* dS, double* part, cudaStream_t st) {
    k_train_loss<<<kTrainLossBlocks, 256, 0, st>>>(f, v, lay, M, C, kappa, alpha_row, sd, g_scale, dS, part);
    SWF_LAUNCH_CHECK();
}
void axpy_f32(const float* x, i64 n, float a, float* y, cudaStream_t st) {
    k_axpy<<<unsigned(std::min<i64>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(x, n, a, y);
    SWF_LAUNCH_CHECK();
}

void preload_bwd_kernels() {
    cudaFuncAttributes a;
    const void* k[] = {(const void*)k_gemm_strided, (const void*)k_norm_bwd_rows, (const void*)k_norm_bwd_cols,
                       (const void*)k_colsum, (const void*)k_swiglu_bwd, (const void*)k_swiglu_bwd4, (const void*)k_relayout,
                       (const void*)k_relayout_push, (const void*)k_attn_bwd_q, (const void*)k_attn_bwd_kv,
                       (const void*)k_attn_bwd_pack, (const void*)k_ada_bwd, (const void*)k_time_bwd,
                       (const void*)k_train_prep, (const void*)k_train_loss, (const void*)k_axpy,
                       (const void*)k_norm_bwd_cols_sum, (const void*)k_colsum_sum, (const void*)k_to_bf16, (const void*)k_to_bf16_2d,
                       (const void*)k_to_f32, (const void*)k_vt_bf16, (const void*)k_attn_bwd_D};
    for (const void* f : k) SWF_CUDA(cudaFuncGetAttributes(&a, f));
    int dev = 0, mx = 0;
    SWF_CUDA(cudaGetDevice(&dev));
    SWF_CUDA(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    for (const void* f : {(const void*)k_attn_bwd_q, (const void*)k_attn_bwd_kv})
        SWF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
}

}  // namespace swf
