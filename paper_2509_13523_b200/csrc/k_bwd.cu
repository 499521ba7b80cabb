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
#include "kernels.cuh"

namespace swf {

namespace {

constexpr int TB = 64, TK = 16;

// C[i][j] = beta * C[i][j] + sum_k A(i,k) B(k,j); A(i,k) = A[i*sai + k*sak], B(k,j) = B[k*sbk + j*sbj],
// C row stride ldc. 256 threads, 64 x 64 tile, 4 x 4 per thread.
__global__ void __launch_bounds__(256) k_gemm_strided(int M, int N, int K, const float* __restrict__ A, i64 sai,
                                                      i64 sak, const float* __restrict__ B, i64 sbk, i64 sbj,
                                                      float* __restrict__ C, i64 ldc, float beta) {
    __shared__ float As[TK][TB + 1], Bs[TK][TB + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * TB, j0 = blockIdx.x * TB;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int t = threadIdx.x; t < TB * TK; t += 256) {
            const int r = t / TK, k = t % TK;  // A: row r of the tile, column k
            const int gi = i0 + r, gk = k0 + k;
            As[k][r] = (gi < M && gk < K) ? A[gi * sai + gk * sak] : 0.f;
            const int c = t / TK, kk = t % TK;
            const int gj = j0 + c, gk2 = k0 + kk;
            Bs[kk][c] = (gj < N && gk2 < K) ? B[gk2 * sbk + gj * sbj] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = As[k][ty * 4 + u];
                b[u] = Bs[k][tx * 4 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int gi = i0 + ty * 4 + u;
        if (gi >= M) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int gj = j0 + tx * 4 + v;
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
    for (int i = lane; i < h; i += 32) {
        const float du = dxm[i] * (gate ? gate[i] : 1.f) * (a ? 1.f + a[i] : 1.f) * g[i];
        dx[i] += du / r - x[i] * c;
    }
    if (lane == 0) rms[j] = r;
}

// per-channel pass: dg[i] += sum_j dxm gate (1+a) u ; da[i] += sum_j dxm gate g u ; db[i] += sum_j dxm gate ;
// dgate[i] += sum_j dxm (g u (1+a) + b), u = x / r. One thread per channel, tokens in order.
__global__ void k_norm_bwd_cols(const float* __restrict__ X, int ldx, const float* __restrict__ dXM, int lddxm,
                                const float* __restrict__ rms, i64 M, int h, const float* __restrict__ g,
                                const float* __restrict__ a, const float* __restrict__ b,
                                const float* __restrict__ gate, float* __restrict__ dg, float* __restrict__ da,
                                float* __restrict__ db, float* __restrict__ dgate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h) return;
    const float gi = g[i], ai = a ? a[i] : 0.f, bi = b ? b[i] : 0.f, qi = gate ? gate[i] : 1.f;
    float sg = 0.f, sa = 0.f, sb = 0.f, sq = 0.f;
    for (i64 j = 0; j < M; ++j) {
        const float u = X[j * ldx + i] / rms[j];
        const float dxm = dXM[j * lddxm + i];
        const float gu = gi * u;
        sa = fmaf(dxm * qi, gu, sa);
        sb = fmaf(dxm, qi, sb);
        sq = fmaf(dxm, gu * (1.f + ai) + bi, sq);
        sg = fmaf(dxm * qi * (1.f + ai), u, sg);
    }
    dg[i] += sg;
    if (da) da[i] += sa;
    if (db) db[i] += sb;
    if (dgate) dgate[i] += sq;
}

// column sums (bias gradients): out[i] += sum_j X[j][i]
__global__ void k_colsum(const float* __restrict__ X, int ldx, i64 M, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float s = 0.f;
    for (i64 j = 0; j < M; ++j) s += X[j * ldx + i];
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
__global__ void k_attn_bwd_q(AttnBwd p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, head = blockIdx.y, lw = blockIdx.z;
    if (i >= p.s) return;
    const int s = p.s, d = p.d;
    const i64 base = (i64(lw) * p.heads + head) * s;
    const float* qi = p.q + (base + i) * d;
    int split;
    bool masked;
    seam(p, lw, split, masked);
    const int gq = i < split ? 0 : 1;
    float m = -INFINITY;
    for (int j = 0; j < s; ++j) {
        if (masked && (j < split ? 0 : 1) != gq) continue;
        const float* kj = p.k + (base + j) * d;
        float acc = 0.f;
        for (int e = 0; e < d; ++e) acc = fmaf(qi[e], kj[e], acc);
        m = fmaxf(m, acc * p.scale);
    }
    float l = 0.f;
    for (int j = 0; j < s; ++j) {
        if (masked && (j < split ? 0 : 1) != gq) continue;
        const float* kj = p.k + (base + j) * d;
        float acc = 0.f;
        for (int e = 0; e < d; ++e) acc = fmaf(qi[e], kj[e], acc);
        l += expf(acc * p.scale - m);
    }
    const float* oi = p.o + (i64(lw) * s + i) * p.ldo + head * d;
    const float* doi = p.dO + (i64(lw) * s + i) * p.ldo + head * d;
    float D = 0.f;
    for (int e = 0; e < d; ++e) D = fmaf(doi[e], oi[e], D);
    float* dqi = p.dq + (base + i) * d;
    for (int e = 0; e < d; ++e) dqi[e] = 0.f;
    for (int j = 0; j < s; ++j) {
        if (masked && (j < split ? 0 : 1) != gq) continue;
        const float* kj = p.k + (base + j) * d;
        const float* vj = p.v + (base + j) * d;
        float acc = 0.f, dp = 0.f;
        for (int e = 0; e < d; ++e) {
            acc = fmaf(qi[e], kj[e], acc);
            dp = fmaf(doi[e], vj[e], dp);
        }
        const float pij = expf(acc * p.scale - m) / l;
        const float da = pij * (dp - D) * p.scale;
        for (int e = 0; e < d; ++e) dqi[e] = fmaf(da, kj[e], dqi[e]);
    }
    p.m[base + i] = m;
    p.l[base + i] = l;
    p.D[base + i] = D;
}
__global__ void k_attn_bwd_kv(AttnBwd p) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, head = blockIdx.y, lw = blockIdx.z;
    if (j >= p.s) return;
    const int s = p.s, d = p.d;
    const i64 base = (i64(lw) * p.heads + head) * s;
    const float* kj = p.k + (base + j) * d;
    const float* vj = p.v + (base + j) * d;
    int split;
    bool masked;
    seam(p, lw, split, masked);
    const int gk = j < split ? 0 : 1;
    float* dkj = p.dk + (base + j) * d;
    float* dvj = p.dv + (base + j) * d;
    for (int e = 0; e < d; ++e) dkj[e] = dvj[e] = 0.f;
    for (int i = 0; i < s; ++i) {
        if (masked && (i < split ? 0 : 1) != gk) continue;
        const float* qi = p.q + (base + i) * d;
        const float* doi = p.dO + (i64(lw) * s + i) * p.ldo + head * d;
        float acc = 0.f, dp = 0.f;
        for (int e = 0; e < d; ++e) {
            acc = fmaf(qi[e], kj[e], acc);
            dp = fmaf(doi[e], vj[e], dp);
        }
        const float pij = expf(acc * p.scale - p.m[base + i]) / p.l[base + i];
        const float da = pij * (dp - p.D[base + i]) * p.scale;
        for (int e = 0; e < d; ++e) {
            dkj[e] = fmaf(da, qi[e], dkj[e]);
            dvj[e] = fmaf(pij, doi[e], dvj[e]);
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
    dim3 grid(unsigned((N + TB - 1) / TB), unsigned((M + TB - 1) / TB));
    k_gemm_strided<<<grid, 256, 0, st>>>(M, N, K, A, sai, sak, B, sbk, sbj, C, ldc, beta);
    SWF_LAUNCH_CHECK();
}
void norm_bwd(const float* X, int ldx, const float* dXM, int lddxm, i64 M, int h, const float* g, const float* a,
              const float* b, const float* gate, float* dX, int lddx, float* rms, float* dg, float* da, float* db,
              float* dgate, cudaStream_t st) {
    k_norm_bwd_rows<<<unsigned((M + 7) / 8), 256, 0, st>>>(X, ldx, dXM, lddxm, M, h, g, a, gate, dX, lddx, rms);
    SWF_LAUNCH_CHECK();
    k_norm_bwd_cols<<<unsigned((h + 127) / 128), 128, 0, st>>>(X, ldx, dXM, lddxm, rms, M, h, g, a, b, gate, dg, da,
                                                               db, dgate);
    SWF_LAUNCH_CHECK();
}
void colsum_f32(const float* X, int ldx, i64 M, int n, float* out, cudaStream_t st) {
    k_colsum<<<unsigned((n + 127) / 128), 128, 0, st>>>(X, ldx, M, n, out);
    SWF_LAUNCH_CHECK();
}
void swiglu_bwd(const float* gu, int ldgu, const float* dS, int ldds, i64 M, int f, int G, float* act, float* dG,
                float* dU, cudaStream_t st) {
    const i64 n = M * f;
    k_swiglu_bwd<<<unsigned((n + 255) / 256), 256, 0, st>>>(gu, ldgu, dS, ldds, M, f, G, act, dG, dU);
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
    dim3 grid(unsigned((s + 63) / 64), unsigned(heads), unsigned(nloc));
    k_attn_bwd_q<<<grid, 64, 0, st>>>(p);
    SWF_LAUNCH_CHECK();
    k_attn_bwd_kv<<<grid, 64, 0, st>>>(p);
    SWF_LAUNCH_CHECK();
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

}  // namespace swf
