// kernels.cuh -- launch interfaces of the swinflow B200 kernels (all sm_100a).
#pragma once

#include "common.cuh"

namespace swf {

// Which tokens a rank owns under one layout (whole windows, SWiPe-style). loc2glob[lw] is the
// global window id of local window lw; glob2rl[gw] = (owner_rank << 16) | local_window.
struct LayMap {
    Lay g;
    int nloc;              // local windows
    const int* loc2glob;   // device [nloc]
    const int* glob2rl;    // device [n_windows]
    __device__ __forceinline__ i64 loc_to_pix(i64 i) const {
        const int s = g.w * g.w;
        const int lw = int(i / s);
        const int tok = int(i - i64(lw) * s);
        return g.win_to_pix(i64(loc2glob[lw]) * s + tok);
    }
    // pixel -> (owner rank, local token index) under this layout
    __device__ __forceinline__ i64 pix_to_loc(i64 p, int* rank) const {
        const i64 gi = g.pix_to_win(p);
        const int s = g.w * g.w;
        const int gw = int(gi / s);
        const int rl = glob2rl[gw];
        *rank = rl >> 16;
        return i64(rl & 0xffff) * s + (gi - i64(gw) * s);
    }
};

// ------------------------------------------------------------------ GEMM epilogues
enum EpiMode : int {
    EPI_ENCODE = 0,  // x[m][n] = acc + bias[n]                                    (swin.hpp:341-342)
    EPI_QKV = 1,     // RoPE(q,k) + scatter to [lwin][head][tok][d] planes          (swin.hpp:168-175)
    EPI_RESID = 2,   // x[m][n] += acc   (out projection + residual)                (swin.hpp:322)
    EPI_SWIGLU = 3,  // s[m][j] = silu(gate) * up from interleaved columns          (swin.hpp:230-232)
    EPI_DOWN = 4,    // xdst[dest(m)][n] = xsrc[m][n] + acc, dest = next layout     (swin.hpp:324, 356-358)
    EPI_DECODE = 5,  // out[m][n] = (acc + bias[n]) * out_scale, n < cout (local L0 order) (swin.hpp:364-366)
};

struct EpiParams {
    i64 M;           // rows (local tokens)
    int N;           // logical output columns
    float* x;        // fp32 residual [M][h] (ENCODE/RESID dst; DOWN src)
    float* const* xdst;  // DOWN: per-rank destination residual bases (peer-mapped for remote ranks)
    int my_rank;
    const float* bias;
    void* out;       // typed output (QKV planes, SWIGLU s, DECODE out)
    i64 plane;       // QKV: elements per q/k/v plane
    int ld_out;      // SWIGLU: row stride of s; DECODE: cout
    int h, d, heads;
    int G;           // SWIGLU interleave granularity
    const float2* rope_row;  // [d/4][H+w] (cos, sin)
    const float2* rope_col;  // [d/4][W+w]
    int rope_nrow, rope_ncol;
    LayMap cur, nxt;
    float out_scale;
};

// C[M][N] = A[M][K] . B[N][K]^T (both K-major), fp32 SIMT -- the FP32 validation mode GEMM.
void gemm_f32(const float* A, const float* B, i64 M, int N, int K, int mode, const EpiParams& ep,
              cudaStream_t st);

// TMA descriptor (CUtensorMap, 128 B) of a row-major bf16 [rows][kcols] operand, box = box_rows x 64
// with 128-byte swizzle (the canonical K-major SW128 UMMA layout).
struct alignas(64) TmaMap {
    uint64_t bytes[16];
};
void make_tma_bf16(TmaMap* m, const void* base, i64 rows, i64 kcols, int box_rows);
// General 2D bf16 map: inner extent `inner` (elements), `rows` rows, box {box_inner, box_rows},
// swizzle in bytes (64 or 128).
void make_tma_bf16_2d(TmaMap* m, const void* base, i64 rows, i64 inner, int box_inner, int box_rows, int swizzle);

// tcgen05/TMEM/TMA BF16 GEMM (2-CTA pairs, persistent, warp-specialised): C[M][Npad] = A . B^T,
// A = [M][K] (box 128 rows), B = [Npad][K] (box BN/2 rows), BN in {128, 256}, K % 64 == 0.
void gemm_bf16_tc(const TmaMap& A, const TmaMap& B, i64 M, int Npad, int K, int BN, int mode, const EpiParams& ep,
                  cudaStream_t st);

// ------------------------------------------------------------------ attention
struct AttnParams {
    const void* q;  // [nloc][heads][s][d]
    const void* k;  // [nloc][heads][s][d]
    const void* v;  // FP32 path: [nloc][heads][s][d]; BF16 path: V^T [nloc][heads][d][s]
    void* o;        // [nloc*s][ldo] head-concatenated
    int ldo;
    int nloc, heads, s, d, w;
    LayMap lay;     // masked windows: shifted layout, last window row
    float scale;    // 1/sqrt(d)
    const TmaMap* tmq;  // BF16 path: TMA maps of the q / k planes ([rows][d]) and of V^T ([rows][s])
    const TmaMap* tmk;
    const TmaMap* tmv;
};
void attention_f32(const AttnParams& p, cudaStream_t st);
void attention_bf16(const AttnParams& p, cudaStream_t st);

// ------------------------------------------------------------------ elementwise
void time_features(double t, int td, float* feat, cudaStream_t st);
void time_embed(const float* feat, const float* w_time_t, const float* b_time, int td, float* emb,
                cudaStream_t st);
void ada_vectors(const float* emb, const float* w_ada_t, const float* b_ada, int nb, int six_h, int td, float* six,
                 cudaStream_t st);
// Gather owned pixels of a pixel-order [N][C] fp32 field into local window order of `lay`, cast
// to T and zero-pad each row to ldo columns (model input assembly / standardisation prep).
template <class T>
void gather_rows(const float* src_pix, const LayMap& lay, int C, int ldo, i64 M, T* dst, int* flags, int slot,
                 cudaStream_t st);
// Inverse: dst_pix[pix(i)][c] = src[i][c] for the owned rows.
void scatter_rows(const float* src_loc, const LayMap& lay, int C, i64 M, float* dst_pix, cudaStream_t st);
// RMSNorm + AdaLN modulation (prenorm_modulate, swin.hpp:72-85) or plain (prenorm_plain :111-123 when
// a == nullptr): out[m][i] = gate*((g*x/r)*(1+a)+b); non-finite input -> flags[slot].
template <class T>
void rms_modulate(const float* x, i64 M, int h, int ldo, const float* g, const float* a, const float* b,
                  const float* gate, T* out, int* flags, int slot, cudaStream_t st);

// Sampler (diffusion.hpp:207-272) elementwise kernels over the [M][C] fp32 state (local L0 order).
// x0hat = cs*xd - sn*v (x0_hat, diffusion.hpp:219-224) ; y = c1*xa - c2*x0hat ; non-finite y -> flags[slot]
void sampler_update(const float* xa, const float* xd, const float* v, i64 n, float cs, float sn, float c1, float c2,
                    float* y, int* flags, int slot, cudaStream_t st);
// a_in channels [cp, cin): [x_prev_std ; forcings_std] + posenc (static conditioning of the net lambda)
template <class T>
void build_static_input(const float* xprev, const float* forc, const float* pe, i64 M, int cp, int cf, int cin,
                        int kp, T* a_in, cudaStream_t st);
// Model-input channels [0,cp) = x / sigma_d + posenc (assemble_model_input, diffusion.hpp:147-156).
template <class T>
void assemble_state(const float* x, const float* pe, i64 M, int cp, int cin, int kp, float sd, T* a_in,
                    cudaStream_t st);
// noise_field (diffusion.hpp:91-108) generated directly in local window order of the unshifted layout.
void noise_field(u64 zfk, int C, const LayMap& lay0, double sigma_d, float* z, cudaStream_t st);
// churn rotation (diffusion.hpp:255-268): x = c*x + s*sd*gaussian(key, ctr0 + pix*C + ch)
void churn_rotate(float* x, const LayMap& lay0, i64 M, int C, u64 key, u64 ctr0, double sigma_d, float c, float s,
                  cudaStream_t st);
// y = (x - mean) / std  (Standardizer::apply_mat, grid.hpp:127-129)
void standardize(const float* x, i64 M, int C, const float* mean, const float* stdv, float* y, cudaStream_t st);
// y = base + (r * std + mean)  (invert_mat grid.hpp:130-132 + forecast_step diffusion.hpp:318)
void destandardize_add(const float* r, const float* base, i64 M, int C, const float* mean, const float* stdv,
                       float* y, cudaStream_t st);
// Count non-finite values of a buffer into flags[slot] (cheap guard for device-entry inputs).
void check_finite(const float* x, i64 n, int* flags, int slot, cudaStream_t st);

}  // namespace swf
