// kernels.cuh -- launch interfaces of the swinflow B200 kernels (all sm_100a).
#pragma once

#include "common.cuh"

namespace swf {

// Which tokens a rank owns under one layout (SWiPe WP x SP). Whole windows go to a WP rank; with
// sequence parallelism the window's rows are split into SP bands keyed by the global row phase
// ((shift + r) mod w) / (w / sp) (window.hpp:67-79, shift-invariant), so rank = wp * sp + band.
// Local token order: owned window (loc2glob order), then the band's rows in ascending r (the
// reference band_rows order), then column. With sp == 1 this is the canonical window order.
// glob2rl[gw] = (wp_rank << 16) | local_window.
struct LayMap {
    Lay g;
    int nloc;             // local windows
    int sp, band;         // sequence-parallel degree, this rank's band
    const int* loc2glob;  // device [nloc]
    const int* glob2rl;   // device [n_windows]
    __host__ __device__ int s_loc() const { return g.w * g.w / sp; }
    // first rolled-frame row of a band and whether the band's row range wraps past r = w - 1
    __host__ __device__ void band_geom(int b, int& st, int& e, bool& wrap) const {
        const int R = g.w / sp;
        st = b * R - g.shift;
        if (st < 0) st += g.w;
        wrap = st + R > g.w;
        e = wrap ? st + R - g.w : 0;
    }
    // k-th row (ascending r) of band b
    __host__ __device__ int band_row(int b, int k) const {
        int st, e;
        bool wrap;
        band_geom(b, st, e, wrap);
        return wrap ? (k < e ? k : st + (k - e)) : st + k;
    }
    __host__ __device__ int band_of_row(int r) const {
        int ph = g.shift + r;
        if (ph >= g.w) ph -= g.w;
        return ph / (g.w / sp);
    }
    __host__ __device__ int row_index_in_band(int b, int r) const {
        int st, e;
        bool wrap;
        band_geom(b, st, e, wrap);
        return wrap ? (r < e ? r : e + (r - st)) : r - st;
    }
    // local token -> (global window, canonical in-window token r*w+c)
    __device__ __forceinline__ void loc_to_wtok(i64 i, int& gw, int& tok, int& lw) const {
        const int sl = s_loc();
        lw = int(i / sl);
        const int t = int(i - i64(lw) * sl);
        const int k = t / g.w, c = t - (t / g.w) * g.w;
        gw = loc2glob[lw];
        tok = band_row(band, k) * g.w + c;
    }
    __device__ __forceinline__ i64 loc_to_pix(i64 i) const {
        int gw, tok, lw;
        loc_to_wtok(i, gw, tok, lw);
        return g.win_to_pix(i64(gw) * (g.w * g.w) + tok);
    }
    // (local window of the WP group, canonical token) -> (owner rank in WP*SP, its local index)
    __device__ __forceinline__ i64 wtok_to_loc(int wp_rank, int lw, int tok, int* rank) const {
        const int r = tok / g.w, c = tok - (tok / g.w) * g.w;
        const int b = band_of_row(r);
        *rank = wp_rank * sp + b;
        return i64(lw) * s_loc() + i64(row_index_in_band(b, r)) * g.w + c;
    }
    // pixel -> (owner rank, local token index) under this layout
    __device__ __forceinline__ i64 pix_to_loc(i64 p, int* rank) const {
        const i64 gi = g.pix_to_win(p);
        const int s = g.w * g.w;
        const int gw = int(gi / s);
        const int rl = glob2rl[gw];
        return wtok_to_loc(rl >> 16, rl & 0xffff, int(gi - i64(gw) * s), rank);
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
    EPI_STORE = 6,   // x[m][n] = acc, n < N (the backward's plain products; tensor-core kernel only)
    // attention backward on the tensor cores (head_attention_bwd, swin.hpp:189-226), bf16 out[m][n] with
    // row pitch ld_out, n < N (N % 8 == 0); the row's key range: [0, N), or with `masked` [0, split)
    // for rows < split and [split, N) for the others (the seam mask, window.hpp:107-122)
    EPI_SMAX = 7,    // P = 2^(acc * out_scale - rowv[m]) in the key range, else 0 (rowv = log2-sum-exp)
    EPI_DSM = 8,     // dS = P[m][n] * (acc - rowv[m]) * out_scale, P = pin (bf16, pitch ld_out), rowv = D
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
    const float2* rope_row_pm;  // the same tables position-major: [H+w][d/4], [W+w][d/4]
    const float2* rope_col_pm;
    int rope_nrow, rope_ncol;
    LayMap cur, nxt;
    float out_scale;
    // sequence parallelism: QKV planes of every rank of this WP group (peer-mapped), heads per
    // rank, this rank's WP index
    void* const* qkv_dst;
    int heads_loc;
    int wp_rank;
    // RMSNorm + AdaLN fused into the GEMMs (BF16 path; nss == 0 disables it). Producers (ENCODE,
    // RESID, DOWN) also store a bf16 copy of the residual row (operand A of the next normed GEMM) at
    // (bf16*)(xbase + off_xb) + row * hp and the partial sum of squares of their 128 columns at
    // xbase + off_ss + row * nss + slot (slot = 2 * n_tile + half), xbase being ep.x or ep.xdst[rank].
    // Consumers (QKV, SWIGLU, DECODE) scale the accumulator by inv_r[row] = 1 / rms(row) (reduced
    // from the partials by inv_rms) and add beta[col] = (W (gate .* b))[col], the weights having been
    // folded with diag(gate .* g .* (1 + a)) (swin.hpp:72-85).
    int hp, nss;
    i64 off_xb, off_ss;
    const float* inv_r;
    const float* beta;
    // tile counter of the persistent GEMM's dynamic schedule, owned by the context (GEMMs of one
    // context are stream-ordered); nullptr -> a per-device counter (single-stream callers only)
    int* sched;
    // EPI_SMAX / EPI_DSM
    const float* rowv;
    const void* pin;
    int split, masked;
    // plane-batched launches (EPI_STORE / EPI_SMAX / EPI_DSM only): nbatch problems of one shape; problem
    // b shifts the A / B TMA coordinates by b (adx, ady) / (bdx, bdy) and the output (x or out), rowv and
    // pin by b times bst_c, bst_rv, bst_p elements (nbatch 0 = 1)
    int nbatch;
    int adx, ady, bdx, bdy;
    i64 bst_c, bst_rv, bst_p;
};
// inv_r[m] = 1 / sqrt(sum_i ss[m][i] / h + 1e-8) over the nss partials; non-finite rows flag
// flags[slot] (check_finite, swin.hpp:295-300)
void inv_rms(const float* ss, i64 M, int nss, int h, float* inv_r, int* flags, int slot, cudaStream_t st);

// C[M][N] = A[M][K] . B[N][K]^T (both K-major), fp32 SIMT -- the FP32 validation mode GEMM.
void gemm_f32(const float* A, const float* B, i64 M, int N, int K, int mode, const EpiParams& ep,
              cudaStream_t st);
// gemm_f32's epilogue `mode` applied row-wise to a plain fp32 product C = A . B^T ([M][ldc])
void epi_rows_f32(const float* C, int ldc, i64 M, int N, int mode, const EpiParams& ep, cudaStream_t st);

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
// General tensor-core GEMM of the backward: C[M][N] (fp32, row pitch ldc) (+)= A . B with bf16
// operands, A K-major (A[m * lda + k]) or MN-major (A[k * lda + m]), B K-major (B[n * ldb + k]) or
// MN-major (B[k * ldb + n]) -- not A MN-major with B K-major; pitches multiples of 8 elements.
void gemm_bf16_general(const __nv_bfloat16* A, bool a_mn, i64 lda, const __nv_bfloat16* B, bool b_mn, i64 ldb, i64 M,
                       i64 N, i64 K, float* C, i64 ldc, bool accumulate, int* sched, cudaStream_t st);
// Plane-batched plain products: nbatch GEMMs C_b[M][N] = op(A_b) op(B_b) (fp32, pitch ldc), operand maps
// over [a_rows][a_inner] / [b_rows][b_inner] (all problems), problem b at coordinate offsets b (adx, ady),
// b (bdx, bdy) and C_b = C + b bst_c. No K-tail zero fill inside the maps: the caller keeps the K tails
// of one operand zero (or inside the map's inner extent).
void gemm_bf16_batched(const __nv_bfloat16* A, bool a_mn, i64 lda, i64 a_rows, i64 a_inner, const __nv_bfloat16* B,
                       bool b_mn, i64 ldb, i64 b_rows, i64 b_inner, i64 M, i64 N, i64 K, float* C, i64 ldc, int nbatch,
                       int adx, int ady, int bdx, int bdy, i64 bst_c, int* sched, cudaStream_t st);
// The attention backward's row-wise products (both operands K-major, s x s output in bf16, pitch ldo):
// mode EPI_SMAX: out = P from S = A . B^T; EPI_DSM: out = dS from dP = A . B^T (see EpiMode)
// nbatch > 1: problems b = 0.. at A / B row offsets b a_rows_b / b b_rows_b (maps over nbatch of them),
// out / pin + b bst_out, rowv + b s; a_col_b: A column offset per problem instead (dO's head columns)
void gemm_bf16_attn_rows(int mode, const __nv_bfloat16* A, i64 lda, const __nv_bfloat16* B, i64 ldb, int s, int K,
                         __nv_bfloat16* out, int ldo, const float* rowv, const __nv_bfloat16* pin, int split,
                         int masked, float scale, int* sched, cudaStream_t st, int nbatch = 1, i64 a_rows_b = 0,
                         int a_col_b = 0, i64 b_rows_b = 0, i64 bst_out = 0);

// ------------------------------------------------------------------ attention
struct AttnParams {
    const void* q;  // [nloc][heads][s][d]
    const void* k;  // [nloc][heads][s][d]
    const void* v;  // FP32 path: [nloc][heads][s][d]; BF16 path: V^T [nloc][heads][d][s]
    void* o;        // [nloc*s][ldo] head-concatenated (FP32 path, sp == 1)
    void* const* o_dst;  // BF16 path: attention-output buffer of every rank (peer-mapped; own when sp == 1)
    int ldo;
    int nloc, heads, s, d, w;
    int head0;      // first global head of this rank's head group (sequence parallelism)
    int wp_rank;
    LayMap lay;     // masked windows: shifted layout, last window row
    float scale;    // 1/sqrt(d)
    const TmaMap* tmq;  // BF16 path: TMA maps of the q / k planes ([rows][d]) and of V^T ([rows][s])
    const TmaMap* tmk;
    const TmaMap* tmv;
    const TmaMap* tmk2; // BF16 path: K planes with 32-row boxes (the ping-pong kernel's 64-key tiles)
    const TmaMap* tmo;  // BF16 path, sp == 1: map of the own output buffer (box 64 x 128, SW128) for TMA
                        // stores of whole query tiles; nullptr = per-row stores
    int dbg = 0;        // test only (swf_selftest_attention negative control): bit 0 skips the O rescale
    float* lse = nullptr;  // BF16 training mode, ping-pong kernel: per query row [nloc][heads][s] the
                           // log2-sum-exp of the scaled logits (s log2e / sqrt(d)), for the backward's P
};
void attention_f32(const AttnParams& p, cudaStream_t st);
void attention_bf16(const AttnParams& p, cudaStream_t st);

// ------------------------------------------------------------------ backward (k_bwd.cu, FP32 mode)
// C[i][j] = beta C[i][j] + sum_k A[i*sai + k*sak] B[k*sbk + j*sbj]
void gemm_strided_f32(int M, int N, int K, const float* A, i64 sai, i64 sak, const float* B, i64 sbk, i64 sbj,
                      float* C, i64 ldc, float beta, cudaStream_t st);
void to_bf16(const float* x, i64 n, __nv_bfloat16* y, cudaStream_t st);
void to_f32(const __nv_bfloat16* x, i64 n, float* y, cudaStream_t st);
void vt_bf16(const float* v, i64 planes, int s, int d, __nv_bfloat16* vt, cudaStream_t st);
// attention backward on the tensor cores (BF16 training mode): per (window, head) plane, five tcgen05
// GEMMs -- P from S = Q K^T in the GEMM's epilogue with the forward's log2-sum-exp `lse`, dS from
// dP = dO V^T in the next one's with D = rowsum(dO . O) (one pass over all planes into `Dbuf`,
// [nloc][heads][s]); one window's heads per (plane-batched) launch; scratch of attention_bwd_tc_scratch(s, heads) bytes, qkv16 3 M h and dO16 M ldo bf16
// elements; d % 8 == 0, s % 8 == 0
size_t attention_bwd_tc_scratch(int s, int heads);
struct AttnBwdStreams {  // worker streams of the per-plane loop, each with scratch and a GEMM tile counter
    static constexpr int kMax = 4;
    int n = 0;
    cudaStream_t st[kMax];
    cudaEvent_t ev[kMax + 1];
    void* scratch[kMax];
    int* sched[kMax];
};
void attention_bwd_tc(const float* q, const float* k, const float* v, const float* o, const float* dO, int ldo,
                      float* dq, float* dk, float* dv, int nloc, int heads, int s, int d, int w, const LayMap& lay,
                      const EpiParams& ep, float* dqkv, __nv_bfloat16* qkv16, __nv_bfloat16* dO16,
                      const float* lse, float* Dbuf, const AttnBwdStreams& ws, cudaStream_t st);
void gemm_strided_tc(int M, int N, int K, const float* A, i64 sai, i64 sak, const float* B, i64 sbk, i64 sbj, float* C,
                     i64 ldc, float beta, __nv_bfloat16* ta, __nv_bfloat16* tb, int* sched, cudaStream_t st);
// prenorm_modulate_bwd / prenorm_plain_bwd (a, b, gate null): dX += ..., per-channel grads +=
// part: scratch of kNormSlices * 4 * h floats (per-slice channel sums)
constexpr int kNormSlices = 256;
void norm_bwd(const float* X, int ldx, const float* dXM, int lddxm, i64 M, int h, const float* g, const float* a,
              const float* b, const float* gate, float* dX, int lddx, float* rms, float* dg, float* da, float* db,
              float* dgate, float* part, cudaStream_t st);
void colsum_f32(const float* X, int ldx, i64 M, int n, float* out, float* part, cudaStream_t st);  // part: kNormSlices * n
void swiglu_bwd(const float* gu, int ldgu, const float* dS, int ldds, i64 M, int f, int G, float* act, float* dG,
                float* dU, cudaStream_t st);
// WP: row i of A's local order -> dst[owner rank][B-local index] (peer stores)
void relayout_push(const float* src, const LayMap& A, const LayMap& B, i64 M, int h, float* const* dst,
                   cudaStream_t st);
void relayout_rows(const float* src, const LayMap& A, const LayMap& B, i64 M, int h, float* dst, cudaStream_t st);
void attention_bwd_f32(const float* q, const float* k, const float* v, const float* o, const float* dO, int ldo,
                       float* dq, float* dk, float* dv, float* stats, int nloc, int heads, int s, int d, int w,
                       const LayMap& lay, const EpiParams& ep, float* dqkv, cudaStream_t st);
void ada_bwd(const float* d6, const float* emb, const float* Wa, int n6, int td, float* gWa, float* gba, float* demb,
             cudaStream_t st);
// diffusion training loss (diffusion.hpp:57-67, 111-133): x_t / v targets, weighted squared error
// with per-block double partials (kTrainLossBlocks of them) and its gradient into dS, y += a x
constexpr int kTrainLossBlocks = 592;
void train_prep(const float* x0, const float* z, i64 n, float cs, float sn, float* xt, float* v, cudaStream_t st);
void train_loss(const float* f, const float* v, const LayMap& lay, i64 M, int C, const float* kappa,
                const float* alpha_row, float sd, float g_scale, float* dS, double* part, cudaStream_t st);
void axpy_f32(const float* x, i64 n, float a, float* y, cudaStream_t st);
void time_bwd(const float* demb, const float* feat, const float* Wt, const float* bt, int td, float* gWt, float* gbt,
              cudaStream_t st);

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
// Fused-norm operands of residual rows written by the host (block_window_forward): bf16 copy [M][hp]
// and the per-row sum of squares (partial slot 0; inv_rms sums all nss slots)
void prep_residual(const float* x, i64 M, int h, int hp, int nss, __nv_bfloat16* xb, float* ss, cudaStream_t st);
// dst[k][c] = src[local index of pix[k]][c] for the pixels `rank` owns under `lay` (others untouched)
void rows_at_pixels(const float* src_loc, const LayMap& lay, int rank, int C, const i64* pix, i64 n, float* dst,
                    cudaStream_t st);
// RMSNorm + AdaLN modulation (prenorm_modulate, swin.hpp:72-85) or plain (prenorm_plain :111-123 when
// a == nullptr): out[m][i] = gate*((g*x/r)*(1+a)+b); non-finite input -> flags[slot].
// AdaLN folding for the fused norm (BF16 path): Wf[n][k] = bf16(Wm[n][k] * s[k]) and
// beta[n] = sum_k Wm[n][k] c[k] with s = gate .* g .* (1 + a), c = gate .* b (a, b, gate may be null
// = 0, 0, 1), Wm the fp32 master in the repacked [Np][ld] layout.
void fold_adaln(const float* Wm, int Np, int K, int ld, const float* g, const float* a, const float* b,
                const float* gate, __nv_bfloat16* Wf, float* beta, cudaStream_t st);
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
void churn_rotate(float* x, const LayMap& lay0, i64 M, int C, const u64* key, u64 ctr0, double sigma_d, float c, float s,
                  cudaStream_t st);
// y = (x - mean) / std  (Standardizer::apply_mat, grid.hpp:127-129)
void standardize(const float* x, i64 M, int C, const float* mean, const float* stdv, float* y, cudaStream_t st);
// y = base + (r * std + mean)  (invert_mat grid.hpp:130-132 + forecast_step diffusion.hpp:318)
void destandardize_add(const float* r, const float* base, i64 M, int C, const float* mean, const float* stdv,
                       float* y, cudaStream_t st);
// Count non-finite values of a buffer into flags[slot] (cheap guard for device-entry inputs).
void check_finite(const float* x, i64 n, int* flags, int slot, cudaStream_t st);

// Load every kernel into the current device's context (cudaFuncGetAttributes per kernel). CUDA's
// lazy module loading would otherwise load a kernel at its first launch, which needs the context idle
// -- and with ranks of one process meeting in spin barriers on a shared GPU, a rank's first launch of
// a kernel can wait behind a peer's barrier that waits for that rank: a deadlock.
void preload_elem_kernels();
// the calling thread's swf_last_error() message (ctx.cu)
void set_last_error(const std::string& m);
// load all kernels and set their shared-memory limits on `device`, once per process (ctx.cu)
void ensure_device(int device);
void preload_bwd_kernels();
void preload_simt_kernels();
void preload_gemm_kernels();
void preload_attn_kernels();

}  // namespace swf
