/* swinflow_capi.h -- C-ABI of the B200-native swinflow denoiser hot path.
 *
 * Drop-in boundary for the reference's header-only C++ API (arxiv 2509.13523 / AERIS,
 * /root/reference/proj/include/swinflow). Each entry point cites the reference interface it
 * replaces. Plain pointers and sizes only; no torch / Eigen types cross this boundary.
 *
 * Data layout (identical to the reference's Eigen column-major storage):
 *   a C x N field (C channels, N = H*W pixels, pixel index y*W + x) is N*C contiguous values
 *   with the C channels of one pixel adjacent ("[N][C]"); a weight W (out x in) is in*out
 *   values, column k (input k) contiguous ("[in][out]").
 *
 * Errors: every int-returning call returns SWF_OK (0) or a code below; swf_last_error() gives a
 * thread-local message. Codes mirror the reference CLI exit codes (swinflow_main.cpp:705-718):
 *   SWF_ERR_NUMERICS (1) <- NumericsError  (non-finite activation / solver divergence)
 *   SWF_ERR_CONFIG   (2) <- ConfigError    (shape / divisibility / channel mismatch)
 *   SWF_ERR_IO       (3) <- IoError
 *   SWF_ERR_CUDA     (4)    device / driver failure (no CPU fallback exists)
 *
 * Threading: one stream and one workspace per context; a context must not be used from two
 * threads at once (use one context per thread, as reference_train_step_mt's pool would).
 */
#ifndef SWINFLOW_CAPI_H
#define SWINFLOW_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWF_OK 0
#define SWF_ERR_NUMERICS 1
#define SWF_ERR_CONFIG 2
#define SWF_ERR_IO 3
#define SWF_ERR_CUDA 4

/* precision of the device path */
#define SWF_PREC_BF16 0 /* BF16 tensor-core operands, FP32 accumulate + FP32 residual stream */
#define SWF_PREC_FP32 1 /* FP32 validation mode (SIMT FP32 on the GPU; <= 1e-4 vs the oracle) */

/* host buffer element types */
#define SWF_F32 0
#define SWF_F64 1

/* ownership of windows across ranks (SWiPe window parallelism) */
#define SWF_OWN_CONTIGUOUS 0 /* contiguous window blocks (performance default, least exchange) */
#define SWF_OWN_ROUND_ROBIN 1 /* reference window_owner (topology.hpp:107-109) */

/* swinflow::ModelConfig (model.hpp:21-62) */
typedef struct swf_model_cfg {
    int hidden_dim, n_heads, ffn_dim, n_layers, blocks_per_layer, window_px, in_channels, out_channels, time_dim;
} swf_model_cfg;

/* swinflow::DiffusionConfig (diffusion.hpp:29-46) with ChurnSchedule::amount */
typedef struct swf_diffusion_cfg {
    double sigma_d, sigma_min, sigma_max;
    int solver_steps;
    double churn;
} swf_diffusion_cfg;

/* Standardizer pairs (grid.hpp:85-133): mean/std arrays of the state (C_out), residual (C_out)
 * and forcing (C_in - 2*C_out) channels, element type given by the call's dtype. */
typedef struct swf_standardizers {
    const void *state_mean, *state_std, *resid_mean, *resid_std, *forcing_mean, *forcing_std;
} swf_standardizers;

typedef struct swf_ctx swf_ctx;

const char* swf_last_error(void);
const char* swf_version(void);

/* Create a context for a model on an H x W grid on CUDA device `device`.
 * Replaces ModelConfig::validate_grid (model.hpp:48-52) + the implicit state of forward(). */
int swf_create(const swf_model_cfg* cfg, int grid_h, int grid_w, int device, int precision, swf_ctx** out);
void swf_destroy(swf_ctx* ctx);

/* Window-parallel topology (topology.hpp:74-132): this context is rank `rank` of a wp_a x wp_b
 * window-parallel grid times sp sequence-parallel bands (rank = wp_rank * sp + band). Each WP
 * rank owns whole windows of both the unshifted and the shifted layout; with sp > 1 its windows'
 * rows are split into SP bands by global row phase (window.hpp:67-79), heads into sp groups
 * (heads % sp == 0 and window_px % sp == 0, topology.hpp:95-102). Must precede parameter loading. */
int swf_set_topology(swf_ctx* ctx, int wp_a, int wp_b, int sp, int rank, int ownership);
/* Single-process multi-GPU (SURVEY.md §8(b) swf_set_topology(ctx, wp_a, wp_b, sp, device_ids)): this
 * context becomes rank 0 of a wp_a x wp_b x sp topology whose rank r runs on CUDA device
 * device_ids[r] (device_ids[0] = the context's device; a device may host several ranks). The context
 * creates and owns the other ranks; every call on it (load / init params, forward, forward_hidden,
 * solve_pf_ode, forecast_step[_chunked], rollout_ensemble, backward, training, noise_field) runs all
 * ranks from one host call, each rank on its own host thread, and returns the complete result: each
 * rank writes its owned pixels of the output fields, partial sums (losses, gradients) are added in
 * rank order. Peers are mapped directly (same address space; cudaDeviceEnablePeerAccess across
 * GPUs) -- no IPC and no external process group. The reference-signature forward() / forecast_step()
 * (include/swinflow/b200.hpp) therefore drive every GPU from one thread. Must precede parameter
 * loading. */
int swf_set_topology_devices(swf_ctx* ctx, int wp_a, int wp_b, int sp, int ownership, const int* device_ids);
int swf_group_size(swf_ctx* ctx);                /* ranks driven by this context (1 without a group) */
swf_ctx* swf_group_rank(swf_ctx* ctx, int rank); /* rank context (0 = ctx itself), for per-rank queries */
/* Export this rank's IPC handles (residual buffers x2, barrier flags, attention planes, attention
 * output: 5 x 64 bytes) / map all ranks' handles (world x 320 bytes, rank order). After connecting, the down-projection epilogue
 * stores owner-changed tokens straight into the peer's residual buffer over NVLink (the
 * shifted-layer regroup of send_boundary, simulator.hpp:781-824) and a release/acquire flag
 * barrier over the same mapping orders block boundaries. */
int swf_ipc_handles(swf_ctx* ctx, void* out320);
int swf_connect_peers(swf_ctx* ctx, const void* all_handles);
/* Host-only planning (no GPU): owner rank of every window (row-major window id) and the tokens
 * each rank sends each other rank at a shift_from -> shift_to block boundary (sent[src*world+dst]),
 * i.e. shift_transfer_plan (topology.hpp:149-188) aggregated per rank pair. */
int swf_plan_owners(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int ownership, int* owner);
int swf_plan_tokens(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int sp, int ownership, int rank,
                    long long* pixels); /* pixel of every local token of `rank`, layout 0, device order */
int swf_plan_exchange(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int ownership, int shift_from,
                      int shift_to, long long* sent);

/* Parameters in canonical parameter_arrays order (model.hpp:140-168), each array Eigen
 * column-major, element type dtype. Replaces Parameters<T> / load_params. */
int swf_load_params(swf_ctx* ctx, const void* const* arrays, int n_arrays, int dtype);
int swf_load_params_flat(swf_ctx* ctx, const void* flat, long long count, int dtype);
long long swf_param_count(const swf_model_cfg* cfg); /* parameter_count_formula (model.hpp:118-129) */
/* load_params(base, p) (checkpoint.hpp:84-89 / load_named_arrays :50-80): `base`.manifest (dtype
 * line, then `name RxC offset fnv1a64` per array in canonical order) + `base`.bin, strict name /
 * shape / dtype / checksum checks (rc 3 on any mismatch), streamed into the device repack. */
int swf_load_checkpoint(swf_ctx* ctx, const char* base);
/* The same checks on the host only (no GPU needed). */
int swf_verify_checkpoint(const swf_model_cfg* cfg, const char* base);
/* fnv1a64 of n bytes continuing from h (0xcbf29ce484222325 to start; checkpoint.hpp / chunked_file.cpp
 * checksums), for writers of either format. Host only. */
uint64_t swf_fnv1a64(const void* data, size_t n, uint64_t h);
/* parameter_arrays (model.hpp:140-168): name and shape (rows x cols, column-major) of canonical
 * array i; rc 2 past the last array. */
int swf_param_array(const swf_model_cfg* cfg, int i, char* name, int name_len, long long* rows, long long* cols);
/* init_parameters (model.hpp:185-209) generated on the device with the reference counter RNG:
 * mode 0 = init_parameters(seed); 1 = init_parameters_random(seed, scale) (model.hpp:213-223);
 * 2 = init_parameters(seed) + scale*N(0,1) added only to the arrays it leaves at zero except the
 * encode/time biases (ada.w, ada.b, decode.w, decode.b) -- synthetic benchmark weights with live
 * AdaLN and decode paths. */
int swf_init_params(swf_ctx* ctx, uint64_t seed, int mode, double scale);

/* forward(p, input, t, H, W) (swin.hpp:327-368): input C_in x N, output C_out x N, host memory.
 * Under a multi-rank topology each rank writes only the pixels it owns (see swf_owned_pixels). */
int swf_forward(swf_ctx* ctx, const void* input, double t, void* output, int dtype);
/* forward() stopped after the first n_blocks blocks (0 = right after the encode, n_blocks = all
 * blocks, before the decode): the FP32 residual stream (ForwardCache::blocks[n_blocks].x_in /
 * the final x of swin.hpp:273-291,344-362) for the listed pixels, hidden = n_pix x hidden_dim.
 * Under a multi-rank topology only the rows of pixels this rank owns are written. */
int swf_forward_hidden(swf_ctx* ctx, const void* input, double t, int n_blocks, const long long* pixels,
                       long long n_pix, float* hidden, int dtype);
/* block_window_forward(bp, ada, layout, wy, wx, n_heads, wc) (swin.hpp:306-325) with the context's
 * block `block` (its layout: shift 0 on even, w/2 on odd blocks, window.hpp:83-85) and ada vectors
 * at time t: x_in / x_out are one window's h x s_w residual columns (s_w = w*w tokens in canonical
 * r*w + c order, column-major = [token][h]). Single-rank contexts. */
int swf_block_window_forward(swf_ctx* ctx, int block, int wy, int wx, double t, const void* x_in, void* x_out,
                             int dtype);
/* Same, on device pointers (fp32, [N][C]) on the context stream, without synchronising;
 * numerics flags are checked by swf_sync(). */
int swf_forward_device(swf_ctx* ctx, const float* d_input, double t, float* d_output);
/* backward(p, fc, d_output) (swin.hpp:419-467) of forward(p, input, t) (f3, FP32 validation mode,
 * one rank): parameter gradients in the canonical parameter_arrays order and column-major layout
 * (model.hpp:140-168; swf_param_count elements) and, if d_input is not NULL, the input gradient
 * (C_in x N). The forward is re-run with its block inputs saved; each block's internals are
 * recomputed from them in the backward (no s x s probabilities are stored). */
int swf_backward(swf_ctx* ctx, const void* input, double t, const void* d_output, void* grads, void* d_input,
                 int dtype);
/* Arithmetic of the backward's linears (not a reference interface; the reference backward runs in T,
 * swin.hpp:370-467): SWF_PREC_FP32 (default, FP32 validation mode, SIMT) or SWF_PREC_BF16 -- the
 * data and weight gradients of the QKV, out, gate/up and down projections as tcgen05 GEMMs with bf16
 * operands and fp32 accumulation (weight gradients with MN-major operands, K = tokens). Applies to
 * swf_backward, swf_diffusion_loss_sample and the training entry points; hidden_dim and ffn_dim must
 * be multiples of 8. */
int swf_set_backward_precision(swf_ctx* ctx, int precision);

/* LossWeights (grid.hpp:76-96): alpha_row = per-row latitude weights (H entries, unit mean),
 * kappa = per-variable weights (C_out entries, > 0); element type given by the call's dtype. */
typedef struct swf_loss_weights {
    const void *alpha_row, *kappa;
} swf_loss_weights;
/* diffusion_loss_sample(p, sb, w, dc, t_key, z, pos_enc, H, W) (diffusion.hpp:168-192), FP32
 * validation mode, one rank: t from sample_noise_draw(t_key), x_t / v_t from the standardized
 * residual target x0 (C_out x N) and noise z (C_out x N), the weighted v-prediction loss into *loss
 * and, if grads is not NULL, the parameter gradients (canonical order, swf_param_count elements). */
int swf_diffusion_loss_sample(swf_ctx* ctx, const void* x_prev, const void* x0, const void* forcings,
                              const swf_loss_weights* w, const swf_diffusion_cfg* dc, uint64_t t_key, const void* z,
                              double* loss, void* grads, int dtype);
/* One microbatch of reference_train_step (simulator.hpp:50-86): z = noise_field(seeds, sample_id)
 * and t_key = SeedProtocol::t_key(sample_id) (rng.hpp:72-80) for run_seed, loss into *loss, the
 * gradient added to the device accumulator. swf_train_reset zeroes it; swf_train_grads exposes it
 * (FP32 device pointer + element count) for an in-place all-reduce across data-parallel ranks;
 * swf_train_read copies it out multiplied by scale. */
int swf_train_accumulate(swf_ctx* ctx, const void* x_prev, const void* x0, const void* forcings,
                         const swf_loss_weights* w, const swf_diffusion_cfg* dc, uint64_t run_seed,
                         uint64_t sample_id, double* loss, int dtype);
int swf_train_reset(swf_ctx* ctx);
int swf_train_grads(swf_ctx* ctx, float** dev_ptr, long long* n);
int swf_train_read(swf_ctx* ctx, double scale, void* grads, int dtype);
int swf_sync(swf_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for callers that enqueue their own copies. */
void* swf_stream(swf_ctx* ctx);

/* solve_pf_ode(net, x_init, dc, churn_key) (diffusion.hpp:207-272) with net = the denoiser
 * conditioned on standardized x_prev (C_out x N) and forcings ((C_in-2C_out) x N), as in the
 * forecast_step net lambda (diffusion.hpp:304-311). Host buffers. f_evals may be NULL. */
int swf_solve_pf_ode(swf_ctx* ctx, const void* x_init, const void* x_prev_std, const void* forcings_std,
                     const swf_diffusion_cfg* dc, uint64_t churn_key, void* x_out, int* f_evals, int dtype);
/* forecast_step (diffusion.hpp:295-319): standardize, window-keyed noise z_init, solve, invert
 * the residual standardization and add to x_prev_phys. Host buffers. */
int swf_forecast_step(swf_ctx* ctx, const void* x_prev_phys, const void* forcing_phys,
                      const swf_standardizers* stds, const swf_diffusion_cfg* dc, uint64_t run_seed,
                      uint64_t noise_event, void* out, int dtype);
/* Per-rank input loading (f4; ChunkedReader::read_window_slice, chunked_file.cpp:156-188): forecast_step
 * with x_prev and forcings read from chunked containers (format of write_chunked, chunked_file.cpp:44-99).
 * Each rank reads only the chunks covering its own windows (its SP band rows), with parallel readers,
 * checksum-verified, straight into pinned staging in its local token order. swf_prefetch_chunked starts
 * that read on a background thread (two slots), so the next step's fields load while the current step
 * computes; a forecast call with the same paths consumes the prefetched slot. rc 3 on a checksum /
 * format error, rc 2 on a grid or channel mismatch. */
int swf_prefetch_chunked(swf_ctx* ctx, const char* state_path, const char* forcing_path);
int swf_forecast_step_chunked(swf_ctx* ctx, const char* state_path, const char* forcing_path,
                              const swf_standardizers* stds, const swf_diffusion_cfg* dc, uint64_t run_seed,
                              uint64_t noise_event, void* out, int dtype);
long long swf_last_chunk_reads(swf_ctx* ctx); /* chunks read by the last chunked forecast */

/* The chunked container itself (host only; chunked_file.hpp). Fields are C x (H*W) column-major
 * ([pixel][channel]), as FieldTensor<float>::values. read fills an h x w rect as [h*w][C].
 * A rect outside the grid is rc 2 (the reference's std::out_of_range), a checksum mismatch rc 3
 * (IntegrityError). */
typedef struct swf_chunked swf_chunked;
int swf_chunked_write(const char* path, const float* field, int channels, int height, int width, int chunk_h,
                      int chunk_w);
int swf_chunked_open(const char* path, swf_chunked** out);
void swf_chunked_close(swf_chunked* r);
int swf_chunked_info(swf_chunked* r, int* channels, int* height, int* width, int* chunk_h, int* chunk_w);
int swf_chunked_read(swf_chunked* r, int y0, int x0, int h, int w, float* out);
int swf_chunked_cover(swf_chunked* r, int y0, int x0, int h, int w, long long* n_chunks);
long long swf_chunked_reads(swf_chunked* r);
void swf_chunked_reset_reads(swf_chunked* r);

/* rollout_ensemble (diffusion.hpp:323-339): members x steps, out is members*steps fields
 * (member-major), forcings is steps fields. */
int swf_rollout_ensemble(swf_ctx* ctx, const void* x_init_phys, const void* forcings_phys, int n_members,
                         int n_steps, const swf_standardizers* stds, const swf_diffusion_cfg* dc,
                         uint64_t run_seed, uint64_t rollout_id, void* out, int dtype);

/* Diagnostics: local token count, owned-pixel list (pixel index per local token, window order of
 * the unshifted layout), and the number of kernels launched by the last forward. */
long long swf_local_tokens(swf_ctx* ctx);
int swf_owned_pixels(swf_ctx* ctx, long long* pixels);
long long swf_kernel_launches(swf_ctx* ctx);
/* Per-kernel-class device time from CUDA events recorded on the context stream around each
 * launch while enabled. Classes: 0 encode GEMM, 1 RMS+AdaLN, 2 QKV GEMM, 3 attention, 4 out GEMM,
 * 5 gate/up GEMM, 6 down GEMM, 7 decode GEMM, 8 other. swf_profile resets the counters. */
int swf_profile(swf_ctx* ctx, int enable);
/* CUDA-graph replay of the sampler's 2*S evaluations (default on; not a reference interface):
 * the first solve with a diffusion config runs eagerly, the second captures, later ones replay.
 * Disabled while profiling or while the forward saves activations. */
int swf_set_graphs(swf_ctx* ctx, int enable);
int swf_profile_read(swf_ctx* ctx, double* ms, long long* launches, int n_classes);
int swf_profile_launches(swf_ctx* ctx, int* classes, double* ms, int max_n, int* n_out);
/* Replay one kernel class (1..6 above) reps times back-to-back on the resident buffers of the
 * last forward for block blk; *ms = mean device time per launch (kernel isolation at steady clocks). */
int swf_bench_kernel(swf_ctx* ctx, int kernel_class, int block, int reps, double* ms);
/* Noise field (diffusion.hpp:91-108) for (run_seed, event) into a host C x N buffer (fp32). */
int swf_noise_field(swf_ctx* ctx, uint64_t run_seed, uint64_t event, int channels, double sigma_d, float* out);
/* Leaves of the reference's ops namespace (swin.hpp:49-234), as the SWiPe simulator calls them per
 * sequence band (simulator.hpp:466-506): standalone device calls on host buffers, column-major like
 * the reference (a C x n matrix is n*C floats, token j's C values contiguous). precision selects the
 * BF16 tensor-core or the FP32 SIMT arithmetic.
 *   linear_cols(W, X) = W X           W: out x in (W[k*out + o]), X: in x n, Y: out x n  (swin.hpp:49-54)
 *   prenorm_modulate(x; g, a, b, gate) = gate*((g*x/rms(x))*(1+a)+b), rms with eps 1e-8;
 *                                      a = b = gate = NULL for prenorm_plain      (swin.hpp:72-85,111-123)
 *   swiglu_fwd(x) = W_down (silu(W_gate x) * (W_up x))                              (swin.hpp:228-234)
 * head_attention_fwd's attention core is swf_selftest_attention below (flags 0). */
int swf_op_linear_cols(int device, int precision, const float* W, int out, int in, const float* X, long long n,
                       float* Y);
int swf_op_prenorm_modulate(int device, const float* X, int h, long long n, const float* g, const float* a,
                            const float* b, const float* gate, float* Y);
int swf_op_swiglu_fwd(int device, int precision, const float* W_gate, const float* W_up, const float* W_down,
                      int h, int f, const float* X, long long n, float* Y);
/* Test hook for the backward's tensor-core GEMM (gemm_bf16_general, not a reference interface):
 * C[M][N] (+)= A . B with A = [M][lda] and B = [N][ldb] (K-major, mn_major = 0) or A = [K][lda] and
 * B = [K][ldb] (MN-major, mn_major = 1); operands rounded to bf16, fp32 accumulation. */
int swf_op_gemm_bf16(int device, int mn_major, long long M, long long N, long long K, const float* A, long long lda,
                     const float* B, long long ldb, float* C, long long ldc, int accumulate);
/* Run one bf16 GEMM self-test of the tcgen05 kernel: C = A.B^T on device, returns max |err|
 * against an fp32 SIMT product of the same bf16 operands (used by the parity tests). */
int swf_selftest_gemm(int device, long long M, int N, int K, double* max_abs_err, double* max_ref);
/* Run the windowed attention kernel alone (head_attention_fwd, swin.hpp:161-188) on the windows of
 * an (n_wy*w) x (n_wx*w) grid under cyclic shift `shift` (the last window row seam-masked when
 * shift > 0, window.hpp:107-122): q, k, v are [n_win][heads][w*w][d] fp32 host arrays (rounded to
 * bf16 for SWF_PREC_BF16), o receives [n_win][w*w][heads*d] (head-concatenated, swin.hpp:319-320).
 * flags bit 0 (negative control for the tests): skip the online-softmax O rescale. */
int swf_selftest_attention(int device, int precision, int n_wy, int n_wx, int w, int shift, int heads, int d,
                           const float* q, const float* k, const float* v, float* o, int flags);

#ifdef __cplusplus
}
#endif
#endif /* SWINFLOW_CAPI_H */
