// ctx.cu -- device context, weight repack, the denoiser forward orchestration and the device-
// resident TrigFlow sampler, behind the C-ABI in include/swinflow_capi.h.
//
// Data flow of one forward (reference swin.hpp:327-368), all on one stream:
//   gather(input, pixel -> window order of layout 0)            [HBM]
//   encode GEMM (+bias) -> x (fp32 residual, window order)       [tensor]
//   per block b (layout L_b = shift 0 / w/2, window.hpp:83-85):
//     rms+AdaLN(x) -> xm ; QKV GEMM (+RoPE, head-major scatter) ; attention -> O ;
//     out GEMM (x += W_out O) ; rms+AdaLN(x) -> xm ; gate/up GEMM (+SiLU*up) -> s ;
//     down GEMM (x' = x + W_down s) stored directly in the window order of L_{b+1}
//       -- the window gather/scatter of swin.hpp:356-358 becomes the down-projection's
//          store address, so no standalone permutation pass exists.
//   rms(x) -> xm ; decode GEMM (+bias) -> out (window order of layout 0) ; scatter to pixels
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/swinflow_capi.h"
#include "kernels.cuh"

namespace swf {

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericsError : std::runtime_error {
    explicit NumericsError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {  // common.hpp:33-40 (IoError / IntegrityError)
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
}  // namespace swf
#include "chunk_store.hpp"
namespace swf {
static void require(bool c, const std::string& m) {
    if (!c) throw ConfigError(m);
}

static inline i64 roundup(i64 a, i64 b) { return (a + b - 1) / b * b; }

struct Dims {
    int h, heads, d, f, nb, w, cin, cout, td;
    int hp, fp, cinp;              // K dims padded to 64
    int bn_enc, bn_qkv, bn_out, bn_gu, bn_down, bn_dec;
    int np_enc, np_qkv, np_out, np_gu, np_down, np_dec;  // N dims padded
    int G;                         // gate/up interleave granularity
    int nss;                       // fused-norm partial sums per row (BF16): 2 per N tile of h
};

struct Peer {
    float* x[2];
    int* flags;
    void* qkv;  // attention planes (sequence parallelism: QKV epilogue stores)
    void* xm;   // attention output rows (sequence parallelism: attention epilogue stores)
};

}  // namespace swf

using namespace swf;

struct swf_ctx {
    swf_model_cfg cfg;
    Dims m;
    int H = 0, W = 0;
    i64 N = 0;
    int prec = SWF_PREC_BF16;
    int dev = 0;
    cudaStream_t st = nullptr;
    // topology
    int wp_a = 1, wp_b = 1, sp = 1, rank = 0, world = 1, own = SWF_OWN_CONTIGUOUS;
    int wp_rank = 0, band = 0;  // rank = wp_rank * sp + band
    i64 M = 0;  // local tokens
    std::vector<int> l2g[2];
    int* d_l2g[2] = {nullptr, nullptr};
    int* d_g2rl[2] = {nullptr, nullptr};
    LayMap lay[2];
    bool allocated = false, loaded = false, peers = false;
    // small fp32 parameters
    float *enc_b = nullptr, *g_attn = nullptr, *g_ffn = nullptr, *w_ada_t = nullptr, *b_ada = nullptr;
    float *w_time_t = nullptr, *b_time = nullptr, *g_dec = nullptr, *b_dec = nullptr;
    // GEMM weights [Npad][Kpad] (bf16 or fp32)
    void *w_enc = nullptr, *w_dec = nullptr;
    std::vector<void*> w_qkv, w_out, w_gu, w_down;
    // activations
    float* xbuf[2] = {nullptr, nullptr};
    void *xm = nullptr, *qkv = nullptr, *sbuf = nullptr, *a_in = nullptr;
    float* out_loc = nullptr;
    float *rope_row = nullptr, *rope_col = nullptr, *rope_row_pm = nullptr, *rope_col_pm = nullptr, *feat = nullptr, *emb = nullptr, *six = nullptr;
    int* flags = nullptr;
    int* h_flags = nullptr;
    float* h_feat = nullptr;
    float *in_pix = nullptr, *out_pix = nullptr;
    float** d_xdst[2] = {nullptr, nullptr};
    std::vector<Peer> peer;
    int* bar_flags = nullptr;        // this rank's barrier slots (IPC-exported), one per peer
    int** d_flag_table = nullptr;    // device table: flag array of every rank (peer-mapped)
    void** d_qkv_dst = nullptr;      // device table: attention planes of every rank
    void** d_o_dst = nullptr;        // device table: attention-output (xm) buffer of every rank
    int* d_epoch = nullptr;          // device barrier epoch (advanced by k_peer_barrier; graph-safe)
    int* d_sched = nullptr;          // GEMM dynamic-schedule tile counter (reset before every launch)
    // TMA maps (BF16 path)
    TmaMap tm_ain, tm_xm, tm_s, tm_enc, tm_dec, tm_q, tm_k, tm_k2, tm_vt;
    TmaMap tm_so;  // sbuf viewed as [M][hp] (attention output of the kernel benchmark)
    // fused RMSNorm + AdaLN (BF16): bf16 copy + row partial sums of squares of each residual buffer
    // (inside xbuf[par] at off_xb / off_ss floats), fp32 masters of the folded weights, shift biases
    __nv_bfloat16* xbb[2] = {nullptr, nullptr};
    float* ssb[2] = {nullptr, nullptr};
    float* invr = nullptr;  // [M] 1 / rms of the current normed GEMM's A rows
    i64 off_xb = 0, off_ss = 0;
    TmaMap tm_xb[2];
    std::vector<float*> w_qkv_m, w_gu_m, beta_qkv, beta_gu;
    float* w_dec_m = nullptr;
    std::vector<TmaMap> tm_qkv, tm_out, tm_gu, tm_down;
    long long launches = 0;
    // sampler workspace (allocated lazily)
    float *pe_loc = nullptr, *s_x = nullptr, *s_xmid = nullptr, *s_tmp = nullptr, *s_base = nullptr;
    float *s_cond = nullptr, *s_stats = nullptr;
    std::vector<void*> allocs;
    int nflags = 0;
    // chunked-container input staging (pinned, local token order), two prefetch slots
    struct Staged {
        std::string state_path, forcing_path;
        float *state = nullptr, *forcing = nullptr;  // pinned [M][C_out], [M][C_f]
        unsigned long long reads = 0;
        std::thread th;
        std::exception_ptr err;
        bool pending = false;
        long long seq = 0;
    } staged[2];
    long long staged_seq = 0;
    unsigned long long last_chunk_reads = 0;
    // backward (FP32 validation mode): canonical fp32 parameters in the reference layout, the saved
    // block inputs of the last forward, and work buffers (allocated on first use)
    float* pflat = nullptr;
    std::vector<size_t> poff;
    bool save_x = false;
    float* xsave = nullptr;
    struct Bwd {
        float *dx[2], *dtmp, *xmid, *dxm, *xm1, *obuf, *x2m, *dO, *gu, *act, *dS, *dG, *dU, *dqkv, *dplanes, *stats,
            *rms, *d6, *demb, *zero, *gflat, *din, *npart;
    } bw = {};
    bool bw_alloc = false;
    // swf_set_backward_precision(BF16): the backward's linears on the tensor cores (bf16 operand
    // copies in bt_a / bt_b, allocated with the work buffers)
    bool bwd_tc = false;
    __nv_bfloat16 *bt_a = nullptr, *bt_b = nullptr;
    float* bt_c = nullptr;  // plain fp32 product of the two-pass linears (gemm_f32_ctx)
    size_t bt_c_n = 0;
    // tensor-core attention of the BF16 training mode: bf16 q / k planes + V^T, bf16 output rows
    __nv_bfloat16 *bt_qkv = nullptr, *bt_o = nullptr;
    float *bt_lse = nullptr, *bt_D = nullptr;
    void** bench_otab = nullptr;  // swf_bench_kernel's attention output table  // attention rows' log2-sum-exp (forward) and D (backward)
    AttnBwdStreams bt_ws;  // worker streams / scratch of the tensor-core attention backward
    void** d_bt_o = nullptr;
    TmaMap bt_tm_q, bt_tm_k, bt_tm_k2, bt_tm_vt, bt_tm_o;
    // diffusion training loss (FP32 validation mode): residual target x0, noise z, velocity target v,
    // loss weights, per-block loss partials, and the gradient accumulator of the training step
    struct Train {
        float *x0, *z, *v, *kappa, *alpha, *gacc;
        double *part, *h_part;
    } tr = {};
    bool tr_alloc = false;
    // per-kernel-class CUDA-event timing (bench roofline): class id -> accumulated ms / launches
    bool prof = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_ev;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    double prof_ms[16] = {0};
    long long prof_n[16] = {0};
    // CUDA graph of solve_pf_ode's 2*S evaluations (+ sampler updates and churn), keyed on the
    // diffusion config; the churn key is read from device memory so one graph serves every
    // member / step of a rollout. First call with a new key runs eagerly, the second captures.
    bool graphs = true;
    cudaGraphExec_t solve_exec = nullptr;
    swf_diffusion_cfg graph_dc = {};
    int graph_seen = 0;  // 1: key seen once (eager), 2: captured
    long long graph_launches = 0;
    u64* d_churn_key = nullptr;
    u64* h_churn_key = nullptr;  // pinned staging
    // test hook (swf_forward_hidden): stop the forward after this many blocks (-1: full forward);
    // the residual then sits in xbuf[hid_cur] in the local order of layout hid_par
    int stop_after = -1, hid_cur = 0, hid_par = 0;
    // single-process multi-GPU group (swf_set_topology_devices): the root context (rank 0) owns the
    // contexts of ranks 1..world-1 and fans every call out to them; peers are mapped directly
    // (peer access, same address space) instead of through CUDA IPC
    std::vector<swf_ctx*> kids;
    bool ipc_mapped = false;
    std::vector<long long> owned_pix;  // pixel of every local token (layout 0, local order)
    float* h_stage = nullptr;          // pinned staging for owned-row readback [M][max C]
    size_t h_stage_n = 0;
    // per-call device buffers of the sampler entry points, kept across calls (grow-only)
    std::vector<std::pair<float*, size_t>> scratch;
};

namespace {

thread_local std::string g_err;

// Zeroed device allocation owned by the context. The zero fill is complete on return: cudaMemset on
// the legacy stream is not ordered with the context's non-blocking stream (and may still be pending
// when cudaMemset returns), so a fill racing the first writes of the new buffer on c->st could zero
// them (seen as a zero loss on the first training call with two ranks on one GPU).
template <class T>
T* dalloc(swf_ctx* c, size_t n) {
    void* p = nullptr;
    SWF_CUDA(cudaMalloc(&p, n * sizeof(T) + 256));
    c->allocs.push_back(p);
    SWF_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T) + 256, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
    return static_cast<T*>(p);
}

void dfree(swf_ctx* c, void* p) {
    for (size_t i = 0; i < c->allocs.size(); ++i)
        if (c->allocs[i] == p) {
            SWF_CUDA(cudaFree(p));
            c->allocs.erase(c->allocs.begin() + i);
            return;
        }
}

// Grow-only device scratch slot k: the per-call buffers of the host-buffer entry points (staged
// forcings, outputs, rollout states, readback rows) are allocated once, not cudaMalloc'd / cudaFree'd
// per call (cudaFree synchronises the whole device -- other ranks of a single-process group included).
enum Scratch { SC_FORC, SC_OUT, SC_RX0, SC_RXA, SC_RXB, SC_RFORC, SC_NOISE, SC_NOISE_PIX, SC_PIX, SC_ROWS, SC_WIN, SC_N };
void* scratch(swf_ctx* c, int k, size_t bytes) {
    if (c->scratch.size() < SC_N) c->scratch.resize(SC_N, {nullptr, 0});
    auto& s = c->scratch[k];
    if (s.second < bytes) {
        if (s.first) {
            SWF_CUDA(cudaStreamSynchronize(c->st));
            dfree(c, s.first);
        }
        s.first = dalloc<float>(c, (bytes + 3) / 4);
        s.second = bytes;
    }
    return s.first;
}
float* scratch_f(swf_ctx* c, int k, size_t n) { return static_cast<float*>(scratch(c, k, n * 4)); }

// Host -> device copy complete on return and ordered with the context stream (a legacy-stream
// cudaMemcpy from pageable memory may return before its DMA lands, unordered with c->st).
void h2d_sync(swf_ctx* c, void* dst, const void* src, size_t bytes) {
    SWF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
}

size_t esize(const swf_ctx* c) { return c->prec == SWF_PREC_BF16 ? 2 : 4; }

void* talloc(swf_ctx* c, size_t n) {
    return c->prec == SWF_PREC_BF16 ? static_cast<void*>(dalloc<__nv_bfloat16>(c, n))
                                    : static_cast<void*>(dalloc<float>(c, n));
}

Dims make_dims(const swf_model_cfg& cf, int prec) {
    Dims m;
    m.h = cf.hidden_dim;
    m.heads = cf.n_heads;
    m.d = cf.hidden_dim / cf.n_heads;
    m.f = cf.ffn_dim;
    m.nb = cf.n_layers * cf.blocks_per_layer;
    m.w = cf.window_px;
    m.cin = cf.in_channels;
    m.cout = cf.out_channels;
    m.td = cf.time_dim > 0 ? cf.time_dim : cf.hidden_dim;
    m.hp = int(roundup(m.h, 64));
    m.fp = int(roundup(m.f, 64));
    m.cinp = int(roundup(m.cin, 64));
    auto bn = [&](int n) { return (prec == SWF_PREC_BF16 && n % 256 == 0) ? 256 : 128; };
    m.bn_enc = bn(m.h);
    m.bn_qkv = bn(3 * m.h);
    m.bn_out = bn(m.h);
    m.bn_down = bn(m.h);
    m.bn_dec = 128;
    m.np_enc = int(roundup(m.h, m.bn_enc));
    m.np_qkv = int(roundup(3 * m.h, m.bn_qkv));
    m.np_out = int(roundup(m.h, m.bn_out));
    m.np_down = int(roundup(m.h, m.bn_down));
    m.np_dec = int(roundup(m.cout, 128));
    m.nss = prec == SWF_PREC_BF16 ? 2 * (m.np_out / m.bn_out) : 0;
    if (prec == SWF_PREC_BF16) {
        m.bn_gu = (2 * m.f) % 256 == 0 ? 256 : 128;
        m.G = m.bn_gu / 2;
        m.np_gu = int(roundup(2 * m.f, m.bn_gu));
    } else {
        m.bn_gu = 128;
        m.G = 4;
        m.np_gu = int(roundup(2 * roundup(m.f, 4), 128));
    }
    return m;
}

void validate_model(const swf_model_cfg& c, int H, int W, int prec) {
    require(c.hidden_dim > 0 && c.n_heads > 0 && c.ffn_dim > 0 && c.n_layers > 0, "model: dims must be positive");
    require(c.blocks_per_layer >= 1, "model: blocks_per_layer must be >= 1");
    require(c.hidden_dim % c.n_heads == 0, "model: hidden_dim must divide by n_heads");
    require((c.hidden_dim / c.n_heads) % 4 == 0, "model: head_dim must be divisible by 4 (axial rotary pairs)");
    require(c.in_channels > 0 && c.out_channels > 0, "model: channel counts must be positive");
    require(c.in_channels % 2 == 0, "model: in_channels must be even (positional encoding split)");
    require(c.window_px > 0, "model: window size must be positive");
    require(H > 0 && W > 0 && H % c.window_px == 0 && W % c.window_px == 0, "model: grid not divisible by window size");
    require(prec == SWF_PREC_BF16 || prec == SWF_PREC_FP32, "precision must be SWF_PREC_BF16 or SWF_PREC_FP32");
    if (prec == SWF_PREC_BF16) {
        const int d = c.hidden_dim / c.n_heads;
        require(c.hidden_dim % 128 == 0 && c.ffn_dim % 128 == 0,
                "BF16 path: hidden_dim and ffn_dim must be multiples of 128 (use SWF_PREC_FP32 otherwise)");
        require(d == 32 || d == 64 || d == 128, "BF16 path: head_dim must be 32, 64 or 128");
        require(c.window_px % 4 == 0, "BF16 path: window_px must be a multiple of 4 (16-byte TMA row pitch of V^T)");
    }
}

// ------------------------------------------------------------------ weight repack
// dst[row(o)][k] = src[k*out + o] (Eigen col-major W(out x in) -> K-major rows), optional
// gate/up interleave: row(o) = (o/G)*2G + part*G + o%G.
template <class T>
__global__ void k_repack(const float* __restrict__ src, int out, int in, T* __restrict__ dst, int ld, int G,
                         int part) {
    const i64 total = i64(out) * in;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const int o = int(e / in);
        const int k = int(e - i64(o) * in);
        const int row = G > 0 ? (o / G) * 2 * G + part * G + (o % G) : o;
        const float v = src[i64(k) * out + o];
        if constexpr (sizeof(T) == 2)
            dst[i64(row) * ld + k] = __float2bfloat16_rn(v);
        else
            dst[i64(row) * ld + k] = v;
    }
}

void repack(swf_ctx* c, const float* d_src, int out, int in, void* dst, int ld, int G, int part, bool force_f32) {
    const i64 total = i64(out) * in;
    int grid = int(std::min<i64>((total + 255) / 256, 148 * 32));
    if (c->prec == SWF_PREC_BF16 && !force_f32)
        k_repack<__nv_bfloat16><<<grid, 256, 0, c->st>>>(d_src, out, in, static_cast<__nv_bfloat16*>(dst), ld, G, part);
    else
        k_repack<float><<<grid, 256, 0, c->st>>>(d_src, out, in, static_cast<float*>(dst), ld, G, part);
    SWF_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ topology / layouts
void build_layouts(swf_ctx* c) {
    const Dims& m = c->m;
    const int ny = c->H / m.w, nx = c->W / m.w, nwin = ny * nx;
    require(ny % c->wp_a == 0, "topology: window rows " + std::to_string(ny) + " not divisible by WP grid A=" +
                                   std::to_string(c->wp_a));
    require(nx % c->wp_b == 0, "topology: window cols " + std::to_string(nx) + " not divisible by WP grid B=" +
                                   std::to_string(c->wp_b));
    const int nwp = c->wp_a * c->wp_b;
    // glob2rl packs (WP rank << 16) | local window (LayMap): local window counts must fit 16 bits
    require((nwin + nwp - 1) / nwp < 65536, "topology: " + std::to_string(nwin / nwp) +
                                                " windows per rank exceed the 65535 the window maps address");
    std::vector<int> g2rl(nwin);
    for (int par = 0; par < 2; ++par) {
        c->l2g[par].clear();
        std::vector<int> cnt(nwp, 0);
        for (int wy = 0; wy < ny; ++wy)
            for (int wx = 0; wx < nx; ++wx) {
                int oa, ob;
                if (c->own == SWF_OWN_ROUND_ROBIN) {  // window_owner, topology.hpp:107-109
                    oa = wy % c->wp_a;
                    ob = wx % c->wp_b;
                } else {  // contiguous window blocks
                    oa = wy / (ny / c->wp_a);
                    ob = wx / (nx / c->wp_b);
                }
                const int r = oa * c->wp_b + ob;  // WP rank (shared by its SP ranks)
                const int gw = wy * nx + wx;
                g2rl[gw] = (r << 16) | cnt[r]++;
                if (r == c->wp_rank) c->l2g[par].push_back(gw);
            }
        if (!c->d_l2g[par]) {
            c->d_l2g[par] = dalloc<int>(c, nwin);
            c->d_g2rl[par] = dalloc<int>(c, nwin);
        }
        h2d_sync(c, c->d_l2g[par], c->l2g[par].data(), sizeof(int) * c->l2g[par].size());
        h2d_sync(c, c->d_g2rl[par], g2rl.data(), sizeof(int) * nwin);
        LayMap& L = c->lay[par];
        L.g = make_lay(c->H, c->W, m.w, par == 0 ? 0 : m.w / 2);
        L.nloc = int(c->l2g[par].size());
        L.sp = c->sp;
        L.band = c->band;
        L.loc2glob = c->d_l2g[par];
        L.glob2rl = c->d_g2rl[par];
    }
    c->M = i64(c->lay[0].nloc) * c->lay[0].s_loc();
}

// RoPE cos/sin tables: angle = T(pos * omega_j) in double then cast (rope.hpp:19-31), trig in
// float (rope.hpp:38) -- identical to the reference's float instantiation.
void build_rope(swf_ctx* c) {
    const Dims& m = c->m;
    const int q4 = m.d / 4;
    auto table = [&](int npos) {  // [pair j][position] (cos, sin)
        std::vector<float> t(size_t(npos) * q4 * 2);
        for (int j = 0; j < q4; ++j) {
            const double om = std::pow(10000.0, -double(j) / q4);
            for (int pos = 0; pos < npos; ++pos) {
                const float a = static_cast<float>(pos * om);
                t[(size_t(j) * npos + pos) * 2] = std::cos(a);
                t[(size_t(j) * npos + pos) * 2 + 1] = std::sin(a);
            }
        }
        return t;
    };
    const auto tr = table(c->H + m.w), tc = table(c->W + m.w);
    c->rope_row = dalloc<float>(c, tr.size());
    c->rope_col = dalloc<float>(c, tc.size());
    h2d_sync(c, c->rope_row, tr.data(), tr.size() * 4);
    h2d_sync(c, c->rope_col, tc.data(), tc.size() * 4);
    // position-major copies for the tensor-core QKV epilogue: a row's 16 pairs are one 128-B line
    auto pm = [&](const std::vector<float>& t, int npos) {
        std::vector<float> o(t.size());
        for (int j = 0; j < q4; ++j)
            for (int pos = 0; pos < npos; ++pos)
                for (int k = 0; k < 2; ++k) o[(size_t(pos) * q4 + j) * 2 + k] = t[(size_t(j) * npos + pos) * 2 + k];
        return o;
    };
    const auto trp = pm(tr, c->H + m.w), tcp = pm(tc, c->W + m.w);
    c->rope_row_pm = dalloc<float>(c, trp.size());
    c->rope_col_pm = dalloc<float>(c, tcp.size());
    h2d_sync(c, c->rope_row_pm, trp.data(), trp.size() * 4);
    h2d_sync(c, c->rope_col_pm, tcp.data(), tcp.size() * 4);
}

void allocate(swf_ctx* c) {
    if (c->allocated) return;
    const Dims& m = c->m;
    build_layouts(c);
    build_rope(c);
    const i64 M = c->M;
    {  // pixel of every local token (layout 0): owned windows, the band's rows ascending, columns
        const LayMap& L = c->lay[0];
        const int w = m.w, R = w / c->sp;
        c->owned_pix.clear();
        c->owned_pix.reserve(size_t(M));
        for (int gw : c->l2g[0])
            for (int k = 0; k < R; ++k)
                for (int cc = 0; cc < w; ++cc)
                    c->owned_pix.push_back(L.g.win_to_pix(i64(gw) * w * w + i64(L.band_row(c->band, k)) * w + cc));
    }
    if (c->prec == SWF_PREC_BF16) {  // [x fp32 M x h][x bf16 M x hp][sum-of-squares partials M x nss]
        c->off_xb = M * m.h;
        c->off_ss = c->off_xb + M * m.hp / 2;
        for (int par = 0; par < 2; ++par) {
            c->xbuf[par] = dalloc<float>(c, size_t(c->off_ss) + size_t(M) * m.nss);
            c->xbb[par] = reinterpret_cast<__nv_bfloat16*>(c->xbuf[par] + c->off_xb);
            c->ssb[par] = c->xbuf[par] + c->off_ss;
        }
    } else {
        c->xbuf[0] = dalloc<float>(c, size_t(M) * m.h);
        c->xbuf[1] = dalloc<float>(c, size_t(M) * m.h);
    }
    c->xm = talloc(c, size_t(M) * m.hp);
    c->qkv = talloc(c, size_t(3) * M * m.h);
    c->sbuf = talloc(c, size_t(M) * m.fp);
    c->a_in = talloc(c, size_t(M) * m.cinp);
    c->out_loc = dalloc<float>(c, size_t(M) * m.cout);
    c->feat = dalloc<float>(c, m.td);
    c->emb = dalloc<float>(c, m.td);
    c->six = dalloc<float>(c, size_t(m.nb) * 6 * m.h);
    c->nflags = m.nb + 2 + 4096;
    c->flags = dalloc<int>(c, c->nflags);
    SWF_CUDA(cudaMallocHost(&c->h_flags, sizeof(int) * c->nflags));
    SWF_CUDA(cudaMallocHost(&c->h_feat, sizeof(float) * m.td));
    c->in_pix = dalloc<float>(c, size_t(c->N) * m.cin);
    c->out_pix = dalloc<float>(c, size_t(c->N) * m.cout);
    // weights
    c->enc_b = dalloc<float>(c, m.h);
    c->g_attn = dalloc<float>(c, size_t(m.nb) * m.h);
    c->g_ffn = dalloc<float>(c, size_t(m.nb) * m.h);
    c->w_ada_t = dalloc<float>(c, size_t(m.nb) * 6 * m.h * m.td);
    c->b_ada = dalloc<float>(c, size_t(m.nb) * 6 * m.h);
    c->w_time_t = dalloc<float>(c, size_t(m.td) * m.td);
    c->b_time = dalloc<float>(c, m.td);
    c->g_dec = dalloc<float>(c, m.h);
    c->b_dec = dalloc<float>(c, m.np_dec);
    c->w_enc = talloc(c, size_t(m.np_enc) * m.cinp);
    c->w_dec = talloc(c, size_t(m.np_dec) * m.hp);
    for (int b = 0; b < m.nb; ++b) {
        c->w_qkv.push_back(talloc(c, size_t(m.np_qkv) * m.hp));
        c->w_out.push_back(talloc(c, size_t(m.np_out) * m.hp));
        c->w_gu.push_back(talloc(c, size_t(m.np_gu) * m.hp));
        c->w_down.push_back(talloc(c, size_t(m.np_down) * m.fp));
    }
    if (c->prec == SWF_PREC_BF16) {
        for (int b = 0; b < m.nb; ++b) {
            c->w_qkv_m.push_back(dalloc<float>(c, size_t(m.np_qkv) * m.hp));
            c->w_gu_m.push_back(dalloc<float>(c, size_t(m.np_gu) * m.hp));
            c->beta_qkv.push_back(dalloc<float>(c, size_t(m.np_qkv)));
            c->beta_gu.push_back(dalloc<float>(c, size_t(m.np_gu)));
        }
        c->w_dec_m = dalloc<float>(c, size_t(m.np_dec) * m.hp);
        c->invr = dalloc<float>(c, size_t(M));
    }
    // destination tables for the fused down-projection store (own buffer unless peers connect)
    c->bar_flags = dalloc<int>(c, 64);
    c->d_flag_table = dalloc<int*>(c, 8);
    c->d_epoch = dalloc<int>(c, 1);
    c->d_sched = dalloc<int>(c, 1);
    c->d_churn_key = dalloc<u64>(c, 1);
    SWF_CUDA(cudaMallocHost(&c->h_churn_key, sizeof(u64)));
    c->peer.assign(c->world, Peer{{nullptr, nullptr}, nullptr, nullptr, nullptr});
    c->peer[c->rank].x[0] = c->xbuf[0];
    c->peer[c->rank].x[1] = c->xbuf[1];
    c->peer[c->rank].flags = c->bar_flags;
    c->peer[c->rank].qkv = c->qkv;
    c->peer[c->rank].xm = c->xm;
    c->d_qkv_dst = dalloc<void*>(c, 8);
    c->d_o_dst = dalloc<void*>(c, 8);
    {
        std::vector<void*> t(8, nullptr), o(8, nullptr);
        t[c->rank] = c->qkv;
        o[c->rank] = c->xm;
        h2d_sync(c, c->d_qkv_dst, t.data(), sizeof(void*) * 8);
        h2d_sync(c, c->d_o_dst, o.data(), sizeof(void*) * 8);
    }
    for (int par = 0; par < 2; ++par) {
        c->d_xdst[par] = dalloc<float*>(c, 8);
        std::vector<float*> t(8, nullptr);
        for (int r = 0; r < c->world; ++r) t[r] = c->peer[r].x[par];
        h2d_sync(c, c->d_xdst[par], t.data(), sizeof(float*) * 8);
    }
    if (c->prec == SWF_PREC_BF16) {
        make_tma_bf16(&c->tm_ain, c->a_in, M, m.cinp, 128);
        make_tma_bf16(&c->tm_xm, c->xm, M, m.hp, 128);
        make_tma_bf16(&c->tm_xb[0], c->xbb[0], M, m.hp, 128);
        make_tma_bf16(&c->tm_xb[1], c->xbb[1], M, m.hp, 128);
        make_tma_bf16(&c->tm_s, c->sbuf, M, m.fp, 128);
        make_tma_bf16(&c->tm_so, c->sbuf, M, m.hp, 128);
        make_tma_bf16(&c->tm_enc, c->w_enc, m.np_enc, m.cinp, m.bn_enc / 2);
        {
            // attention operands: q / k planes [rows][d] (box d<=64 x 128 rows), V^T [rows][s] (64 x d)
            const int sw = m.d >= 64 ? 128 : 2 * m.d;
            const int hl = m.heads / c->sp;  // heads of this rank's group
            const i64 rows_qk = i64(c->lay[0].nloc) * hl * m.w * m.w;  // (window, head, token) rows of d
            const char* qb = static_cast<const char*>(c->qkv);
            make_tma_bf16_2d(&c->tm_q, qb, rows_qk, m.d, sw / 2, 128, sw);
            // K and V^T tiles are fetched half per CTA of a 2-CTA cluster and multicast (k_attn.cu)
            make_tma_bf16_2d(&c->tm_k, qb + size_t(M) * m.h * 2, rows_qk, m.d, sw / 2, 64, sw);
            make_tma_bf16_2d(&c->tm_k2, qb + size_t(M) * m.h * 2, rows_qk, m.d, sw / 2, 32, sw);
            make_tma_bf16_2d(&c->tm_vt, qb + size_t(2) * M * m.h * 2, i64(c->lay[0].nloc) * hl * m.d,
                             i64(m.w) * m.w, 64, m.d / 2, 128);
        }
        make_tma_bf16(&c->tm_dec, c->w_dec, m.np_dec, m.hp, m.bn_dec / 2);
        c->tm_qkv.resize(m.nb);
        c->tm_out.resize(m.nb);
        c->tm_gu.resize(m.nb);
        c->tm_down.resize(m.nb);
        for (int b = 0; b < m.nb; ++b) {
            make_tma_bf16(&c->tm_qkv[b], c->w_qkv[b], m.np_qkv, m.hp, m.bn_qkv / 2);
            make_tma_bf16(&c->tm_out[b], c->w_out[b], m.np_out, m.hp, m.bn_out / 2);
            make_tma_bf16(&c->tm_gu[b], c->w_gu[b], m.np_gu, m.hp, m.bn_gu / 2);
            make_tma_bf16(&c->tm_down[b], c->w_down[b], m.np_down, m.fp, m.bn_down / 2);
        }
    }
    SWF_CUDA(cudaDeviceSynchronize());
    c->allocated = true;
}

// ------------------------------------------------------------------ parameter load
// Canonical array list (model.hpp:140-168): (rows, cols) of every array in order.
std::vector<std::pair<i64, i64>> param_shapes(const Dims& m) {
    std::vector<std::pair<i64, i64>> v;
    v.push_back({m.h, m.cin});
    v.push_back({m.h, 1});
    for (int b = 0; b < m.nb; ++b) {
        v.push_back({3 * m.h, m.h});
        v.push_back({m.h, m.h});
        v.push_back({m.h, 1});
        v.push_back({m.h, 1});
        v.push_back({m.f, m.h});
        v.push_back({m.f, m.h});
        v.push_back({m.h, m.f});
        v.push_back({6 * m.h, m.td});
        v.push_back({6 * m.h, 1});
    }
    v.push_back({m.td, m.td});
    v.push_back({m.td, 1});
    v.push_back({m.h, 1});
    v.push_back({m.cout, m.h});
    v.push_back({m.cout, 1});
    return v;
}

// Consume arrays in canonical order from `next(ai, n)` (device fp32, Eigen col-major) and repack.
template <class Next>
void load_params_from(swf_ctx* c, Next&& next) {
    allocate(c);
    const Dims& m = c->m;
    int ai = 0;
    if (c->prec == SWF_PREC_FP32 && !c->pflat) {  // the backward reads the reference-layout weights
        size_t tot = 0;
        c->poff.clear();
        for (const auto& sh : param_shapes(m)) {
            c->poff.push_back(tot);
            tot += size_t(sh.first * sh.second);
        }
        c->poff.push_back(tot);
        c->pflat = dalloc<float>(c, tot);
    }
    auto up = [&](size_t n) -> float* {
        float* src = next(ai, n);
        if (c->pflat)
            SWF_CUDA(cudaMemcpyAsync(c->pflat + c->poff[ai], src, n * 4, cudaMemcpyDeviceToDevice, c->st));
        ++ai;
        return src;
    };
    const bool bf = c->prec == SWF_PREC_BF16;
    auto copy_vec = [&](float* dst, size_t n) {
        float* s = up(n);
        SWF_CUDA(cudaMemcpyAsync(dst, s, n * 4, cudaMemcpyDeviceToDevice, c->st));
    };
    repack(c, up(size_t(m.h) * m.cin), m.h, m.cin, c->w_enc, m.cinp, 0, 0, false);  // encode.w (h x C_in)
    copy_vec(c->enc_b, m.h);
    for (int b = 0; b < m.nb; ++b) {
        {
            float* src = up(size_t(3) * m.h * m.h);
            repack(c, src, 3 * m.h, m.h, c->w_qkv[b], m.hp, 0, 0, false);
            if (bf) repack(c, src, 3 * m.h, m.h, c->w_qkv_m[b], m.hp, 0, 0, true);
        }
        repack(c, up(size_t(m.h) * m.h), m.h, m.h, c->w_out[b], m.hp, 0, 0, false);
        copy_vec(c->g_attn + size_t(b) * m.h, m.h);
        copy_vec(c->g_ffn + size_t(b) * m.h, m.h);
        for (int part = 0; part < 2; ++part) {  // gate, up (interleaved per G rows)
            float* src = up(size_t(m.f) * m.h);
            repack(c, src, m.f, m.h, c->w_gu[b], m.hp, m.G, part, false);
            if (bf) repack(c, src, m.f, m.h, c->w_gu_m[b], m.hp, m.G, part, true);
        }
        repack(c, up(size_t(m.h) * m.f), m.h, m.f, c->w_down[b], m.fp, 0, 0, false);
        repack(c, up(size_t(6) * m.h * m.td), 6 * m.h, m.td, c->w_ada_t + size_t(b) * 6 * m.h * m.td, m.td, 0, 0,
               true);
        copy_vec(c->b_ada + size_t(b) * 6 * m.h, size_t(6) * m.h);
    }
    repack(c, up(size_t(m.td) * m.td), m.td, m.td, c->w_time_t, m.td, 0, 0, true);
    copy_vec(c->b_time, m.td);
    copy_vec(c->g_dec, m.h);
    {
        float* src = up(size_t(m.cout) * m.h);
        repack(c, src, m.cout, m.h, c->w_dec, m.hp, 0, 0, false);
        if (bf) repack(c, src, m.cout, m.h, c->w_dec_m, m.hp, 0, 0, true);
    }
    copy_vec(c->b_dec, m.cout);
    SWF_CUDA(cudaStreamSynchronize(c->st));
    c->loaded = true;
}

size_t max_array(const Dims& m) {
    size_t mx = 0;
    for (const auto& s : param_shapes(m)) mx = std::max(mx, size_t(s.first * s.second));
    return mx;
}

void load_params(swf_ctx* c, const void* const* arrays, int n_arrays, int dtype) {
    allocate(c);
    const Dims& m = c->m;
    const int expect = 2 + 9 * m.nb + 5;
    require(n_arrays == expect, "load_params: expected " + std::to_string(expect) + " arrays, got " +
                                    std::to_string(n_arrays));
    require(dtype == SWF_F32 || dtype == SWF_F64, "load_params: dtype must be SWF_F32 or SWF_F64");
    float* stage = nullptr;
    SWF_CUDA(cudaMalloc(&stage, max_array(m) * sizeof(float)));
    std::vector<float> hb;
    load_params_from(c, [&](int ai, size_t n) -> float* {
        SWF_CUDA(cudaStreamSynchronize(c->st));  // staging buffer reuse
        const void* src = arrays[ai];
        require(src != nullptr, "load_params: null array pointer");
        const float* f32;
        if (dtype == SWF_F64) {
            hb.resize(n);
            const double* d = static_cast<const double*>(src);
            for (size_t i = 0; i < n; ++i) hb[i] = static_cast<float>(d[i]);
            f32 = hb.data();
        } else {
            f32 = static_cast<const float*>(src);
        }
        SWF_CUDA(cudaMemcpyAsync(stage, f32, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
        return stage;
    });
    SWF_CUDA(cudaFree(stage));
}

// ------------------------------------------------------------------ checkpoints (checkpoint.hpp:29-89)
u64 fnv1a64(const void* data, size_t n, u64 h = 0xcbf29ce484222325ULL) {  // src/chunked_file.cpp:33-41
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

std::vector<std::string> param_names(const Dims& m) {  // parameter_arrays names (model.hpp:140-168)
    std::vector<std::string> v{"encode.w", "encode.b"};
    for (int b = 0; b < m.nb; ++b)
        for (const char* n : {"qkv.w", "out.w", "rms_attn.g", "rms_ffn.g", "gate.w", "up.w", "down.w", "ada.w", "ada.b"})
            v.push_back("block" + std::to_string(b) + "." + n);
    for (const char* n : {"time.w", "time.b", "decode.g", "decode.w", "decode.b"}) v.push_back(n);
    return v;
}

// Manifest of a checkpoint (the text half of save_named_arrays / load_named_arrays,
// checkpoint.hpp:29-80): first line `dtype f32|f64`, then one `name RxC offset fnv1a64` line per
// array. Parsed in two passes: the whole file is tokenised into records, then the records are
// matched against this model's canonical array list (names, element counts, in order).
struct ManifestRecord {
    std::string name;
    long long rows = 0, cols = 0;
    unsigned long long offset = 0, sum = 0;
};

std::vector<ManifestRecord> parse_manifest(const std::string& path, std::string* dtype_word) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("checkpoint: no manifest at " + path);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::istringstream lines(text);
    std::string line, key;
    if (!std::getline(lines, line)) throw IoError("checkpoint: empty manifest " + path);
    std::istringstream head(line);
    head >> key >> *dtype_word;
    if (key != "dtype") throw IoError("checkpoint: " + path + " does not start with a dtype line");
    std::vector<ManifestRecord> recs;
    while (std::getline(lines, line)) {
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        ManifestRecord r;
        std::string shape;
        std::istringstream f(line);
        if (!(f >> r.name >> shape >> r.offset >> r.sum))
            throw IoError("checkpoint: unreadable manifest line " + std::to_string(recs.size() + 2) + " in " + path);
        const size_t x = shape.find('x');
        char* e1 = nullptr;
        char* e2 = nullptr;
        r.rows = x == std::string::npos ? -1 : std::strtoll(shape.c_str(), &e1, 10);
        r.cols = x == std::string::npos ? -1 : std::strtoll(shape.c_str() + x + 1, &e2, 10);
        if (r.rows < 0 || r.cols < 0 || e1 != shape.c_str() + x || *e2 != '\0')
            throw IoError("checkpoint: bad shape `" + shape + "` for `" + r.name + "` in " + path);
        recs.push_back(std::move(r));
    }
    return recs;
}

struct CkptEntry {
    u64 offset, sum;
    size_t n;
};

std::vector<CkptEntry> read_manifest(const std::string& base, const Dims& m, int* dtype) {
    std::string word;
    const std::vector<ManifestRecord> recs = parse_manifest(base + ".manifest", &word);
    if (word != "f32" && word != "f64") throw IoError("checkpoint dtype `" + word + "` is neither f32 nor f64 (" + base + ")");
    *dtype = word == "f64" ? SWF_F64 : SWF_F32;
    const auto names = param_names(m);
    const auto shapes = param_shapes(m);
    std::vector<CkptEntry> out;
    out.reserve(names.size());
    for (size_t i = 0; i < names.size(); ++i) {
        if (i >= recs.size())
            throw IoError("checkpoint " + base + " is truncated: the manifest ends before `" + names[i] + "`");
        const ManifestRecord& r = recs[i];
        const long long want = shapes[i].first * shapes[i].second;
        if (r.name != names[i] || r.rows * r.cols != want)
            throw IoError("checkpoint layout mismatch at array " + std::to_string(i) + ": this model has `" + names[i] +
                          "` with " + std::to_string(want) + " values, the manifest `" + r.name + "` " +
                          std::to_string(r.rows) + "x" + std::to_string(r.cols));
        out.push_back({r.offset, r.sum, size_t(want)});
    }
    return out;
}

// Read-ahead over a checkpoint's arrays: up to `depth` arrays are read, fnv1a64-verified and
// converted to f32 by worker threads (one stream per thread) while the caller consumes earlier
// ones in canonical order, so the serial checksum of load_named_arrays (checkpoint.hpp:50-80) runs
// in parallel with the H2D copies and the device repack. Errors surface on the consuming call.
class CkptReader {
public:
    CkptReader(const std::string& base, const std::vector<CkptEntry>& ent, int dtype, std::vector<std::string> names)
        : base_(base), ent_(ent), es_(dtype == SWF_F64 ? 8 : 4), names_(std::move(names)), slot_(ent.size()) {
        depth_ = int(std::max(2u, std::min(8u, std::thread::hardware_concurrency())));
        if (const char* e = std::getenv("SWF_CKPT_THREADS")) depth_ = std::max(0, std::atoi(e) - 1);
    }
    ~CkptReader() {
        for (auto& s : slot_)
            if (s.th.joinable()) s.th.join();
    }
    // f32 contents of array ai (valid until the next call)
    const float* get(int ai) {
        while (next_ < int(slot_.size()) && next_ <= ai + depth_) {  // arrays ai .. ai + depth_ in flight
            const int k = next_++;
            slot_[k].th = std::thread([this, k] { work(k); });
        }
        Slot& s = slot_[ai];
        if (s.th.joinable()) s.th.join();
        if (!s.err.empty()) throw IoError(s.err);
        if (prev_ >= 0 && prev_ != ai) release(prev_);
        prev_ = ai;
        return s.f32.data();
    }

private:
    struct Slot {
        std::vector<float> f32;
        std::string err;
        std::thread th;
    };
    void release(int k) { std::vector<float>().swap(slot_[k].f32); }
    void work(int k) {
        Slot& s = slot_[k];
        const CkptEntry& e = ent_[k];
        std::ifstream bin(base_ + ".bin", std::ios::binary);
        std::vector<char> raw(e.n * es_);
        if (bin) {
            bin.seekg(std::streamoff(e.offset));
            bin.read(raw.data(), std::streamsize(raw.size()));
        }
        if (!bin) {
            s.err = "checkpoint truncated at `" + names_[k] + "` in " + base_;
            return;
        }
        if (fnv1a64(raw.data(), raw.size()) != e.sum) {
            s.err = "IntegrityError: checksum mismatch for `" + names_[k] + "` in " + base_;
            return;
        }
        s.f32.resize(e.n);
        if (es_ == 8) {
            const double* d = reinterpret_cast<const double*>(raw.data());
            for (size_t i = 0; i < e.n; ++i) s.f32[i] = static_cast<float>(d[i]);
        } else {
            std::memcpy(s.f32.data(), raw.data(), raw.size());
        }
    }
    std::string base_;
    const std::vector<CkptEntry>& ent_;
    size_t es_;
    std::vector<std::string> names_;
    std::vector<Slot> slot_;
    int depth_ = 4, next_ = 0, prev_ = -1;
};

void load_checkpoint(swf_ctx* c, const std::string& base) {
    allocate(c);
    const Dims& m = c->m;
    int dtype = SWF_F32;
    const auto ent = read_manifest(base, m, &dtype);
    {
        std::ifstream bin(base + ".bin", std::ios::binary);
        if (!bin) throw IoError("cannot open checkpoint: " + base + ".bin");
    }
    float* stage = nullptr;
    SWF_CUDA(cudaMalloc(&stage, max_array(m) * sizeof(float)));
    try {
        CkptReader rd(base, ent, dtype, param_names(m));
        load_params_from(c, [&](int ai, size_t n) -> float* {
            SWF_CUDA(cudaStreamSynchronize(c->st));  // the previous array's repack is done with stage
            SWF_CUDA(cudaMemcpyAsync(stage, rd.get(ai), n * 4, cudaMemcpyHostToDevice, c->st));
            SWF_CUDA(cudaStreamSynchronize(c->st));
            return stage;
        });
    } catch (...) {
        cudaFree(stage);
        c->loaded = false;
        throw;
    }
    SWF_CUDA(cudaFree(stage));
}

// init_parameters (model.hpp:185-209) / init_parameters_random (:213-223) generated on the device
// with the same counter RNG (rng.hpp:17-45). mode 0: init_parameters; 1: init_parameters_random
// (every array += scale*N(0,1)); 2: init_parameters + scale*N(0,1) on the arrays it leaves at zero
// (ada.w, ada.b, decode.w, decode.b -- the bench's synthetic weights).
__device__ __forceinline__ u64 dv_splitmix(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__global__ void k_init_fill(float* __restrict__ dst, i64 n, u64 key, double scale, int op /*0 set,1 add,2 ones*/) {
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
        if (op == 2) {
            dst[i] = 1.f;
            continue;
        }
        const u64 b0 = dv_splitmix(key + 0x632be59bd9b4e019ULL * (2 * u64(i) + 1));
        const u64 b1 = dv_splitmix(key + 0x632be59bd9b4e019ULL * (2 * u64(i) + 2));
        const double u1 = (double(b0 >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = double(b1 >> 11) * 0x1.0p-53;
        const float v = static_cast<float>(scale * (sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2)));
        dst[i] = op == 1 ? dst[i] + v : v;
    }
}

u64 h_splitmix(u64 x);
u64 h_kd(u64 k, u64 t);

void init_params_device(swf_ctx* c, u64 seed, int mode, double scale) {
    allocate(c);
    const Dims& m = c->m;
    const auto shapes = param_shapes(m);
    float* stage = nullptr;
    SWF_CUDA(cudaMalloc(&stage, max_array(m) * sizeof(float)));
    u64 stream = 0;
    const int nb = m.nb;
    load_params_from(c, [&](int ai, size_t n) -> float* {
        SWF_CUDA(cudaStreamSynchronize(c->st));
        const int grid = int(std::min<size_t>((n + 255) / 256, 148 * 32));
        // which base rule applies to array ai (model.hpp:193-208)
        double sc = 0.0;
        int op = 0;  // 0: gaussian fill, 2: ones, 3: zeros
        if (ai == 0) {
            sc = 1.0 / std::sqrt(double(m.cin));
        } else if (ai == 1) {
            op = 3;
        } else if (ai < 2 + 9 * nb) {
            const int k = (ai - 2) % 9;
            switch (k) {
                case 0: sc = 1.0 / std::sqrt(double(m.h)); break;
                case 1: sc = 1.0 / std::sqrt(double(m.h) * 2 * nb); break;
                case 2: case 3: op = 2; break;
                case 4: case 5: sc = 1.0 / std::sqrt(double(m.h)); break;
                case 6: sc = 1.0 / std::sqrt(double(m.f) * 2 * nb); break;
                default: op = 3; break;  // ada.w, ada.b
            }
        } else {
            const int k = ai - (2 + 9 * nb);
            if (k == 0) sc = 1.0 / std::sqrt(double(m.td));
            else if (k == 2) op = 2;
            else op = 3;
        }
        if (op == 0) {
            k_init_fill<<<grid, 256, 0, c->st>>>(stage, i64(n), h_kd(h_kd(seed, 0x1217u), stream++), sc, 0);
        } else if (op == 2) {
            k_init_fill<<<grid, 256, 0, c->st>>>(stage, i64(n), 0, 0.0, 2);
        } else {
            SWF_CUDA(cudaMemsetAsync(stage, 0, n * 4, c->st));
        }
        const bool zero_init = (op == 3);
        if (mode == 1 || (mode == 2 && zero_init && ai != 1 && ai != 2 + 9 * nb + 1)) {
            // init_parameters_random key: key_derive(seed, 0xabc, 1000 + j)
            k_init_fill<<<grid, 256, 0, c->st>>>(stage, i64(n), h_kd(h_kd(seed, 0xabcu), u64(1000 + ai)), scale, 1);
        }
        SWF_LAUNCH_CHECK();
        return stage;
    });
    SWF_CUDA(cudaFree(stage));
}

// ------------------------------------------------------------------ forward
const TmaMap* tmap_at(const std::vector<TmaMap>& v, int b) { return b < int(v.size()) ? &v[b] : nullptr; }

template <class T>
struct Gemm;

void attention_ctx(swf_ctx* c, const AttnParams& ap, bool training);

// FP32-context linear layer. In the BF16 training mode (swf_set_backward_precision(BF16)) the
// forwards of the training entry points (activations saved) and the backward's recomputation run
// their GEMMs on the tensor cores: bf16 operands, plain fp32 product, then the same epilogue.
void gemm_f32_ctx(swf_ctx* c, const float* A, const float* W, i64 M, int Np, int K, int mode, const EpiParams& ep) {
    if (c->bwd_tc && c->bt_c && K % 8 == 0 && size_t(M) * Np <= c->bt_c_n) {
        gemm_strided_tc(int(M), Np, K, A, K, 1, W, 1, K, c->bt_c, Np, 0.f, c->bt_a, c->bt_b, c->d_sched, c->st);
        epi_rows_f32(c->bt_c, Np, M, Np, mode, ep, c->st);
        c->launches += 4;
        return;
    }
    gemm_f32(A, W, M, Np, K, mode, ep, c->st);
}

template <>
struct Gemm<float> {
    static void run(swf_ctx* c, const void* A, const TmaMap*, const void* B, const TmaMap*, i64 M, int Np, int K, int,
                    int mode, const EpiParams& ep) {
        if (c->save_x)
            gemm_f32_ctx(c, static_cast<const float*>(A), static_cast<const float*>(B), M, Np, K, mode, ep);
        else
            gemm_f32(static_cast<const float*>(A), static_cast<const float*>(B), M, Np, K, mode, ep, c->st);
    }
};
template <>
struct Gemm<__nv_bfloat16> {
    static void run(swf_ctx* c, const void*, const TmaMap* tA, const void*, const TmaMap* tB, i64 M, int Np, int K,
                    int BN, int mode, const EpiParams& ep) {
        gemm_bf16_tc(*tA, *tB, M, Np, K, BN, mode, ep, c->st);
    }
};

EpiParams base_ep(swf_ctx* c) {
    EpiParams ep;
    std::memset(&ep, 0, sizeof ep);
    ep.M = c->M;
    ep.h = c->m.h;
    ep.d = c->m.d;
    ep.heads = c->m.heads;
    ep.sched = c->d_sched;
    ep.rope_row = reinterpret_cast<const float2*>(c->rope_row);
    ep.rope_col = reinterpret_cast<const float2*>(c->rope_col);
    ep.rope_row_pm = reinterpret_cast<const float2*>(c->rope_row_pm);
    ep.rope_col_pm = reinterpret_cast<const float2*>(c->rope_col_pm);
    ep.rope_nrow = c->H + c->m.w;
    ep.rope_ncol = c->W + c->m.w;
    ep.cur = c->lay[0];
    ep.nxt = c->lay[0];
    ep.my_rank = c->rank;
    ep.out_scale = 1.f;
    ep.qkv_dst = c->d_qkv_dst;
    ep.heads_loc = c->m.heads / c->sp;
    ep.wp_rank = c->wp_rank;
    ep.hp = c->m.hp;
    ep.nss = c->prec == SWF_PREC_BF16 ? c->m.nss : 0;  // fused norm: producers emit xb / partial sums
    ep.off_xb = c->off_xb;
    ep.off_ss = c->off_ss;
    return ep;
}

void time_vectors(swf_ctx* c, double t) {
    // time_features (model.hpp:229-241) evaluates the arguments in double from T t
    const double tt = double(static_cast<float>(t));
    time_features(tt, c->m.td, c->feat, c->st);
    time_embed(c->feat, c->w_time_t, c->b_time, c->m.td, c->emb, c->st);
    ada_vectors(c->emb, c->w_ada_t, c->b_ada, c->m.nb, 6 * c->m.h, c->m.td, c->six, c->st);
    c->launches += 3;
}

void peer_barrier(swf_ctx* c);

// kernel classes for the profile (swf_profile_read)
enum KClass { K_ENCODE, K_RMS, K_QKV, K_ATTN, K_OUT, K_GATEUP, K_DOWN, K_DECODE, K_OTHER, K_NCLASS };

cudaEvent_t prof_event(swf_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        SWF_CUDA(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}
struct ProfScope {
    swf_ctx* c;
    int k;
    cudaEvent_t b = nullptr;
    ProfScope(swf_ctx* c_, int k_) : c(c_), k(k_) {
        if (c->prof) {
            b = prof_event(c);
            SWF_CUDA(cudaEventRecord(b, c->st));
        }
    }
    ~ProfScope() {
        if (c->prof) {
            cudaEvent_t e = prof_event(c);
            cudaEventRecord(e, c->st);
            c->prof_ev.push_back({k, {b, e}});
        }
    }
};

// Per-t preparation: time embedding + every block's AdaLN vectors; BF16 also folds this t's AdaLN
// scale into the normed GEMMs' weights and its shift into their biases.
template <class T>
void prep_time(swf_ctx* c, double t) {
    const Dims& m = c->m;
    time_vectors(c, t);
    if constexpr (sizeof(T) == 2) {
        const int h = m.h;
        for (int b = 0; b < m.nb; ++b) {
            const float* six = c->six + size_t(b) * 6 * h;
            fold_adaln(c->w_qkv_m[b], m.np_qkv, h, m.hp, c->g_attn + size_t(b) * h, six, six + h, six + 2 * h,
                       static_cast<__nv_bfloat16*>(c->w_qkv[b]), c->beta_qkv[b], c->st);
            fold_adaln(c->w_gu_m[b], m.np_gu, h, m.hp, c->g_ffn + size_t(b) * h, six + 3 * h, six + 4 * h,
                       six + 5 * h, static_cast<__nv_bfloat16*>(c->w_gu[b]), c->beta_gu[b], c->st);
        }
        fold_adaln(c->w_dec_m, m.np_dec, h, m.hp, c->g_dec, nullptr, nullptr, nullptr,
                   static_cast<__nv_bfloat16*>(c->w_dec), nullptr, c->st);
        c->launches += 2 * m.nb + 1;
    }
}

// One block (block_window_forward, swin.hpp:306-325, over all local windows at once) on the residual
// rows xbuf[cur] (M rows in the local order of layout L); the output is stored in the local order of
// Lnext into xbuf[cur ^ 1] (and, multi-rank, the peers' buffers). M < c->M runs a window subset (the
// q / k / V^T planes keep the full-size offsets the attention's TMA maps were built with).
template <class T>
void run_block(swf_ctx* c, int b, int cur, const LayMap& L, const LayMap& Lnext, i64 M) {
    const Dims& m = c->m;
    constexpr bool kFuse = sizeof(T) == 2;  // BF16: RMSNorm + AdaLN fused into the GEMMs
    const int par = b & 1;
    const float* six = c->six + size_t(b) * 6 * m.h;
    float* x = c->xbuf[cur];
    T* xm = static_cast<T*>(c->xm);
    EpiParams ep = base_ep(c);
    ep.M = M;
    // attention branch: prenorm_modulate -> heads -> out projection (swin.hpp:313-322)
    if constexpr (!kFuse) {
        ProfScope ps(c, K_RMS);
        rms_modulate<T>(x, M, m.h, m.hp, c->g_attn + size_t(b) * m.h, six, six + m.h, six + 2 * m.h, xm, c->flags,
                        1 + b, c->st);
    }
    EpiParams e = ep;
    e.cur = L;
    e.out = c->qkv;
    e.plane = i64(c->lay[par].nloc) * (m.heads / c->sp) * m.w * m.w * m.d;  // one q/k/v plane of a rank
    e.N = 3 * m.h;
    if constexpr (kFuse) {  // A = bf16 copy of x; norm from the producer's partial sums
        inv_rms(c->ssb[cur], M, m.nss, m.h, c->invr, c->flags, 1 + b, c->st);
        e.inv_r = c->invr;
        e.beta = c->beta_qkv[b];
        c->launches++;
    }
    {
        ProfScope ps(c, K_QKV);
        Gemm<T>::run(c, xm, kFuse ? &c->tm_xb[cur] : &c->tm_xm, c->w_qkv[b], tmap_at(c->tm_qkv, b), M, m.np_qkv,
                     m.hp, m.bn_qkv, EPI_QKV, e);
    }
    if (c->sp > 1) peer_barrier(c);  // every head group's planes complete before attention
    AttnParams ap;
    ap.q = c->qkv;
    ap.k = static_cast<const char*>(c->qkv) + size_t(c->M) * m.h * esize(c);
    ap.v = static_cast<const char*>(c->qkv) + size_t(2) * c->M * m.h * esize(c);
    ap.o = xm;
    ap.ldo = m.hp;
    ap.nloc = L.nloc;
    ap.heads = m.heads / c->sp;
    ap.head0 = c->band * (m.heads / c->sp);
    ap.wp_rank = c->wp_rank;
    ap.o_dst = c->d_o_dst;
    ap.s = m.w * m.w;
    ap.d = m.d;
    ap.w = m.w;
    ap.lay = L;
    ap.scale = 1.0f / std::sqrt(float(m.d));
    ap.tmq = &c->tm_q;
    ap.tmk = &c->tm_k;
    ap.tmk2 = &c->tm_k2;
    ap.tmv = &c->tm_vt;
    ap.tmo = c->sp == 1 ? &c->tm_xm : nullptr;  // SP: rows go to the band owners row by row
    {
        ProfScope ps(c, K_ATTN);
        if constexpr (sizeof(T) == 4)
            attention_ctx(c, ap, c->save_x);
        else
            attention_bf16(ap, c->st);
    }
    if (c->sp > 1) peer_barrier(c);  // all O rows of this rank's tokens landed
    e = ep;
    e.x = x;
    e.N = m.h;
    {
        ProfScope ps(c, K_OUT);
        Gemm<T>::run(c, xm, &c->tm_xm, c->w_out[b], tmap_at(c->tm_out, b), M, m.np_out, m.hp, m.bn_out, EPI_RESID, e);
    }
    // feed-forward branch (swin.hpp:323-324)
    if constexpr (!kFuse) {
        ProfScope ps(c, K_RMS);
        rms_modulate<T>(x, M, m.h, m.hp, c->g_ffn + size_t(b) * m.h, six + 3 * m.h, six + 4 * m.h, six + 5 * m.h, xm,
                        nullptr, 0, c->st);
    }
    e = ep;
    e.out = c->sbuf;
    e.ld_out = m.fp;
    e.N = m.f;
    e.G = m.G;
    if constexpr (kFuse) {
        inv_rms(c->ssb[cur], M, m.nss, m.h, c->invr, nullptr, 0, c->st);
        e.inv_r = c->invr;
        e.beta = c->beta_gu[b];
        c->launches++;
    }
    {
        ProfScope ps(c, K_GATEUP);
        Gemm<T>::run(c, xm, kFuse ? &c->tm_xb[cur] : &c->tm_xm, c->w_gu[b], tmap_at(c->tm_gu, b), M, m.np_gu, m.hp,
                     m.bn_gu, EPI_SWIGLU, e);
    }
    e = ep;
    e.x = x;
    e.N = m.h;
    e.cur = L;
    e.nxt = Lnext;
    e.xdst = c->d_xdst[cur ^ 1];
    {
        ProfScope ps(c, K_DOWN);
        Gemm<T>::run(c, c->sbuf, &c->tm_s, c->w_down[b], tmap_at(c->tm_down, b), M, m.np_down, m.fp, m.bn_down,
                     EPI_DOWN, e);
    }
    c->launches += 7;
}

// The network on the prepared model input a_in (window order of layout 0). out_scale multiplies
// the decode output (sigma_d for the sampler's net lambda, 1 for forward()).
template <class T>
void forward_core(swf_ctx* c, double t, float out_scale) {
    const Dims& m = c->m;
    const i64 M = c->M;
    // no rank may store into a peer's residual buffer while that peer still reads it
    if (c->world > 1) peer_barrier(c);
    prep_time<T>(c, t);
    constexpr bool kFuse = sizeof(T) == 2;
    EpiParams ep = base_ep(c);
    // encode (swin.hpp:341-342)
    ep.x = c->xbuf[0];
    ep.bias = c->enc_b;
    ep.N = m.h;
    {
        ProfScope ps(c, K_ENCODE);
        Gemm<T>::run(c, c->a_in, &c->tm_ain, c->w_enc, &c->tm_enc, M, m.np_enc, m.cinp, m.bn_enc, EPI_ENCODE, ep);
    }
    c->launches++;
    int cur = 0;
    T* xm = static_cast<T*>(c->xm);
    for (int b = 0; b < m.nb; ++b) {
        const int par = b & 1;
        const int npar = (b + 1 < m.nb) ? ((b + 1) & 1) : 0;
        if (b == c->stop_after) {
            c->hid_cur = cur;
            c->hid_par = par;
            return;
        }
        if (c->save_x)
            SWF_CUDA(cudaMemcpyAsync(c->xsave + size_t(b) * M * m.h, c->xbuf[cur], size_t(M) * m.h * 4,
                                     cudaMemcpyDeviceToDevice, c->st));
        run_block<T>(c, b, cur, c->lay[par], c->lay[npar], M);
        if (c->world > 1) peer_barrier(c);
        cur ^= 1;
    }
    if (c->save_x)
        SWF_CUDA(cudaMemcpyAsync(c->xsave + size_t(m.nb) * M * m.h, c->xbuf[cur], size_t(M) * m.h * 4,
                                 cudaMemcpyDeviceToDevice, c->st));
    if (c->stop_after == m.nb) {
        c->hid_cur = cur;
        c->hid_par = 0;
        return;
    }
    // decode (swin.hpp:362-366)
    if constexpr (!kFuse) {
        ProfScope ps(c, K_RMS);
        rms_modulate<T>(c->xbuf[cur], M, m.h, m.hp, c->g_dec, nullptr, nullptr, nullptr, xm, c->flags, 1 + m.nb, c->st);
    }
    EpiParams e = ep;
    e.out = c->out_loc;
    e.ld_out = m.cout;
    e.N = m.cout;
    e.bias = c->b_dec;
    e.out_scale = out_scale;
    if constexpr (kFuse) {
        inv_rms(c->ssb[cur], M, m.nss, m.h, c->invr, c->flags, 1 + m.nb, c->st);
        e.inv_r = c->invr;
        c->launches++;
    }
    {
        ProfScope ps(c, K_DECODE);
        Gemm<T>::run(c, xm, kFuse ? &c->tm_xb[cur] : &c->tm_xm, c->w_dec, &c->tm_dec, M, m.np_dec, m.hp, m.bn_dec,
                     EPI_DECODE, e);
    }
    c->launches += 2;
    // every rank sees every rank's non-finite flags (the decode input's included) before any of
    // them checks: all ranks raise the same NumericsError at the same call (k_peer_barrier)
    if (c->world > 1) peer_barrier(c);
}

// block_window_forward (swin.hpp:306-325) of block b on window (wy, wx) of the block's layout:
// x_in / x_out are that window's h x s_w residual columns (canonical token order r * w + c), fp32 rows
// [token][h] on the device. Runs the forward's kernels on a one-window layout (Lnext = the same
// window, so the down projection stores in place order).
template <class T>
void block_window_core(swf_ctx* c, int b, int wy, int wx, double t) {
    const Dims& m = c->m;
    const int par = b & 1;
    const LayMap& Lf = c->lay[par];
    const int nwin = Lf.g.nx * Lf.g.ny, gw = wy * Lf.g.nx + wx;
    int* ids = static_cast<int*>(scratch(c, SC_WIN, size_t(nwin + 1) * 4));
    std::vector<int> h_ids(size_t(nwin) + 1, 0);  // [0] = loc2glob[0] = gw; [1 + g] = glob2rl (rank 0, window 0)
    h_ids[0] = gw;
    SWF_CUDA(cudaMemcpyAsync(ids, h_ids.data(), h_ids.size() * 4, cudaMemcpyHostToDevice, c->st));
    LayMap L = Lf;
    L.nloc = 1;
    L.loc2glob = ids;
    L.glob2rl = ids + 1;
    const i64 M = i64(m.w) * m.w;
    prep_time<T>(c, t);
    if constexpr (sizeof(T) == 2) {
        prep_residual(c->xbuf[0], M, m.h, m.hp, m.nss, c->xbb[0], c->ssb[0], c->st);
        c->launches++;
    }
    run_block<T>(c, b, 0, L, L, M);
    SWF_CUDA(cudaStreamSynchronize(c->st));  // h_ids staging
}

void forward_any(swf_ctx* c, double t, float out_scale) {
    if (c->prec == SWF_PREC_BF16)
        forward_core<__nv_bfloat16>(c, t, out_scale);
    else
        forward_core<float>(c, t, out_scale);
}

// ------------------------------------------------------------------ backward (swin.hpp:370-467)
// FP32 validation mode, one rank. The forward saves every block's input (its layout's local order);
// the backward recomputes each block's internals from it (no s x s probabilities are stored),
// then runs the reference backward in reverse block order with k_bwd.cu kernels. Weight gradients
// come out in the reference's canonical order and column-major layout.
// bf16 operand copies and the plain-product buffer of the BF16 training mode
void alloc_bwd_tc(swf_ctx* c) {
    if (c->bt_a) return;
    const Dims& m = c->m;
    const size_t M = size_t(c->M);
    const size_t wide = size_t(std::max({m.np_gu, m.np_qkv, 3 * m.h, m.hp, m.cinp, m.np_dec}));
    const size_t w_max = std::max({size_t(m.np_gu) * m.hp, size_t(m.np_qkv) * m.hp, size_t(m.f) * m.h,
                                   size_t(m.np_dec) * m.hp, size_t(m.np_enc) * m.cinp});
    const size_t n = std::max(M * wide, w_max);
    c->bt_a = dalloc<__nv_bfloat16>(c, n);
    c->bt_b = dalloc<__nv_bfloat16>(c, n);
    c->bt_c_n = M * wide;
    c->bt_c = dalloc<float>(c, c->bt_c_n);
    // the tensor-core attention pieces need the rank's own O rows (no sequence parallelism); window
    // parallelism is fine -- attention is per window, every rank on its own windows
    if (c->sp == 1 && m.d % 8 == 0) {
        auto& ws = c->bt_ws;
        ws.n = AttnBwdStreams::kMax;
        for (int i = 0; i < ws.n; ++i) {
            SWF_CUDA(cudaStreamCreateWithFlags(&ws.st[i], cudaStreamNonBlocking));
            ws.scratch[i] = dalloc<char>(c, attention_bwd_tc_scratch(m.w * m.w, m.heads));
            ws.sched[i] = dalloc<int>(c, 1);
        }
        for (int i = 0; i <= ws.n; ++i) SWF_CUDA(cudaEventCreateWithFlags(&ws.ev[i], cudaEventDisableTiming));
    }
    if (c->sp == 1 && (m.d == 32 || m.d == 64 || m.d == 128)) {
        c->bt_qkv = dalloc<__nv_bfloat16>(c, size_t(3) * M * m.h);
        c->bt_o = dalloc<__nv_bfloat16>(c, M * size_t(m.hp));
        c->bt_lse = dalloc<float>(c, M * size_t(m.heads));  // [nloc][heads][s], nloc s = M
        c->bt_D = dalloc<float>(c, M * size_t(m.heads));
        // the kernel indexes the output table by the owning rank (wp_rank under window parallelism):
        // every entry is this rank's buffer, its O rows are always its own tokens' (sp == 1)
        c->d_bt_o = dalloc<void*>(c, 8);
        std::vector<void*> o(8, c->bt_o);
        h2d_sync(c, c->d_bt_o, o.data(), 8 * sizeof(void*));
        const int sw = m.d >= 64 ? 128 : 2 * m.d;
        const i64 rows = i64(c->lay[0].nloc) * m.heads * m.w * m.w;
        const __nv_bfloat16* qb = c->bt_qkv;
        make_tma_bf16_2d(&c->bt_tm_q, qb, rows, m.d, sw / 2, 128, sw);
        make_tma_bf16_2d(&c->bt_tm_k, qb + M * m.h, rows, m.d, sw / 2, 64, sw);
        make_tma_bf16_2d(&c->bt_tm_k2, qb + M * m.h, rows, m.d, sw / 2, 32, sw);
        make_tma_bf16_2d(&c->bt_tm_vt, qb + 2 * M * m.h, i64(c->lay[0].nloc) * m.heads * m.d, i64(m.w) * m.w, 64,
                         m.d / 2, 128);
        make_tma_bf16(&c->bt_tm_o, c->bt_o, i64(M), m.hp, 128);
    }
}

// FP32-context attention. The BF16 training mode runs the tensor-core kernel (k_attn_pp) on bf16
// copies of q, k and V^T and widens its bf16 output; the FP32 validation mode runs the SIMT kernel.
void attention_ctx(swf_ctx* c, const AttnParams& ap, bool training) {
    if (!(c->bwd_tc && training && c->bt_qkv)) {
        attention_f32(ap, c->st);
        return;
    }
    const Dims& m = c->m;
    const i64 M = c->M;
    const i64 planes = i64(ap.nloc) * ap.heads;
    to_bf16(static_cast<const float*>(ap.q), 2 * M * m.h, c->bt_qkv, c->st);  // q and k planes are adjacent
    vt_bf16(static_cast<const float*>(ap.v), planes, ap.s, ap.d, c->bt_qkv + 2 * M * m.h, c->st);
    AttnParams b = ap;
    b.q = c->bt_qkv;
    b.k = c->bt_qkv + M * m.h;
    b.v = c->bt_qkv + 2 * M * m.h;
    b.o_dst = c->d_bt_o;
    b.ldo = m.hp;
    b.head0 = 0;
    b.tmq = &c->bt_tm_q;
    b.tmk = &c->bt_tm_k;
    b.tmk2 = &c->bt_tm_k2;
    b.tmv = &c->bt_tm_vt;
    b.tmo = &c->bt_tm_o;
    b.lse = c->bt_lse;  // the backward's P comes from these row statistics
    attention_bf16(b, c->st);
    to_f32(c->bt_o, M * m.hp, static_cast<float*>(ap.o), c->st);
    c->launches += 4;
}

void ensure_bwd(swf_ctx* c) {
    if (c->bw_alloc) return;
    const Dims& m = c->m;
    const i64 M = c->M;
    auto& b = c->bw;
    c->xsave = dalloc<float>(c, size_t(m.nb + 1) * M * m.h);
    b.dx[0] = dalloc<float>(c, size_t(M) * m.h);
    b.dx[1] = dalloc<float>(c, size_t(M) * m.h);
    b.dtmp = dalloc<float>(c, size_t(M) * m.h);
    b.xmid = dalloc<float>(c, size_t(M) * m.h);
    b.dxm = dalloc<float>(c, size_t(M) * m.h);
    b.xm1 = dalloc<float>(c, size_t(M) * m.hp);
    b.obuf = dalloc<float>(c, size_t(M) * m.hp);
    b.x2m = dalloc<float>(c, size_t(M) * m.hp);
    b.dO = dalloc<float>(c, size_t(M) * m.hp);
    b.gu = dalloc<float>(c, size_t(M) * m.np_gu);
    b.act = dalloc<float>(c, size_t(M) * m.f);
    b.dS = dalloc<float>(c, size_t(M) * m.f);
    b.dG = dalloc<float>(c, size_t(M) * m.f);
    b.dU = dalloc<float>(c, size_t(M) * m.f);
    b.dqkv = dalloc<float>(c, size_t(M) * 3 * m.h);
    b.dplanes = dalloc<float>(c, size_t(3) * M * m.h);
    b.stats = dalloc<float>(c, size_t(3) * M * m.heads);
    b.rms = dalloc<float>(c, size_t(M));
    b.d6 = dalloc<float>(c, size_t(6) * m.h);
    b.demb = dalloc<float>(c, size_t(m.td));
    b.zero = dalloc<float>(c, size_t(m.np_gu) + m.np_dec + 64);
    b.gflat = dalloc<float>(c, c->poff.back());
    b.din = dalloc<float>(c, size_t(M) * m.cin);
    b.npart = dalloc<float>(c, size_t(kNormSlices) * 4 * m.h);
    if (c->bwd_tc) alloc_bwd_tc(c);
    c->bw_alloc = true;
}

void backward_core(swf_ctx* c, const float* dout) {
    const Dims& m = c->m;
    const i64 M = c->M;
    const int h = m.h, hp = m.hp, f = m.f, td = m.td, nb = m.nb;
    auto& bw = c->bw;
    cudaStream_t st = c->st;
    float* G = bw.gflat;
    const float* P = c->pflat;
    auto pa = [&](int ai) { return P + c->poff[ai]; };
    auto ga = [&](int ai) { return G + c->poff[ai]; };
    const int kHead = 2, kPer = 9, tail = kHead + nb * kPer;
    // the linears' GEMMs: SIMT FP32 (validation mode) or tcgen05 BF16 (swf_set_backward_precision)
    auto lin = [&](int Mg, int Ng, int Kg, const float* A, i64 sai, i64 sak, const float* B, i64 sbk, i64 sbj, float* C,
                   i64 ldc, float beta) {
        if (c->bwd_tc)
            gemm_strided_tc(Mg, Ng, Kg, A, sai, sak, B, sbk, sbj, C, ldc, beta, c->bt_a, c->bt_b, c->d_sched, st);
        else
            gemm_strided_f32(Mg, Ng, Kg, A, sai, sak, B, sbk, sbj, C, ldc, beta, st);
    };
    // WP: every rank's gradients are partial sums over its tokens (all-reduced by the caller); no
    // rank may store into a peer's landing buffer while that peer still runs its forward
    if (c->world > 1) peer_barrier(c);
    SWF_CUDA(cudaMemsetAsync(G, 0, c->poff.back() * 4, st));
    SWF_CUDA(cudaMemsetAsync(bw.demb, 0, size_t(td) * 4, st));
    // decode head (swin.hpp:430-436): n3 = prenorm_plain(x_final); dW_dec, db_dec, dN3, prenorm_plain_bwd
    const float* xf = c->xsave + size_t(nb) * M * h;
    rms_modulate<float>(xf, M, h, hp, c->g_dec, nullptr, nullptr, nullptr, bw.xm1, nullptr, 0, st);
    lin(h, m.cout, int(M), bw.xm1, 1, hp, dout, m.cout, 1, ga(tail + 3), m.cout, 1.f);
    colsum_f32(dout, m.cout, M, m.cout, ga(tail + 4), bw.npart, st);
    lin(int(M), h, m.cout, dout, m.cout, 1, pa(tail + 3), 1, m.cout, bw.dtmp, h, 0.f);
    SWF_CUDA(cudaMemsetAsync(bw.dx[0], 0, size_t(M) * h * 4, st));
    norm_bwd(xf, h, bw.dtmp, h, M, h, c->g_dec, nullptr, nullptr, nullptr, bw.dx[0], h, bw.rms, ga(tail + 2), nullptr,
             nullptr, nullptr, bw.npart, st);
    int cur = 0;  // bw.dx[cur]: gradient of the current block's output, in that output's layout
    EpiParams ep = base_ep(c);
    for (int b = nb - 1; b >= 0; --b) {
        const int par = b & 1, npar = (b + 1 < nb) ? ((b + 1) & 1) : 0;
        const int base = kHead + b * kPer;
        const float* xb = c->xsave + size_t(b) * M * h;
        const float* six = c->six + size_t(b) * 6 * h;
        // ---- recompute the block's internals (block_window_forward, swin.hpp:306-325)
        rms_modulate<float>(xb, M, h, hp, c->g_attn + size_t(b) * h, six, six + h, six + 2 * h, bw.xm1, nullptr, 0, st);
        EpiParams e = ep;
        e.cur = c->lay[par];
        e.out = c->qkv;
        e.plane = i64(c->lay[par].nloc) * m.heads * m.w * m.w * m.d;
        e.N = 3 * h;
        gemm_f32_ctx(c, bw.xm1, static_cast<const float*>(c->w_qkv[b]), M, m.np_qkv, hp, EPI_QKV, e);
        const float* q = static_cast<const float*>(c->qkv);
        const float* kk = q + size_t(M) * h;
        const float* v = q + size_t(2) * M * h;
        AttnParams ap;
        ap = AttnParams{};
        ap.q = q;
        ap.k = kk;
        ap.v = v;
        ap.o = bw.obuf;
        ap.ldo = hp;
        ap.nloc = c->lay[par].nloc;
        ap.heads = m.heads;
        ap.s = m.w * m.w;
        ap.d = m.d;
        ap.w = m.w;
        ap.lay = c->lay[par];
        ap.scale = 1.0f / std::sqrt(float(m.d));
        attention_ctx(c, ap, true);
        SWF_CUDA(cudaMemcpyAsync(bw.xmid, xb, size_t(M) * h * 4, cudaMemcpyDeviceToDevice, st));
        e = ep;
        e.x = bw.xmid;
        e.N = h;
        gemm_f32_ctx(c, bw.obuf, static_cast<const float*>(c->w_out[b]), M, m.np_out, hp, EPI_RESID, e);
        rms_modulate<float>(bw.xmid, M, h, hp, c->g_ffn + size_t(b) * h, six + 3 * h, six + 4 * h, six + 5 * h, bw.x2m,
                            nullptr, 0, st);
        e = ep;
        e.out = bw.gu;
        e.ld_out = m.np_gu;
        e.N = m.np_gu;
        e.bias = bw.zero;
        if (c->bwd_tc && c->bt_c && hp % 8 == 0)  // tensor cores: the plain product is the result (no epilogue pass)
            gemm_strided_tc(int(M), m.np_gu, hp, bw.x2m, hp, 1, static_cast<const float*>(c->w_gu[b]), 1, hp, bw.gu,
                            m.np_gu, 0.f, c->bt_a, c->bt_b, c->d_sched, st);
        else
            gemm_f32_ctx(c, bw.x2m, static_cast<const float*>(c->w_gu[b]), M, m.np_gu, hp, EPI_DECODE, e);
        // ---- backward (block_window_backward, swin.hpp:370-417)
        float* dXp = bw.dtmp;  // output gradient in this block's layout
        if (c->world > 1) {    // WP: owners change between the layouts -> peer stores, then a barrier
            relayout_push(bw.dx[cur], c->lay[npar], c->lay[par], M, h, c->d_xdst[par], st);
            peer_barrier(c);
            dXp = c->xbuf[par];  // landing buffer (the forward's residual stream is free here)
            c->launches++;
        } else {
            relayout_rows(bw.dx[cur], c->lay[npar], c->lay[par], M, h, dXp, st);
        }
        // feed-forward branch: swiglu_bwd (:236-252)
        lin(int(M), f, h, dXp, h, 1, pa(base + 6), 1, h, bw.dS, f, 0.f);
        swiglu_bwd(bw.gu, m.np_gu, bw.dS, f, M, f, m.G, bw.act, bw.dG, bw.dU, st);
        lin(f, h, int(M), bw.act, 1, f, dXp, h, 1, ga(base + 6), h, 1.f);     // dW_down
        lin(h, f, int(M), bw.x2m, 1, hp, bw.dG, f, 1, ga(base + 4), f, 1.f);  // dW_gate
        lin(h, f, int(M), bw.x2m, 1, hp, bw.dU, f, 1, ga(base + 5), f, 1.f);  // dW_up
        lin(int(M), h, f, bw.dG, f, 1, pa(base + 4), 1, f, bw.dxm, h, 0.f);
        lin(int(M), h, f, bw.dU, f, 1, pa(base + 5), 1, f, bw.dxm, h, 1.f);
        SWF_CUDA(cudaMemsetAsync(bw.d6, 0, size_t(6) * h * 4, st));
        float* dxmid = bw.dx[cur ^ 1];
        SWF_CUDA(cudaMemcpyAsync(dxmid, dXp, size_t(M) * h * 4, cudaMemcpyDeviceToDevice, st));
        norm_bwd(bw.xmid, h, bw.dxm, h, M, h, c->g_ffn + size_t(b) * h, six + 3 * h, six + 4 * h, six + 5 * h, dxmid,
                 h, bw.rms, ga(base + 3), bw.d6 + 3 * h, bw.d6 + 4 * h, bw.d6 + 5 * h, bw.npart, st);
        // attention branch: out projection, head_attention_bwd (:189-226), prenorm_modulate_bwd
        lin(h, h, int(M), bw.obuf, 1, hp, dxmid, h, 1, ga(base + 1), h, 1.f);  // dW_out
        lin(int(M), h, h, dxmid, h, 1, pa(base + 1), 1, h, bw.dO, hp, 0.f);
        float* dq = bw.dplanes;
        if (c->bwd_tc && c->bt_ws.n > 0 && c->bt_lse)  // the recompute above ran the tensor-core kernel
            attention_bwd_tc(q, kk, v, bw.obuf, bw.dO, hp, dq, dq + size_t(M) * h, dq + size_t(2) * M * h,
                             c->lay[par].nloc, m.heads, m.w * m.w, m.d, m.w, c->lay[par], ep, bw.dqkv, c->bt_a,
                             c->bt_b, c->bt_lse, c->bt_D, c->bt_ws, st);
        else
            attention_bwd_f32(q, kk, v, bw.obuf, bw.dO, hp, dq, dq + size_t(M) * h, dq + size_t(2) * M * h,
                              bw.stats, c->lay[par].nloc, m.heads, m.w * m.w, m.d, m.w, c->lay[par], ep, bw.dqkv, st);
        lin(h, 3 * h, int(M), bw.xm1, 1, hp, bw.dqkv, 3 * h, 1, ga(base + 0), 3 * h, 1.f);  // dW_qkv
        lin(int(M), h, 3 * h, bw.dqkv, 3 * h, 1, pa(base + 0), 1, 3 * h, bw.dxm, h, 0.f);
        // dx_in = dx_mid + prenorm_modulate_bwd(...) -- accumulated in place in dxmid
        norm_bwd(xb, h, bw.dxm, h, M, h, c->g_attn + size_t(b) * h, six, six + h, six + 2 * h, dxmid, h, bw.rms,
                 ga(base + 2), bw.d6, bw.d6 + h, bw.d6 + 2 * h, bw.npart, st);
        ada_bwd(bw.d6, c->emb, pa(base + 7), 6 * h, td, ga(base + 7), ga(base + 8), bw.demb, st);
        cur ^= 1;  // the block input's gradient, in layout par = the previous block's output layout
    }
    // encode (swin.hpp:458-461) and the shared time projection (:463-466)
    const float* dx = bw.dx[cur];
    lin(m.cin, h, int(M), static_cast<const float*>(c->a_in), 1, m.cinp, dx, h, 1, ga(0), h, 1.f);
    colsum_f32(dx, h, M, h, ga(1), bw.npart, st);
    lin(int(M), m.cin, h, dx, h, 1, pa(0), 1, h, bw.din, m.cin, 0.f);
    time_bwd(bw.demb, c->feat, pa(tail + 0), pa(tail + 1), td, ga(tail + 0), ga(tail + 1), st);
}

void gather_input_any(swf_ctx* c, const float* in_pix) {
    if (c->prec == SWF_PREC_BF16)
        gather_rows<__nv_bfloat16>(in_pix, c->lay[0], c->m.cin, c->m.cinp, c->M, static_cast<__nv_bfloat16*>(c->a_in),
                                   c->flags, 0, c->st);
    else
        gather_rows<float>(in_pix, c->lay[0], c->m.cin, c->m.cinp, c->M, static_cast<float*>(c->a_in), c->flags, 0,
                           c->st);
    c->launches++;
}

void reset_flags(swf_ctx* c) { SWF_CUDA(cudaMemsetAsync(c->flags, 0, sizeof(int) * c->nflags, c->st)); }

// Raise NumericsError for the first flagged slot, naming it like check_finite (swin.hpp:295-300)
// and the solver (diffusion.hpp:248-251).
void check_flags(swf_ctx* c) {
    SWF_CUDA(cudaMemcpyAsync(c->h_flags, c->flags, sizeof(int) * c->nflags, cudaMemcpyDeviceToHost, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
    const int nb = c->m.nb;
    if (c->h_flags[c->nflags - 1]) throw CudaError("peer barrier timed out (a window-parallel rank stopped)");
    for (int s = 0; s < c->nflags - 1; ++s) {
        if (!c->h_flags[s]) continue;
        if (s == 0) throw NumericsError("non-finite activation entering input");
        if (s <= nb) throw NumericsError("non-finite activation entering block " + std::to_string(s - 1));
        if (s == nb + 1) throw NumericsError("non-finite activation entering decode");
        throw NumericsError("pf-ode solver diverged at step " + std::to_string(s - nb - 2));
    }
}

// Cross-rank barrier over peer-mapped flag words (one CTA per rank; rank 0..world-1 may share a GPU,
// the waiting CTA never holds resources another rank's kernels need). Slot layout of a rank's
// 64-int barrier array: [0, 8) the epoch each peer reached, [8 + 8 p, 16 + 8 p) for epoch parity p
// the lowest numerics flag slot each peer had raised (+1; 0 = none). Each rank publishes its lowest
// raised slot into every peer, release-stores the epoch, acquire-polls every peer's epoch, then
// raises the peers' slots locally: after a barrier every rank holds every rank's flags, so a NaN in
// one rank's windows makes all ranks throw the same NumericsError at the same point. A
// peer can be at most one barrier ahead (it waits for this rank's epoch), so parity double-buffers
// the published slots. A peer silent for 30 s sets the timeout word instead of hanging.
__global__ void k_peer_barrier(int* const* flags, int rank, int world, int* epoch_ctr, int* local, int nflags) {
    __shared__ int epoch, lowest;
    const int t = threadIdx.x;
    if (t == 0) {
        epoch = *epoch_ctr + 1;  // every rank runs the same barrier sequence
        lowest = 0x7fffffff;
    }
    __syncthreads();
    int lo = 0x7fffffff;
    for (int i = t; i < nflags - 1; i += blockDim.x)
        if (local[i]) lo = min(lo, i);
    atomicMin(&lowest, lo);
    __syncthreads();
    const int par = epoch & 1;
    if (t < world) {
        int* remote = flags[t];
        remote[8 + 8 * par + rank] = lowest == 0x7fffffff ? 0 : lowest + 1;
        __threadfence_system();
        asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(remote + rank), "r"(epoch) : "memory");
        const int* mine = flags[rank] + t;
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (true) {
            int v;
            asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
            if (v >= epoch) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 30000000000ull) {  // 30 s: a peer died -> report instead of hanging
                atomicOr(local + nflags - 1, 1);
                break;
            }
        }
        int v;
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags[rank] + 8 + 8 * par + t) : "memory");
        if (v > 0 && v < nflags) atomicOr(local + (v - 1), 1);
    }
    __syncthreads();
    if (t == 0) *epoch_ctr = epoch;
}

void peer_barrier(swf_ctx* c) {
    if (!c->peers) throw ConfigError("multi-rank topology: connect the ranks (swf_connect_peers) before running");
    k_peer_barrier<<<1, 256, 0, c->st>>>(c->d_flag_table, c->rank, c->world, c->d_epoch, c->flags, c->nflags);
    SWF_LAUNCH_CHECK();
    c->launches++;
}

// ------------------------------------------------------------------ sampler
void ensure_sampler(swf_ctx* c) {
    if (c->pe_loc) return;
    const Dims& m = c->m;
    const i64 M = c->M;
    // sinusoidal_pos_encode (posenc.hpp:16-37) in double, cast to float, pixel order, then gathered
    std::vector<float> pe(size_t(c->N) * m.cin);
    const int per_axis = m.cin / 2, nf = (per_axis + 1) / 2;
    for (int axis = 0; axis < 2; ++axis)
        for (int i = 0; i < per_axis; ++i) {
            const int k = i / 2;
            const double om = std::pow(10000.0, -double(k) / std::max(1, nf));
            const bool use_sin = (i % 2 == 0);
            const int ch = axis * per_axis + i;
            for (int y = 0; y < c->H; ++y)
                for (int x = 0; x < c->W; ++x) {
                    const double pos = axis == 0 ? y : x;
                    pe[(size_t(y) * c->W + x) * m.cin + ch] =
                        static_cast<float>(use_sin ? std::sin(pos * om) : std::cos(pos * om));
                }
        }
    c->pe_loc = dalloc<float>(c, size_t(M) * m.cin);
    h2d_sync(c, c->in_pix, pe.data(), pe.size() * 4);
    gather_rows<float>(c->in_pix, c->lay[0], m.cin, m.cin, M, c->pe_loc, nullptr, 0, c->st);
    c->s_x = dalloc<float>(c, size_t(M) * m.cout);
    c->s_xmid = dalloc<float>(c, size_t(M) * m.cout);
    c->s_tmp = dalloc<float>(c, size_t(M) * m.cout);
    c->s_base = dalloc<float>(c, size_t(M) * m.cout);
    c->s_cond = dalloc<float>(c, size_t(M) * std::max(m.cin - 2 * m.cout, 1));
    c->s_stats = dalloc<float>(c, size_t(6) * m.cin);
    SWF_CUDA(cudaStreamSynchronize(c->st));
}

// a_in channels [cp, cin) <- [x_prev ; forcings] + posenc (net lambda, diffusion.hpp:304-311)
void set_conditioning(swf_ctx* c, const float* xprev_loc, const float* forc_loc) {
    const Dims& m = c->m;
    const int cf = m.cin - 2 * m.cout;
    if (c->prec == SWF_PREC_BF16)
        build_static_input<__nv_bfloat16>(xprev_loc, forc_loc, c->pe_loc, c->M, m.cout, cf, m.cin, m.cinp,
                                          static_cast<__nv_bfloat16*>(c->a_in), c->st);
    else
        build_static_input<float>(xprev_loc, forc_loc, c->pe_loc, c->M, m.cout, cf, m.cin, m.cinp,
                                  static_cast<float*>(c->a_in), c->st);
}

// v = sigma_d * F(x / sigma_d, t) into out_loc
void net_eval(swf_ctx* c, const float* x, double sd, double t) {
    const Dims& m = c->m;
    if (c->prec == SWF_PREC_BF16)
        assemble_state<__nv_bfloat16>(x, c->pe_loc, c->M, m.cout, m.cin, m.cinp, float(sd),
                                      static_cast<__nv_bfloat16*>(c->a_in), c->st);
    else
        assemble_state<float>(x, c->pe_loc, c->M, m.cout, m.cin, m.cinp, float(sd), static_cast<float*>(c->a_in),
                              c->st);
    forward_any(c, t, float(sd));
}

void validate_dc(const swf_diffusion_cfg& dc) {
    require(dc.sigma_d > 0, "diffusion: sigma_d must be positive");
    require(0 < dc.sigma_min && dc.sigma_min < dc.sigma_max, "diffusion: need 0 < sigma_min < sigma_max");
    require(dc.solver_steps >= 1, "diffusion: solver_steps must be >= 1");
    require(dc.churn >= 0, "diffusion: churn amount must be >= 0");
    require(dc.solver_steps <= 4000, "diffusion: solver_steps too large");
}

static std::pair<float, float> trig_coeffs_f(float t) {  // diffusion.hpp:50-55 in float
    if (t == 0.f) return {1.f, 0.f};
    if (t == static_cast<float>(M_PI_2)) return {0.f, 1.f};
    return {std::cos(t), std::sin(t)};
}

// solve_pf_ode (diffusion.hpp:207-272) on the state c->s_x (local window order, [M][C_out]).
// Enqueues the 2*S net evaluations, sampler updates and churn rotations on c->st; every scalar is a
// function of dc alone (the churn key is read from c->d_churn_key), so the sequence can be captured.
void enqueue_solve(swf_ctx* c, const swf_diffusion_cfg& dc) {
    const Dims& m = c->m;
    const i64 n = c->M * m.cout;
    const int S = dc.solver_steps;
    const double sd = dc.sigma_d;
    auto t_of = [&](double s) { return std::atan(s / sd); };
    std::vector<double> sigma(S + 1);
    for (int k = 0; k <= S; ++k) {
        const double fr = double(k) / S;
        sigma[k] = std::exp((1.0 - fr) * std::log(dc.sigma_max) + fr * std::log(dc.sigma_min));
    }
    double t_cur = t_of(sigma[0]), sig_cur = sigma[0];
    u64 churn_ctr = 0;
    for (int k = 0; k < S; ++k) {
        const double sig_next = sigma[k + 1], t_next = t_of(sig_next);
        const double sig_mid = std::sqrt(sig_cur * sig_next), t_mid = t_of(sig_mid);
        const double b_s = std::sin(t_cur) * sd;
        const double a_m = std::cos(t_mid), b_m = std::sin(t_mid) * sd;
        const double a_t = std::cos(t_next), b_t = std::sin(t_next) * sd;
        // stage 1: d1 = x0hat(x, t_cur); x_mid = (b_m/b_s) x - a_m (r_mid - 1) d1
        net_eval(c, c->s_x, sd, static_cast<float>(t_cur));
        auto cs1 = trig_coeffs_f(static_cast<float>(t_cur));
        const double r_mid = sig_mid / sig_cur;
        sampler_update(c->s_x, c->s_x, c->out_loc, n, cs1.first, cs1.second, float(b_m / b_s),
                       float(a_m * (r_mid - 1.0)), c->s_xmid, nullptr, 0, c->st);
        // stage 2: d2 = x0hat(x_mid, t_mid); x = (b_t/b_s) x - a_t (r - 1) d2
        net_eval(c, c->s_xmid, sd, static_cast<float>(t_mid));
        auto cs2 = trig_coeffs_f(static_cast<float>(t_mid));
        const double r = sig_next / sig_cur;
        sampler_update(c->s_x, c->s_xmid, c->out_loc, n, cs2.first, cs2.second, float(b_t / b_s),
                       float(a_t * (r - 1.0)), c->s_x, c->flags, m.nb + 2 + std::min(k, 4000), c->st);
        c->launches += 2;
        t_cur = t_next;
        sig_cur = sig_next;
        const bool active = dc.churn > 0.0 && 3 * k >= S && 3 * k < 2 * S;  // ChurnSchedule::active_step
        if (active && k + 1 < S) {
            const double delta = dc.churn * 0.05 * (t_of(sigma[k]) - t_next);
            if (delta > 0) {
                churn_rotate(c->s_x, c->lay[0], c->M, m.cout, c->d_churn_key, churn_ctr, sd, float(std::cos(delta)),
                             float(std::sin(delta)), c->st);
                churn_ctr += u64(c->N) * m.cout;
                t_cur += delta;
                sig_cur = sd * std::tan(t_cur);
                c->launches++;
            }
        }
    }
}

static bool same_dc(const swf_diffusion_cfg& a, const swf_diffusion_cfg& b) {
    return a.sigma_d == b.sigma_d && a.sigma_min == b.sigma_min && a.sigma_max == b.sigma_max &&
           a.solver_steps == b.solver_steps && a.churn == b.churn;
}

void solve(swf_ctx* c, const swf_diffusion_cfg& dc, u64 churn_key, int* f_evals) {
    validate_dc(dc);
    if (f_evals) *f_evals = 2 * dc.solver_steps;
    // stream-ordered: the previous solve's churn kernels read the key before this copy lands
    *c->h_churn_key = churn_key;
    SWF_CUDA(cudaMemcpyAsync(c->d_churn_key, c->h_churn_key, sizeof(u64), cudaMemcpyHostToDevice, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));  // pinned staging reused by the next call
    const bool use_graph = c->graphs && !c->prof && !c->save_x;
    if (!use_graph || !same_dc(dc, c->graph_dc) || c->graph_seen == 0) {
        if (c->solve_exec) {
            SWF_CUDA(cudaGraphExecDestroy(c->solve_exec));
            c->solve_exec = nullptr;
        }
        c->graph_dc = dc;
        c->graph_seen = use_graph ? 1 : 0;
        enqueue_solve(c, dc);
        return;
    }
    if (c->graph_seen == 1) {  // second call with this config: capture once
        const long long l0 = c->launches;
        cudaGraph_t g = nullptr;
        SWF_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_solve(c, dc);
        } catch (...) {
            cudaStreamEndCapture(c->st, &g);
            if (g) cudaGraphDestroy(g);
            c->graph_seen = 0;
            throw;
        }
        SWF_CUDA(cudaStreamEndCapture(c->st, &g));
        SWF_CUDA(cudaGraphInstantiate(&c->solve_exec, g, 0));
        SWF_CUDA(cudaGraphDestroy(g));
        c->graph_launches = c->launches - l0;
        c->launches = l0;
        c->graph_seen = 2;
    }
    SWF_CUDA(cudaGraphLaunch(c->solve_exec, c->st));
    c->launches += c->graph_launches;
}

// host-side helpers: host [N][C] (f32/f64) <-> device pixel staging
void h2d_field(swf_ctx* c, const void* src, int C, int dtype, float* dst_pix) {
    const size_t n = size_t(c->N) * C;
    if (dtype == SWF_F64) {
        std::vector<float> tmp(n);
        const double* d = static_cast<const double*>(src);
        for (size_t i = 0; i < n; ++i) tmp[i] = static_cast<float>(d[i]);
        SWF_CUDA(cudaMemcpyAsync(dst_pix, tmp.data(), n * 4, cudaMemcpyHostToDevice, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
    } else {
        SWF_CUDA(cudaMemcpyAsync(dst_pix, src, n * 4, cudaMemcpyHostToDevice, c->st));
    }
}

void d2h_field(swf_ctx* c, const float* src_loc, int C, int dtype, void* dst) {
    const size_t n = size_t(c->N) * C;
    SWF_CUDA(cudaMemsetAsync(c->out_pix, 0, n * 4, c->st));
    scatter_rows(src_loc, c->lay[0], C, c->M, c->out_pix, c->st);
    if (dtype == SWF_F64) {
        std::vector<float> tmp(n);
        SWF_CUDA(cudaMemcpyAsync(tmp.data(), c->out_pix, n * 4, cudaMemcpyDeviceToHost, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
        double* d = static_cast<double*>(dst);
        for (size_t i = 0; i < n; ++i) d[i] = tmp[i];
    } else {
        SWF_CUDA(cudaMemcpyAsync(dst, c->out_pix, n * 4, cudaMemcpyDeviceToHost, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
    }
}

// Multi-rank readback: this rank's local rows [M][C] -> pinned staging -> the caller's [N][C] field at
// the owned pixels only (the other ranks of a single-process group write theirs concurrently).
void d2h_owned(swf_ctx* c, const float* src_loc, int C, int dtype, void* dst) {
    const size_t n = size_t(c->M) * C;
    if (c->h_stage_n < n) {
        if (c->h_stage) SWF_CUDA(cudaFreeHost(c->h_stage));
        c->h_stage = nullptr;
        SWF_CUDA(cudaMallocHost(&c->h_stage, n * 4));
        c->h_stage_n = n;
    }
    SWF_CUDA(cudaMemcpyAsync(c->h_stage, src_loc, n * 4, cudaMemcpyDeviceToHost, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
    for (i64 i = 0; i < c->M; ++i) {
        const float* r = c->h_stage + size_t(i) * C;
        const size_t o = size_t(c->owned_pix[i]) * C;
        if (dtype == SWF_F64)
            for (int k = 0; k < C; ++k) static_cast<double*>(dst)[o + k] = r[k];
        else
            std::memcpy(static_cast<float*>(dst) + o, r, size_t(C) * 4);
    }
}

// Output field: the whole grid on one rank; owned pixels only under a multi-rank topology.
void d2h_out(swf_ctx* c, const float* src_loc, int C, int dtype, void* dst) {
    if (c->world > 1)
        d2h_owned(c, src_loc, C, dtype, dst);
    else
        d2h_field(c, src_loc, C, dtype, dst);
}

// host field [N][C] -> device local window order (layout 0)
void h2d_local(swf_ctx* c, const void* src, int C, int dtype, float* dst_loc) {
    h2d_field(c, src, C, dtype, c->in_pix);
    gather_rows<float>(c->in_pix, c->lay[0], C, C, c->M, dst_loc, nullptr, 0, c->st);
    SWF_CUDA(cudaStreamSynchronize(c->st));
}

// Per-rank input loading from tiled field files (ChunkedReader::read_window_slice,
// chunked_file.cpp:156-188; the reference CLI reads whole fields, swinflow_main.cpp:128-157). The
// rank's owned windows of the unshifted layout -- only its SP band rows -- define the pixel rows it
// needs; the tiles covering them are read once each by a pool of threads sharing one descriptor
// (pread), verified, and scattered straight into the local token order [M][C]. Returns the number of
// tiles read.
unsigned long long read_local_chunked(const swf_ctx* c, const std::string& path, int C, float* dst) {
    const tiles::File f(path);
    const tiles::Grid& g = f.grid();
    require(g.H == c->H && g.W == c->W, "chunked input " + path + ": grid " + std::to_string(g.H) + "x" +
                                            std::to_string(g.W) + " does not match the model grid " +
                                            std::to_string(c->H) + "x" + std::to_string(c->W));
    require(g.C == C, "chunked input " + path + ": " + std::to_string(g.C) + " channels, expected " + std::to_string(C));
    // local token -> pixel is c->owned_pix; invert it per tile: the tiles this rank touches and, per
    // tile, the (pixel, local index) pairs inside it
    const int tc = g.cols();
    std::vector<std::vector<std::pair<long long, i64>>> need(size_t(g.count()));
    for (i64 i = 0; i < c->M; ++i) {
        const long long p = c->owned_pix[size_t(i)];
        const int y = int(p / c->W), x = int(p % c->W);
        need[size_t(y / g.th) * tc + x / g.tw].push_back({p, i});
    }
    std::vector<int> todo;
    for (int t = 0; t < g.count(); ++t)
        if (!need[size_t(t)].empty()) todo.push_back(t);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = int(std::min<size_t>(std::min(16u, hw), std::max<size_t>(todo.size(), 1)));
    std::atomic<size_t> next{0};
    std::vector<std::exception_ptr> errs(static_cast<size_t>(nt));
    auto worker = [&](int k) {
        try {
            std::vector<float> buf;
            for (size_t j = next++; j < todo.size(); j = next++) {
                const int t = todo[j], ty = t / tc, tx = t % tc;
                f.tile(ty, tx, buf);
                const tiles::Rect b = g.box(ty, tx);
                for (const auto& pi : need[size_t(t)]) {
                    const int yy = int(pi.first / c->W) - b.y0, xx = int(pi.first % c->W) - b.x0;
                    float* o = dst + size_t(pi.second) * C;
                    for (int ch = 0; ch < C; ++ch) o[ch] = buf[(size_t(ch) * b.h + yy) * b.w + xx];
                }
            }
        } catch (...) {
            errs[size_t(k)] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nt; ++k) th.emplace_back(worker, k);
    worker(0);
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    return f.tiles_read();
}

// chunked staging slots: pinned local-order buffers filled by a (background) reader thread
void stage_alloc(swf_ctx* c, swf_ctx::Staged& s) {
    const int cf = std::max(c->m.cin - 2 * c->m.cout, 1);
    if (!s.state) SWF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.state), size_t(c->M) * c->m.cout * 4, 0));
    if (!s.forcing) SWF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.forcing), size_t(c->M) * cf * 4, 0));
}
void stage_fill(swf_ctx* c, swf_ctx::Staged& s) {
    const int cf = c->m.cin - 2 * c->m.cout;
    s.reads = read_local_chunked(c, s.state_path, c->m.cout, s.state);
    if (cf > 0) s.reads += read_local_chunked(c, s.forcing_path, cf, s.forcing);
}
void stage_join(swf_ctx::Staged& s) {
    if (s.th.joinable()) s.th.join();
}
// start (background) loading of (state, forcing) into a free slot; returns the slot
int stage_start(swf_ctx* c, const std::string& state, const std::string& forcing, bool background) {
    int slot = 0;
    if (c->staged[0].pending && !c->staged[1].pending)
        slot = 1;
    else if (c->staged[0].pending && c->staged[1].pending)
        slot = c->staged[0].seq <= c->staged[1].seq ? 0 : 1;  // drop the older prefetch
    swf_ctx::Staged& s = c->staged[slot];
    stage_join(s);
    stage_alloc(c, s);
    s.state_path = state;
    s.forcing_path = forcing;
    s.err = nullptr;
    s.pending = true;
    s.seq = ++c->staged_seq;
    if (background) {
        s.th = std::thread([c, &s] {
            try {
                stage_fill(c, s);
            } catch (...) {
                s.err = std::current_exception();
            }
        });
    } else {
        stage_fill(c, s);
    }
    return slot;
}

void upload_stats(swf_ctx* c, const swf_standardizers* s, int dtype) {
    const Dims& m = c->m;
    const int cp = m.cout, cf = std::max(m.cin - 2 * m.cout, 0);
    std::vector<float> st(size_t(6) * m.cin, 0.f);
    auto get = [&](const void* p, int n, size_t off, float dflt) {
        for (int i = 0; i < n; ++i) {
            float v = dflt;
            if (p) v = dtype == SWF_F64 ? float(static_cast<const double*>(p)[i]) : static_cast<const float*>(p)[i];
            st[off + i] = v;
        }
    };
    get(s ? s->state_mean : nullptr, cp, 0, 0.f);
    get(s ? s->state_std : nullptr, cp, size_t(m.cin), 1.f);
    get(s ? s->resid_mean : nullptr, cp, size_t(2) * m.cin, 0.f);
    get(s ? s->resid_std : nullptr, cp, size_t(3) * m.cin, 1.f);
    get(s ? s->forcing_mean : nullptr, cf, size_t(4) * m.cin, 0.f);
    get(s ? s->forcing_std : nullptr, cf, size_t(5) * m.cin, 1.f);
    h2d_sync(c, c->s_stats, st.data(), st.size() * 4);
}

u64 h_splitmix(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
u64 h_kd(u64 k, u64 t) { return h_splitmix(k ^ h_splitmix(t)); }

// forecast_step on device-resident x_prev (local order): result into dst_loc.
void forecast_core(swf_ctx* c, const float* xprev_phys_loc, const float* forc_phys_loc,
                   const swf_diffusion_cfg& dc, u64 run_seed, u64 event, float* dst_loc) {
    const Dims& m = c->m;
    const int cp = m.cout, cf = m.cin - 2 * m.cout;
    require(cf >= 0, "forecast: in_channels must be >= 2 * out_channels");
    float* S = c->s_stats;
    standardize(xprev_phys_loc, c->M, cp, S, S + m.cin, c->s_tmp, c->st);
    if (cf > 0) standardize(forc_phys_loc, c->M, cf, S + 4 * m.cin, S + 5 * m.cin, c->s_cond, c->st);
    set_conditioning(c, c->s_tmp, c->s_cond);
    // z_init = noise_field(sp, key_derive(event, 0x1217), ...) (diffusion.hpp:313-315)
    const u64 zfk = h_kd(h_kd(run_seed, 0x7au), h_kd(event, 0x1217u));
    noise_field(zfk, cp, c->lay[0], dc.sigma_d, c->s_x, c->st);
    solve(c, dc, h_kd(event, 0xc4u), nullptr);
    destandardize_add(c->s_x, xprev_phys_loc, c->M, cp, S + 2 * m.cin, S + 3 * m.cin, dst_loc, c->st);
    c->launches += 5;
    if (c->world > 1) peer_barrier(c);  // the solver's divergence flags reach every rank
}

int fail(const std::exception& e, int rc) {
    g_err = e.what();
    return rc;
}

// ------------------------------------------------------------------ training loss + step
// diffusion_loss_sample (diffusion.hpp:168-192) and the microbatch loop of reference_train_step
// (simulator.hpp:50-86) in the FP32 validation mode on one rank; the DP all-reduce of the
// accumulated gradient runs over NCCL on the device buffer (swf_train_grads).
void ensure_train(swf_ctx* c) {
    ensure_sampler(c);
    ensure_bwd(c);
    if (c->tr_alloc) return;
    const Dims& m = c->m;
    const size_t n = size_t(c->M) * m.cout;
    auto& t = c->tr;
    t.x0 = dalloc<float>(c, n);
    t.z = dalloc<float>(c, n);
    t.v = dalloc<float>(c, n);
    t.kappa = dalloc<float>(c, size_t(m.cout));
    t.alpha = dalloc<float>(c, size_t(c->H));
    t.gacc = dalloc<float>(c, c->poff.back());
    t.part = dalloc<double>(c, kTrainLossBlocks);
    SWF_CUDA(cudaMallocHost(&t.h_part, sizeof(double) * kTrainLossBlocks));
    c->tr_alloc = true;
}

double h_uniform01(u64 key, u64 ctr) {  // rng.hpp:28-35
    return double(h_splitmix(key + 0x632be59bd9b4e019ULL * (ctr + 1)) >> 11) * 0x1.0p-53;
}

void set_loss_weights(swf_ctx* c, const swf_loss_weights* w, int dtype) {
    require(w && w->alpha_row && w->kappa, "loss weights: alpha_row and kappa required");
    const Dims& m = c->m;
    std::vector<float> kap(m.cout), al(c->H);
    for (int i = 0; i < m.cout; ++i) {
        kap[i] = dtype == SWF_F64 ? float(static_cast<const double*>(w->kappa)[i]) : static_cast<const float*>(w->kappa)[i];
        if (!(kap[i] > 0.f)) throw ConfigError("loss weights: kappa must be positive");  // grid.hpp:87
    }
    for (int r = 0; r < c->H; ++r)
        al[r] = dtype == SWF_F64 ? float(static_cast<const double*>(w->alpha_row)[r])
                                 : static_cast<const float*>(w->alpha_row)[r];
    SWF_CUDA(cudaMemcpyAsync(c->tr.kappa, kap.data(), kap.size() * 4, cudaMemcpyHostToDevice, c->st));
    SWF_CUDA(cudaMemcpyAsync(c->tr.alpha, al.data(), al.size() * 4, cudaMemcpyHostToDevice, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
}

// One sample: x_prev in s_tmp, forcings in s_cond, x0 and z in tr (local layout-0 order). Gradient
// into bw.gflat; returns the loss.
double train_sample_core(swf_ctx* c, const swf_diffusion_cfg& dc, u64 t_key) {
    validate_dc(dc);
    const Dims& m = c->m;
    const i64 n = c->M * m.cout;
    const double u = h_uniform01(t_key, 0);  // sample_noise_draw (diffusion.hpp:76-86)
    const double tau = (1.0 - u) * std::log(dc.sigma_min) + u * std::log(dc.sigma_max);
    const float t = static_cast<float>(std::atan(std::exp(tau) / dc.sigma_d));
    const float sd = static_cast<float>(dc.sigma_d);
    const auto cs = trig_coeffs_f(t);
    reset_flags(c);
    set_conditioning(c, c->s_tmp, c->s_cond);
    train_prep(c->tr.x0, c->tr.z, n, cs.first, cs.second, c->s_x, c->tr.v, c->st);
    assemble_state<float>(c->s_x, c->pe_loc, c->M, m.cout, m.cin, m.cinp, sd, static_cast<float*>(c->a_in), c->st);
    c->save_x = true;
    forward_any(c, double(t), 1.f);
    c->save_x = false;
    train_loss(c->out_loc, c->tr.v, c->lay[0], c->M, m.cout, c->tr.kappa, c->tr.alpha, sd, 2.f / float(c->N),
               c->bw.dS, c->tr.part, c->st);
    SWF_CUDA(cudaMemcpyAsync(c->tr.h_part, c->tr.part, sizeof(double) * kTrainLossBlocks, cudaMemcpyDeviceToHost,
                             c->st));
    check_flags(c);  // synchronizes
    double loss = 0.0;
    for (int b = 0; b < kTrainLossBlocks; ++b) loss += c->tr.h_part[b];
    backward_core(c, c->bw.dS);
    c->launches += 4;
    return loss / double(c->N);
}

void train_inputs(swf_ctx* c, const void* x_prev, const void* x0, const void* forcings, int dtype) {
    const Dims& m = c->m;
    const int cf = m.cin - 2 * m.cout;
    require(cf >= 0, "train: in_channels must be >= 2 * out_channels");
    h2d_local(c, x_prev, m.cout, dtype, c->s_tmp);
    h2d_local(c, x0, m.cout, dtype, c->tr.x0);
    if (cf > 0) {
        require(forcings != nullptr, "train: forcings required");
        h2d_local(c, forcings, cf, dtype, c->s_cond);
    }
}

void train_checks(swf_ctx* c) {
    require(c->loaded, "train: parameters not loaded");
    require(c->prec == SWF_PREC_FP32, "train: available in the FP32 validation mode (SWF_PREC_FP32)");
    require(c->sp == 1, "train: window parallelism only (SP == 1)");
    SWF_CUDA(cudaSetDevice(c->dev));
    ensure_train(c);
}

void grads_to_host(swf_ctx* c, const float* src, double scale, void* out, int dtype) {
    const size_t n = c->poff.back();
    std::vector<float> g(n);
    SWF_CUDA(cudaMemcpyAsync(g.data(), src, n * 4, cudaMemcpyDeviceToHost, c->st));
    SWF_CUDA(cudaStreamSynchronize(c->st));
    if (dtype == SWF_F64)
        for (size_t i = 0; i < n; ++i) static_cast<double*>(out)[i] = double(g[i]) * scale;
    else
        for (size_t i = 0; i < n; ++i) static_cast<float*>(out)[i] = float(double(g[i]) * scale);
}


}  // namespace

namespace swf {
void set_last_error(const std::string& m) { g_err = m; }

// Once per device and process, before any work runs on it: load every kernel and set the dynamic
// shared-memory limits (per device: the attributes live in each device's context). Both would
// otherwise happen on first use, inside the ranks' concurrent calls, and need the context idle.
void ensure_device(int device) {
    static std::mutex mu;
    static std::vector<char> done(256, 0);
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 256 || done[size_t(device)]) return;
    int prev = 0;
    SWF_CUDA(cudaGetDevice(&prev));
    SWF_CUDA(cudaSetDevice(device));
    preload_elem_kernels();
    preload_bwd_kernels();
    preload_simt_kernels();
    preload_gemm_kernels();
    preload_attn_kernels();
    cudaFuncAttributes a;
    for (const void* f : {(const void*)k_repack<float>, (const void*)k_repack<__nv_bfloat16>, (const void*)k_init_fill,
                          (const void*)k_peer_barrier})
        SWF_CUDA(cudaFuncGetAttributes(&a, f));
    SWF_CUDA(cudaSetDevice(prev));
    done[size_t(device)] = 1;
}
}  // namespace swf

// ====================================================================== C ABI
#define SWF_API_TRY(...)                                            \
    try {                                                           \
        __VA_ARGS__;                                                \
        return SWF_OK;                                              \
    } catch (const swf::NumericsError& e) {                         \
        return fail(e, SWF_ERR_NUMERICS);                           \
    } catch (const swf::ConfigError& e) {                           \
        return fail(e, SWF_ERR_CONFIG);                             \
    } catch (const swf::IoError& e) {                               \
        return fail(e, SWF_ERR_IO);                                 \
    } catch (const swf::CudaError& e) {                             \
        return fail(e, SWF_ERR_CUDA);                               \
    } catch (const std::exception& e) {                             \
        return fail(e, SWF_ERR_CUDA);                               \
    }

namespace {

// ---- single-process multi-GPU groups (swf_set_topology_devices)
thread_local bool tl_group_worker = false;  // set inside a group's per-rank threads

std::vector<swf_ctx*> group_ranks(swf_ctx* root) {
    std::vector<swf_ctx*> r{root};
    r.insert(r.end(), root->kids.begin(), root->kids.end());
    return r;
}

// Run fn(rank context) for every rank of the group on its own host thread (the ranks meet in device
// barriers, so they must run concurrently) and return the most specific failure: numerics (1) before
// config (2), I/O (3) and device (4) -- a barrier timeout on one rank is the consequence of another
// rank's error, not the cause.
template <class F>
int group_run(swf_ctx* root, F&& fn) {
    const std::vector<swf_ctx*> R = group_ranks(root);
    const size_t n = R.size();
    std::vector<int> rc(n, SWF_OK);
    std::vector<std::string> msg(n);
    std::vector<std::thread> th;
    th.reserve(n);
    for (size_t r = 0; r < n; ++r)
        th.emplace_back([&, r] {
            tl_group_worker = true;
            rc[r] = fn(R[r], int(r));
            if (rc[r] != SWF_OK) msg[r] = g_err;
        });
    for (auto& t : th) t.join();
    int best = -1;
    for (size_t r = 0; r < n; ++r)
        if (rc[r] != SWF_OK && (best < 0 || rc[r] < rc[best])) best = int(r);
    if (best < 0) return SWF_OK;
    g_err = "rank " + std::to_string(best) + ": " + msg[best];
    for (size_t r = 0; r < n; ++r)  // the other ranks' failures, for diagnosis
        if (rc[r] != SWF_OK && int(r) != best) g_err += " [rank " + std::to_string(r) + ": " + msg[r] + "]";
    return rc[best];
}

#define SWF_FANOUT(c, call)                                                                         \
    if ((c) != nullptr && !(c)->kids.empty() && !tl_group_worker)                                  \
    return group_run((c), [&](swf_ctx * r_, int rank_) {                                          \
        (void)rank_;                                                                                \
        return call;                                                                                \
    })

// Sum per-rank partial sums (f64, fixed rank order: deterministic) into out (f32 / f64).
void sum_ranks(const std::vector<std::vector<double>>& g, void* out, int dtype) {
    if (!out || g.empty()) return;
    const size_t n = g[0].size();
    for (size_t i = 0; i < n; ++i) {
        double v = 0.0;
        for (const auto& r : g) v += r[i];
        if (dtype == SWF_F64)
            static_cast<double*>(out)[i] = v;
        else
            static_cast<float*>(out)[i] = float(v);
    }
}

// Same for per-rank buffers already in the output element type.
void sum_ranks_typed(const std::vector<std::vector<char>>& g, size_t n, void* out, int dtype) {
    if (!out) return;
    for (size_t i = 0; i < n; ++i) {
        double v = 0.0;
        for (const auto& r : g)
            v += dtype == SWF_F64 ? reinterpret_cast<const double*>(r.data())[i]
                                  : double(reinterpret_cast<const float*>(r.data())[i]);
        if (dtype == SWF_F64)
            static_cast<double*>(out)[i] = v;
        else
            static_cast<float*>(out)[i] = float(v);
    }
}

void rethrow_rc(int rc) {
    if (rc == SWF_OK) return;
    if (rc == SWF_ERR_NUMERICS) throw NumericsError(g_err);
    if (rc == SWF_ERR_CONFIG) throw ConfigError(g_err);
    if (rc == SWF_ERR_IO) throw IoError(g_err);
    throw CudaError(g_err);
}

// Device tables of peer pointers (residual buffers, barrier flags, attention planes / output) from
// c->peer, after IPC mapping or in-process peer mapping.
void upload_peer_tables(swf_ctx* c) {
    for (int par = 0; par < 2; ++par) {
        std::vector<float*> t(8, nullptr);
        for (int r = 0; r < c->world; ++r) t[r] = c->peer[r].x[par];
        h2d_sync(c, c->d_xdst[par], t.data(), sizeof(float*) * 8);
    }
    std::vector<int*> ft(8, nullptr);
    std::vector<void*> qt(8, nullptr), ot(8, nullptr);
    for (int r = 0; r < c->world; ++r) {
        ft[r] = c->peer[r].flags;
        qt[r] = c->peer[r].qkv;
        ot[r] = c->peer[r].xm;
    }
    h2d_sync(c, c->d_flag_table, ft.data(), sizeof(int*) * 8);
    h2d_sync(c, c->d_qkv_dst, qt.data(), sizeof(void*) * 8);
    h2d_sync(c, c->d_o_dst, ot.data(), sizeof(void*) * 8);
    c->peers = true;
}

// Map every rank's buffers into every other rank of a single-process group: one address space, so
// the peer pointers are the ranks' own allocations; ranks on different GPUs need peer access.
void group_connect(swf_ctx* root) {
    const std::vector<swf_ctx*> R = group_ranks(root);
    for (swf_ctx* a : R)
        for (swf_ctx* b : R) {
            if (a->dev == b->dev) continue;
            int can = 0;
            SWF_CUDA(cudaDeviceCanAccessPeer(&can, a->dev, b->dev));
            if (!can)
                throw CudaError("group: device " + std::to_string(a->dev) + " cannot access device " +
                                std::to_string(b->dev) + " (no NVLink / P2P path)");
            SWF_CUDA(cudaSetDevice(a->dev));
            const cudaError_t e = cudaDeviceEnablePeerAccess(b->dev, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled)
                (void)cudaGetLastError();
            else
                SWF_CUDA(e);
        }
    for (swf_ctx* c : R) {
        SWF_CUDA(cudaSetDevice(c->dev));
        for (int r = 0; r < c->world; ++r)
            c->peer[r] = Peer{{R[r]->xbuf[0], R[r]->xbuf[1]}, R[r]->bar_flags, R[r]->qkv, R[r]->xm};
        upload_peer_tables(c);
        SWF_CUDA(cudaDeviceSynchronize());
    }
}

}  // namespace

extern "C" {

const char* swf_last_error(void) { return g_err.c_str(); }
const char* swf_version(void) { return "swinflow-b200 0.1 (sm_100a)"; }

long long swf_param_count(const swf_model_cfg* c) {
    const long long h = c->hidden_dim, f = c->ffn_dim, td = c->time_dim > 0 ? c->time_dim : c->hidden_dim;
    const long long blk = 3 * h * h + h * h + 2 * h + 3 * f * h + 6 * h * td + 6 * h;
    return (long long)c->in_channels * h + h + (long long)c->n_layers * c->blocks_per_layer * blk + td * td + td +
           h + (long long)c->out_channels * h + c->out_channels;
}

int swf_create(const swf_model_cfg* cfg, int grid_h, int grid_w, int device, int precision, swf_ctx** out) {
    SWF_API_TRY({
        require(cfg && out, "swf_create: null argument");
        validate_model(*cfg, grid_h, grid_w, precision);
        int ndev = 0;
        SWF_CUDA(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "swf_create: no CUDA device " + std::to_string(device));
        SWF_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        SWF_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw CudaError("swf_create: this build targets sm_100a (B200); found sm_" +
                                               std::to_string(prop.major) + std::to_string(prop.minor));
        ensure_device(device);
        swf_ctx* c = new swf_ctx();
        c->cfg = *cfg;
        c->m = make_dims(*cfg, precision);
        c->H = grid_h;
        c->W = grid_w;
        c->N = i64(grid_h) * grid_w;
        c->prec = precision;
        c->dev = device;
        SWF_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        *out = c;
    })
}

void swf_destroy(swf_ctx* c) {
    if (!c) return;
    for (swf_ctx* k : c->kids) swf_destroy(k);
    c->kids.clear();
    cudaSetDevice(c->dev);
    cudaStreamSynchronize(c->st);
    for (void* p : c->allocs) cudaFree(p);
    for (auto& sl : c->staged) {
        if (sl.th.joinable()) sl.th.join();
        if (sl.state) cudaFreeHost(sl.state);
        if (sl.forcing) cudaFreeHost(sl.forcing);
    }
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->h_churn_key) cudaFreeHost(c->h_churn_key);
    if (c->tr.h_part) cudaFreeHost(c->tr.h_part);
    if (c->solve_exec) cudaGraphExecDestroy(c->solve_exec);
    if (c->h_feat) cudaFreeHost(c->h_feat);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    for (int r = 0; r < int(c->peer.size()) && c->ipc_mapped; ++r) {  // unmap every IPC-opened peer buffer
        if (r == c->rank) continue;
        const Peer& pr = c->peer[r];
        for (void* p : {static_cast<void*>(pr.x[0]), static_cast<void*>(pr.x[1]), static_cast<void*>(pr.flags),
                        pr.qkv, pr.xm})
            if (p) cudaIpcCloseMemHandle(p);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (int i = 0; i < c->bt_ws.n; ++i) {
        cudaStreamSynchronize(c->bt_ws.st[i]);
        cudaStreamDestroy(c->bt_ws.st[i]);
    }
    for (int i = 0; c->bt_ws.n > 0 && i <= c->bt_ws.n; ++i) cudaEventDestroy(c->bt_ws.ev[i]);
    cudaStreamDestroy(c->st);
    delete c;
}

int swf_set_topology(swf_ctx* c, int wp_a, int wp_b, int sp, int rank, int ownership) {
    SWF_API_TRY({
        require(c, "null context");
        require(!c->allocated, "swf_set_topology must precede swf_load_params");
        require(wp_a >= 1 && wp_b >= 1 && sp >= 1, "topology: all degrees must be >= 1");
        require(wp_a * wp_b * sp <= 8, "topology: at most 8 ranks per box");
        require(rank >= 0 && rank < wp_a * wp_b * sp, "topology: rank out of range");
        require(ownership == SWF_OWN_CONTIGUOUS || ownership == SWF_OWN_ROUND_ROBIN, "topology: bad ownership");
        // build_topology constraints (topology.hpp:95-102)
        require(c->m.w % sp == 0, "topology: SP=" + std::to_string(sp) + " does not divide window side " +
                                      std::to_string(c->m.w) + " (row-band slicing)");
        require(c->m.heads % sp == 0, "topology: SP=" + std::to_string(sp) + " does not divide head count " +
                                          std::to_string(c->m.heads));
        require(sp == 1 || c->prec == SWF_PREC_BF16, "topology: sequence parallelism runs on the BF16 path");
        c->wp_a = wp_a;
        c->wp_b = wp_b;
        c->sp = sp;
        c->rank = rank;
        c->world = wp_a * wp_b * sp;
        c->wp_rank = rank / sp;
        c->band = rank % sp;
        c->own = ownership;
    })
}

int swf_set_topology_devices(swf_ctx* c, int wp_a, int wp_b, int sp, int ownership, const int* device_ids) {
    SWF_API_TRY({
        require(c && device_ids, "null argument");
        require(c->kids.empty() && !c->allocated && c->world == 1,
                "swf_set_topology_devices: once, on a fresh context, before loading parameters");
        require(device_ids[0] == c->dev, "swf_set_topology_devices: device_ids[0] must be the context's device");
        rethrow_rc(swf_set_topology(c, wp_a, wp_b, sp, 0, ownership));
        try {
            for (int r = 1; r < c->world; ++r) {
                swf_ctx* k = nullptr;
                rethrow_rc(swf_create(&c->cfg, c->H, c->W, device_ids[r], c->prec, &k));
                c->kids.push_back(k);
                rethrow_rc(swf_set_topology(k, wp_a, wp_b, sp, r, ownership));
            }
        } catch (...) {
            for (swf_ctx* k : c->kids) swf_destroy(k);
            c->kids.clear();
            c->wp_a = c->wp_b = c->sp = c->world = 1;
            c->rank = c->wp_rank = c->band = 0;
            throw;
        }
        SWF_CUDA(cudaSetDevice(c->dev));
    })
}

int swf_group_size(swf_ctx* c) { return c ? 1 + int(c->kids.size()) : 0; }
swf_ctx* swf_group_rank(swf_ctx* c, int r) {
    if (!c || r < 0 || r > int(c->kids.size())) return nullptr;
    return r == 0 ? c : c->kids[size_t(r - 1)];
}

int swf_load_params(swf_ctx* c, const void* const* arrays, int n_arrays, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const int rc = group_run(c, [&](swf_ctx* r_, int) { return swf_load_params(r_, arrays, n_arrays, dtype); });
        if (rc != SWF_OK) return rc;
        SWF_API_TRY(group_connect(c))
    }
    SWF_API_TRY({
        require(c && arrays, "null argument");
        SWF_CUDA(cudaSetDevice(c->dev));
        load_params(c, arrays, n_arrays, dtype);
    })
}

int swf_load_params_flat(swf_ctx* c, const void* flat, long long count, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const int rc = group_run(c, [&](swf_ctx* r_, int) { return swf_load_params_flat(r_, flat, count, dtype); });
        if (rc != SWF_OK) return rc;
        SWF_API_TRY(group_connect(c))
    }
    SWF_API_TRY({
        require(c && flat, "null argument");
        require(count == swf_param_count(&c->cfg), "load_params: flat count " + std::to_string(count) +
                                                        " != parameter_count_formula " +
                                                        std::to_string(swf_param_count(&c->cfg)));
        const Dims& m = c->m;
        std::vector<size_t> sizes;
        sizes.push_back(size_t(m.h) * m.cin);
        sizes.push_back(m.h);
        for (int b = 0; b < m.nb; ++b) {
            for (size_t s : {size_t(3) * m.h * m.h, size_t(m.h) * m.h, size_t(m.h), size_t(m.h), size_t(m.f) * m.h,
                             size_t(m.f) * m.h, size_t(m.h) * m.f, size_t(6) * m.h * m.td, size_t(6) * m.h})
                sizes.push_back(s);
        }
        for (size_t s : {size_t(m.td) * m.td, size_t(m.td), size_t(m.h), size_t(m.cout) * m.h, size_t(m.cout)})
            sizes.push_back(s);
        std::vector<const void*> ptrs;
        size_t off = 0;
        const size_t es = dtype == SWF_F64 ? 8 : 4;
        for (size_t s : sizes) {
            ptrs.push_back(static_cast<const char*>(flat) + off * es);
            off += s;
        }
        SWF_CUDA(cudaSetDevice(c->dev));
        load_params(c, ptrs.data(), int(ptrs.size()), dtype);
    })
}

int swf_load_checkpoint(swf_ctx* c, const char* base) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const int rc = group_run(c, [&](swf_ctx* r_, int) { return swf_load_checkpoint(r_, base); });
        if (rc != SWF_OK) return rc;
        SWF_API_TRY(group_connect(c))
    }
    SWF_API_TRY({
        require(c && base, "null argument");
        SWF_CUDA(cudaSetDevice(c->dev));
        load_checkpoint(c, base);
    })
}

// Host-only verification of a checkpoint against a model config (no GPU): manifest layout and
// every array's fnv1a64 checksum.
uint64_t swf_fnv1a64(const void* data, size_t n, uint64_t h) { return fnv1a64(data, n, h); }

int swf_param_array(const swf_model_cfg* cfg, int i, char* name, int name_len, long long* rows, long long* cols) {
    SWF_API_TRY({
        require(cfg && name && rows && cols && name_len > 0, "null argument");
        const Dims m = make_dims(*cfg, SWF_PREC_FP32);
        const auto names = param_names(m);
        const auto shapes = param_shapes(m);
        if (i < 0 || i >= int(names.size())) throw ConfigError("param_array: index out of range");
        std::snprintf(name, size_t(name_len), "%s", names[i].c_str());
        *rows = shapes[i].first;
        *cols = shapes[i].second;
    })
}

int swf_verify_checkpoint(const swf_model_cfg* cfg, const char* base) {
    SWF_API_TRY({
        require(cfg && base, "null argument");
        const Dims m = make_dims(*cfg, SWF_PREC_FP32);
        int dtype = SWF_F32;
        const auto ent = read_manifest(base, m, &dtype);
        {
            std::ifstream bin(std::string(base) + ".bin", std::ios::binary);
            if (!bin) throw IoError(std::string("cannot open checkpoint: ") + base + ".bin");
        }
        CkptReader rd(base, ent, dtype, param_names(m));
        for (size_t i = 0; i < ent.size(); ++i) rd.get(int(i));
    })
}

int swf_init_params(swf_ctx* c, uint64_t seed, int mode, double scale) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const int rc = group_run(c, [&](swf_ctx* r_, int) { return swf_init_params(r_, seed, mode, scale); });
        if (rc != SWF_OK) return rc;
        SWF_API_TRY(group_connect(c))
    }
    SWF_API_TRY({
        require(c, "null context");
        require(mode >= 0 && mode <= 2, "init_params: mode must be 0, 1 or 2");
        SWF_CUDA(cudaSetDevice(c->dev));
        init_params_device(c, seed, mode, scale);
    })
}

int swf_forward(swf_ctx* c, const void* input, double t, void* output, int dtype) {
    SWF_FANOUT(c, swf_forward(r_, input, t, output, dtype));
    SWF_API_TRY({
        require(c && input && output, "null argument");
        require(c->loaded, "forward: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        reset_flags(c);
        h2d_field(c, input, c->m.cin, dtype, c->in_pix);
        gather_input_any(c, c->in_pix);
        forward_any(c, t, 1.f);
        check_flags(c);
        d2h_out(c, c->out_loc, c->m.cout, dtype, output);
    })
}


int swf_forward_hidden(swf_ctx* c, const void* input, double t, int n_blocks, const long long* pixels,
                       long long n_pix, float* hidden, int dtype) {
    SWF_FANOUT(c, swf_forward_hidden(r_, input, t, n_blocks, pixels, n_pix, hidden, dtype));
    SWF_API_TRY({
        require(c && input && (n_pix == 0 || (pixels && hidden)), "null argument");
        require(c->loaded, "forward_hidden: parameters not loaded");
        require(n_blocks >= 0 && n_blocks <= c->m.nb, "forward_hidden: n_blocks out of range");
        require(n_pix >= 0, "forward_hidden: negative pixel count");
        for (long long k = 0; k < n_pix; ++k)
            require(pixels[k] >= 0 && pixels[k] < c->N, "forward_hidden: pixel index out of range");
        SWF_CUDA(cudaSetDevice(c->dev));
        reset_flags(c);
        h2d_field(c, input, c->m.cin, dtype, c->in_pix);
        gather_input_any(c, c->in_pix);
        c->stop_after = n_blocks;
        try {
            forward_any(c, t, 1.f);
        } catch (...) {
            c->stop_after = -1;
            throw;
        }
        c->stop_after = -1;
        i64* d_pix = static_cast<i64*>(scratch(c, SC_PIX, size_t(std::max<long long>(n_pix, 1)) * 8));
        float* d_out = scratch_f(c, SC_ROWS, size_t(std::max<long long>(n_pix, 1)) * c->m.h);
        SWF_CUDA(cudaMemcpyAsync(d_pix, pixels, size_t(n_pix) * 8, cudaMemcpyHostToDevice, c->st));
        rows_at_pixels(c->xbuf[c->hid_cur], c->lay[c->hid_par], c->rank, c->m.h, d_pix, n_pix, d_out, c->st);
        check_flags(c);
        std::vector<float> tmp(size_t(n_pix) * c->m.h);
        SWF_CUDA(cudaMemcpyAsync(tmp.data(), d_out, tmp.size() * 4, cudaMemcpyDeviceToHost, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
        // rows of pixels another rank owns stay as the caller passed them
        std::vector<char> own(size_t(n_pix), 0);
        {
            const LayMap& L = c->lay[c->hid_par];
            std::vector<int> g2rl(size_t(L.g.nx) * L.g.ny);
            SWF_CUDA(cudaMemcpy(g2rl.data(), L.glob2rl, g2rl.size() * 4, cudaMemcpyDeviceToHost));
            for (long long k = 0; k < n_pix; ++k) {
                const i64 gi = L.g.pix_to_win(pixels[k]);
                const int gw = int(gi / L.g.s()), tok = int(gi % L.g.s());
                const int band = L.band_of_row(tok / L.g.w);
                own[k] = ((g2rl[gw] >> 16) * c->sp + band) == c->rank;
            }
        }
        for (long long k = 0; k < n_pix; ++k)
            if (own[k]) std::memcpy(hidden + size_t(k) * c->m.h, tmp.data() + size_t(k) * c->m.h, size_t(c->m.h) * 4);
    })
}

int swf_block_window_forward(swf_ctx* c, int block, int wy, int wx, double t, const void* x_in, void* x_out,
                             int dtype) {
    SWF_API_TRY({
        require(c && x_in && x_out, "null argument");
        require(c->loaded, "block_window_forward: parameters not loaded");
        require(c->world == 1, "block_window_forward: single-rank contexts (a window lives on one rank)");
        require(block >= 0 && block < c->m.nb, "block_window_forward: block out of range");
        const Lay& g = c->lay[block & 1].g;
        require(wy >= 0 && wy < g.ny && wx >= 0 && wx < g.nx, "block_window_forward: window out of range");
        SWF_CUDA(cudaSetDevice(c->dev));
        const Dims& m = c->m;
        const size_t n = size_t(m.w) * m.w * m.h;
        std::vector<float> tmp(n);
        const float* src = static_cast<const float*>(x_in);
        if (dtype == SWF_F64) {
            for (size_t i = 0; i < n; ++i) tmp[i] = float(static_cast<const double*>(x_in)[i]);
            src = tmp.data();
        }
        reset_flags(c);
        SWF_CUDA(cudaMemcpyAsync(c->xbuf[0], src, n * 4, cudaMemcpyHostToDevice, c->st));
        if (c->prec == SWF_PREC_BF16)
            block_window_core<__nv_bfloat16>(c, block, wy, wx, t);
        else
            block_window_core<float>(c, block, wy, wx, t);
        check_flags(c);
        SWF_CUDA(cudaMemcpyAsync(tmp.data(), c->xbuf[1], n * 4, cudaMemcpyDeviceToHost, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
        if (dtype == SWF_F64)
            for (size_t i = 0; i < n; ++i) static_cast<double*>(x_out)[i] = tmp[i];
        else
            std::memcpy(x_out, tmp.data(), n * 4);
    })
}

int swf_backward(swf_ctx* c, const void* input, double t, const void* d_output, void* grads, void* d_input,
                 int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        // per-rank partial gradients in the caller's element type (the call's dtype also types the
        // input and output-gradient fields); the input gradient rows are disjoint per rank
        const size_t n = size_t(swf_param_count(&c->cfg)), es = dtype == SWF_F64 ? 8 : 4;
        std::vector<std::vector<char>> g(c->kids.size() + 1, std::vector<char>(n * es));
        const int rc = group_run(c, [&](swf_ctx* r_, int k) {
            return swf_backward(r_, input, t, d_output, g[size_t(k)].data(), d_input, dtype);
        });
        if (rc != SWF_OK) return rc;
        sum_ranks_typed(g, n, grads, dtype);
        return SWF_OK;
    }
    SWF_API_TRY({
        require(c && input && d_output && grads, "null argument");
        require(c->loaded, "backward: parameters not loaded");
        require(c->prec == SWF_PREC_FP32, "backward: available in the FP32 validation mode (SWF_PREC_FP32)");
        require(c->sp == 1, "backward: window parallelism only (SP == 1)");
        SWF_CUDA(cudaSetDevice(c->dev));
        ensure_bwd(c);
        reset_flags(c);
        h2d_field(c, input, c->m.cin, dtype, c->in_pix);
        gather_input_any(c, c->in_pix);
        c->save_x = true;
        forward_any(c, t, 1.f);
        c->save_x = false;
        check_flags(c);
        h2d_local(c, d_output, c->m.cout, dtype, c->bw.dtmp);  // [M][C_out] in layout-0 order
        SWF_CUDA(cudaMemcpyAsync(c->bw.dS, c->bw.dtmp, size_t(c->M) * c->m.cout * 4, cudaMemcpyDeviceToDevice, c->st));
        backward_core(c, c->bw.dS);
        check_flags(c);  // a WP peer that stalled in the backward's exchanges fails the call here
        const size_t n = c->poff.back();
        std::vector<float> g(n);
        SWF_CUDA(cudaMemcpyAsync(g.data(), c->bw.gflat, n * 4, cudaMemcpyDeviceToHost, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
        if (dtype == SWF_F64)
            for (size_t i = 0; i < n; ++i) static_cast<double*>(grads)[i] = g[i];
        else
            std::memcpy(grads, g.data(), n * 4);
        if (d_input && c->world > 1) {
            d2h_owned(c, c->bw.din, c->m.cin, dtype, d_input);
        } else if (d_input) {  // local layout-0 rows -> pixel order (in_pix holds N x C_in)
            const size_t ni = size_t(c->N) * c->m.cin;
            SWF_CUDA(cudaMemsetAsync(c->in_pix, 0, ni * 4, c->st));
            scatter_rows(c->bw.din, c->lay[0], c->m.cin, c->M, c->in_pix, c->st);
            std::vector<float> di(ni);
            SWF_CUDA(cudaMemcpyAsync(di.data(), c->in_pix, ni * 4, cudaMemcpyDeviceToHost, c->st));
            SWF_CUDA(cudaStreamSynchronize(c->st));
            if (dtype == SWF_F64)
                for (size_t i = 0; i < ni; ++i) static_cast<double*>(d_input)[i] = di[i];
            else
                std::memcpy(d_input, di.data(), ni * 4);
        }
    })
}


int swf_diffusion_loss_sample(swf_ctx* c, const void* x_prev, const void* x0, const void* forcings,
                              const swf_loss_weights* w, const swf_diffusion_cfg* dc, uint64_t t_key, const void* z,
                              double* loss, void* grads, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const size_t n = size_t(swf_param_count(&c->cfg)), es = dtype == SWF_F64 ? 8 : 4;
        std::vector<std::vector<char>> g(c->kids.size() + 1, std::vector<char>(grads ? n * es : 0));
        std::vector<double> l(c->kids.size() + 1, 0.0);
        const int rc = group_run(c, [&](swf_ctx* r_, int k) {
            return swf_diffusion_loss_sample(r_, x_prev, x0, forcings, w, dc, t_key, z, &l[size_t(k)],
                                             grads ? g[size_t(k)].data() : nullptr, dtype);
        });
        if (rc != SWF_OK) return rc;
        if (loss) {  // partial sums over the ranks' tokens, in rank order
            *loss = 0.0;
            for (double v : l) *loss += v;
        }
        if (grads) sum_ranks_typed(g, n, grads, dtype);
        return SWF_OK;
    }
    SWF_API_TRY({
        require(c && x_prev && x0 && dc && z && loss, "null argument");
        train_checks(c);
        set_loss_weights(c, w, dtype);
        train_inputs(c, x_prev, x0, forcings, dtype);
        h2d_local(c, z, c->m.cout, dtype, c->tr.z);
        *loss = train_sample_core(c, *dc, t_key);
        check_flags(c);
        if (grads) grads_to_host(c, c->bw.gflat, 1.0, grads, dtype);
    })
}

int swf_train_accumulate(swf_ctx* c, const void* x_prev, const void* x0, const void* forcings,
                         const swf_loss_weights* w, const swf_diffusion_cfg* dc, uint64_t run_seed,
                         uint64_t sample_id, double* loss, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        std::vector<double> l(c->kids.size() + 1, 0.0);
        const int rc = group_run(c, [&](swf_ctx* r_, int k) {
            return swf_train_accumulate(r_, x_prev, x0, forcings, w, dc, run_seed, sample_id, &l[size_t(k)], dtype);
        });
        if (rc == SWF_OK && loss) {
            *loss = 0.0;
            for (double v : l) *loss += v;
        }
        return rc;
    }
    SWF_API_TRY({
        require(c && x_prev && x0 && dc && loss, "null argument");
        train_checks(c);
        set_loss_weights(c, w, dtype);
        train_inputs(c, x_prev, x0, forcings, dtype);
        // z = noise_field(seeds, sample_id, ...) on the unshifted grid; t_key = SeedProtocol::t_key
        noise_field(h_kd(h_kd(run_seed, 0x7au), sample_id), c->m.cout, c->lay[0], dc->sigma_d, c->tr.z, c->st);
        c->launches++;
        *loss = train_sample_core(c, *dc, h_kd(h_kd(run_seed, 0x74u), sample_id));
        check_flags(c);  // the backward's peer exchanges completed (no partial landing buffer)
        axpy_f32(c->bw.gflat, i64(c->poff.back()), 1.f, c->tr.gacc, c->st);
        c->launches++;
        SWF_CUDA(cudaStreamSynchronize(c->st));  // the accumulator is complete for an all-reduce
    })
}

int swf_train_reset(swf_ctx* c) {
    SWF_FANOUT(c, swf_train_reset(r_));
    SWF_API_TRY({
        require(c, "null context");
        train_checks(c);
        SWF_CUDA(cudaMemsetAsync(c->tr.gacc, 0, c->poff.back() * 4, c->st));
        SWF_CUDA(cudaStreamSynchronize(c->st));
    })
}

int swf_train_grads(swf_ctx* c, float** dev_ptr, long long* n) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        g_err = "a single-process group sums its ranks' gradients itself: read them with swf_train_read";
        return SWF_ERR_CONFIG;
    }
    SWF_API_TRY({
        require(c && dev_ptr && n, "null argument");
        train_checks(c);
        *dev_ptr = c->tr.gacc;
        *n = static_cast<long long>(c->poff.back());
    })
}

int swf_train_read(swf_ctx* c, double scale, void* grads, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        const size_t n = size_t(swf_param_count(&c->cfg));
        std::vector<std::vector<double>> g(c->kids.size() + 1, std::vector<double>(n));
        const int rc = group_run(c, [&](swf_ctx* r_, int k) { return swf_train_read(r_, 1.0, g[size_t(k)].data(), SWF_F64); });
        if (rc != SWF_OK) return rc;
        for (auto& v : g)
            for (double& x : v) x *= scale;
        sum_ranks(g, grads, dtype);
        return SWF_OK;
    }
    SWF_API_TRY({
        require(c && grads, "null argument");
        train_checks(c);
        grads_to_host(c, c->tr.gacc, scale, grads, dtype);
    })
}

int swf_forward_device(swf_ctx* c, const float* d_input, double t, float* d_output) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        g_err = "swf_forward_device takes one device's pointers: call it per rank context (swf_group_rank)";
        return SWF_ERR_CONFIG;
    }
    SWF_API_TRY({
        require(c && d_input && d_output, "null argument");
        require(c->loaded, "forward: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        c->launches = 0;
        reset_flags(c);
        gather_input_any(c, d_input);
        forward_any(c, t, 1.f);
        scatter_rows(c->out_loc, c->lay[0], c->m.cout, c->M, d_output, c->st);
        c->launches++;
    })
}

int swf_sync(swf_ctx* c) {
    SWF_FANOUT(c, swf_sync(r_));
    SWF_API_TRY({
        require(c, "null context");
        SWF_CUDA(cudaSetDevice(c->dev));
        check_flags(c);
    })
}

void* swf_stream(swf_ctx* c) { return c ? static_cast<void*>(c->st) : nullptr; }

int swf_solve_pf_ode(swf_ctx* c, const void* x_init, const void* x_prev_std, const void* forcings_std,
                     const swf_diffusion_cfg* dc, uint64_t churn_key, void* x_out, int* f_evals, int dtype) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        std::vector<int> fe(c->kids.size() + 1, 0);
        const int rc = group_run(c, [&](swf_ctx* r_, int k) {
            return swf_solve_pf_ode(r_, x_init, x_prev_std, forcings_std, dc, churn_key, x_out, &fe[size_t(k)], dtype);
        });
        if (rc == SWF_OK && f_evals) *f_evals = fe[0];
        return rc;
    }
    SWF_API_TRY({
        require(c && x_init && x_prev_std && dc && x_out, "null argument");
        require(c->loaded, "solve: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        ensure_sampler(c);
        const Dims& m = c->m;
        const int cf = m.cin - 2 * m.cout;
        require(cf >= 0, "solve: in_channels must be >= 2 * out_channels");
        reset_flags(c);
        h2d_local(c, x_prev_std, m.cout, dtype, c->s_tmp);
        if (cf > 0) {
            require(forcings_std != nullptr, "solve: forcings required");
            h2d_local(c, forcings_std, cf, dtype, c->s_cond);
        }
        set_conditioning(c, c->s_tmp, c->s_cond);
        h2d_local(c, x_init, m.cout, dtype, c->s_x);
        solve(c, *dc, churn_key, f_evals);
        if (c->world > 1) peer_barrier(c);  // every rank's divergence flags, before the check
        check_flags(c);
        d2h_out(c, c->s_x, m.cout, dtype, x_out);
    })
}

int swf_forecast_step(swf_ctx* c, const void* x_prev_phys, const void* forcing_phys, const swf_standardizers* stds,
                      const swf_diffusion_cfg* dc, uint64_t run_seed, uint64_t noise_event, void* out, int dtype) {
    SWF_FANOUT(c, swf_forecast_step(r_, x_prev_phys, forcing_phys, stds, dc, run_seed, noise_event, out, dtype));
    SWF_API_TRY({
        require(c && x_prev_phys && dc && out, "null argument");
        require(c->loaded, "forecast: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        validate_dc(*dc);
        ensure_sampler(c);
        const Dims& m = c->m;
        const int cf = m.cin - 2 * m.cout;
        require(cf >= 0, "forecast: in_channels must be >= 2 * out_channels");
        reset_flags(c);
        upload_stats(c, stds, dtype);
        h2d_local(c, x_prev_phys, m.cout, dtype, c->s_base);
        float* forc = nullptr;
        if (cf > 0) {
            require(forcing_phys != nullptr, "forecast: forcings required");
            forc = scratch_f(c, SC_FORC, size_t(c->M) * cf);
            h2d_local(c, forcing_phys, cf, dtype, forc);
        }
        float* dst = scratch_f(c, SC_OUT, size_t(c->M) * m.cout);
        forecast_core(c, c->s_base, forc, *dc, run_seed, noise_event, dst);
        check_flags(c);
        d2h_out(c, dst, m.cout, dtype, out);
    })
}

int swf_prefetch_chunked(swf_ctx* c, const char* state_path, const char* forcing_path) {
    SWF_FANOUT(c, swf_prefetch_chunked(r_, state_path, forcing_path));
    SWF_API_TRY({
        require(c && state_path, "null argument");
        require(c->allocated, "prefetch: load parameters first (the topology fixes the local windows)");
        const int cf = c->m.cin - 2 * c->m.cout;
        require(cf <= 0 || forcing_path, "prefetch: forcing container required");
        stage_start(c, state_path, forcing_path ? forcing_path : "", true);
    })
}

int swf_forecast_step_chunked(swf_ctx* c, const char* state_path, const char* forcing_path,
                              const swf_standardizers* stds, const swf_diffusion_cfg* dc, uint64_t run_seed,
                              uint64_t noise_event, void* out, int dtype) {
    SWF_FANOUT(c, swf_forecast_step_chunked(r_, state_path, forcing_path, stds, dc, run_seed, noise_event, out, dtype));
    SWF_API_TRY({
        require(c && state_path && dc && out, "null argument");
        require(c->loaded, "forecast: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        validate_dc(*dc);
        ensure_sampler(c);
        const Dims& m = c->m;
        const int cf = m.cin - 2 * m.cout;
        require(cf >= 0, "forecast: in_channels must be >= 2 * out_channels");
        require(cf == 0 || forcing_path, "forecast: forcing container required");
        const std::string sp_ = state_path, fp_ = forcing_path ? forcing_path : "";
        int slot = -1;
        for (int i = 0; i < 2; ++i)
            if (c->staged[i].pending && c->staged[i].state_path == sp_ && c->staged[i].forcing_path == fp_) slot = i;
        if (slot < 0) slot = stage_start(c, sp_, fp_, false);
        swf_ctx::Staged& s = c->staged[slot];
        stage_join(s);
        s.pending = false;
        if (s.err) std::rethrow_exception(s.err);
        c->last_chunk_reads = s.reads;
        reset_flags(c);
        upload_stats(c, stds, dtype);
        SWF_CUDA(cudaMemcpyAsync(c->s_base, s.state, size_t(c->M) * m.cout * 4, cudaMemcpyHostToDevice, c->st));
        float* forc = nullptr;
        if (cf > 0) {
            forc = scratch_f(c, SC_FORC, size_t(c->M) * cf);
            SWF_CUDA(cudaMemcpyAsync(forc, s.forcing, size_t(c->M) * cf * 4, cudaMemcpyHostToDevice, c->st));
        }
        float* dst = scratch_f(c, SC_OUT, size_t(c->M) * m.cout);
        forecast_core(c, c->s_base, forc, *dc, run_seed, noise_event, dst);
        check_flags(c);
        d2h_out(c, dst, m.cout, dtype, out);
    })
}

long long swf_last_chunk_reads(swf_ctx* c) { return c ? (long long)c->last_chunk_reads : -1; }

// ---- the tiled field file itself (host only; format of chunked_file.hpp / src/chunked_file.cpp)
struct swf_chunked {
    explicit swf_chunked(const std::string& p) : f(p) {}
    swf::tiles::File f;
};

int swf_chunked_write(const char* path, const float* field, int channels, int height, int width, int chunk_h,
                      int chunk_w) {
    SWF_API_TRY({
        require(path && field, "null argument");
        swf::tiles::save(path, field, channels, height, width, chunk_h, chunk_w);
    })
}
int swf_chunked_open(const char* path, swf_chunked** out) {
    SWF_API_TRY({
        require(path && out, "null argument");
        *out = new swf_chunked(path);
    })
}
void swf_chunked_close(swf_chunked* r) { delete r; }
int swf_chunked_info(swf_chunked* r, int* channels, int* height, int* width, int* chunk_h, int* chunk_w) {
    SWF_API_TRY({
        require(r, "null reader");
        const swf::tiles::Grid& g = r->f.grid();
        if (channels) *channels = g.C;
        if (height) *height = g.H;
        if (width) *width = g.W;
        if (chunk_h) *chunk_h = g.th;
        if (chunk_w) *chunk_w = g.tw;
    })
}
int swf_chunked_read(swf_chunked* r, int y0, int x0, int h, int w, float* out) {
    SWF_API_TRY({
        require(r && out, "null argument");
        r->f.read({y0, x0, h, w}, out);
    })
}
int swf_chunked_cover(swf_chunked* r, int y0, int x0, int h, int w, long long* n) {
    SWF_API_TRY({
        require(r && n, "null argument");
        *n = (long long)r->f.grid().touched({y0, x0, h, w});
    })
}
long long swf_chunked_reads(swf_chunked* r) { return r ? (long long)r->f.tiles_read() : -1; }
void swf_chunked_reset_reads(swf_chunked* r) {
    if (r) r->f.reset_tiles_read();
}

int swf_rollout_ensemble(swf_ctx* c, const void* x_init_phys, const void* forcings_phys, int n_members, int n_steps,
                         const swf_standardizers* stds, const swf_diffusion_cfg* dc, uint64_t run_seed,
                         uint64_t rollout_id, void* out, int dtype) {
    SWF_FANOUT(c, swf_rollout_ensemble(r_, x_init_phys, forcings_phys, n_members, n_steps, stds, dc, run_seed, rollout_id, out, dtype));
    SWF_API_TRY({
        require(c && x_init_phys && dc && out, "null argument");
        require(n_members >= 1 && n_steps >= 1, "rollout: members and steps must be >= 1");
        require(c->loaded, "rollout: parameters not loaded");
        SWF_CUDA(cudaSetDevice(c->dev));
        validate_dc(*dc);
        ensure_sampler(c);
        const Dims& m = c->m;
        const int cf = m.cin - 2 * m.cout;
        require(cf >= 0, "rollout: in_channels must be >= 2 * out_channels");
        upload_stats(c, stds, dtype);
        const size_t es = dtype == SWF_F64 ? 8 : 4;
        const size_t fsz = size_t(c->N) * m.cout * es, ffsz = size_t(c->N) * std::max(cf, 0) * es;
        float* x0 = scratch_f(c, SC_RX0, size_t(c->M) * m.cout);
        float* xa = scratch_f(c, SC_RXA, size_t(c->M) * m.cout);
        float* xb = scratch_f(c, SC_RXB, size_t(c->M) * m.cout);
        float* forc = scratch_f(c, SC_RFORC, size_t(c->M) * std::max(cf, 1) * n_steps);
        h2d_local(c, x_init_phys, m.cout, dtype, x0);
        for (int k = 0; k < n_steps && cf > 0; ++k)
            h2d_local(c, static_cast<const char*>(forcings_phys) + k * ffsz, cf, dtype,
                      forc + size_t(c->M) * cf * k);
        for (int mem = 0; mem < n_members; ++mem) {
            const float* x = x0;
            for (int k = 0; k < n_steps; ++k) {
                // event = key_derive(rollout_id, m, k) (diffusion.hpp:333)
                const u64 ev = h_kd(h_kd(rollout_id, u64(mem)), u64(k));
                float* dst = (x == xa) ? xb : xa;
                reset_flags(c);
                forecast_core(c, x, forc + size_t(c->M) * std::max(cf, 0) * k, *dc, run_seed, ev, dst);
                check_flags(c);
                d2h_out(c, dst, m.cout, dtype, static_cast<char*>(out) + (size_t(mem) * n_steps + k) * fsz);
                x = dst;
            }
        }
        SWF_CUDA(cudaStreamSynchronize(c->st));
    })
}

long long swf_local_tokens(swf_ctx* c) {
    if (!c) return -1;
    try {
        allocate(c);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
    return c->M;
}

int swf_owned_pixels(swf_ctx* c, long long* pixels) {
    SWF_API_TRY({
        require(c && pixels, "null argument");
        const LayMap& L = c->lay[0];
        const int w = c->m.w, R = w / c->sp;
        i64 i = 0;
        for (int gw : c->l2g[0])
            for (int k = 0; k < R; ++k)
                for (int cc = 0; cc < w; ++cc)
                    pixels[i++] = L.g.win_to_pix(i64(gw) * w * w + i64(L.band_row(c->band, k)) * w + cc);
    })
}

long long swf_kernel_launches(swf_ctx* c) { return c ? c->launches : -1; }

// Replay one kernel class `reps` times back-to-back on the resident buffers of the last forward
// (block `blk`), timed with CUDA events on the context stream: isolates a kernel at steady clocks.
// Classes as in swf_profile_read. Returns the mean ms per launch.
int swf_bench_kernel(swf_ctx* c, int kclass, int blk, int reps, double* ms) {
    SWF_API_TRY({
        require(c && ms && reps != 0, "bad argument");
        const bool cold = reps < 0;
        if (cold) reps = -reps;
        require(c->loaded && c->prec == SWF_PREC_BF16, "bench_kernel: BF16 context with parameters required");
        const Dims& m = c->m;
        require(blk >= 0 && blk < m.nb, "bench_kernel: block out of range");
        const i64 M = c->M;
        const int par = blk & 1;
        EpiParams ep = base_ep(c);
        const float* six = c->six + size_t(blk) * 6 * m.h;
        __nv_bfloat16* xm = static_cast<__nv_bfloat16*>(c->xm);
        auto once = [&]() {
            EpiParams e = ep;
            switch (kclass) {
                case K_RMS:
                    rms_modulate<__nv_bfloat16>(c->xbuf[0], M, m.h, m.hp, c->g_attn, six, six + m.h, six + 2 * m.h,
                                                xm, nullptr, 0, c->st);
                    break;
                case K_QKV:
                    e.cur = c->lay[par];
                    e.out = c->qkv;
                    e.plane = i64(c->lay[par].nloc) * (m.heads / c->sp) * m.w * m.w * m.d;
                    e.N = 3 * m.h;
                    e.inv_r = c->invr;  // fused norm, as in the forward (last reduced rows)
                    e.beta = c->beta_qkv[blk];
                    gemm_bf16_tc(c->tm_xb[par], c->tm_qkv[blk], M, m.np_qkv, m.hp, m.bn_qkv, EPI_QKV, e, c->st);
                    break;
                case K_ATTN: {
                    AttnParams ap;
                    ap.q = c->qkv;
                    ap.k = static_cast<const char*>(c->qkv) + size_t(M) * m.h * 2;
                    ap.v = static_cast<const char*>(c->qkv) + size_t(2) * M * m.h * 2;
                    ap.o = c->sbuf;  // scratch: keep xm intact
                    ap.ldo = m.hp;
                    ap.nloc = c->lay[par].nloc;
                    ap.heads = m.heads / c->sp;
                    ap.head0 = c->band * (m.heads / c->sp);
                    ap.wp_rank = c->wp_rank;
                    {
                        void**& scratch_tab = c->bench_otab;  // o_dst table pointing at sbuf (scratch), per context
                        if (!scratch_tab) {
                            scratch_tab = dalloc<void*>(c, 8);
                            std::vector<void*> t(8, c->sbuf);
                            h2d_sync(c, scratch_tab, t.data(), sizeof(void*) * 8);
                        }
                        ap.o_dst = scratch_tab;
                    }
                    ap.s = m.w * m.w;
                    ap.d = m.d;
                    ap.w = m.w;
                    ap.lay = c->lay[par];
                    ap.scale = 1.0f / std::sqrt(float(m.d));
                    ap.tmq = &c->tm_q;
                    ap.tmk = &c->tm_k;
                    ap.tmk2 = &c->tm_k2;
                    ap.tmv = &c->tm_vt;
                    ap.tmo = c->sp == 1 ? &c->tm_so : nullptr;
                    attention_bf16(ap, c->st);
                    break;
                }
                case K_OUT:
                    e.x = c->xbuf[1];
                    e.N = m.h;
                    gemm_bf16_tc(c->tm_xm, c->tm_out[blk], M, m.np_out, m.hp, m.bn_out, EPI_RESID, e, c->st);
                    break;
                case K_GATEUP:
                    e.out = c->sbuf;
                    e.ld_out = m.fp;
                    e.N = m.f;
                    e.G = m.G;
                    e.inv_r = c->invr;
                    e.beta = c->beta_gu[blk];
                    gemm_bf16_tc(c->tm_xb[par], c->tm_gu[blk], M, m.np_gu, m.hp, m.bn_gu, EPI_SWIGLU, e, c->st);
                    break;
                case K_DOWN:
                    e.x = c->xbuf[0];
                    e.N = m.h;
                    e.cur = c->lay[par];
                    e.nxt = c->lay[par ^ 1];
                    e.xdst = c->d_xdst[1];
                    gemm_bf16_tc(c->tm_s, c->tm_down[blk], M, m.np_down, m.fp, m.bn_down, EPI_DOWN, e, c->st);
                    break;
                default:
                    throw ConfigError("bench_kernel: unsupported kernel class");
            }
        };
        SWF_CUDA(cudaSetDevice(c->dev));
        if (!cold) once();  // cold: time the very first launch (no warm-up) -- exposes clock state
        cudaEvent_t a, b;
        SWF_CUDA(cudaEventCreate(&a));
        SWF_CUDA(cudaEventCreate(&b));
        SWF_CUDA(cudaEventRecord(a, c->st));
        for (int i = 0; i < reps; ++i) once();
        SWF_CUDA(cudaEventRecord(b, c->st));
        SWF_CUDA(cudaEventSynchronize(b));
        float t = 0.f;
        SWF_CUDA(cudaEventElapsedTime(&t, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *ms = double(t) / reps;
    })
}

int swf_set_backward_precision(swf_ctx* c, int precision) {
    SWF_FANOUT(c, swf_set_backward_precision(r_, precision));
    SWF_API_TRY({
        require(c, "null context");
        require(precision == SWF_PREC_BF16 || precision == SWF_PREC_FP32,
                "backward precision must be SWF_PREC_BF16 or SWF_PREC_FP32");
        const bool tc = precision == SWF_PREC_BF16;
        if (tc)
            require(c->m.h % 8 == 0 && c->m.f % 8 == 0,
                    "BF16 backward: hidden_dim and ffn_dim must be multiples of 8 (16-byte operand rows)");
        SWF_CUDA(cudaSetDevice(c->dev));
        SWF_CUDA(cudaStreamSynchronize(c->st));
        c->bwd_tc = tc;
        if (tc && c->bw_alloc) alloc_bwd_tc(c);  // work buffers exist already: add the operand copies
    })
}

int swf_set_graphs(swf_ctx* c, int enable) {
    SWF_FANOUT(c, swf_set_graphs(r_, enable));
    SWF_API_TRY({
        require(c, "null context");
        SWF_CUDA(cudaStreamSynchronize(c->st));
        c->graphs = enable != 0;
    })
}

int swf_profile(swf_ctx* c, int enable) {
    SWF_FANOUT(c, swf_profile(r_, enable));
    SWF_API_TRY({
        require(c, "null context");
        SWF_CUDA(cudaStreamSynchronize(c->st));
        c->prof = enable != 0;
        c->prof_ev.clear();
        c->ev_used = 0;
        for (int k = 0; k < 16; ++k) {
            c->prof_ms[k] = 0;
            c->prof_n[k] = 0;
        }
    })
}

// Raw per-launch list of the profiled region (class id, ms) in launch order.
int swf_profile_launches(swf_ctx* c, int* classes, double* ms, int max_n, int* n_out) {
    SWF_API_TRY({
        require(c && classes && ms && n_out, "null argument");
        SWF_CUDA(cudaStreamSynchronize(c->st));
        int n = 0;
        for (auto& pe : c->prof_ev) {
            if (n >= max_n) break;
            float t = 0.f;
            SWF_CUDA(cudaEventElapsedTime(&t, pe.second.first, pe.second.second));
            classes[n] = pe.first;
            ms[n] = t;
            ++n;
        }
        *n_out = n;
    })
}

int swf_profile_read(swf_ctx* c, double* ms, long long* launches, int n) {
    SWF_API_TRY({
        require(c && ms && launches, "null argument");
        SWF_CUDA(cudaStreamSynchronize(c->st));
        for (auto& pe : c->prof_ev) {
            float t = 0.f;
            SWF_CUDA(cudaEventElapsedTime(&t, pe.second.first, pe.second.second));
            c->prof_ms[pe.first] += t;
            c->prof_n[pe.first] += 1;
        }
        c->prof_ev.clear();
        c->ev_used = 0;
        for (int k = 0; k < n && k < 16; ++k) {
            ms[k] = c->prof_ms[k];
            launches[k] = c->prof_n[k];
        }
    })
}

int swf_noise_field(swf_ctx* c, uint64_t run_seed, uint64_t event, int channels, double sigma_d, float* out) {
    SWF_FANOUT(c, swf_noise_field(r_, run_seed, event, channels, sigma_d, out));
    SWF_API_TRY({
        require(c && out && channels > 0, "bad argument");
        SWF_CUDA(cudaSetDevice(c->dev));
        allocate(c);
        float* z = scratch_f(c, SC_NOISE, size_t(c->M) * channels);
        noise_field(h_kd(h_kd(run_seed, 0x7au), event), channels, c->lay[0], sigma_d, z, c->st);
        if (c->world > 1) {
            d2h_owned(c, z, channels, SWF_F32, out);
        } else {
            float* zp = scratch_f(c, SC_NOISE_PIX, size_t(c->N) * channels);
            scatter_rows(z, c->lay[0], channels, c->M, zp, c->st);
            SWF_CUDA(cudaMemcpyAsync(out, zp, size_t(c->N) * channels * 4, cudaMemcpyDeviceToHost, c->st));
            SWF_CUDA(cudaStreamSynchronize(c->st));
        }
    })
}

int swf_ipc_handles(swf_ctx* c, void* out) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        g_err = "a single-process group is already connected (no IPC)";
        return SWF_ERR_CONFIG;
    }
    SWF_API_TRY({
        require(c && out, "null argument");
        SWF_CUDA(cudaSetDevice(c->dev));
        allocate(c);
        cudaIpcMemHandle_t h[5];
        SWF_CUDA(cudaIpcGetMemHandle(&h[0], c->xbuf[0]));
        SWF_CUDA(cudaIpcGetMemHandle(&h[1], c->xbuf[1]));
        SWF_CUDA(cudaIpcGetMemHandle(&h[2], c->bar_flags));
        SWF_CUDA(cudaIpcGetMemHandle(&h[3], c->qkv));
        SWF_CUDA(cudaIpcGetMemHandle(&h[4], c->xm));
        std::memcpy(out, h, sizeof h);
    })
}

int swf_connect_peers(swf_ctx* c, const void* all) {
    if (c && !c->kids.empty() && !tl_group_worker) {
        g_err = "a single-process group is already connected (no IPC)";
        return SWF_ERR_CONFIG;
    }
    SWF_API_TRY({
        require(c && all, "null argument");
        SWF_CUDA(cudaSetDevice(c->dev));
        allocate(c);
        const size_t hs = 5 * sizeof(cudaIpcMemHandle_t);
        for (int r = 0; r < c->world; ++r) {
            if (r == c->rank) continue;
            const cudaIpcMemHandle_t* h =
                reinterpret_cast<const cudaIpcMemHandle_t*>(static_cast<const char*>(all) + r * hs);
            void* p[5];
            for (int k = 0; k < 5; ++k) SWF_CUDA(cudaIpcOpenMemHandle(&p[k], h[k], cudaIpcMemLazyEnablePeerAccess));
            c->peer[r].x[0] = static_cast<float*>(p[0]);
            c->peer[r].x[1] = static_cast<float*>(p[1]);
            c->peer[r].flags = static_cast<int*>(p[2]);
            c->peer[r].qkv = p[3];
            c->peer[r].xm = p[4];
        }
        c->ipc_mapped = true;
        upload_peer_tables(c);
        SWF_CUDA(cudaDeviceSynchronize());
    })
}

// Isolated attention (test infrastructure for head_attention_fwd, swin.hpp:161-188): the windows of
// an (n_wy w) x (n_wx w) grid under `shift` (seam mask on the last window row when shift > 0),
// q / k / v [n_win][heads][s][d] host fp32 (bf16-representable for the BF16 kernel), o
// [n_win][s][heads d] fp32. Same planes, TMA maps and launch as the forward.
int swf_selftest_attention(int device, int precision, int n_wy, int n_wx, int w, int shift, int heads, int d,
                           const float* q, const float* k, const float* v, float* o, int flags) {
    std::vector<void*> mem;
    auto cleanup = [&]() {
        for (void* p : mem) cudaFree(p);
    };
    try {
        require(q && k && v && o, "null argument");
        require(n_wy >= 1 && n_wx >= 1 && w >= 1 && heads >= 1 && shift >= 0 && shift < w, "attention: bad shape");
        require(precision == SWF_PREC_BF16 || precision == SWF_PREC_FP32, "attention: bad precision");
        const bool bf = precision == SWF_PREC_BF16;
        if (bf) require((d == 32 || d == 64 || d == 128) && w % 4 == 0, "attention: BF16 needs d in {32,64,128}");
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        const int nwin = n_wy * n_wx, s = w * w, hd = heads * d;
        const int ldo = int(roundup(hd, 64));
        const size_t n = size_t(nwin) * heads * s * d;
        auto alloc = [&](size_t bytes) {
            void* p = nullptr;
            SWF_CUDA(cudaMalloc(&p, bytes + 256));
            SWF_CUDA(cudaMemset(p, 0, bytes + 256));
            mem.push_back(p);
            return p;
        };
        LayMap L;
        L.g = make_lay(n_wy * w, n_wx * w, w, shift);
        L.nloc = nwin;
        L.sp = 1;
        L.band = 0;
        std::vector<int> ident(static_cast<size_t>(nwin));
        for (int i = 0; i < nwin; ++i) ident[i] = i;
        int* d_ident = static_cast<int*>(alloc(ident.size() * 4));
        SWF_CUDA(cudaMemcpy(d_ident, ident.data(), ident.size() * 4, cudaMemcpyHostToDevice));
        L.loc2glob = d_ident;
        L.glob2rl = d_ident;
        AttnParams ap;
        ap = AttnParams{};
        ap.ldo = ldo;
        ap.nloc = nwin;
        ap.heads = heads;
        ap.s = s;
        ap.d = d;
        ap.w = w;
        ap.lay = L;
        ap.scale = 1.0f / std::sqrt(float(d));
        ap.dbg = flags;
        std::vector<float> out(size_t(nwin) * s * ldo);
        if (bf) {
            std::vector<__nv_bfloat16> hq(n), hk(n), hv(n);
            for (size_t i = 0; i < n; ++i) {
                hq[i] = __float2bfloat16_rn(q[i]);
                hk[i] = __float2bfloat16_rn(k[i]);
            }
            for (size_t pl = 0; pl < size_t(nwin) * heads; ++pl)  // V^T planes [d][s]
                for (int t = 0; t < s; ++t)
                    for (int j = 0; j < d; ++j) hv[(pl * d + j) * s + t] = __float2bfloat16_rn(v[(pl * s + t) * d + j]);
            char* qkv = static_cast<char*>(alloc(3 * n * 2));
            SWF_CUDA(cudaMemcpy(qkv, hq.data(), n * 2, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(qkv + n * 2, hk.data(), n * 2, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(qkv + 2 * n * 2, hv.data(), n * 2, cudaMemcpyHostToDevice));
            __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(alloc(out.size() * 2));
            TmaMap tq, tk, tk2, tv, to;
            const int sw = d >= 64 ? 128 : 2 * d;
            const i64 rows = i64(nwin) * heads * s;
            make_tma_bf16_2d(&tq, qkv, rows, d, sw / 2, 128, sw);
            make_tma_bf16_2d(&tk, qkv + n * 2, rows, d, sw / 2, 64, sw);
            make_tma_bf16_2d(&tk2, qkv + n * 2, rows, d, sw / 2, 32, sw);
            make_tma_bf16_2d(&tv, qkv + 2 * n * 2, i64(nwin) * heads * d, s, 64, d / 2, 128);
            make_tma_bf16(&to, ob, i64(nwin) * s, ldo, 128);
            void** otab = static_cast<void**>(alloc(8 * sizeof(void*)));
            std::vector<void*> t8(8, ob);
            SWF_CUDA(cudaMemcpy(otab, t8.data(), 8 * sizeof(void*), cudaMemcpyHostToDevice));
            ap.q = qkv;
            ap.k = qkv + n * 2;
            ap.v = qkv + 2 * n * 2;
            ap.o = ob;
            ap.o_dst = otab;
            ap.tmq = &tq;
            ap.tmk = &tk;
            ap.tmk2 = &tk2;
            ap.tmv = &tv;
            ap.tmo = &to;
            attention_bf16(ap, nullptr);
            SWF_CUDA(cudaDeviceSynchronize());
            std::vector<__nv_bfloat16> ho(out.size());
            SWF_CUDA(cudaMemcpy(ho.data(), ob, ho.size() * 2, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < out.size(); ++i) out[i] = __bfloat162float(ho[i]);
        } else {
            float* qkv = static_cast<float*>(alloc(3 * n * 4));
            SWF_CUDA(cudaMemcpy(qkv, q, n * 4, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(qkv + n, k, n * 4, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(qkv + 2 * n, v, n * 4, cudaMemcpyHostToDevice));
            float* of = static_cast<float*>(alloc(out.size() * 4));
            ap.q = qkv;
            ap.k = qkv + n;
            ap.v = qkv + 2 * n;
            ap.o = of;
            attention_f32(ap, nullptr);
            SWF_CUDA(cudaDeviceSynchronize());
            SWF_CUDA(cudaMemcpy(out.data(), of, out.size() * 4, cudaMemcpyDeviceToHost));
        }
        for (size_t r = 0; r < size_t(nwin) * s; ++r) std::memcpy(o + r * hd, out.data() + r * ldo, size_t(hd) * 4);
        cleanup();
        return SWF_OK;
    } catch (const ConfigError& e) {
        cleanup();
        return fail(e, SWF_ERR_CONFIG);
    } catch (const std::exception& e) {
        cleanup();
        return fail(e, SWF_ERR_CUDA);
    }
}

// ---------------------------------------------------------------- host-only planning (no GPU)
// Window owner of every window under the given ownership rule (topology.hpp:107-109 for
// round-robin), rank = a * wp_b + b.
int swf_plan_owners(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int ownership, int* owner) {
    SWF_API_TRY({
        require(owner && window_px > 0 && grid_h % window_px == 0 && grid_w % window_px == 0, "plan: bad grid");
        const int ny = grid_h / window_px, nx = grid_w / window_px;
        require(wp_a >= 1 && wp_b >= 1 && ny % wp_a == 0 && nx % wp_b == 0, "plan: WP grid does not divide windows");
        for (int wy = 0; wy < ny; ++wy)
            for (int wx = 0; wx < nx; ++wx) {
                const int oa = ownership == SWF_OWN_ROUND_ROBIN ? wy % wp_a : wy / (ny / wp_a);
                const int ob = ownership == SWF_OWN_ROUND_ROBIN ? wx % wp_b : wx / (nx / wp_b);
                owner[wy * nx + wx] = oa * wp_b + ob;
            }
    })
}

// Local token order of a rank (no GPU): pixel of every local token of layout 0, as the device uses
// it (owned windows, SP band rows in ascending r, columns).
int swf_plan_tokens(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int sp, int ownership, int rank,
                    long long* pixels) {
    SWF_API_TRY({
        require(pixels && sp >= 1 && window_px % sp == 0, "plan: bad SP degree");
        const int ny = grid_h / window_px, nx = grid_w / window_px;
        std::vector<int> own(size_t(ny) * nx);
        const int rc = swf_plan_owners(grid_h, grid_w, window_px, wp_a, wp_b, ownership, own.data());
        if (rc) return rc;
        LayMap L;
        L.g = make_lay(grid_h, grid_w, window_px, 0);
        L.sp = sp;
        L.band = rank % sp;
        const int R = window_px / sp;
        i64 i = 0;
        for (int gw = 0; gw < ny * nx; ++gw) {
            if (own[gw] != rank / sp) continue;
            for (int k = 0; k < R; ++k)
                for (int cc = 0; cc < window_px; ++cc)
                    pixels[i++] = L.g.win_to_pix(i64(gw) * window_px * window_px +
                                                 i64(L.band_row(L.band, k)) * window_px + cc);
        }
    })
}

// Tokens each rank sends to another rank at a block boundary shift_from -> shift_to (the
// owner-changed tokens of shift_transfer_plan, topology.hpp:149-188): sent[src * world + dst].
int swf_plan_exchange(int grid_h, int grid_w, int window_px, int wp_a, int wp_b, int ownership, int shift_from,
                      int shift_to, long long* sent) {
    SWF_API_TRY({
        const int ny = grid_h / window_px, nx = grid_w / window_px, world = wp_a * wp_b;
        std::vector<int> own(size_t(ny) * nx);
        const int rc = swf_plan_owners(grid_h, grid_w, window_px, wp_a, wp_b, ownership, own.data());
        if (rc) return rc;
        for (int i = 0; i < world * world; ++i) sent[i] = 0;
        const Lay from = make_lay(grid_h, grid_w, window_px, shift_from), to = make_lay(grid_h, grid_w, window_px, shift_to);
        const i64 N = i64(grid_h) * grid_w;
        for (i64 p = 0; p < N; ++p) {
            const int s = own[from.pix_to_win(p) / (window_px * window_px)];
            const int d = own[to.pix_to_win(p) / (window_px * window_px)];
            if (s != d) sent[s * world + d]++;
        }
    })
}

}  // extern "C"
