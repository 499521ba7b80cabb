// swf_oracle.cpp -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// CPU restatement of the reference swinflow denoiser hot path (arxiv 2509.13523 / AERIS,
// /root/reference/proj/include/swinflow/*), written without Eigen so that it builds with
// plain g++ here and on the GPU box. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.
//
// Parity pin: the reference itself cannot be compiled in this image (it needs Eigen3 and
// the un-vendored doctest/CLI11, proj/CMakeLists.txt:10-11), so this restatement is pinned
// on the reference's own frozen golden values (tests/test_oracle_golden.py):
//   * forward golden probe y(1,77) = 1.2440901490316572 (proj/tests/test_swin_core.cpp:415-422)
//   * parameter count 1,324,144,198 (test_swin_core.cpp:157-173)
//   * sampler contraction 0.968827, t endpoints (test_trigflow.cpp:58-81, 296-306)
//   * index-map KATs (test_swin_core.cpp:76-113, test_topology.cpp:128-235)
//
// Layout conventions follow the reference's Eigen column-major storage: a C x N field is
// stored as [N][C] (token-major), a weight W (out x in) as [in][out].
//
// Every function names the reference file:line it restates.

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;

namespace orc {

// ---------------------------------------------------------------- errors
// common.hpp:28-55 -- ConfigError (rc 2), NumericsError (rc 1).
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericsError : std::runtime_error {
    explicit NumericsError(const std::string& m) : std::runtime_error(m) {}
};
static void require(bool c, const std::string& m) {
    if (!c) throw ConfigError(m);
}

// ---------------------------------------------------------------- rng.hpp:17-45
static inline u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static inline u64 kd(u64 key, u64 tag) { return splitmix64(key ^ splitmix64(tag)); }
static inline u64 kd2(u64 key, u64 a, u64 b) { return kd(kd(key, a), b); }
static inline u64 rbits(u64 key, u64 ctr) { return splitmix64(key + 0x632be59bd9b4e019ULL * (ctr + 1)); }
static inline double uniform01(u64 key, u64 ctr) { return double(rbits(key, ctr) >> 11) * 0x1.0p-53; }
static inline double gaussian(u64 key, u64 ctr) {
    const double u1 = (double(rbits(key, 2 * ctr) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = double(rbits(key, 2 * ctr + 1) >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// ---------------------------------------------------------------- config (model.hpp:21-62)
struct Cfg {
    int hidden_dim, n_heads, ffn_dim, n_layers, blocks_per_layer, window_px, in_channels, out_channels,
        time_dim;
    int nb() const { return n_layers * blocks_per_layer; }
    int hd() const { return hidden_dim / n_heads; }
    int td() const { return time_dim > 0 ? time_dim : hidden_dim; }
    void validate() const {
        require(hidden_dim > 0 && n_heads > 0 && ffn_dim > 0 && n_layers > 0, "model: dims must be positive");
        require(blocks_per_layer >= 1, "model: blocks_per_layer must be >= 1");
        require(hidden_dim % n_heads == 0, "model: hidden_dim must divide by n_heads");
        require(hd() % 4 == 0, "model: head_dim must be divisible by 4 (axial rotary pairs)");
        require(in_channels > 0 && out_channels > 0, "model: channel counts must be positive");
        require(in_channels % 2 == 0, "model: in_channels must be even (positional encoding split)");
        require(window_px > 0, "model: window size must be positive");
    }
    void validate_grid(int H, int W) const {
        validate();
        require(H % window_px == 0 && W % window_px == 0, "model: grid not divisible by window size");
    }
};

// ---------------------------------------------------------------- window.hpp:26-85
struct Layout {
    int H, W, w, shift;
    int ny() const { return H / w; }
    int nx() const { return W / w; }
    int nwin() const { return ny() * nx(); }
    int s() const { return w * w; }
    i64 pixel_of(int wy, int wx, int r, int c) const {  // window.hpp:46-50
        const int y = (wy * w + shift + r) % H;
        const int x = (wx * w + shift + c) % W;
        return i64(y) * W + x;
    }
    bool seam(int wy) const { return shift > 0 && wy == ny() - 1; }  // :60
    int seam_group(int r) const { return r < w - shift ? 0 : 1; }    // :65
    int band_of_row(int r, int sp) const { return ((shift + r) % w) / (w / sp); }  // :69
};
static int shift_for_block(int b, int w) { return (b % 2 == 0) ? 0 : w / 2; }  // window.hpp:83-85

// ---------------------------------------------------------------- parameter layout (model.hpp:140-168)
struct ArrDesc {
    std::string name;
    i64 rows, cols;
};
static std::vector<ArrDesc> param_arrays(const Cfg& c) {
    const i64 h = c.hidden_dim, f = c.ffn_dim, td = c.td();
    std::vector<ArrDesc> a;
    a.push_back({"encode.w", h, c.in_channels});
    a.push_back({"encode.b", h, 1});
    for (int b = 0; b < c.nb(); ++b) {
        const std::string p = "block" + std::to_string(b) + ".";
        a.push_back({p + "qkv.w", 3 * h, h});
        a.push_back({p + "out.w", h, h});
        a.push_back({p + "rms_attn.g", h, 1});
        a.push_back({p + "rms_ffn.g", h, 1});
        a.push_back({p + "gate.w", f, h});
        a.push_back({p + "up.w", f, h});
        a.push_back({p + "down.w", h, f});
        a.push_back({p + "ada.w", 6 * h, td});
        a.push_back({p + "ada.b", 6 * h, 1});
    }
    a.push_back({"time.w", td, td});
    a.push_back({"time.b", td, 1});
    a.push_back({"decode.g", h, 1});
    a.push_back({"decode.w", c.out_channels, h});
    a.push_back({"decode.b", c.out_channels, 1});
    return a;
}
static const int kPerBlock = 9;
static const int kHead = 2;  // encode.w, encode.b

// parameter_count_formula, model.hpp:118-129
static i64 param_count_formula(const Cfg& c) {
    const i64 h = c.hidden_dim, f = c.ffn_dim, td = c.td();
    const i64 blk = 3 * h * h + h * h + 2 * h + 3 * f * h + 6 * h * td + 6 * h;
    return i64(c.in_channels) * h + h + c.nb() * blk + td * td + td + h + i64(c.out_channels) * h +
           c.out_channels;
}

// Views of a flat parameter vector laid out in canonical order.
template <class T>
struct Params {
    Cfg cfg;
    std::vector<const T*> arr;
    const T* enc_w() const { return arr[0]; }
    const T* enc_b() const { return arr[1]; }
    const T* blk(int b, int k) const { return arr[kHead + b * kPerBlock + k]; }
    const T* tail(int k) const { return arr[kHead + cfg.nb() * kPerBlock + k]; }
};
template <class T>
static Params<T> view(const Cfg& c, const T* flat) {
    Params<T> p;
    p.cfg = c;
    i64 off = 0;
    for (const auto& a : param_arrays(c)) {
        p.arr.push_back(flat + off);
        off += a.rows * a.cols;
    }
    return p;
}

// init_parameters (model.hpp:185-209) and init_parameters_random (:213-223).
template <class T>
static void init_params(const Cfg& c, u64 seed, int random, double scale, T* flat) {
    const auto arrs = param_arrays(c);
    std::vector<T*> ptr;
    i64 off = 0;
    for (const auto& a : arrs) {
        ptr.push_back(flat + off);
        off += a.rows * a.cols;
    }
    std::memset(flat, 0, sizeof(T) * off);
    const int h = c.hidden_dim, f = c.ffn_dim, td = c.td();
    u64 stream = 0;
    auto fill = [&](int ai, double sc) {
        const u64 key = kd2(seed, 0x1217u, stream++);
        const i64 n = arrs[ai].rows * arrs[ai].cols;
        for (i64 i = 0; i < n; ++i) ptr[ai][i] = static_cast<T>(sc * gaussian(key, u64(i)));
    };
    auto ones = [&](int ai) {
        for (i64 i = 0; i < arrs[ai].rows; ++i) ptr[ai][i] = T(1);
    };
    fill(0, 1.0 / std::sqrt(double(c.in_channels)));
    for (int b = 0; b < c.nb(); ++b) {
        const int base = kHead + b * kPerBlock;
        fill(base + 0, 1.0 / std::sqrt(double(h)));
        fill(base + 1, 1.0 / std::sqrt(double(h) * 2 * c.nb()));
        ones(base + 2);
        ones(base + 3);
        fill(base + 4, 1.0 / std::sqrt(double(h)));
        fill(base + 5, 1.0 / std::sqrt(double(h)));
        fill(base + 6, 1.0 / std::sqrt(double(f) * 2 * c.nb()));
    }
    const int tb = kHead + c.nb() * kPerBlock;
    fill(tb + 0, 1.0 / std::sqrt(double(td)));
    ones(tb + 2);
    if (random) {
        u64 st = 1000;
        for (std::size_t j = 0; j < arrs.size(); ++j) {
            const u64 key = kd2(seed, 0xabcu, st++);
            const i64 n = arrs[j].rows * arrs[j].cols;
            for (i64 i = 0; i < n; ++i) ptr[j][i] += static_cast<T>(scale * gaussian(key, u64(i)));
        }
    }
}

// ---------------------------------------------------------------- small dense helpers
// Y[n][out] = sum_k W(out,k) X[n][k]  (+ b). W column-major (out x in) => Wm[k*out + o].
// Restates ops::linear_cols (swin.hpp:49-54): each output column is an independent GEMV,
// blocked here over tokens and outputs for cache reuse; the per-column K order is k=0..in-1.
template <class T>
static void linear(const T* Wm, const T* b, int out, int in, const T* X, i64 n, T* Y) {
    const int TB = 16, OB = 256;
#pragma omp parallel for schedule(static)
    for (i64 n0 = 0; n0 < n; n0 += TB) {
        const int nt = int(std::min<i64>(TB, n - n0));
        T acc[TB][OB];
        for (int o0 = 0; o0 < out; o0 += OB) {
            const int ot = std::min(OB, out - o0);
            for (int j = 0; j < nt; ++j)
                for (int o = 0; o < ot; ++o) acc[j][o] = T(0);
            for (int k = 0; k < in; ++k) {
                const T* wr = Wm + i64(k) * out + o0;
                for (int j = 0; j < nt; ++j) {
                    const T xv = X[(n0 + j) * in + k];
                    T* a = acc[j];
#pragma omp simd
                    for (int o = 0; o < ot; ++o) a[o] += wr[o] * xv;
                }
            }
            for (int j = 0; j < nt; ++j)
                for (int o = 0; o < ot; ++o) Y[(n0 + j) * out + o0 + o] = b ? acc[j][o] + b[o0 + o] : acc[j][o];
        }
    }
}

template <class T>
static T silu(T x) {
    return x / (T(1) + std::exp(-x));  // model.hpp:243-246
}

// time_features + time_embed (model.hpp:229-241, 261-269)
template <class T>
static std::vector<T> time_embed(const Params<T>& p, T t) {
    const int td = p.cfg.td();
    std::vector<T> f(td), lin(td);
    const int nf = td / 2;
    for (int k = 0; k < nf; ++k) {
        const double om = std::pow(10000.0, -double(k) / nf);
        const double arg = double(t) * 636.6197723675814 * om;
        f[2 * k] = static_cast<T>(std::sin(arg));
        f[2 * k + 1] = static_cast<T>(std::cos(arg));
    }
    if (td % 2 == 1) f[td - 1] = T(1);
    const T* Wt = p.tail(0);
    const T* bt = p.tail(1);
    for (int o = 0; o < td; ++o) {
        T acc = T(0);
        for (int k = 0; k < td; ++k) acc += Wt[i64(k) * td + o] * f[k];
        lin[o] = acc + bt[o];
    }
    for (int o = 0; o < td; ++o) lin[o] = silu(lin[o]);
    return lin;
}

// ada_vectors (swin.hpp:28-41): six = b_ada + W_ada * embed, split [a1,b1,g1,a2,b2,g2].
template <class T>
static std::vector<T> ada_six(const Params<T>& p, int blk, const std::vector<T>& emb) {
    const int h = p.cfg.hidden_dim, td = p.cfg.td();
    const T* Wa = p.blk(blk, 7);
    const T* ba = p.blk(blk, 8);
    std::vector<T> six(6 * h);
    for (int o = 0; o < 6 * h; ++o) {
        T acc = T(0);
        for (int k = 0; k < td; ++k) acc += Wa[i64(k) * 6 * h + o] * emb[k];
        six[o] = ba[o] + acc;
    }
    return six;
}

// prenorm_modulate (swin.hpp:72-85), kRmsEps = 1e-8 (:45)
template <class T>
static void prenorm_modulate(const T* X, i64 n, int h, const T* g, const T* a, const T* b, const T* gate, T* XM) {
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; ++j) {
        const T* x = X + j * h;
        T ss = T(0);
        for (int i = 0; i < h; ++i) ss += x[i] * x[i];
        const T r = std::sqrt(ss / T(h) + T(1e-8));
        for (int i = 0; i < h; ++i) {
            const T u = x[i] / r;
            XM[j * h + i] = gate[i] * ((g[i] * u) * (T(1) + a[i]) + b[i]);
        }
    }
}

// prenorm_plain (swin.hpp:111-123)
template <class T>
static void prenorm_plain(const T* X, i64 n, int h, const T* g, T* N) {
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; ++j) {
        const T* x = X + j * h;
        T ss = T(0);
        for (int i = 0; i < h; ++i) ss += x[i] * x[i];
        const T r = std::sqrt(ss / T(h) + T(1e-8));
        for (int i = 0; i < h; ++i) N[j * h + i] = g[i] * (x[i] / r);
    }
}

// rope_angles (rope.hpp:19-31) for the unwrapped window position (window.hpp:54-56), as used
// by window_rope_angles (swin.hpp:139-150): angle in double, cast to T.
template <class T>
static void rope_angles(int d, int row, int col, T* ang) {
    const int per_axis = d / 4;
    for (int j = 0; j < per_axis; ++j) {
        const double om = std::pow(10000.0, -double(j) / per_axis);
        ang[j] = static_cast<T>(row * om);
        ang[per_axis + j] = static_cast<T>(col * om);
    }
}

// One window, one block: block_window_forward (swin.hpp:306-325) with head_attention_fwd
// (:161-188). xin/xout: [s][h] in canonical in-window token order.
template <class T>
static void block_window(const Params<T>& p, int blk, const std::vector<T>& six, const Layout& lay, int wy,
                         int wx, const T* xin, T* xout) {
    const Cfg& c = p.cfg;
    const int h = c.hidden_dim, d = c.hd(), f = c.ffn_dim, heads = c.n_heads, w = lay.w, s = lay.s();
    const T *a1 = &six[0], *b1 = &six[h], *g1 = &six[2 * h], *a2 = &six[3 * h], *b2 = &six[4 * h],
            *g2 = &six[5 * h];
    // angles (d/2 x s)
    std::vector<T> ang(size_t(s) * (d / 2));
    for (int r = 0; r < w; ++r)
        for (int cc = 0; cc < w; ++cc)
            rope_angles<T>(d, wy * w + lay.shift + r, wx * w + lay.shift + cc, &ang[size_t(r * w + cc) * (d / 2)]);
    const bool masked = lay.seam(wy);

    std::vector<T> xm(size_t(s) * h), qkv(size_t(s) * 3 * h), concat(size_t(s) * h), tmp(size_t(s) * h);
    prenorm_modulate<T>(xin, s, h, p.blk(blk, 2), a1, b1, g1, xm.data());
    linear<T>(p.blk(blk, 0), nullptr, 3 * h, h, xm.data(), s, qkv.data());  // rows [q;k;v], head-major
    const T scale = T(1) / std::sqrt(T(d));
#pragma omp parallel for schedule(dynamic)
    for (int hd = 0; hd < heads; ++hd) {
        std::vector<T> q(size_t(s) * d), k(size_t(s) * d), v(size_t(s) * d), lg(s);
        for (int j = 0; j < s; ++j) {
            for (int e = 0; e < d; ++e) {
                q[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + hd * d + e];
                k[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + h + hd * d + e];
                v[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + 2 * h + hd * d + e];
            }
            // rope_rotate (rope.hpp:34-44): cos/sin evaluated in T
            for (int pr = 0; pr < d / 2; ++pr) {
                const T an = ang[size_t(j) * (d / 2) + pr];
                const T cs = std::cos(an), sn = std::sin(an);
                T* qq = &q[size_t(j) * d + 2 * pr];
                T* kk = &k[size_t(j) * d + 2 * pr];
                T x0 = qq[0], y0 = qq[1];
                qq[0] = cs * x0 - sn * y0;
                qq[1] = sn * x0 + cs * y0;
                x0 = kk[0], y0 = kk[1];
                kk[0] = cs * x0 - sn * y0;
                kk[1] = sn * x0 + cs * y0;
            }
        }
        const T ninf = -std::numeric_limits<T>::infinity();
        for (int i = 0; i < s; ++i) {
            // logits row i = (q_i . k_j) * scale + mask (swin.hpp:176-180)
            const T* qi = &q[size_t(i) * d];
            const int gq = masked ? lay.seam_group(i / w) : 0;
            T m = ninf;
            for (int j = 0; j < s; ++j) {
                const T* kj = &k[size_t(j) * d];
                T acc = T(0);
                for (int e = 0; e < d; ++e) acc += qi[e] * kj[e];
                T l = acc * scale;
                if (masked && lay.seam_group(j / w) != gq) l = l + ninf;
                lg[j] = l;
                if (l > m) m = l;
            }
            // softmax with max subtraction (:181-185)
            T sum = T(0);
            for (int j = 0; j < s; ++j) {
                lg[j] = std::exp(lg[j] - m);
                sum += lg[j];
            }
            for (int j = 0; j < s; ++j) lg[j] = lg[j] / sum;
            // O(:, i) = sum_j v(:, j) P(i, j)  (:186)
            T* o = &concat[size_t(i) * h + hd * d];
            for (int e = 0; e < d; ++e) o[e] = T(0);
            for (int j = 0; j < s; ++j) {
                const T pj = lg[j];
                const T* vj = &v[size_t(j) * d];
                for (int e = 0; e < d; ++e) o[e] += vj[e] * pj;
            }
        }
    }
    // x_mid = x_in + W_out * concat (:322)
    std::vector<T> xmid(size_t(s) * h);
    linear<T>(p.blk(blk, 1), nullptr, h, h, concat.data(), s, tmp.data());
    for (size_t i = 0; i < size_t(s) * h; ++i) xmid[i] = xin[i] + tmp[i];
    // FFN branch: swiglu_fwd (:228-234)
    prenorm_modulate<T>(xmid.data(), s, h, p.blk(blk, 3), a2, b2, g2, xm.data());
    std::vector<T> gp(size_t(s) * f), up(size_t(s) * f);
    linear<T>(p.blk(blk, 4), nullptr, f, h, xm.data(), s, gp.data());
    linear<T>(p.blk(blk, 5), nullptr, f, h, xm.data(), s, up.data());
    for (size_t i = 0; i < size_t(s) * f; ++i) gp[i] = silu(gp[i]) * up[i];
    linear<T>(p.blk(blk, 6), nullptr, h, f, gp.data(), s, tmp.data());
    for (size_t i = 0; i < size_t(s) * h; ++i) xout[i] = xmid[i] + tmp[i];
}

template <class T>
static bool all_finite(const T* x, i64 n) {
    for (i64 i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) return false;
    return true;
}

// forward (swin.hpp:327-368). input: [N][C_in]; out: [N][C_out]. first_block/n_blocks allow
// running a contiguous sub-range of blocks (used by spot checks); full forward = (0, nb()).
template <class T>
static void forward(const Params<T>& p, const T* input, T t, int H, int W, T* out, int nblocks_override = -1,
                    T* hidden_out = nullptr) {
    const Cfg& c = p.cfg;
    c.validate_grid(H, W);
    const i64 N = i64(H) * W;
    const int h = c.hidden_dim;
    if (!all_finite(input, N * c.in_channels)) throw NumericsError("non-finite activation entering input");
    const std::vector<T> emb = time_embed(p, t);
    std::vector<T> x(size_t(N) * h);
    linear<T>(p.enc_w(), p.enc_b(), h, c.in_channels, input, N, x.data());
    const int nb = nblocks_override >= 0 ? nblocks_override : c.nb();
    for (int blk = 0; blk < nb; ++blk) {
        if (!all_finite(x.data(), N * h))
            throw NumericsError("non-finite activation entering block " + std::to_string(blk));
        const Layout lay{H, W, c.window_px, shift_for_block(blk, c.window_px)};
        const std::vector<T> six = ada_six(p, blk, emb);
        const int s = lay.s();
        std::vector<T> xin(size_t(s) * h), xo(size_t(s) * h);
        // Windows are disjoint, so processing them in order with in-place scatter
        // (swin.hpp:353-360) equals gathering all from the block input first.
        for (int wy = 0; wy < lay.ny(); ++wy)
            for (int wx = 0; wx < lay.nx(); ++wx) {
                for (int tk = 0; tk < s; ++tk) {
                    const i64 pix = lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w);
                    std::memcpy(&xin[size_t(tk) * h], &x[size_t(pix) * h], sizeof(T) * h);
                }
                block_window<T>(p, blk, six, lay, wy, wx, xin.data(), xo.data());
                for (int tk = 0; tk < s; ++tk) {
                    const i64 pix = lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w);
                    std::memcpy(&x[size_t(pix) * h], &xo[size_t(tk) * h], sizeof(T) * h);
                }
            }
    }
    if (!all_finite(x.data(), N * h)) throw NumericsError("non-finite activation entering decode");
    if (hidden_out) std::memcpy(hidden_out, x.data(), sizeof(T) * N * h);
    std::vector<T> nrm(size_t(N) * h);
    prenorm_plain<T>(x.data(), N, h, p.tail(2), nrm.data());
    linear<T>(p.tail(3), p.tail(4), c.out_channels, h, nrm.data(), N, out);
}

// ---------------------------------------------------------------- backward (swin.hpp:370-467)
// Gradient buffers mirror the flat canonical parameter vector (accumulated, +=).
template <class T>
struct Grads {
    std::vector<T*> arr;
    T* blk(int b, int k) const { return arr[kHead + b * kPerBlock + k]; }
};
template <class T>
static Grads<T> gview(const Cfg& c, T* flat) {
    Grads<T> g;
    i64 off = 0;
    for (const auto& a : param_arrays(c)) {
        g.arr.push_back(flat + off);
        off += a.rows * a.cols;
    }
    return g;
}
template <class T>
static T silu_grad(T x) {  // model.hpp:248-252
    const T s = T(1) / (T(1) + std::exp(-x));
    return s * (T(1) + x * (T(1) - s));
}
// linear_cols_t (swin.hpp:57-62): Y[n][in] = W^T X[n][out], W col-major out x in
template <class T>
static void linear_t(const T* Wm, int out, int in, const T* X, i64 n, T* Y) {
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; ++j)
        for (int k = 0; k < in; ++k) {
            T acc = T(0);
            const T* wc = Wm + i64(k) * out;
            for (int o = 0; o < out; ++o) acc += wc[o] * X[j * out + o];
            Y[j * in + k] = acc;
        }
}
// accum_outer (swin.hpp:64-68): G(out x in, col-major) += sum_j dY[j][out] X[j][in]^T, row_off
// selects a row block of a taller matrix with ld rows.
template <class T>
static void accum_outer(T* G, int ld, int row_off, int out, int in, const T* dY, int ldy, const T* X, int ldx, i64 n) {
#pragma omp parallel for schedule(static)
    for (int k = 0; k < in; ++k)
        for (int o = 0; o < out; ++o) {
            T acc = T(0);
            for (i64 j = 0; j < n; ++j) acc += dY[j * ldy + o] * X[j * ldx + k];
            G[i64(k) * ld + row_off + o] += acc;
        }
}
// prenorm_modulate_bwd (swin.hpp:86-107)
template <class T>
static void prenorm_modulate_bwd(const T* X, i64 n, int h, const T* g, const T* a, const T* b, const T* gate,
                                 const T* dXM, T* dX, T* dg, T* da, T* db, T* dgate) {
    for (i64 j = 0; j < n; ++j) {
        const T* x = X + j * h;
        T ss = T(0);
        for (int i = 0; i < h; ++i) ss += x[i] * x[i];
        const T r = std::sqrt(ss / T(h) + T(1e-8));
        std::vector<T> du(h);
        T xdotdu = T(0);
        for (int i = 0; i < h; ++i) {
            const T u = x[i] / r, dxm = dXM[j * h + i], gu = g[i] * u;
            da[i] += dxm * gate[i] * gu;
            db[i] += dxm * gate[i];
            dgate[i] += dxm * (gu * (T(1) + a[i]) + b[i]);
            const T dgu = dxm * gate[i] * (T(1) + a[i]);
            dg[i] += dgu * u;
            du[i] = dgu * g[i];
            xdotdu += x[i] * du[i];
        }
        for (int i = 0; i < h; ++i) dX[j * h + i] += du[i] / r - x[i] * (xdotdu / (T(h) * r * r * r));
    }
}
// prenorm_plain_bwd (swin.hpp:125-136)
template <class T>
static void prenorm_plain_bwd(const T* X, i64 n, int h, const T* g, const T* dN, T* dX, T* dg) {
    for (i64 j = 0; j < n; ++j) {
        const T* x = X + j * h;
        T ss = T(0);
        for (int i = 0; i < h; ++i) ss += x[i] * x[i];
        const T r = std::sqrt(ss / T(h) + T(1e-8));
        T xdotdu = T(0);
        std::vector<T> du(h);
        for (int i = 0; i < h; ++i) {
            dg[i] += dN[j * h + i] * (x[i] / r);
            du[i] = dN[j * h + i] * g[i];
            xdotdu += x[i] * du[i];
        }
        for (int i = 0; i < h; ++i) dX[j * h + i] += du[i] / r - x[i] * (xdotdu / (T(h) * r * r * r));
    }
}

// block_window_backward (swin.hpp:370-417) with head_attention_bwd (:189-226) and swiglu_bwd
// (:236-252). The window's forward internals are recomputed from its block input (no cache of the
// s x s probabilities is kept across windows). xin, dX: [s][h]; returns dxin; d6 accumulates
// [da1, db1, dg1, da2, db2, dg2].
template <class T>
static void block_window_backward(const Params<T>& p, const Grads<T>& G, int blk, const std::vector<T>& six,
                                  const Layout& lay, int wy, int wx, const T* xin, const T* dX, T* dxin, T* d6) {
    const Cfg& c = p.cfg;
    const int h = c.hidden_dim, d = c.hd(), f = c.ffn_dim, heads = c.n_heads, w = lay.w, s = lay.s();
    const T *a1 = &six[0], *b1 = &six[h], *g1 = &six[2 * h], *a2 = &six[3 * h], *b2 = &six[4 * h],
            *g2 = &six[5 * h];
    std::vector<T> ang(size_t(s) * (d / 2));
    for (int r = 0; r < w; ++r)
        for (int cc = 0; cc < w; ++cc)
            rope_angles<T>(d, wy * w + lay.shift + r, wx * w + lay.shift + cc, &ang[size_t(r * w + cc) * (d / 2)]);
    const bool masked = lay.seam(wy);
    const T scale = T(1) / std::sqrt(T(d));
    // ---- forward recompute
    std::vector<T> xm(size_t(s) * h), qkv(size_t(s) * 3 * h), concat(size_t(s) * h), tmp(size_t(s) * h);
    prenorm_modulate<T>(xin, s, h, p.blk(blk, 2), a1, b1, g1, xm.data());
    linear<T>(p.blk(blk, 0), nullptr, 3 * h, h, xm.data(), s, qkv.data());
    std::vector<std::vector<T>> Q(heads), K(heads), V(heads), P(heads);
    for (int hd = 0; hd < heads; ++hd) {
        std::vector<T>&q = Q[hd], &k = K[hd], &v = V[hd], &pr = P[hd];
        q.resize(size_t(s) * d);
        k.resize(size_t(s) * d);
        v.resize(size_t(s) * d);
        pr.resize(size_t(s) * s);
        for (int j = 0; j < s; ++j) {
            for (int e = 0; e < d; ++e) {
                q[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + hd * d + e];
                k[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + h + hd * d + e];
                v[size_t(j) * d + e] = qkv[size_t(j) * 3 * h + 2 * h + hd * d + e];
            }
            for (int pp = 0; pp < d / 2; ++pp) {
                const T an = ang[size_t(j) * (d / 2) + pp];
                const T cs = std::cos(an), sn = std::sin(an);
                for (T* z : {&q[size_t(j) * d + 2 * pp], &k[size_t(j) * d + 2 * pp]}) {
                    const T x0 = z[0], y0 = z[1];
                    z[0] = cs * x0 - sn * y0;
                    z[1] = sn * x0 + cs * y0;
                }
            }
        }
        const T ninf = -std::numeric_limits<T>::infinity();
        for (int i = 0; i < s; ++i) {
            const int gq = masked ? lay.seam_group(i / w) : 0;
            T m = ninf;
            T* row = &pr[size_t(i) * s];
            for (int j = 0; j < s; ++j) {
                T acc = T(0);
                for (int e = 0; e < d; ++e) acc += q[size_t(i) * d + e] * k[size_t(j) * d + e];
                T l = acc * scale;
                if (masked && lay.seam_group(j / w) != gq) l = l + ninf;
                row[j] = l;
                if (l > m) m = l;
            }
            T sum = T(0);
            for (int j = 0; j < s; ++j) {
                row[j] = std::exp(row[j] - m);
                sum += row[j];
            }
            for (int j = 0; j < s; ++j) row[j] = row[j] / sum;
            T* o = &concat[size_t(i) * h + hd * d];
            for (int e = 0; e < d; ++e) o[e] = T(0);
            for (int j = 0; j < s; ++j)
                for (int e = 0; e < d; ++e) o[e] += v[size_t(j) * d + e] * row[j];
        }
    }
    std::vector<T> xmid(size_t(s) * h);
    linear<T>(p.blk(blk, 1), nullptr, h, h, concat.data(), s, tmp.data());
    for (size_t i = 0; i < size_t(s) * h; ++i) xmid[i] = xin[i] + tmp[i];
    std::vector<T> x2m(size_t(s) * h), gp(size_t(s) * f), up(size_t(s) * f), act(size_t(s) * f);
    prenorm_modulate<T>(xmid.data(), s, h, p.blk(blk, 3), a2, b2, g2, x2m.data());
    linear<T>(p.blk(blk, 4), nullptr, f, h, x2m.data(), s, gp.data());
    linear<T>(p.blk(blk, 5), nullptr, f, h, x2m.data(), s, up.data());
    for (size_t i = 0; i < size_t(s) * f; ++i) act[i] = silu(gp[i]) * up[i];
    // ---- feed-forward branch backward (swiglu_bwd + prenorm_modulate_bwd)
    std::vector<T> dxmid(dX, dX + size_t(s) * h);
    accum_outer<T>(G.blk(blk, 6), h, 0, h, f, dX, h, act.data(), f, s);
    std::vector<T> dS(size_t(s) * f), dG(size_t(s) * f), dU(size_t(s) * f);
    linear_t<T>(p.blk(blk, 6), h, f, dX, s, dS.data());
    for (size_t i = 0; i < size_t(s) * f; ++i) {
        dG[i] = dS[i] * up[i] * silu_grad(gp[i]);
        dU[i] = dS[i] * silu(gp[i]);
    }
    accum_outer<T>(G.blk(blk, 4), f, 0, f, h, dG.data(), f, x2m.data(), h, s);
    accum_outer<T>(G.blk(blk, 5), f, 0, f, h, dU.data(), f, x2m.data(), h, s);
    std::vector<T> dx2m(size_t(s) * h), t2(size_t(s) * h);
    linear_t<T>(p.blk(blk, 4), f, h, dG.data(), s, dx2m.data());
    linear_t<T>(p.blk(blk, 5), f, h, dU.data(), s, t2.data());
    for (size_t i = 0; i < size_t(s) * h; ++i) dx2m[i] += t2[i];
    prenorm_modulate_bwd<T>(xmid.data(), s, h, p.blk(blk, 3), a2, b2, g2, dx2m.data(), dxmid.data(), G.blk(blk, 3),
                            d6 + 3 * h, d6 + 4 * h, d6 + 5 * h);
    // ---- attention branch backward
    for (size_t i = 0; i < size_t(s) * h; ++i) dxin[i] = dxmid[i];
    accum_outer<T>(G.blk(blk, 1), h, 0, h, h, dxmid.data(), h, concat.data(), h, s);
    std::vector<T> dOc(size_t(s) * h), dXm(size_t(s) * h, T(0));
    linear_t<T>(p.blk(blk, 1), h, h, dxmid.data(), s, dOc.data());
    std::vector<T> dqkv(size_t(s) * 3 * h, T(0));  // [s][3h] like qkv
    for (int hd = 0; hd < heads; ++hd) {
        const std::vector<T>&q = Q[hd], &k = K[hd], &v = V[hd], &pr = P[hd];
        std::vector<T> dV(size_t(s) * d, T(0)), dQ(size_t(s) * d, T(0)), dK(size_t(s) * d, T(0)), dA(size_t(s) * s);
        for (int i = 0; i < s; ++i) {  // dP(i,j) = dO_i . v_j ; dA = P .* (dP - rowdot)
            const T* dOi = &dOc[size_t(i) * h + hd * d];
            T dot = T(0);
            for (int j = 0; j < s; ++j) {
                T acc = T(0);
                for (int e = 0; e < d; ++e) acc += dOi[e] * v[size_t(j) * d + e];
                dA[size_t(i) * s + j] = acc;
                dot += acc * pr[size_t(i) * s + j];
            }
            for (int j = 0; j < s; ++j) dA[size_t(i) * s + j] = pr[size_t(i) * s + j] * (dA[size_t(i) * s + j] - dot);
            for (int j = 0; j < s; ++j)  // dV_j += dO_i P(i,j)
                for (int e = 0; e < d; ++e) dV[size_t(j) * d + e] += dOi[e] * pr[size_t(i) * s + j];
        }
        for (int i = 0; i < s; ++i)
            for (int j = 0; j < s; ++j) {
                const T a = dA[size_t(i) * s + j];
                for (int e = 0; e < d; ++e) {
                    dQ[size_t(i) * d + e] += k[size_t(j) * d + e] * a;
                    dK[size_t(j) * d + e] += q[size_t(i) * d + e] * a;
                }
            }
        for (int j = 0; j < s; ++j) {
            for (int e = 0; e < d; ++e) {
                dQ[size_t(j) * d + e] *= scale;
                dK[size_t(j) * d + e] *= scale;
            }
            for (int pp = 0; pp < d / 2; ++pp) {  // rope_rotate(..., inverse=true)
                const T an = -ang[size_t(j) * (d / 2) + pp];
                const T cs = std::cos(an), sn = std::sin(an);
                for (T* z : {&dQ[size_t(j) * d + 2 * pp], &dK[size_t(j) * d + 2 * pp]}) {
                    const T x0 = z[0], y0 = z[1];
                    z[0] = cs * x0 - sn * y0;
                    z[1] = sn * x0 + cs * y0;
                }
            }
            for (int e = 0; e < d; ++e) {
                dqkv[size_t(j) * 3 * h + hd * d + e] = dQ[size_t(j) * d + e];
                dqkv[size_t(j) * 3 * h + h + hd * d + e] = dK[size_t(j) * d + e];
                dqkv[size_t(j) * 3 * h + 2 * h + hd * d + e] = dV[size_t(j) * d + e];
            }
        }
    }
    accum_outer<T>(G.blk(blk, 0), 3 * h, 0, 3 * h, h, dqkv.data(), 3 * h, xm.data(), h, s);
    linear_t<T>(p.blk(blk, 0), 3 * h, h, dqkv.data(), s, dXm.data());
    prenorm_modulate_bwd<T>(xin, s, h, p.blk(blk, 2), a1, b1, g1, dXm.data(), dxin, G.blk(blk, 2), d6, d6 + h,
                            d6 + 2 * h);
}

// backward (swin.hpp:419-467) of the full forward for output gradient dout [N][C_out]: parameter
// gradients in canonical flat order (overwritten) and the input gradient [N][C_in].
template <class T>
static void backward(const Params<T>& p, const T* input, T t, int H, int W, const T* dout, T* gflat, T* din) {
    const Cfg& c = p.cfg;
    c.validate_grid(H, W);
    const i64 N = i64(H) * W;
    const int h = c.hidden_dim, td = c.td(), nb = c.nb();
    i64 total = 0;
    for (const auto& a : param_arrays(c)) total += a.rows * a.cols;
    std::memset(gflat, 0, sizeof(T) * total);
    const Grads<T> G = gview<T>(c, gflat);
    // forward, keeping every block's input (pixel order)
    const std::vector<T> emb = time_embed(p, t);
    std::vector<std::vector<T>> xb(nb + 1, std::vector<T>(size_t(N) * h));
    linear<T>(p.enc_w(), p.enc_b(), h, c.in_channels, input, N, xb[0].data());
    for (int blk = 0; blk < nb; ++blk) {
        const Layout lay{H, W, c.window_px, shift_for_block(blk, c.window_px)};
        const std::vector<T> six = ada_six(p, blk, emb);
        const int s = lay.s();
        std::vector<T> xin(size_t(s) * h), xo(size_t(s) * h);
        xb[blk + 1] = xb[blk];
        for (int wy = 0; wy < lay.ny(); ++wy)
            for (int wx = 0; wx < lay.nx(); ++wx) {
                for (int tk = 0; tk < s; ++tk)
                    std::memcpy(&xin[size_t(tk) * h], &xb[blk][size_t(lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w)) * h],
                                sizeof(T) * h);
                block_window<T>(p, blk, six, lay, wy, wx, xin.data(), xo.data());
                for (int tk = 0; tk < s; ++tk)
                    std::memcpy(&xb[blk + 1][size_t(lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w)) * h],
                                &xo[size_t(tk) * h], sizeof(T) * h);
            }
    }
    const std::vector<T>& xf = xb[nb];
    // decode head
    std::vector<T> n3(size_t(N) * h), dn3(size_t(N) * h), dx(size_t(N) * h, T(0));
    prenorm_plain<T>(xf.data(), N, h, p.tail(2), n3.data());
    T* gdw = G.arr[kHead + nb * kPerBlock + 3];
    T* gdb = G.arr[kHead + nb * kPerBlock + 4];
    accum_outer<T>(gdw, c.out_channels, 0, c.out_channels, h, dout, c.out_channels, n3.data(), h, N);
    for (i64 j = 0; j < N; ++j)
        for (int o = 0; o < c.out_channels; ++o) gdb[o] += dout[j * c.out_channels + o];
    linear_t<T>(p.tail(3), c.out_channels, h, dout, N, dn3.data());
    prenorm_plain_bwd<T>(xf.data(), N, h, p.tail(2), dn3.data(), dx.data(), G.arr[kHead + nb * kPerBlock + 2]);
    // blocks in reverse
    std::vector<T> d_embed(td, T(0));
    for (int blk = nb - 1; blk >= 0; --blk) {
        const Layout lay{H, W, c.window_px, shift_for_block(blk, c.window_px)};
        const std::vector<T> six = ada_six(p, blk, emb);
        const int s = lay.s();
        std::vector<T> d6(6 * h, T(0)), dxn(size_t(N) * h, T(0)), xin(size_t(s) * h), dwin(size_t(s) * h),
            dwin_in(size_t(s) * h);
        for (int wy = 0; wy < lay.ny(); ++wy)
            for (int wx = 0; wx < lay.nx(); ++wx) {
                for (int tk = 0; tk < s; ++tk) {
                    const i64 pix = lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w);
                    std::memcpy(&xin[size_t(tk) * h], &xb[blk][size_t(pix) * h], sizeof(T) * h);
                    std::memcpy(&dwin[size_t(tk) * h], &dx[size_t(pix) * h], sizeof(T) * h);
                }
                block_window_backward<T>(p, G, blk, six, lay, wy, wx, xin.data(), dwin.data(), dwin_in.data(),
                                         d6.data());
                for (int tk = 0; tk < s; ++tk)
                    std::memcpy(&dxn[size_t(lay.pixel_of(wy, wx, tk / lay.w, tk % lay.w)) * h],
                                &dwin_in[size_t(tk) * h], sizeof(T) * h);
            }
        dx.swap(dxn);
        // ada: six = b_ada + W_ada embed (W_ada 6h x td col-major)
        T* gwa = G.blk(blk, 7);
        T* gba = G.blk(blk, 8);
        const T* Wa = p.blk(blk, 7);
        for (int k = 0; k < td; ++k)
            for (int o = 0; o < 6 * h; ++o) {
                gwa[i64(k) * 6 * h + o] += d6[o] * emb[k];
                d_embed[k] += Wa[i64(k) * 6 * h + o] * d6[o];
            }
        for (int o = 0; o < 6 * h; ++o) gba[o] += d6[o];
    }
    // encode
    accum_outer<T>(G.arr[0], h, 0, h, c.in_channels, dx.data(), h, input, c.in_channels, N);
    for (i64 j = 0; j < N; ++j)
        for (int o = 0; o < h; ++o) G.arr[1][o] += dx[j * h + o];
    if (din) linear_t<T>(p.enc_w(), h, c.in_channels, dx.data(), N, din);
    // shared time projection: embed = silu(lin), lin = W_time feat + b_time
    std::vector<T> feat(td), lin(td);
    const int nf = td / 2;
    for (int k = 0; k < nf; ++k) {
        const double om = std::pow(10000.0, -double(k) / nf);
        const double arg = double(t) * 636.6197723675814 * om;
        feat[2 * k] = static_cast<T>(std::sin(arg));
        feat[2 * k + 1] = static_cast<T>(std::cos(arg));
    }
    if (td % 2 == 1) feat[td - 1] = T(1);
    for (int o = 0; o < td; ++o) {
        T acc = T(0);
        for (int k = 0; k < td; ++k) acc += p.tail(0)[i64(k) * td + o] * feat[k];
        lin[o] = acc + p.tail(1)[o];
    }
    T* gwt = G.arr[kHead + nb * kPerBlock + 0];
    T* gbt = G.arr[kHead + nb * kPerBlock + 1];
    for (int o = 0; o < td; ++o) {
        const T dl = d_embed[o] * silu_grad(lin[o]);
        for (int k = 0; k < td; ++k) gwt[i64(k) * td + o] += dl * feat[k];
        gbt[o] += dl;
    }
}

// ---------------------------------------------------------------- posenc.hpp:16-37
template <class T>
static void posenc(int H, int W, int C, T* enc) {
    require(C > 0 && C % 2 == 0, "positional encoding: channel count must be even");
    const int per_axis = C / 2, nf = (per_axis + 1) / 2;
    for (int axis = 0; axis < 2; ++axis)
        for (int i = 0; i < per_axis; ++i) {
            const int k = i / 2;
            const double om = std::pow(10000.0, -double(k) / std::max(1, nf));
            const bool use_sin = (i % 2 == 0);
            const int ch = axis * per_axis + i;
            for (int y = 0; y < H; ++y)
                for (int x = 0; x < W; ++x) {
                    const double pos = axis == 0 ? y : x;
                    enc[(i64(y) * W + x) * C + ch] = static_cast<T>(use_sin ? std::sin(pos * om) : std::cos(pos * om));
                }
        }
}

// ---------------------------------------------------------------- diffusion.hpp
struct DCfg {
    double sigma_d, sigma_min, sigma_max;
    int solver_steps;
    double churn;
    double t_of_sigma(double s) const { return std::atan(s / sigma_d); }
};

template <class T>
static std::pair<T, T> trig_coeffs(T t) {  // diffusion.hpp:50-55
    if (t == T(0)) return {T(1), T(0)};
    if (t == static_cast<T>(M_PI_2)) return {T(0), T(1)};
    return {std::cos(t), std::sin(t)};
}

// noise_field (diffusion.hpp:91-108) with SeedProtocol::z_cell_key (rng.hpp:88-90)
template <class T>
static void noise_field(u64 run_seed, u64 event, int C, int H, int W, int w, double sigma_d, T* z) {
    const Layout lay{H, W, w, 0};
    const u64 zfk = kd2(run_seed, 0x7au, event);
    for (int wy = 0; wy < lay.ny(); ++wy)
        for (int wx = 0; wx < lay.nx(); ++wx) {
            const u64 wid = u64(wy) * lay.nx() + wx;
            for (int tok = 0; tok < lay.s(); ++tok) {
                const u64 key = kd2(zfk, wid, u64(tok));
                const i64 pix = lay.pixel_of(wy, wx, tok / w, tok % w);
                for (int c = 0; c < C; ++c) z[pix * C + c] = static_cast<T>(sigma_d * gaussian(key, u64(c)));
            }
        }
}

// solve_pf_ode (diffusion.hpp:207-272). net(x, t) -> sigma_d * F(x / sigma_d, t).
template <class T>
static std::vector<T> solve_pf_ode(const std::function<std::vector<T>(const std::vector<T>&, T)>& net,
                                   const std::vector<T>& x_init, const DCfg& dc, u64 churn_key, int* f_evals) {
    require(dc.sigma_d > 0, "diffusion: sigma_d must be positive");
    require(0 < dc.sigma_min && dc.sigma_min < dc.sigma_max, "diffusion: need 0 < sigma_min < sigma_max");
    require(dc.solver_steps >= 1, "diffusion: solver_steps must be >= 1");
    require(dc.churn >= 0, "diffusion: churn amount must be >= 0");
    const int S = dc.solver_steps;
    const double sd = dc.sigma_d;
    std::vector<double> sigma(S + 1);
    for (int k = 0; k <= S; ++k) {
        const double fr = double(k) / S;
        sigma[k] = std::exp((1.0 - fr) * std::log(dc.sigma_max) + fr * std::log(dc.sigma_min));
    }
    const size_t n = x_init.size();
    auto x0_hat = [&](const std::vector<T>& x, double t) {
        const auto cs = trig_coeffs(static_cast<T>(t));
        std::vector<T> v = net(x, static_cast<T>(t));
        if (f_evals) ++*f_evals;
        std::vector<T> r(n);
        for (size_t i = 0; i < n; ++i) r[i] = cs.first * x[i] - cs.second * v[i];
        return r;
    };
    std::vector<T> x = x_init;
    double t_cur = dc.t_of_sigma(sigma[0]), sig_cur = sigma[0];
    u64 churn_ctr = 0;
    for (int k = 0; k < S; ++k) {
        const double sig_next = sigma[k + 1], t_next = dc.t_of_sigma(sig_next);
        const double sig_mid = std::sqrt(sig_cur * sig_next), t_mid = dc.t_of_sigma(sig_mid);
        const double b_s = std::sin(t_cur) * sd;
        const double a_m = std::cos(t_mid), b_m = std::sin(t_mid) * sd;
        const double a_t = std::cos(t_next), b_t = std::sin(t_next) * sd;
        const std::vector<T> d1 = x0_hat(x, t_cur);
        const double r_mid = sig_mid / sig_cur;
        const T c1 = static_cast<T>(b_m / b_s), c2 = static_cast<T>(a_m * (r_mid - 1.0));
        std::vector<T> xm(n);
        for (size_t i = 0; i < n; ++i) xm[i] = c1 * x[i] - c2 * d1[i];
        const std::vector<T> d2 = x0_hat(xm, t_mid);
        const double r = sig_next / sig_cur;
        const T c3 = static_cast<T>(b_t / b_s), c4 = static_cast<T>(a_t * (r - 1.0));
        for (size_t i = 0; i < n; ++i) x[i] = c3 * x[i] - c4 * d2[i];
        if (!all_finite(x.data(), i64(n)))
            throw NumericsError("pf-ode solver diverged at step " + std::to_string(k) + " (t=" + std::to_string(t_next) + ")");
        t_cur = t_next;
        sig_cur = sig_next;
        const bool active = dc.churn > 0.0 && 3 * k >= S && 3 * k < 2 * S;  // ChurnSchedule :24-26
        if (active && k + 1 < S) {
            const double delta = dc.churn * 0.05 * (dc.t_of_sigma(sigma[k]) - t_next);
            if (delta > 0) {
                const double cc = std::cos(delta), ss = std::sin(delta);
                for (size_t i = 0; i < n; ++i) {
                    const T zeta = static_cast<T>(sd * gaussian(churn_key, churn_ctr++));
                    x[i] = static_cast<T>(cc) * x[i] + static_cast<T>(ss) * zeta;
                }
                t_cur += delta;
                sig_cur = sd * std::tan(t_cur);
            }
        }
    }
    return x;
}

// forecast_step (diffusion.hpp:295-319) with Standardizer apply/invert (grid.hpp:127-132) and
// the net lambda (diffusion.hpp:304-311). Standardizers are passed as (mean, std) arrays.
template <class T>
static void forecast_step(const Params<T>& p, const DCfg& dc, int H, int W, const T* x_prev_phys,
                          const T* forc_phys, const T* st_mean, const T* st_std, const T* rs_mean,
                          const T* rs_std, const T* fo_mean, const T* fo_std, u64 run_seed, u64 noise_event,
                          T* out, int* f_evals) {
    const Cfg& c = p.cfg;
    const i64 N = i64(H) * W;
    const int Cp = c.out_channels, Cin = c.in_channels, Cf = Cin - 2 * Cp;
    require(Cf >= 0, "forecast: in_channels must be >= 2 * out_channels");
    std::vector<T> xp(size_t(N) * Cp), fo(size_t(N) * std::max(Cf, 1)), pe(size_t(N) * Cin);
    for (i64 j = 0; j < N; ++j) {
        for (int i = 0; i < Cp; ++i) xp[j * Cp + i] = (x_prev_phys[j * Cp + i] - st_mean[i]) / st_std[i];
        for (int i = 0; i < Cf; ++i) fo[j * Cf + i] = (forc_phys[j * Cf + i] - fo_mean[i]) / fo_std[i];
    }
    posenc<T>(H, W, Cin, pe.data());
    const T sdT = static_cast<T>(dc.sigma_d);
    auto net = [&](const std::vector<T>& xs, T t) {
        std::vector<T> in(size_t(N) * Cin), o(size_t(N) * Cp);
        for (i64 j = 0; j < N; ++j) {
            for (int i = 0; i < Cp; ++i) in[j * Cin + i] = xs[j * Cp + i] / sdT;
            for (int i = 0; i < Cp; ++i) in[j * Cin + Cp + i] = xp[j * Cp + i];
            for (int i = 0; i < Cf; ++i) in[j * Cin + 2 * Cp + i] = fo[j * Cf + i];
            for (int i = 0; i < Cin; ++i) in[j * Cin + i] += pe[j * Cin + i];
        }
        forward<T>(p, in.data(), t, H, W, o.data());
        for (auto& v : o) v = sdT * v;
        return o;
    };
    std::vector<T> z(size_t(N) * Cp);
    noise_field<T>(run_seed, kd(noise_event, 0x1217u), Cp, H, W, c.window_px, dc.sigma_d, z.data());
    const std::vector<T> r = solve_pf_ode<T>(net, z, dc, kd(noise_event, 0xc4u), f_evals);
    for (i64 j = 0; j < N; ++j)
        for (int i = 0; i < Cp; ++i) out[j * Cp + i] = x_prev_phys[j * Cp + i] + (r[j * Cp + i] * rs_std[i] + rs_mean[i]);
}

// solve_pf_ode with the forecast_step net lambda (diffusion.hpp:304-311) on given standardized
// conditioning: used to check the device solver without the noise / standardisation steps.
template <class T>
static void solve_net(const Params<T>& p, const DCfg& dc, int H, int W, const T* x_init, const T* xp, const T* fo,
                      u64 churn_key, T* out, int* f_evals) {
    const Cfg& c = p.cfg;
    const i64 N = i64(H) * W;
    const int Cp = c.out_channels, Cin = c.in_channels, Cf = Cin - 2 * Cp;
    std::vector<T> pe(size_t(N) * Cin);
    posenc<T>(H, W, Cin, pe.data());
    const T sdT = static_cast<T>(dc.sigma_d);
    auto net = [&](const std::vector<T>& xs, T t) {
        std::vector<T> in(size_t(N) * Cin), o(size_t(N) * Cp);
        for (i64 j = 0; j < N; ++j) {
            for (int i = 0; i < Cp; ++i) in[j * Cin + i] = xs[j * Cp + i] / sdT;
            for (int i = 0; i < Cp; ++i) in[j * Cin + Cp + i] = xp[j * Cp + i];
            for (int i = 0; i < Cf; ++i) in[j * Cin + 2 * Cp + i] = fo[j * Cf + i];
            for (int i = 0; i < Cin; ++i) in[j * Cin + i] += pe[j * Cin + i];
        }
        forward<T>(p, in.data(), t, H, W, o.data());
        for (auto& v : o) v = sdT * v;
        return o;
    };
    std::vector<T> x0(x_init, x_init + N * Cp);
    const auto r = solve_pf_ode<T>(net, x0, dc, churn_key, f_evals);
    std::memcpy(out, r.data(), sizeof(T) * N * Cp);
}

// ---------------------------------------------------------------- topology.hpp:74-188
static std::pair<int, int> window_owner(int wy, int wx, int a, int b) { return {wy % a, wx % b}; }

}  // namespace orc

// ====================================================================== C ABI (for ctypes)
using namespace orc;

extern "C" {

typedef struct {
    int hidden_dim, n_heads, ffn_dim, n_layers, blocks_per_layer, window_px, in_channels, out_channels, time_dim;
} orc_cfg;

static thread_local char g_err[512];
const char* orc_last_error() { return g_err; }

static Cfg to_cfg(const orc_cfg* c) {
    return Cfg{c->hidden_dim, c->n_heads, c->ffn_dim, c->n_layers, c->blocks_per_layer, c->window_px,
               c->in_channels, c->out_channels, c->time_dim};
}

#define ORC_TRY(...)                                                    \
    try {                                                               \
        __VA_ARGS__;                                                    \
        return 0;                                                       \
    } catch (const orc::NumericsError& e) {                             \
        std::snprintf(g_err, sizeof g_err, "NumericsError: %s", e.what()); \
        return 1;                                                       \
    } catch (const orc::ConfigError& e) {                               \
        std::snprintf(g_err, sizeof g_err, "ConfigError: %s", e.what()); \
        return 2;                                                       \
    } catch (const std::exception& e) {                                 \
        std::snprintf(g_err, sizeof g_err, "error: %s", e.what());      \
        return 3;                                                       \
    }

u64 orc_splitmix64(u64 x) { return splitmix64(x); }
u64 orc_key_derive(u64 key, u64 tag) { return kd(key, tag); }
double orc_gaussian(u64 key, u64 ctr) { return gaussian(key, ctr); }
double orc_uniform01(u64 key, u64 ctr) { return uniform01(key, ctr); }
void orc_gaussian_fill(u64 key, i64 n, double* out) {
    for (i64 i = 0; i < n; ++i) out[i] = gaussian(key, u64(i));
}

int orc_validate(const orc_cfg* c, int H, int W) { ORC_TRY(to_cfg(c).validate_grid(H, W)) }

long long orc_param_count_formula(const orc_cfg* c) { return param_count_formula(to_cfg(c)); }

// Returns the number of arrays; fills rows/cols if non-null.
int orc_param_arrays(const orc_cfg* c, long long* rows, long long* cols) {
    const auto a = param_arrays(to_cfg(c));
    for (size_t i = 0; i < a.size(); ++i) {
        if (rows) rows[i] = a[i].rows;
        if (cols) cols[i] = a[i].cols;
    }
    return int(a.size());
}
int orc_param_name(const orc_cfg* c, int i, char* buf, int len) {
    const auto a = param_arrays(to_cfg(c));
    if (i < 0 || i >= int(a.size())) return -1;
    std::snprintf(buf, len, "%s", a[i].name.c_str());
    return 0;
}

void orc_init_params_f64(const orc_cfg* c, u64 seed, int random, double scale, double* flat) {
    init_params<double>(to_cfg(c), seed, random, scale, flat);
}
void orc_init_params_f32(const orc_cfg* c, u64 seed, int random, double scale, float* flat) {
    init_params<float>(to_cfg(c), seed, random, scale, flat);
}

int orc_forward_f64(const orc_cfg* c, const double* params, const double* input, double t, int H, int W,
                    double* out) {
    ORC_TRY(forward<double>(view<double>(to_cfg(c), params), input, t, H, W, out))
}
int orc_forward_f32(const orc_cfg* c, const float* params, const float* input, float t, int H, int W, float* out) {
    ORC_TRY(forward<float>(view<float>(to_cfg(c), params), input, t, H, W, out))
}
// Hidden state after the first nblocks blocks (pixel order, [N][h]) -- for per-block checks.
int orc_hidden_f64(const orc_cfg* c, const double* params, const double* input, double t, int H, int W,
                   int nblocks, double* hidden, double* out) {
    ORC_TRY(forward<double>(view<double>(to_cfg(c), params), input, t, H, W, out, nblocks, hidden))
}
int orc_hidden_f32(const orc_cfg* c, const float* params, const float* input, float t, int H, int W, int nblocks,
                   float* hidden, float* out) {
    ORC_TRY(forward<float>(view<float>(to_cfg(c), params), input, t, H, W, out, nblocks, hidden))
}

// One block on one window, input xin [s][h] canonical order -> xout (block_window_forward).
int orc_block_window_f32(const orc_cfg* c, const float* params, float t, int H, int W, int blk, int wy, int wx,
                         const float* xin, float* xout) {
    ORC_TRY({
        const Cfg cf = to_cfg(c);
        const auto p = view<float>(cf, params);
        const auto emb = time_embed(p, t);
        const auto six = ada_six(p, blk, emb);
        const Layout lay{H, W, cf.window_px, shift_for_block(blk, cf.window_px)};
        block_window<float>(p, blk, six, lay, wy, wx, xin, xout);
    })
}

// backward (swin.hpp:419-467): parameter gradients (canonical flat order) and input gradient for
// an output gradient dout [N][C_out] at the given input / t.
int orc_backward_f64(const orc_cfg* c, const double* params, const double* input, double t, int H, int W,
                     const double* dout, double* grads, double* din) {
    ORC_TRY(backward<double>(view<double>(to_cfg(c), params), input, t, H, W, dout, grads, din))
}
int orc_backward_f32(const orc_cfg* c, const float* params, const float* input, float t, int H, int W,
                     const float* dout, float* grads, float* din) {
    ORC_TRY(backward<float>(view<float>(to_cfg(c), params), input, t, H, W, dout, grads, din))
}

// Time embedding (td) and all blocks' ada vectors ([nb][6h]).
void orc_time_embed_f64(const orc_cfg* c, const double* params, double t, double* emb, double* six_all) {
    const Cfg cf = to_cfg(c);
    const auto p = view<double>(cf, params);
    const auto e = time_embed(p, t);
    std::memcpy(emb, e.data(), sizeof(double) * e.size());
    if (six_all)
        for (int b = 0; b < cf.nb(); ++b) {
            const auto s = ada_six(p, b, e);
            std::memcpy(six_all + size_t(b) * s.size(), s.data(), sizeof(double) * s.size());
        }
}

long long orc_pixel_of(int H, int W, int w, int shift, int wy, int wx, int r, int c) {
    return Layout{H, W, w, shift}.pixel_of(wy, wx, r, c);
}
// perm[window-order index] = pixel, window order = (wy, wx) row-major then (r, c) row-major.
void orc_window_perm(int H, int W, int w, int shift, long long* perm) {
    const Layout lay{H, W, w, shift};
    i64 i = 0;
    for (int wy = 0; wy < lay.ny(); ++wy)
        for (int wx = 0; wx < lay.nx(); ++wx)
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c) perm[i++] = lay.pixel_of(wy, wx, r, c);
}
// window_gather / window_scatter (window.hpp:88-103) over all windows of a [N][C] field.
void orc_window_gather_f64(int H, int W, int w, int shift, int C, const double* tokens, double* win_order) {
    const Layout lay{H, W, w, shift};
    i64 i = 0;
    for (int wy = 0; wy < lay.ny(); ++wy)
        for (int wx = 0; wx < lay.nx(); ++wx)
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c, ++i)
                    std::memcpy(win_order + i * C, tokens + lay.pixel_of(wy, wx, r, c) * C, sizeof(double) * C);
}
void orc_window_scatter_f64(int H, int W, int w, int shift, int C, const double* win_order, double* tokens) {
    const Layout lay{H, W, w, shift};
    i64 i = 0;
    for (int wy = 0; wy < lay.ny(); ++wy)
        for (int wx = 0; wx < lay.nx(); ++wx)
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c, ++i)
                    std::memcpy(tokens + lay.pixel_of(wy, wx, r, c) * C, win_order + i * C, sizeof(double) * C);
}
// seam_mask (window.hpp:107-122): dense s x s additive mask (0 / -inf); returns 0 if none needed.
int orc_seam_mask_f64(int H, int W, int w, int shift, int wy, double* m) {
    const Layout lay{H, W, w, shift};
    if (!lay.seam(wy)) return 0;
    const int s = lay.s();
    for (int q = 0; q < s; ++q)
        for (int k = 0; k < s; ++k)
            m[i64(q) * s + k] = lay.seam_group(q / w) == lay.seam_group(k / w) ? 0.0 : -INFINITY;
    return 1;
}
int orc_band_of_row(int H, int W, int w, int shift, int r, int sp) { return Layout{H, W, w, shift}.band_of_row(r, sp); }

void orc_rope_angles_f64(int d, int row, int col, double* ang) { rope_angles<double>(d, row, col, ang); }

void orc_posenc_f64(int H, int W, int C, double* enc) { posenc<double>(H, W, C, enc); }
void orc_posenc_f32(int H, int W, int C, float* enc) { posenc<float>(H, W, C, enc); }

void orc_noise_field_f64(u64 run_seed, u64 event, int C, int H, int W, int w, double sigma_d, double* z) {
    noise_field<double>(run_seed, event, C, H, W, w, sigma_d, z);
}
void orc_noise_field_f32(u64 run_seed, u64 event, int C, int H, int W, int w, double sigma_d, float* z) {
    noise_field<float>(run_seed, event, C, H, W, w, sigma_d, z);
}

// solve_pf_ode with the analytic Gaussian oracle velocity (test_trigflow.cpp:44-54) -- used to
// pin the solver on the reference's KATs.
int orc_solve_gaussian(double mu, double s0, double sdd, double sigma_d, double sigma_min, double sigma_max,
                       int steps, double churn, u64 churn_key, const double* x_init, i64 n, double* out,
                       int* f_evals) {
    ORC_TRY({
        DCfg dc{sigma_d, sigma_min, sigma_max, steps, churn};
        auto net = [&](const std::vector<double>& x, double t) {
            const double c = std::cos(t), s = std::sin(t);
            const double den = c * c * s0 * s0 + s * s * sdd * sdd;
            std::vector<double> v(x.size());
            for (size_t i = 0; i < x.size(); ++i) {
                const double dev = x[i] - c * mu;
                const double ex0 = mu + (c * s0 * s0 / den) * dev;
                const double ez = (s * sdd * sdd / den) * dev;
                v[i] = c * ez - s * ex0;
            }
            return v;
        };
        std::vector<double> x0(x_init, x_init + n);
        const auto r = solve_pf_ode<double>(net, x0, dc, churn_key, f_evals);
        std::memcpy(out, r.data(), sizeof(double) * n);
    })
}
// Elementwise solver with an affine velocity v = alpha*x + beta (divergence tests).
int orc_solve_affine(double alpha, double beta, double sigma_d, double sigma_min, double sigma_max, int steps,
                     const double* x_init, i64 n, double* out) {
    ORC_TRY({
        DCfg dc{sigma_d, sigma_min, sigma_max, steps, 0.0};
        auto net = [&](const std::vector<double>& x, double) {
            std::vector<double> v(x.size());
            for (size_t i = 0; i < x.size(); ++i) v[i] = alpha * x[i] + beta;
            return v;
        };
        std::vector<double> x0(x_init, x_init + n);
        const auto r = solve_pf_ode<double>(net, x0, dc, 0, nullptr);
        std::memcpy(out, r.data(), sizeof(double) * n);
    })
}

double orc_t_of_sigma(double sigma, double sigma_d) { return std::atan(sigma / sigma_d); }

#define ORC_FORECAST(T, SUF)                                                                                 \
    int orc_forecast_step_##SUF(const orc_cfg* c, const T* params, double sigma_d, double sigma_min,           \
                                double sigma_max, int steps, double churn, int H, int W, const T* x_prev,      \
                                const T* forc, const T* st_mean, const T* st_std, const T* rs_mean,            \
                                const T* rs_std, const T* fo_mean, const T* fo_std, u64 run_seed, u64 event,   \
                                T* out, int* f_evals) {                                                        \
        ORC_TRY({                                                                                              \
            const Cfg cf = to_cfg(c);                                                                          \
            DCfg dc{sigma_d, sigma_min, sigma_max, steps, churn};                                              \
            forecast_step<T>(view<T>(cf, params), dc, H, W, x_prev, forc, st_mean, st_std, rs_mean, rs_std,   \
                             fo_mean, fo_std, run_seed, event, out, f_evals);                                  \
        })                                                                                                     \
    }
ORC_FORECAST(double, f64)
ORC_FORECAST(float, f32)

int orc_solve_net_f64(const orc_cfg* c, const double* params, double sigma_d, double sigma_min, double sigma_max,
                      int steps, double churn, int H, int W, const double* x_init, const double* xp,
                      const double* fo, u64 churn_key, double* out, int* f_evals) {
    ORC_TRY({
        DCfg dc{sigma_d, sigma_min, sigma_max, steps, churn};
        solve_net<double>(view<double>(to_cfg(c), params), dc, H, W, x_init, xp, fo, churn_key, out, f_evals);
    })
}

// window_owner (topology.hpp:107-109)
void orc_window_owner(int wy, int wx, int a, int b, int* oa, int* ob) {
    const auto o = window_owner(wy, wx, a, b);
    *oa = o.first;
    *ob = o.second;
}
// shift_transfer_plan (topology.hpp:149-188): total displaced tokens and per-(src rank) counts
// for round-robin ownership on an a x b WP grid and sp bands. counts: [a*b] tokens sent.
long long orc_shift_transfer_total(int H, int W, int w, int shift_from, int shift_to, int a, int b, int sp,
                                   long long* sent_per_rank) {
    const Layout from{H, W, w, shift_from}, to{H, W, w, shift_to};
    long long total = 0;
    if (sent_per_rank)
        for (int i = 0; i < a * b; ++i) sent_per_rank[i] = 0;
    for (int wy = 0; wy < to.ny(); ++wy)
        for (int wx = 0; wx < to.nx(); ++wx) {
            const auto d = window_owner(wy, wx, a, b);
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c) {
                    const i64 pix = to.pixel_of(wy, wx, r, c);
                    const int y = int(pix / W), x = int(pix % W);
                    const int sy = (y - from.shift + H) % H, sx = (x - from.shift + W) % W;
                    const auto s = window_owner(sy / w, sx / w, a, b);
                    if (from.band_of_row(sy % w, sp) != to.band_of_row(r, sp)) return -1;
                    if (s != d) {
                        ++total;
                        if (sent_per_rank) ++sent_per_rank[s.first * b + s.second];
                    }
                }
        }
    return total;
}

int orc_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {  // torchrun exports OMP_NUM_THREADS=1: the CPU baselines undo it
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

}  // extern "C"
