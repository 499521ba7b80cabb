// swinflow/b200.hpp -- C++ host API of the B200 denoiser path, mirroring the reference's
// proj/include/swinflow signatures so callers of the hot path switch by changing one include:
//
//   reference (swin.hpp:327-329)           here
//   MatX<T> forward(const Parameters<T>&,  MatX<T> forward(const Parameters<T>&,
//                   const MatX<T>& input,                  const MatX<T>& input,
//                   T t, int H, int W,                     T t, int H, int W)
//                   ForwardCache<T>* = nullptr)            (no cache: the GPU path keeps no s x s probs)
//   solve_pf_ode(net, x_init, dc, churn)   solve_pf_ode(DeviceNet&, x_init, dc, churn)  (diffusion.hpp:207)
//   forecast_step(fm, x_prev, forc, sp, ev) forecast_step(fm, x_prev, forc, sp, ev)     (diffusion.hpp:295)
//   rollout_ensemble(...)                  rollout_ensemble(...)                        (diffusion.hpp:323)
//
// Everything runs on the GPU through the C-ABI (swinflow_capi.h); exceptions mirror the
// reference's (ConfigError, NumericsError, common.hpp:28-55) and there is no CPU fallback.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../swinflow_capi.h"

namespace swinflow {

using u64 = std::uint64_t;
using i64 = std::int64_t;

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericsError : std::runtime_error {
    explicit NumericsError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check_rc(int rc) {
    if (rc == SWF_OK) return;
    const std::string msg = swf_last_error();
    if (rc == SWF_ERR_NUMERICS) throw NumericsError(msg);
    if (rc == SWF_ERR_CONFIG) throw ConfigError(msg);
    throw DeviceError(msg);
}

// Minimal column-major dense matrix with the Eigen subset the hot path's callers use
// (rows/cols/size/data/operator()/Zero); storage order identical to Eigen::Matrix.
template <class T>
class MatX {
public:
    MatX() = default;
    MatX(i64 r, i64 c) : r_(r), c_(c), d_(size_t(r * c)) {}
    static MatX Zero(i64 r, i64 c) { return MatX(r, c); }
    i64 rows() const { return r_; }
    i64 cols() const { return c_; }
    i64 size() const { return r_ * c_; }
    T* data() { return d_.data(); }
    const T* data() const { return d_.data(); }
    T& operator()(i64 i, i64 j) { return d_[size_t(j * r_ + i)]; }
    T operator()(i64 i, i64 j) const { return d_[size_t(j * r_ + i)]; }
    T& operator[](i64 i) { return d_[size_t(i)]; }
    T operator[](i64 i) const { return d_[size_t(i)]; }
    void resize(i64 r, i64 c) {
        r_ = r;
        c_ = c;
        d_.assign(size_t(r * c), T(0));
    }
    void setOnes() { std::fill(d_.begin(), d_.end(), T(1)); }
    void setZero() { std::fill(d_.begin(), d_.end(), T(0)); }

private:
    i64 r_ = 0, c_ = 0;
    std::vector<T> d_;
};
template <class T>
using VecX = MatX<T>;  // column vector (n x 1)

struct ModelConfig {  // model.hpp:21-62
    int hidden_dim = 0, n_heads = 0, ffn_dim = 0, n_layers = 0, blocks_per_layer = 1, window_px = 0;
    int patch_size = 1, in_channels = 0, out_channels = 0, time_dim = 0;
    int n_blocks() const { return n_layers * blocks_per_layer; }
    int head_dim() const { return hidden_dim / n_heads; }
    int tdim() const { return time_dim > 0 ? time_dim : hidden_dim; }
    swf_model_cfg c() const {
        return swf_model_cfg{hidden_dim, n_heads, ffn_dim, n_layers, blocks_per_layer, window_px,
                             in_channels, out_channels, time_dim};
    }
};

template <class T>
struct BlockParams {  // model.hpp:64-74
    MatX<T> w_qkv, w_out;
    VecX<T> g_attn, g_ffn;
    MatX<T> w_gate, w_up, w_down, w_ada;
    VecX<T> b_ada;
};

template <class T>
struct Parameters {  // model.hpp:76-115
    ModelConfig cfg;
    MatX<T> w_encode;
    VecX<T> b_encode;
    std::vector<BlockParams<T>> blocks;
    MatX<T> w_time;
    VecX<T> b_time;
    VecX<T> g_decode;
    MatX<T> w_decode;
    VecX<T> b_decode;

    static Parameters zeros(const ModelConfig& cfg) {
        const int h = cfg.hidden_dim, f = cfg.ffn_dim, td = cfg.tdim();
        Parameters p;
        p.cfg = cfg;
        p.w_encode.resize(h, cfg.in_channels);
        p.b_encode.resize(h, 1);
        p.blocks.resize(cfg.n_blocks());
        for (auto& b : p.blocks) {
            b.w_qkv.resize(3 * h, h);
            b.w_out.resize(h, h);
            b.g_attn.resize(h, 1);
            b.g_ffn.resize(h, 1);
            b.w_gate.resize(f, h);
            b.w_up.resize(f, h);
            b.w_down.resize(h, f);
            b.w_ada.resize(6 * h, td);
            b.b_ada.resize(6 * h, 1);
        }
        p.w_time.resize(td, td);
        p.b_time.resize(td, 1);
        p.g_decode.resize(h, 1);
        p.w_decode.resize(cfg.out_channels, h);
        p.b_decode.resize(cfg.out_channels, 1);
        return p;
    }
};

// Counter RNG (rng.hpp:17-45) -- host side, for parameter init and synthetic fields.
inline u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline u64 key_derive(u64 key, u64 tag) { return splitmix64(key ^ splitmix64(tag)); }
inline u64 key_derive(u64 key, u64 a, u64 b) { return key_derive(key_derive(key, a), b); }
inline double gaussian(u64 key, u64 counter) {
    auto bits = [&](u64 c) { return splitmix64(key + 0x632be59bd9b4e019ULL * (c + 1)); };
    const double u1 = (double(bits(2 * counter) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = double(bits(2 * counter + 1) >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// parameter_arrays (model.hpp:140-168): canonical-order raw pointers.
template <class T>
std::vector<const void*> parameter_arrays(const Parameters<T>& p) {
    std::vector<const void*> a{p.w_encode.data(), p.b_encode.data()};
    for (const auto& b : p.blocks)
        for (const MatX<T>* m : {&b.w_qkv, &b.w_out, &b.g_attn, &b.g_ffn, &b.w_gate, &b.w_up, &b.w_down, &b.w_ada,
                                 &b.b_ada})
            a.push_back(m->data());
    for (const MatX<T>* m : {&p.w_time, &p.b_time, &p.g_decode, &p.w_decode, &p.b_decode}) a.push_back(m->data());
    return a;
}

// init_parameters (model.hpp:185-209) / init_parameters_random (model.hpp:213-223).
template <class T>
Parameters<T> init_parameters(const ModelConfig& cfg, u64 seed) {
    Parameters<T> p = Parameters<T>::zeros(cfg);
    const int h = cfg.hidden_dim, f = cfg.ffn_dim, td = cfg.tdim();
    u64 stream = 0;
    auto fill = [&](MatX<T>& m, double scale) {
        const u64 key = key_derive(seed, 0x1217u, stream++);
        for (i64 i = 0; i < m.size(); ++i) m.data()[i] = static_cast<T>(scale * gaussian(key, u64(i)));
    };
    fill(p.w_encode, 1.0 / std::sqrt(double(cfg.in_channels)));
    for (auto& b : p.blocks) {
        fill(b.w_qkv, 1.0 / std::sqrt(double(h)));
        fill(b.w_out, 1.0 / std::sqrt(double(h) * 2 * cfg.n_blocks()));
        b.g_attn.setOnes();
        b.g_ffn.setOnes();
        fill(b.w_gate, 1.0 / std::sqrt(double(h)));
        fill(b.w_up, 1.0 / std::sqrt(double(h)));
        fill(b.w_down, 1.0 / std::sqrt(double(f) * 2 * cfg.n_blocks()));
    }
    fill(p.w_time, 1.0 / std::sqrt(double(td)));
    p.g_decode.setOnes();
    return p;
}

template <class T>
Parameters<T> init_parameters_random(const ModelConfig& cfg, u64 seed, double scale = 0.25) {
    Parameters<T> p = init_parameters<T>(cfg, seed);
    u64 stream = 1000;
    std::vector<MatX<T>*> arr{&p.w_encode, &p.b_encode};
    for (auto& b : p.blocks)
        for (MatX<T>* m : {&b.w_qkv, &b.w_out, &b.g_attn, &b.g_ffn, &b.w_gate, &b.w_up, &b.w_down, &b.w_ada, &b.b_ada})
            arr.push_back(m);
    for (MatX<T>* m : {&p.w_time, &p.b_time, &p.g_decode, &p.w_decode, &p.b_decode}) arr.push_back(m);
    for (MatX<T>* m : arr) {
        const u64 key = key_derive(seed, 0xabcu, stream++);
        for (i64 i = 0; i < m->size(); ++i) m->data()[i] += static_cast<T>(scale * gaussian(key, u64(i)));
    }
    return p;
}

template <class T>
constexpr int dtype_of() {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "float or double");
    return sizeof(T) == 8 ? SWF_F64 : SWF_F32;
}

// Window / sequence parallelism of one process over several GPUs (swf_set_topology_devices):
// rank r of the wp_a x wp_b x sp topology runs on device_ids[r] (a device may host several ranks).
struct Topology {
    int wp_a = 1, wp_b = 1, sp = 1, ownership = SWF_OWN_CONTIGUOUS;
    std::vector<int> device_ids{0};
    int world() const { return wp_a * wp_b * sp; }
    bool operator<(const Topology& o) const {
        return std::tie(wp_a, wp_b, sp, ownership, device_ids) < std::tie(o.wp_a, o.wp_b, o.sp, o.ownership, o.device_ids);
    }
};

// One device context per (parameter set, grid, precision, topology): weights are uploaded once and
// kept resident; one mutex per context serialises concurrent callers (one stream per context).
class Context {
public:
    Context(const ModelConfig& cfg, int H, int W, int device = 0, int precision = SWF_PREC_BF16,
            const Topology* topo = nullptr)
        : cfg_(cfg) {
        const swf_model_cfg c = cfg.c();
        swf_ctx* p = nullptr;
        const int dev0 = topo ? topo->device_ids.at(0) : device;
        check_rc(swf_create(&c, H, W, dev0, precision, &p));
        ctx_.reset(p);
        if (topo && topo->world() > 1) {
            if (int(topo->device_ids.size()) != topo->world())
                throw ConfigError("topology: one device id per rank required");
            check_rc(swf_set_topology_devices(p, topo->wp_a, topo->wp_b, topo->sp, topo->ownership,
                                              topo->device_ids.data()));
        }
    }
    template <class T>
    void load(const Parameters<T>& p) {
        const auto a = parameter_arrays(p);
        check_rc(swf_load_params(ctx_.get(), a.data(), int(a.size()), dtype_of<T>()));
    }
    swf_ctx* get() const { return ctx_.get(); }
    const ModelConfig& cfg() const { return cfg_; }
    std::mutex& mutex() { return mu_; }

private:
    struct Del {
        void operator()(swf_ctx* c) const { swf_destroy(c); }
    };
    ModelConfig cfg_;
    std::unique_ptr<swf_ctx, Del> ctx_;
    std::mutex mu_;
};

namespace detail {
struct Key {
    const void* params;
    int H, W, prec;
    Topology topo;
    bool operator<(const Key& o) const {
        return std::tie(params, H, W, prec, topo) < std::tie(o.params, o.H, o.W, o.prec, o.topo);
    }
};
struct Entry {
    std::unique_ptr<Context> ctx;
    u64 fingerprint = 0;
};
// Process-wide (not per thread: a C2 context holds ~46 GB of HBM)
inline std::map<Key, Entry>& cache() {
    static std::map<Key, Entry> c;
    return c;
}
inline std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
inline int& default_precision() {
    static int p = SWF_PREC_BF16;
    return p;
}
inline Topology& default_topology() {
    static Topology t;
    return t;
}
inline u64 mix(u64 h, u64 v) { return splitmix64(h ^ splitmix64(v)); }
// Identity + contents of a parameter set: every array's address and size, and an fnv1a64 of its
// values -- all of them up to 2^22 elements per array, an evenly strided sample of 2^22 above that
// (an optimizer / EMA update rewrites every element, so it cannot hide between the samples).
template <class T>
u64 fingerprint(const Parameters<T>& p) {
    const std::vector<const void*> a = parameter_arrays(p);
    std::vector<i64> n{p.w_encode.size(), p.b_encode.size()};
    for (const auto& b : p.blocks)
        for (const MatX<T>* m : {&b.w_qkv, &b.w_out, &b.g_attn, &b.g_ffn, &b.w_gate, &b.w_up, &b.w_down, &b.w_ada,
                                 &b.b_ada})
            n.push_back(m->size());
    for (const MatX<T>* m : {&p.w_time, &p.b_time, &p.g_decode, &p.w_decode, &p.b_decode}) n.push_back(m->size());
    u64 h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < a.size(); ++i) {
        h = mix(h, reinterpret_cast<std::uintptr_t>(a[i]));
        h = mix(h, u64(n[i]));
        const T* v = static_cast<const T*>(a[i]);
        const i64 stride = std::max<i64>(1, n[i] >> 22);
        u64 f = 0xcbf29ce484222325ULL;
        for (i64 k = 0; k < n[i]; k += stride) {
            u64 bits = 0;
            std::memcpy(&bits, v + k, sizeof(T));
            f = (f ^ bits) * 0x100000001b3ULL;
        }
        h = mix(h, f);
    }
    return h;
}
}  // namespace detail

// Select the device arithmetic for the reference-signature entry points below.
inline void set_precision(int precision) { detail::default_precision() = precision; }
// Run the reference-signature entry points on several GPUs of this process (window / sequence
// parallelism; the results are identical to one device, bitwise).
inline void set_topology(const Topology& t) { detail::default_topology() = t; }

// The context serving `p` on an H x W grid. The parameters are re-uploaded whenever their contents
// changed since the last call (in-place optimizer / EMA updates of the caller's Parameters).
template <class T>
Context& context_for(const Parameters<T>& p, int H, int W) {
    const detail::Key k{&p, H, W, detail::default_precision(), detail::default_topology()};
    const u64 fp = detail::fingerprint(p);
    std::lock_guard<std::mutex> lk(detail::cache_mutex());
    auto& c = detail::cache();
    auto it = c.find(k);
    if (it == c.end()) {
        detail::Entry e;
        e.ctx = std::make_unique<Context>(p.cfg, H, W, 0, k.prec, &k.topo);
        it = c.emplace(k, std::move(e)).first;
    }
    if (!it->second.fingerprint || it->second.fingerprint != fp) {
        std::lock_guard<std::mutex> lk2(it->second.ctx->mutex());
        it->second.ctx->load(p);
        it->second.fingerprint = fp;
    }
    return *it->second.ctx;
}
// Drop the cached contexts (frees their device memory).
inline void release_contexts() {
    std::lock_guard<std::mutex> lk(detail::cache_mutex());
    detail::cache().clear();
}

// forward (swin.hpp:327-368): input C_in x N, returns C_out x N.
template <class T>
MatX<T> forward(const Parameters<T>& p, const MatX<T>& input, T t, int grid_h, int grid_w) {
    if (input.rows() != p.cfg.in_channels) throw ConfigError("forward: input channel mismatch");
    Context& ctx = context_for(p, grid_h, grid_w);
    MatX<T> out(p.cfg.out_channels, i64(grid_h) * grid_w);
    std::lock_guard<std::mutex> lk(ctx.mutex());
    check_rc(swf_forward(ctx.get(), input.data(), double(t), out.data(), dtype_of<T>()));
    return out;
}

// block_window_forward (swin.hpp:306-325): window (wy, wx) of block `block`'s layout (shift 0 / w/2 by
// parity, window.hpp:83-85) at time t; x_in / the result are the window's h x s_w residual columns.
// The reference passes the block's parameters and ada vectors; here they are block `block` of p
// (uploaded once, like forward()) and its ada vectors at t.
template <class T>
MatX<T> block_window_forward(const Parameters<T>& p, int block, T t, int grid_h, int grid_w, int wy, int wx,
                             const MatX<T>& x_in) {
    if (x_in.rows() != p.cfg.hidden_dim || x_in.cols() != i64(p.cfg.window_px) * p.cfg.window_px)
        throw ConfigError("block_window_forward: x_in must be hidden_dim x window_px^2");
    Context& ctx = context_for(p, grid_h, grid_w);
    MatX<T> out(x_in.rows(), x_in.cols());
    std::lock_guard<std::mutex> lk(ctx.mutex());
    check_rc(swf_block_window_forward(ctx.get(), block, wy, wx, double(t), x_in.data(), out.data(), dtype_of<T>()));
    return out;
}

struct DiffusionConfig {  // diffusion.hpp:29-46
    double sigma_d = 1.0, sigma_min = 0.2, sigma_max = 500.0;
    int solver_steps = 10;
    double churn = 0.0;
    swf_diffusion_cfg c() const { return swf_diffusion_cfg{sigma_d, sigma_min, sigma_max, solver_steps, churn}; }
};

// The net callable of solve_pf_ode (diffusion.hpp:204-209) as a device-resident functor:
// sigma_d * F([x/sigma_d; x_prev; forcings] + posenc, t), the forecast_step net lambda.
template <class T>
struct DeviceNet {
    Context* ctx;
    const MatX<T>* x_prev_std;
    const MatX<T>* forcings_std;
};

template <class T>
MatX<T> solve_pf_ode(const DeviceNet<T>& net, const MatX<T>& x_init, const DiffusionConfig& dc, u64 churn_key = 0,
                     int* f_evals = nullptr) {
    MatX<T> out(x_init.rows(), x_init.cols());
    const swf_diffusion_cfg c = dc.c();
    check_rc(swf_solve_pf_ode(net.ctx->get(), x_init.data(), net.x_prev_std->data(),
                              net.forcings_std ? net.forcings_std->data() : nullptr, &c, churn_key, out.data(),
                              f_evals, dtype_of<T>()));
    return out;
}

template <class T>
struct Standardizer {  // grid.hpp:85-133
    VecX<T> mean, std;
};

template <class T>
struct ForecastModel {  // diffusion.hpp:278-291 (grid/posenc are implied by the context)
    Context* ctx;
    Standardizer<T> state_std, resid_std, forcing_std;
    DiffusionConfig dcfg;
};

struct SeedProtocol {  // rng.hpp:77-91
    u64 run_seed = 0;
};

template <class T>
MatX<T> forecast_step(const ForecastModel<T>& fm, const MatX<T>& x_prev_phys, const MatX<T>& forcing_phys,
                      const SeedProtocol& sp, u64 noise_event) {
    MatX<T> out(x_prev_phys.rows(), x_prev_phys.cols());
    const swf_standardizers s{fm.state_std.mean.data(), fm.state_std.std.data(), fm.resid_std.mean.data(),
                              fm.resid_std.std.data(),  fm.forcing_std.mean.data(), fm.forcing_std.std.data()};
    const swf_diffusion_cfg c = fm.dcfg.c();
    check_rc(swf_forecast_step(fm.ctx->get(), x_prev_phys.data(), forcing_phys.data(), &s, &c, sp.run_seed,
                               noise_event, out.data(), dtype_of<T>()));
    return out;
}

template <class T>
std::vector<std::vector<MatX<T>>> rollout_ensemble(const ForecastModel<T>& fm, const MatX<T>& x_init_phys,
                                                   const std::vector<MatX<T>>& forcings_phys, int n_members,
                                                   int n_steps, const SeedProtocol& sp, u64 rollout_id) {
    if (int(forcings_phys.size()) < n_steps) throw ConfigError("rollout: not enough forcing steps");
    const i64 fn = forcings_phys.empty() ? 0 : forcings_phys[0].size();
    std::vector<T> forc(size_t(fn) * n_steps);
    for (int k = 0; k < n_steps; ++k)
        std::copy(forcings_phys[k].data(), forcings_phys[k].data() + fn, forc.begin() + size_t(fn) * k);
    std::vector<T> all(size_t(x_init_phys.size()) * n_members * n_steps);
    const swf_standardizers s{fm.state_std.mean.data(), fm.state_std.std.data(), fm.resid_std.mean.data(),
                              fm.resid_std.std.data(),  fm.forcing_std.mean.data(), fm.forcing_std.std.data()};
    const swf_diffusion_cfg c = fm.dcfg.c();
    check_rc(swf_rollout_ensemble(fm.ctx->get(), x_init_phys.data(), forc.data(), n_members, n_steps, &s, &c,
                                  sp.run_seed, rollout_id, all.data(), dtype_of<T>()));
    std::vector<std::vector<MatX<T>>> out(n_members);
    for (int m = 0; m < n_members; ++m)
        for (int k = 0; k < n_steps; ++k) {
            MatX<T> x(x_init_phys.rows(), x_init_phys.cols());
            std::copy(all.begin() + size_t(x.size()) * (m * n_steps + k),
                      all.begin() + size_t(x.size()) * (m * n_steps + k + 1), x.data());
            out[m].push_back(std::move(x));
        }
    return out;
}

}  // namespace swinflow
