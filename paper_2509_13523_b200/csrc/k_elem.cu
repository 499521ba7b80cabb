// k_elem.cu -- HBM-bound kernels of the denoiser path: time embedding / AdaLN vectors, input
// gather, RMSNorm+modulation, sampler updates, noise field, standardisation.
#include "kernels.cuh"

namespace swf {

namespace {

constexpr int kThreads = 256;

inline bool aligned16(const void* a, const void* b, const void* c, const void* d) {
    return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(c) |
             reinterpret_cast<uintptr_t>(d)) & 15) == 0;
}

inline int grid_for(i64 n, int per_block = kThreads) {
    i64 g = (n + per_block - 1) / per_block;
    if (g > 148 * 64) g = 148 * 64;
    return int(g < 1 ? 1 : g);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- time features (model.hpp:229-241)
// f[2k] = sin(t * 2000/pi * 10000^(-k/(td/2))), f[2k+1] = cos(...), in double, cast to float. t is
// a kernel argument, so back-to-back evaluations at different t never share a staging buffer.
__global__ void k_time_features(double t, int td, float* __restrict__ feat) {
    const int nf = td / 2;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x) {
        const double om = pow(10000.0, -double(k) / nf);
        const double arg = t * 636.6197723675814 * om;
        feat[2 * k] = static_cast<float>(sin(arg));
        feat[2 * k + 1] = static_cast<float>(cos(arg));
    }
    if ((td & 1) && blockIdx.x == 0 && threadIdx.x == 0) feat[td - 1] = 1.f;
}

// ---------------------------------------------------------------- time embedding (model.hpp:261-269)
// emb[o] = silu(sum_k Wt[o][k] feat[k] + b[o]); one warp per output row.
__global__ void k_time_embed(const float* __restrict__ feat, const float* __restrict__ wt,
                             const float* __restrict__ b, int td, float* __restrict__ emb) {
    const int o = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (o >= td) return;
    float acc = 0.f;
    for (int k = lane; k < td; k += 32) acc += wt[i64(o) * td + k] * feat[k];
    acc = warp_sum(acc);
    if (lane == 0) emb[o] = silu_f(acc + b[o]);
}

// ---------------------------------------------------------------- ada vectors (swin.hpp:28-41)
__global__ void k_ada(const float* __restrict__ emb, const float* __restrict__ wt, const float* __restrict__ b,
                      i64 rows, int td, float* __restrict__ six) {
    const i64 o = i64(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (o >= rows) return;
    const float* w = wt + o * td;
    float acc = 0.f;
    for (int k = lane; k < td; k += 32) acc += w[k] * emb[k];
    acc = warp_sum(acc);
    if (lane == 0) six[o] = b[o] + acc;
}

// ---------------------------------------------------------------- gather / scatter rows
template <class T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <class T>
__device__ __forceinline__ void store_cvt4(T* p, float4 v);
template <>
__device__ __forceinline__ void store_cvt4<float>(float* p, float4 v) {
    *reinterpret_cast<float4*>(p) = v;
}
template <>
__device__ __forceinline__ void store_cvt4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
}

// One warp per local row: the row's pixel is resolved once (not per element), then the C source
// values are read as 16-byte vectors (C % 4 == 0 and ldo % 4 == 0) or scalars, cast and zero-padded to
// ldo. Source rows are contiguous [pixel][C] runs, so each warp reads / writes whole rows coalesced.
template <class T>
__global__ void __launch_bounds__(256) k_gather_rows(const float* __restrict__ src, LayMap lay, int C, int ldo, i64 M,
                                                     T* __restrict__ dst, int* flags, int slot) {
    const int lane = threadIdx.x & 31;
    const bool vec = (C % 4 == 0) && (ldo % 4 == 0);
    bool bad = false;
    for (i64 i = i64(blockIdx.x) * 8 + (threadIdx.x >> 5); i < M; i += i64(gridDim.x) * 8) {
        const float* row = src + lay.loc_to_pix(i) * C;
        T* o = dst + i * ldo;
        if (vec) {
            for (int q = lane; q < ldo / 4; q += 32) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (4 * q < C) {
                    v = __ldg(reinterpret_cast<const float4*>(row) + q);
                    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
                }
                store_cvt4<T>(o + 4 * q, v);
            }
        } else {
            for (int c = lane; c < ldo; c += 32) {
                float v = 0.f;
                if (c < C) {
                    v = __ldg(row + c);
                    bad |= !isfinite(v);
                }
                o[c] = cvt<T>(v);
            }
        }
    }
    if (flags && __any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(flags, slot);
}

// One warp per local row, the inverse of k_gather_rows.
__global__ void __launch_bounds__(256) k_scatter_rows(const float* __restrict__ src, LayMap lay, int C, i64 M,
                                                      float* __restrict__ dst) {
    const int lane = threadIdx.x & 31;
    for (i64 i = i64(blockIdx.x) * 8 + (threadIdx.x >> 5); i < M; i += i64(gridDim.x) * 8) {
        float* o = dst + lay.loc_to_pix(i) * C;
        const float* r = src + i * C;
        if (C % 4 == 0)
            for (int q = lane; q < C / 4; q += 32)
                reinterpret_cast<float4*>(o)[q] = __ldg(reinterpret_cast<const float4*>(r) + q);
        else if (C % 2 == 0)  // e.g. the decode output's 70 channels: 8-byte vectors
            for (int q = lane; q < C / 2; q += 32)
                reinterpret_cast<float2*>(o)[q] = __ldg(reinterpret_cast<const float2*>(r) + q);
        else
            for (int c = lane; c < C; c += 32) o[c] = __ldg(r + c);
    }
}

// ---------------------------------------------------------------- RMSNorm + AdaLN (swin.hpp:72-85)
// One warp per token row. r = sqrt(||x||^2/h + 1e-8); u = x / r; out = gate*((g*u)*(1+a)+b).
template <class T>
__device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
    uint2 u;
    u.x = pack_bf16x2(a, b);
    u.y = pack_bf16x2(c, d);
    *reinterpret_cast<uint2*>(p) = u;
}

template <class T>
__global__ void __launch_bounds__(256) k_rms_mod(const float* __restrict__ x, i64 M, int h, int ldo,
                                                 const float* __restrict__ g, const float* __restrict__ a,
                                                 const float* __restrict__ b, const float* __restrict__ gate,
                                                 T* __restrict__ out, int* flags, int slot) {
    const int lane = threadIdx.x & 31;
    const i64 nwarps = i64(gridDim.x) * (blockDim.x / 32);
    for (i64 m = i64(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; m < M; m += nwarps) {
        const float4* xr = reinterpret_cast<const float4*>(x + m * h);
        float ss = 0.f;
        bool bad = false;
        for (int i = lane; i < h / 4; i += 32) {
            const float4 v = xr[i];
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
            bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
        }
        ss = warp_sum(ss);
        if (flags && __any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(flags, slot);
        const float r = sqrtf(ss / float(h) + 1e-8f);
        T* o = out + m * ldo;
        for (int i = lane; i < h / 4; i += 32) {
            const float4 v = xr[i];
            const float4 gg = reinterpret_cast<const float4*>(g)[i];
            float y0 = gg.x * (v.x / r), y1 = gg.y * (v.y / r), y2 = gg.z * (v.z / r), y3 = gg.w * (v.w / r);
            if (a) {
                const float4 aa = reinterpret_cast<const float4*>(a)[i];
                const float4 bb = reinterpret_cast<const float4*>(b)[i];
                const float4 ga = reinterpret_cast<const float4*>(gate)[i];
                y0 = ga.x * (y0 * (1.f + aa.x) + bb.x);
                y1 = ga.y * (y1 * (1.f + aa.y) + bb.y);
                y2 = ga.z * (y2 * (1.f + aa.z) + bb.z);
                y3 = ga.w * (y3 * (1.f + aa.w) + bb.w);
            }
            store4<T>(o + 4 * i, y0, y1, y2, y3);
        }
    }
}

// ---------------------------------------------------------------- sampler
// xa and y may alias (stage 2 updates the state in place): no __restrict__ on either; each element is
// read and written by one thread, in that order
// VEC: 16-byte accesses (all pointers 16-byte aligned, checked by the launcher) plus a scalar tail
template <bool VEC>
__global__ void k_sampler_update(const float* xa, const float* __restrict__ xd, const float* __restrict__ v, i64 n,
                                 float cs, float sn, float c1, float c2, float* y, int* flags, int slot) {
    bool bad = false;
    auto one = [&](float a, float d0, float w) {
        const float d = cs * d0 - sn * w;
        const float r = c1 * a - c2 * d;
        bad |= !isfinite(r);
        return r;
    };
    const i64 stride = i64(gridDim.x) * blockDim.x, t0 = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    i64 done = 0;
    if constexpr (VEC) {
        const i64 n4 = n >> 2;
        for (i64 i = t0; i < n4; i += stride) {
            const float4 a = reinterpret_cast<const float4*>(xa)[i], d = __ldg(reinterpret_cast<const float4*>(xd) + i),
                         w = __ldg(reinterpret_cast<const float4*>(v) + i);
            reinterpret_cast<float4*>(y)[i] =
                make_float4(one(a.x, d.x, w.x), one(a.y, d.y, w.y), one(a.z, d.z, w.z), one(a.w, d.w, w.w));
        }
        done = 4 * n4;
    }
    for (i64 i = done + t0; i < n; i += stride) y[i] = one(xa[i], xd[i], v[i]);
    if (flags && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_nonfinite(flags, slot);
}

template <class T>
__device__ __forceinline__ void store_cvt2(T* p, float a, float b);
template <>
__device__ __forceinline__ void store_cvt2<float>(float* p, float a, float b) {
    *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
template <>
__device__ __forceinline__ void store_cvt2<__nv_bfloat16>(__nv_bfloat16* p, float a, float b) {
    *reinterpret_cast<uint32_t*>(p) = pack_bf16x2(a, b);
}
// The sampler's input assembly, one warp per row and channel pairs (cp, cf, cin, kp even; checked by
// the launchers, which fall back to the element-wise kernels below otherwise).
template <class T>
__global__ void __launch_bounds__(256) k_build_static_rows(const float* __restrict__ xp, const float* __restrict__ fo,
                                                           const float* __restrict__ pe, i64 M, int cp, int cf,
                                                           int cin, int kp, T* __restrict__ a_in) {
    const int lane = threadIdx.x & 31;
    for (i64 i = i64(blockIdx.x) * 8 + (threadIdx.x >> 5); i < M; i += i64(gridDim.x) * 8) {
        for (int c = cp + 2 * lane; c < kp; c += 64) {  // channels [cp, kp): x_prev, forcings, zero pad
            float2 v = make_float2(0.f, 0.f);
            if (c < 2 * cp) {
                const float2 a = __ldg(reinterpret_cast<const float2*>(xp + i * cp + (c - cp)));
                const float2 p = __ldg(reinterpret_cast<const float2*>(pe + i * cin + c));
                v = make_float2(a.x + p.x, a.y + p.y);
            } else if (c < cin) {
                const float2 a = __ldg(reinterpret_cast<const float2*>(fo + i * cf + (c - 2 * cp)));
                const float2 p = __ldg(reinterpret_cast<const float2*>(pe + i * cin + c));
                v = make_float2(a.x + p.x, a.y + p.y);
            }
            store_cvt2<T>(a_in + i * kp + c, v.x, v.y);
        }
    }
}
template <class T>
__global__ void __launch_bounds__(256) k_assemble_state_rows(const float* __restrict__ x, const float* __restrict__ pe,
                                                             i64 M, int cp, int cin, int kp, float sd,
                                                             T* __restrict__ a_in) {
    const int lane = threadIdx.x & 31;
    for (i64 i = i64(blockIdx.x) * 8 + (threadIdx.x >> 5); i < M; i += i64(gridDim.x) * 8) {
        for (int c = 2 * lane; c < cp; c += 64) {
            const float2 a = __ldg(reinterpret_cast<const float2*>(x + i * cp + c));
            const float2 p = __ldg(reinterpret_cast<const float2*>(pe + i * cin + c));
            store_cvt2<T>(a_in + i * kp + c, a.x / sd + p.x, a.y / sd + p.y);
        }
    }
}

template <class T>
__global__ void k_build_static(const float* __restrict__ xp, const float* __restrict__ fo,
                               const float* __restrict__ pe, i64 M, int cp, int cf, int cin, int kp,
                               T* __restrict__ a_in) {
    const int w = kp - cp;
    const i64 total = M * w;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e / w;
        const int c = cp + int(e - i * w);
        float v = 0.f;
        if (c < 2 * cp)
            v = xp[i * cp + (c - cp)] + pe[i * cin + c];
        else if (c < cin)
            v = fo[i * cf + (c - 2 * cp)] + pe[i * cin + c];
        a_in[i * kp + c] = cvt<T>(v);
    }
}

template <class T>
__global__ void k_assemble_state(const float* __restrict__ x, const float* __restrict__ pe, i64 M, int cp, int cin,
                                 int kp, float sd, T* __restrict__ a_in) {
    const i64 total = M * cp;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e / cp;
        const int c = int(e - i * cp);
        a_in[i * kp + c] = cvt<T>(x[e] / sd + pe[i * cin + c]);
    }
}

// counter RNG (rng.hpp:17-45), double-precision Box-Muller as in the reference
__device__ __forceinline__ u64 d_splitmix(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ u64 d_kd(u64 key, u64 tag) { return d_splitmix(key ^ d_splitmix(tag)); }
__device__ __forceinline__ double d_gaussian(u64 key, u64 ctr) {
    const u64 b0 = d_splitmix(key + 0x632be59bd9b4e019ULL * (2 * ctr + 1));
    const u64 b1 = d_splitmix(key + 0x632be59bd9b4e019ULL * (2 * ctr + 2));
    const double u1 = (double(b0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = double(b1 >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

__global__ void k_noise(u64 zfk, int C, LayMap lay, double sd, float* __restrict__ z, i64 M) {
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < M; i += i64(gridDim.x) * blockDim.x) {
        int gw, tok, lw;
        lay.loc_to_wtok(i, gw, tok, lw);
        const u64 key = d_kd(d_kd(zfk, u64(gw)), u64(tok));  // z_cell_key(window, token)
        for (int c = 0; c < C; ++c) z[i * C + c] = float(sd * d_gaussian(key, u64(c)));
    }
}

__global__ void k_churn(float* __restrict__ x, LayMap lay, i64 M, int C, const u64* __restrict__ key_p, u64 ctr0,
                        double sd, float c, float s) {
    const i64 total = M * C;
    const u64 key = *key_p;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e / C;
        const int ch = int(e - i * C);
        const u64 ctr = ctr0 + u64(lay.loc_to_pix(i)) * C + ch;
        const float zeta = float(sd * d_gaussian(key, ctr));
        x[e] = c * x[e] + s * zeta;
    }
}

// per-channel affine maps over [M][C] rows; VEC: 16-byte accesses, one channel modulo per 4 elements
template <bool VEC>
__global__ void k_standardize(const float* __restrict__ x, i64 M, int C, const float* __restrict__ mean,
                              const float* __restrict__ sd, float* __restrict__ y) {
    const i64 total = M * C, stride = i64(gridDim.x) * blockDim.x, t0 = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    auto f = [&](float v, int c) { return (v - mean[c]) / sd[c]; };
    i64 done = 0;
    if constexpr (VEC) {
        for (i64 i = t0; i < (total >> 2); i += stride) {
            int c = int((4 * i) % C);
            const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
            float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[k] = f(o[k], c);
                if (++c == C) c = 0;
            }
            reinterpret_cast<float4*>(y)[i] = make_float4(o[0], o[1], o[2], o[3]);
        }
        done = total & ~i64(3);
    }
    for (i64 e = done + t0; e < total; e += stride) y[e] = f(x[e], int(e % C));
}

template <bool VEC>
__global__ void k_destd_add(const float* __restrict__ r, const float* __restrict__ base, i64 M, int C,
                            const float* __restrict__ mean, const float* __restrict__ sd, float* __restrict__ y) {
    const i64 total = M * C, stride = i64(gridDim.x) * blockDim.x, t0 = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    auto f = [&](float b, float v, int c) { return b + (v * sd[c] + mean[c]); };
    i64 done = 0;
    if constexpr (VEC) {
        for (i64 i = t0; i < (total >> 2); i += stride) {
            int c = int((4 * i) % C);
            const float4 v = __ldg(reinterpret_cast<const float4*>(r) + i),
                         b = __ldg(reinterpret_cast<const float4*>(base) + i);
            float o[4] = {v.x, v.y, v.z, v.w}, bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[k] = f(bb[k], o[k], c);
                if (++c == C) c = 0;
            }
            reinterpret_cast<float4*>(y)[i] = make_float4(o[0], o[1], o[2], o[3]);
        }
        done = total & ~i64(3);
    }
    for (i64 e = done + t0; e < total; e += stride) y[e] = f(base[e], r[e], int(e % C));
}

__global__ void k_check_finite(const float* __restrict__ x, i64 n, int* flags, int slot) {
    bool bad = false;
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_nonfinite(flags, slot);
}

}  // namespace

void time_features(double t, int td, float* feat, cudaStream_t st) {
    k_time_features<<<(td / 2 + 255) / 256 + 1, 256, 0, st>>>(t, td, feat);
    SWF_LAUNCH_CHECK();
}

void time_embed(const float* feat, const float* w_time_t, const float* b_time, int td, float* emb, cudaStream_t st) {
    k_time_embed<<<(td + 7) / 8, 256, 0, st>>>(feat, w_time_t, b_time, td, emb);
    SWF_LAUNCH_CHECK();
}

void ada_vectors(const float* emb, const float* w_ada_t, const float* b_ada, int nb, int six_h, int td, float* six,
                 cudaStream_t st) {
    const i64 rows = i64(nb) * six_h;
    k_ada<<<int((rows + 7) / 8), 256, 0, st>>>(emb, w_ada_t, b_ada, rows, td, six);
    SWF_LAUNCH_CHECK();
}

template <class T>
void gather_rows(const float* src_pix, const LayMap& lay, int C, int ldo, i64 M, T* dst, int* flags, int slot,
                 cudaStream_t st) {
    k_gather_rows<T><<<grid_for(M, 8), kThreads, 0, st>>>(src_pix, lay, C, ldo, M, dst, flags, slot);
    SWF_LAUNCH_CHECK();
}
template void gather_rows<float>(const float*, const LayMap&, int, int, i64, float*, int*, int, cudaStream_t);
template void gather_rows<__nv_bfloat16>(const float*, const LayMap&, int, int, i64, __nv_bfloat16*, int*, int,
                                         cudaStream_t);

void scatter_rows(const float* src_loc, const LayMap& lay, int C, i64 M, float* dst_pix, cudaStream_t st) {
    k_scatter_rows<<<grid_for(M, 8), kThreads, 0, st>>>(src_loc, lay, C, M, dst_pix);
    SWF_LAUNCH_CHECK();
}

namespace {
// one warp per residual row: the bf16 copy (zero-padded to hp) and the row's sum of squares in
// partial slot 0 (others 0) -- what the producing GEMM epilogues emit for the fused norm
__global__ void k_prep_residual(const float* __restrict__ x, i64 M, int h, int hp, int nss,
                                __nv_bfloat16* __restrict__ xb, float* __restrict__ ss) {
    const i64 row = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= M) return;
    const int lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int c = lane; c < hp; c += 32) {
        const float v = c < h ? x[row * h + c] : 0.f;
        xb[row * hp + c] = __float2bfloat16_rn(v);
        acc += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    for (int k = lane; k < nss; k += 32) ss[row * nss + k] = k == 0 ? acc : 0.f;
}

// one warp per requested pixel: its row of the local [M][C] buffer (owned pixels only)
__global__ void k_rows_at_pixels(const float* __restrict__ src, LayMap lay, int rank, int C,
                                 const i64* __restrict__ pix, i64 n, float* __restrict__ dst) {
    const i64 k = i64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= n) return;
    int owner = 0;
    const i64 i = lay.pix_to_loc(pix[k], &owner);
    if (owner != rank) return;
    for (int c = threadIdx.x & 31; c < C; c += 32) dst[k * C + c] = src[i * C + c];
}
}  // namespace

void prep_residual(const float* x, i64 M, int h, int hp, int nss, __nv_bfloat16* xb, float* ss, cudaStream_t st) {
    if (M <= 0) return;
    k_prep_residual<<<int((M + 7) / 8), 256, 0, st>>>(x, M, h, hp, nss, xb, ss);
    SWF_LAUNCH_CHECK();
}

void rows_at_pixels(const float* src_loc, const LayMap& lay, int rank, int C, const i64* pix, i64 n, float* dst,
                    cudaStream_t st) {
    if (n <= 0) return;
    k_rows_at_pixels<<<int((n + 7) / 8), 256, 0, st>>>(src_loc, lay, rank, C, pix, n, dst);
    SWF_LAUNCH_CHECK();
}

namespace {
// one warp per weight row: fold the AdaLN scale into the row and dot it with the shift vector
__global__ void k_fold_adaln(const float* __restrict__ Wm, int Np, int K, int ld, const float* __restrict__ g,
                             const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ gate,
                             __nv_bfloat16* __restrict__ Wf, float* __restrict__ beta) {
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (n >= Np) return;
    const float* w = Wm + i64(n) * ld;
    __nv_bfloat16* o = Wf + i64(n) * ld;
    float acc = 0.f;
    for (int k = lane; k < ld; k += 32) {
        float sk = 0.f, ck = 0.f;
        if (k < K) {
            const float q = gate ? gate[k] : 1.f;
            sk = q * g[k] * (a ? 1.f + a[k] : 1.f);
            ck = b ? q * b[k] : 0.f;
        }
        const float wv = w[k];
        o[k] = __float2bfloat16_rn(wv * sk);
        acc = fmaf(wv, ck, acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (beta && lane == 0) beta[n] = acc;
}
}  // namespace

namespace {
__global__ void k_inv_rms(const float* __restrict__ ss, i64 M, int nss, int h, float* __restrict__ inv_r,
                          int* __restrict__ flags, int slot) {
    const i64 m = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (m >= M) return;
    float sq = 0.f;
    for (int i = 0; i < nss; ++i) sq += ss[m * nss + i];
    inv_r[m] = 1.f / sqrtf(sq / float(h) + 1e-8f);  // kRmsEps, swin.hpp:45
    if (flags && !isfinite(sq)) atomicOr(flags + slot, 1);
}
}  // namespace

void inv_rms(const float* ss, i64 M, int nss, int h, float* inv_r, int* flags, int slot, cudaStream_t st) {
    k_inv_rms<<<unsigned((M + 255) / 256), 256, 0, st>>>(ss, M, nss, h, inv_r, flags, slot);
    SWF_LAUNCH_CHECK();
}

void fold_adaln(const float* Wm, int Np, int K, int ld, const float* g, const float* a, const float* b,
                const float* gate, __nv_bfloat16* Wf, float* beta, cudaStream_t st) {
    k_fold_adaln<<<unsigned((Np + 7) / 8), 256, 0, st>>>(Wm, Np, K, ld, g, a, b, gate, Wf, beta);
    SWF_LAUNCH_CHECK();
}

template <class T>
void rms_modulate(const float* x, i64 M, int h, int ldo, const float* g, const float* a, const float* b,
                  const float* gate, T* out, int* flags, int slot, cudaStream_t st) {
    if (h % 4 != 0) throw CudaError("rms_modulate: h must be a multiple of 4");
    k_rms_mod<T><<<grid_for(M * 32), 256, 0, st>>>(x, M, h, ldo, g, a, b, gate, out, flags, slot);
    SWF_LAUNCH_CHECK();
}
template void rms_modulate<float>(const float*, i64, int, int, const float*, const float*, const float*,
                                  const float*, float*, int*, int, cudaStream_t);
template void rms_modulate<__nv_bfloat16>(const float*, i64, int, int, const float*, const float*, const float*,
                                          const float*, __nv_bfloat16*, int*, int, cudaStream_t);

void sampler_update(const float* xa, const float* xd, const float* v, i64 n, float cs, float sn, float c1, float c2,
                    float* y, int* flags, int slot, cudaStream_t st) {
    if (aligned16(xa, xd, v, y))
        k_sampler_update<true><<<grid_for((n + 3) / 4), kThreads, 0, st>>>(xa, xd, v, n, cs, sn, c1, c2, y, flags, slot);
    else
        k_sampler_update<false><<<grid_for(n), kThreads, 0, st>>>(xa, xd, v, n, cs, sn, c1, c2, y, flags, slot);
    SWF_LAUNCH_CHECK();
}

template <class T>
void build_static_input(const float* xprev, const float* forc, const float* pe, i64 M, int cp, int cf, int cin,
                        int kp, T* a_in, cudaStream_t st) {
    if (cp % 2 == 0 && cf % 2 == 0 && cin % 2 == 0 && kp % 2 == 0 && aligned16(xprev, forc, pe, a_in))
        k_build_static_rows<T><<<grid_for(M, 8), kThreads, 0, st>>>(xprev, forc, pe, M, cp, cf, cin, kp, a_in);
    else
        k_build_static<T><<<grid_for(M * (kp - cp)), kThreads, 0, st>>>(xprev, forc, pe, M, cp, cf, cin, kp, a_in);
    SWF_LAUNCH_CHECK();
}
template void build_static_input<float>(const float*, const float*, const float*, i64, int, int, int, int, float*,
                                        cudaStream_t);
template void build_static_input<__nv_bfloat16>(const float*, const float*, const float*, i64, int, int, int, int,
                                                __nv_bfloat16*, cudaStream_t);

template <class T>
void assemble_state(const float* x, const float* pe, i64 M, int cp, int cin, int kp, float sd, T* a_in,
                    cudaStream_t st) {
    if (cp % 2 == 0 && cin % 2 == 0 && kp % 2 == 0 && aligned16(x, pe, a_in, a_in))
        k_assemble_state_rows<T><<<grid_for(M, 8), kThreads, 0, st>>>(x, pe, M, cp, cin, kp, sd, a_in);
    else
        k_assemble_state<T><<<grid_for(M * cp), kThreads, 0, st>>>(x, pe, M, cp, cin, kp, sd, a_in);
    SWF_LAUNCH_CHECK();
}
template void assemble_state<float>(const float*, const float*, i64, int, int, int, float, float*, cudaStream_t);
template void assemble_state<__nv_bfloat16>(const float*, const float*, i64, int, int, int, float, __nv_bfloat16*,
                                            cudaStream_t);

void noise_field(u64 zfk, int C, const LayMap& lay0, double sigma_d, float* z, cudaStream_t st) {
    const i64 M = i64(lay0.nloc) * lay0.s_loc();
    k_noise<<<grid_for(M), kThreads, 0, st>>>(zfk, C, lay0, sigma_d, z, M);
    SWF_LAUNCH_CHECK();
}

void churn_rotate(float* x, const LayMap& lay0, i64 M, int C, const u64* key, u64 ctr0, double sigma_d, float c, float s,
                  cudaStream_t st) {
    k_churn<<<grid_for(M * C), kThreads, 0, st>>>(x, lay0, M, C, key, ctr0, sigma_d, c, s);
    SWF_LAUNCH_CHECK();
}

void standardize(const float* x, i64 M, int C, const float* mean, const float* stdv, float* y, cudaStream_t st) {
    if (aligned16(x, y, x, y) && C >= 4)
        k_standardize<true><<<grid_for((M * C + 3) / 4), kThreads, 0, st>>>(x, M, C, mean, stdv, y);
    else
        k_standardize<false><<<grid_for(M * C), kThreads, 0, st>>>(x, M, C, mean, stdv, y);
    SWF_LAUNCH_CHECK();
}

void destandardize_add(const float* r, const float* base, i64 M, int C, const float* mean, const float* stdv,
                       float* y, cudaStream_t st) {
    if (aligned16(r, base, y, y) && C >= 4)
        k_destd_add<true><<<grid_for((M * C + 3) / 4), kThreads, 0, st>>>(r, base, M, C, mean, stdv, y);
    else
        k_destd_add<false><<<grid_for(M * C), kThreads, 0, st>>>(r, base, M, C, mean, stdv, y);
    SWF_LAUNCH_CHECK();
}

void check_finite(const float* x, i64 n, int* flags, int slot, cudaStream_t st) {
    k_check_finite<<<grid_for(n), kThreads, 0, st>>>(x, n, flags, slot);
    SWF_LAUNCH_CHECK();
}

// Load every kernel of this file into the current device's context now (see preload_kernels).
void preload_elem_kernels() {
    cudaFuncAttributes a;
    const void* k[] = {
        (const void*)k_time_features, (const void*)k_time_embed, (const void*)k_ada,
        (const void*)k_gather_rows<float>, (const void*)k_gather_rows<__nv_bfloat16>, (const void*)k_scatter_rows,
        (const void*)k_rms_mod<float>, (const void*)k_rms_mod<__nv_bfloat16>, (const void*)k_sampler_update<true>,
        (const void*)k_sampler_update<false>,
        (const void*)k_build_static<float>, (const void*)k_build_static<__nv_bfloat16>,
        (const void*)k_build_static_rows<float>, (const void*)k_build_static_rows<__nv_bfloat16>,
        (const void*)k_assemble_state_rows<float>, (const void*)k_assemble_state_rows<__nv_bfloat16>,
        (const void*)k_assemble_state<float>, (const void*)k_assemble_state<__nv_bfloat16>, (const void*)k_noise,
        (const void*)k_churn, (const void*)k_standardize<true>, (const void*)k_standardize<false>,
        (const void*)k_destd_add<true>, (const void*)k_destd_add<false>, (const void*)k_check_finite,
        (const void*)k_prep_residual, (const void*)k_rows_at_pixels, (const void*)k_fold_adaln, (const void*)k_inv_rms};
    for (const void* f : k) SWF_CUDA(cudaFuncGetAttributes(&a, f));
}

}  // namespace swf
