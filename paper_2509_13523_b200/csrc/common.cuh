// common.cuh -- shared device helpers for the swinflow B200 denoiser path (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#ifndef __CUDACC__
#error "sm_100a CUDA source"
#endif

namespace swf {

typedef int64_t i64;
typedef uint64_t u64;

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

#define SWF_CUDA(x)                                                                                       \
    do {                                                                                                  \
        cudaError_t e_ = (x);                                                                             \
        if (e_ != cudaSuccess)                                                                            \
            throw ::swf::CudaError(std::string(#x) + " failed: " + cudaGetErrorString(e_) + " at " +       \
                                   __FILE__ + ":" + std::to_string(__LINE__));                            \
    } while (0)

#define SWF_LAUNCH_CHECK() SWF_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ window layouts
// Restates WindowLayout::pixel_of (reference window.hpp:46-50) for a full-grid layout, plus
// the window-order <-> pixel maps the kernels use. Window order: index i = win * s + tok with
// win = wy * nx + wx and tok = r * w + c (canonical in-window order, window.hpp:11-14).
struct Lay {
    int H, W, w, shift;
    int nx, ny;  // windows per row / column
    __host__ __device__ int s() const { return w * w; }
    __host__ __device__ i64 win_to_pix(i64 i) const {
        const int ss = w * w;
        const int win = int(i / ss), tok = int(i - i64(win) * ss);
        const int wy = win / nx, wx = win - wy * nx;
        const int r = tok / w, c = tok - r * w;
        int y = wy * w + shift + r;
        if (y >= H) y -= H;
        int x = wx * w + shift + c;
        if (x >= W) x -= W;
        return i64(y) * W + x;
    }
    __host__ __device__ i64 pix_to_win(i64 p) const {
        const int y = int(p / W), x = int(p - i64(y) * W);
        int yy = y - shift;
        if (yy < 0) yy += H;
        int xx = x - shift;
        if (xx < 0) xx += W;
        const int wy = yy / w, r = yy - wy * w, wx = xx / w, c = xx - wx * w;
        return (i64(wy) * nx + wx) * (w * w) + r * w + c;
    }
};

static inline Lay make_lay(int H, int W, int w, int shift) {
    Lay l;
    l.H = H;
    l.W = W;
    l.w = w;
    l.shift = shift;
    l.nx = W / w;
    l.ny = H / w;
    return l;
}

// ------------------------------------------------------------------ small math
__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Non-finite flag (reference check_finite, swin.hpp:295-300): bit per block boundary.
__device__ __forceinline__ void flag_nonfinite(int* flags, int slot) { atomicOr(flags + slot, 1); }

}  // namespace swf
