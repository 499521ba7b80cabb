// ops.cu -- the leaves of the reference's `ops` namespace (swin.hpp:49-234) as standalone device
// calls on host buffers: linear_cols, prenorm_modulate, swiglu_fwd and the windowed attention. The
// reference's SWiPe simulator calls these leaves directly per sequence band (simulator.hpp:466-506);
// here they run the same sm_100a kernels the fused forward uses (tcgen05 GEMM / SIMT FP32 GEMM,
// RMSNorm + AdaLN, SwiGLU epilogue arithmetic). Column-major like the reference: a C x n matrix is
// n * C values with column j (token j) contiguous, i.e. [n][C] rows.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/swinflow_capi.h"
#include "kernels.cuh"

namespace swf {
namespace {

struct OpError : std::runtime_error {
    int rc;
    OpError(int r, const std::string& m) : std::runtime_error(m), rc(r) {}
};
void need(bool c, const std::string& m) {
    if (!c) throw OpError(SWF_ERR_CONFIG, m);
}
inline i64 up(i64 a, i64 b) { return (a + b - 1) / b * b; }

struct DevBuf {  // device allocation released on scope exit
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        SWF_CUDA(cudaMalloc(&p, bytes + 256));
        SWF_CUDA(cudaMemset(p, 0, bytes + 256));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

__global__ void k_silu_mul(const float* __restrict__ g, const float* __restrict__ u, i64 rows, int cols, int ld,
                           float* __restrict__ out, int ldo, int bf16_round) {
    const i64 total = rows * cols;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const i64 r = e / cols;
        const int c = int(e - r * cols);
        float v = silu_f(g[r * ld + c]) * u[r * ld + c];
        if (bf16_round) v = __bfloat162float(__float2bfloat16_rn(v));
        out[r * ldo + c] = v;
    }
}

// Y[n][out] = X[n][in] . W^T with W the reference's out x in column-major array (W[k * out + o]).
// BF16: operands rounded to bf16, FP32 accumulation on the tensor cores; FP32: SIMT FP32.
void linear(int precision, const float* W, int out, int in, const float* X, i64 n, float* Y) {
    need(out > 0 && in > 0 && n > 0, "linear_cols: empty operand");
    const int Kp = int(up(in, 64));
    const bool bf = precision == SWF_PREC_BF16;
    const int BN = bf && up(out, 128) % 256 == 0 ? 256 : 128;
    const int Np = int(up(out, BN));
    const i64 Mp = up(n, 128);
    // host staging: A rows [Mp][Kp] and B rows [Np][Kp] (K-major), zero padded
    std::vector<float> a(size_t(Mp) * Kp, 0.f), b(size_t(Np) * Kp, 0.f);
    for (i64 j = 0; j < n; ++j) std::memcpy(&a[size_t(j) * Kp], X + size_t(j) * in, size_t(in) * 4);
    for (int k = 0; k < in; ++k)
        for (int o = 0; o < out; ++o) b[size_t(o) * Kp + k] = W[size_t(k) * out + o];
    DevBuf dy(size_t(Mp) * Np * 4), dbias(size_t(Np) * 4);
    EpiParams ep;
    std::memset(&ep, 0, sizeof ep);
    ep.M = n;
    ep.N = Np;
    ep.h = Np;
    ep.x = dy.as<float>();
    ep.bias = dbias.as<float>();
    ep.out_scale = 1.f;
    if (bf) {
        std::vector<__nv_bfloat16> ah(a.size()), bh(b.size());
        for (size_t i = 0; i < a.size(); ++i) ah[i] = __float2bfloat16_rn(a[i]);
        for (size_t i = 0; i < b.size(); ++i) bh[i] = __float2bfloat16_rn(b[i]);
        DevBuf da(ah.size() * 2), db(bh.size() * 2), sched(64);
        SWF_CUDA(cudaMemcpy(da.p, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice));
        SWF_CUDA(cudaMemcpy(db.p, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice));
        ep.sched = sched.as<int>();
        TmaMap ta, tb;
        make_tma_bf16(&ta, da.p, Mp, Kp, 128);
        make_tma_bf16(&tb, db.p, Np, Kp, BN / 2);
        gemm_bf16_tc(ta, tb, n, Np, Kp, BN, EPI_ENCODE, ep, nullptr);
    } else {
        DevBuf da(a.size() * 4), db(b.size() * 4);
        SWF_CUDA(cudaMemcpy(da.p, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
        SWF_CUDA(cudaMemcpy(db.p, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
        gemm_f32(da.as<float>(), db.as<float>(), n, Np, Kp, EPI_ENCODE, ep, nullptr);
    }
    SWF_CUDA(cudaDeviceSynchronize());
    std::vector<float> yp(size_t(n) * Np);
    SWF_CUDA(cudaMemcpy(yp.data(), dy.p, yp.size() * 4, cudaMemcpyDeviceToHost));
    for (i64 j = 0; j < n; ++j) std::memcpy(Y + size_t(j) * out, &yp[size_t(j) * Np], size_t(out) * 4);
}

template <class F>
int op_try(F&& f) {
    try {
        f();
        return SWF_OK;
    } catch (const OpError& e) {
        set_last_error(e.what());
        return e.rc;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SWF_ERR_CUDA;
    }
}

}  // namespace
}  // namespace swf

using namespace swf;

extern "C" {

int swf_op_linear_cols(int device, int precision, const float* W, int out, int in, const float* X, long long n,
                       float* Y) {
    return op_try([&] {
        need(W && X && Y, "linear_cols: null argument");
        need(precision == SWF_PREC_BF16 || precision == SWF_PREC_FP32, "linear_cols: bad precision");
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        linear(precision, W, out, in, X, n, Y);
    });
}

int swf_op_prenorm_modulate(int device, const float* X, int h, long long n, const float* g, const float* a,
                            const float* b, const float* gate, float* Y) {
    return op_try([&] {
        need(X && g && Y && h > 0 && n > 0, "prenorm_modulate: bad argument");
        need(h % 4 == 0, "prenorm_modulate: hidden size must be a multiple of 4");
        need((a && b && gate) || (!a && !b && !gate), "prenorm_modulate: a, b, gate all given or all null");
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        const size_t nx = size_t(n) * h;
        DevBuf dx(nx * 4), dy(nx * 4), dv(size_t(4) * h * 4), flags(64);
        SWF_CUDA(cudaMemcpy(dx.p, X, nx * 4, cudaMemcpyHostToDevice));
        float* v = dv.as<float>();
        SWF_CUDA(cudaMemcpy(v, g, size_t(h) * 4, cudaMemcpyHostToDevice));
        if (a) {
            SWF_CUDA(cudaMemcpy(v + h, a, size_t(h) * 4, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(v + 2 * h, b, size_t(h) * 4, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(v + 3 * h, gate, size_t(h) * 4, cudaMemcpyHostToDevice));
        }
        rms_modulate<float>(dx.as<float>(), n, h, h, v, a ? v + h : nullptr, a ? v + 2 * h : nullptr,
                            a ? v + 3 * h : nullptr, dy.as<float>(), flags.as<int>(), 0, nullptr);
        SWF_CUDA(cudaDeviceSynchronize());
        int flag = 0;
        SWF_CUDA(cudaMemcpy(&flag, flags.p, 4, cudaMemcpyDeviceToHost));
        if (flag) throw OpError(SWF_ERR_NUMERICS, "prenorm_modulate: non-finite input");
        SWF_CUDA(cudaMemcpy(Y, dy.p, nx * 4, cudaMemcpyDeviceToHost));
    });
}

int swf_op_swiglu_fwd(int device, int precision, const float* W_gate, const float* W_up, const float* W_down,
                      int h, int f, const float* X, long long n, float* Y) {
    return op_try([&] {
        need(W_gate && W_up && W_down && X && Y && h > 0 && f > 0 && n > 0, "swiglu_fwd: bad argument");
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        std::vector<float> G(size_t(n) * f), U(size_t(n) * f), S(size_t(n) * f);
        linear(precision, W_gate, f, h, X, n, G.data());
        linear(precision, W_up, f, h, X, n, U.data());
        {  // s = silu(gate) * up (swin.hpp:230-232); rounded to bf16 on the BF16 path like the fused epilogue
            DevBuf dg(G.size() * 4), du(U.size() * 4), ds(S.size() * 4);
            SWF_CUDA(cudaMemcpy(dg.p, G.data(), G.size() * 4, cudaMemcpyHostToDevice));
            SWF_CUDA(cudaMemcpy(du.p, U.data(), U.size() * 4, cudaMemcpyHostToDevice));
            const int grid = int(std::min<i64>((i64(G.size()) + 255) / 256, 148 * 32));
            k_silu_mul<<<grid, 256>>>(dg.as<float>(), du.as<float>(), n, f, f, ds.as<float>(), f,
                                      precision == SWF_PREC_BF16);
            SWF_LAUNCH_CHECK();
            SWF_CUDA(cudaDeviceSynchronize());
            SWF_CUDA(cudaMemcpy(S.data(), ds.p, S.size() * 4, cudaMemcpyDeviceToHost));
        }
        linear(precision, W_down, h, f, S.data(), n, Y);
    });
}

// The backward's tensor-core GEMM on host buffers (test hook for gemm_bf16_general): C[M][N] (+)= A . B,
// A = [M][lda] K-major or [K][lda] MN-major, B = [N][ldb] K-major or [K][ldb] MN-major, operands
// rounded to bf16, fp32 accumulation.
int swf_op_gemm_bf16(int device, int mn_major, long long M, long long N, long long K, const float* A, long long lda,
                     const float* B, long long ldb, float* Cm, long long ldc, int accumulate) {
    return op_try([&] {
        need(A && B && Cm && M > 0 && N > 0 && K > 0, "gemm_bf16: bad argument");
        need(lda % 8 == 0 && ldb % 8 == 0 && ldc >= N, "gemm_bf16: operand pitches must be multiples of 8");
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        const size_t na = size_t(mn_major ? K : M) * lda, nb = size_t(mn_major ? K : N) * ldb, nc = size_t(M) * ldc;
        DevBuf da(na * 4), db(nb * 4), dc(nc * 4), ta(na * 2), tb(nb * 2), sched(64);
        SWF_CUDA(cudaMemcpy(da.p, A, na * 4, cudaMemcpyHostToDevice));
        SWF_CUDA(cudaMemcpy(db.p, B, nb * 4, cudaMemcpyHostToDevice));
        SWF_CUDA(cudaMemcpy(dc.p, Cm, nc * 4, cudaMemcpyHostToDevice));
        to_bf16(da.as<float>(), i64(na), ta.as<__nv_bfloat16>(), nullptr);
        to_bf16(db.as<float>(), i64(nb), tb.as<__nv_bfloat16>(), nullptr);
        gemm_bf16_general(ta.as<__nv_bfloat16>(), mn_major != 0, lda, tb.as<__nv_bfloat16>(), mn_major != 0, ldb, M, N,
                          K, dc.as<float>(), ldc, accumulate != 0, sched.as<int>(), nullptr);
        SWF_CUDA(cudaDeviceSynchronize());
        SWF_CUDA(cudaMemcpy(Cm, dc.p, nc * 4, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
