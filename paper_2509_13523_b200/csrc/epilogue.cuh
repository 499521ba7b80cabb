// epilogue.cuh -- GEMM epilogues shared by the SIMT (FP32 validation) and tcgen05 (BF16) GEMMs.
// Each call handles `CNT` consecutive output columns [n0, n0+CNT) of one row m (n0 % CNT == 0).
#pragma once

#include "kernels.cuh"

namespace swf {

template <class T>
__device__ __forceinline__ void st_val(T* p, float v);
template <>
__device__ __forceinline__ void st_val<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st_val<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// RoPE (rope.hpp:34-44) on the pair (v0, v1) of column pair j of a head vector at window token
// position (prow, pcol): pairs j < d/4 rotate with the row coordinate, the rest with the column.
// Tables are [pair][position] (cos, sin), so the 32 lanes of a warp -- 32 consecutive tokens --
// read one broadcast row entry and 32 contiguous column entries.
__device__ __forceinline__ void rope_pair(const EpiParams& ep, int prow, int pcol, int j, float& v0, float& v1) {
    const int q4 = ep.d >> 2;
    const float2 cs = j < q4 ? ep.rope_row[j * ep.rope_nrow + prow] : ep.rope_col[(j - q4) * ep.rope_ncol + pcol];
    const float x = v0, y = v1;
    v0 = cs.x * x - cs.y * y;
    v1 = cs.y * x + cs.x * y;
}

template <int MODE, class OutT, int CNT>
__device__ __forceinline__ void epi_apply(const EpiParams& ep, i64 m, int n0, float* v) {
    if (m >= ep.M) return;
    const int h = ep.h;
    if constexpr (MODE == EPI_ENCODE) {
        float* xr = ep.x + m * h;
#pragma unroll
        for (int j = 0; j < CNT; ++j)
            if (n0 + j < ep.N) xr[n0 + j] = v[j] + ep.bias[n0 + j];
    } else if constexpr (MODE == EPI_RESID) {
        float* xr = ep.x + m * h;
#pragma unroll
        for (int j = 0; j < CNT; ++j)
            if (n0 + j < ep.N) xr[n0 + j] += v[j];
    } else if constexpr (MODE == EPI_DOWN) {
        int rank;
        const i64 li = ep.nxt.pix_to_loc(ep.cur.loc_to_pix(m), &rank);
        const float* xs = ep.x + m * h;
        float* xd = ep.xdst[rank] + li * h;
#pragma unroll
        for (int j = 0; j < CNT; ++j)
            if (n0 + j < ep.N) xd[n0 + j] = xs[n0 + j] + v[j];
    } else if constexpr (MODE == EPI_DECODE) {
        float* o = reinterpret_cast<float*>(ep.out) + m * ep.ld_out;
#pragma unroll
        for (int j = 0; j < CNT; ++j)
            if (n0 + j < ep.N) o[n0 + j] = (v[j] + ep.bias[n0 + j]) * ep.out_scale;
    } else if constexpr (MODE == EPI_QKV) {
        const int s = ep.cur.g.w * ep.cur.g.w;
        int gw, tok, lw;
        ep.cur.loc_to_wtok(m, gw, tok, lw);
        const int wy = gw / ep.cur.g.nx, wx = gw - (gw / ep.cur.g.nx) * ep.cur.g.nx;
        const int w = ep.cur.g.w;
        const int prow = wy * w + ep.cur.g.shift + tok / w;  // unwrapped rope position (window.hpp:54-56)
        const int pcol = wx * w + ep.cur.g.shift + tok % w;
        OutT* base = reinterpret_cast<OutT*>(ep.out);
#pragma unroll
        for (int j = 0; j < CNT; j += 2) {
            const int n = n0 + j;
            if (n >= ep.N) continue;
            const int which = n / h;
            const int e = n - which * h;
            const int head = e / ep.d;
            const int dd = e - head * ep.d;
            float a = v[j], b = v[j + 1];
            if (which < 2) rope_pair(ep, prow, pcol, dd >> 1, a, b);
            OutT* dst = base + which * ep.plane + ((i64(lw) * ep.heads + head) * s + tok) * ep.d + dd;
            st_val<OutT>(dst, a);
            st_val<OutT>(dst + 1, b);
        }
    }
}

// SwiGLU epilogue: gate/up columns for the same CNT ffn units (swin.hpp:230-232).
template <class OutT, int CNT>
__device__ __forceinline__ void epi_swiglu(const EpiParams& ep, i64 m, int j0, const float* g, const float* u) {
    if (m >= ep.M) return;
    OutT* o = reinterpret_cast<OutT*>(ep.out) + m * ep.ld_out;
#pragma unroll
    for (int t = 0; t < CNT; ++t)
        if (j0 + t < ep.N) st_val<OutT>(o + j0 + t, silu_f(g[t]) * u[t]);
}

}  // namespace swf
