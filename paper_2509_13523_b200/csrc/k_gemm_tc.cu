// k_gemm_tc.cu -- BF16 GEMM on the 5th-generation tensor cores (sm_100a):
//   tcgen05.mma.cta_group::2 (UMMA 256 x BN x 16, 2-CTA pairs), operands staged by TMA with
//   128-byte swizzle, FP32 accumulators in TMEM (double-buffered), persistent static tile
//   schedule, warp specialisation (TMA producer / MMA issuer / 4 epilogue warps).
// The epilogue fuses the reference's per-token ops that follow each linear:
//   encode bias, RoPE + head-major scatter (QKV), residual add (out), SiLU*up (gate/up) and the
//   residual add + next-layout window permutation of the down projection (swin.hpp:306-366).
#include <cuda.h>

#include <cstring>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "../../include/swinflow_capi.h"
#include "epilogue.cuh"
#include "tc_ptx.cuh"

namespace swf {

namespace {

constexpr int BM = 128;  // rows per CTA; UMMA M = 256 per CTA pair
constexpr int BK = 64;   // one 128-byte swizzle atom of bf16
constexpr int kThreads = 384;
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quadrant, each draining half of the columns

// The gate/up GEMM (SwiGLU epilogue, no shared-memory transposes) gives the epilogue staging space to a
// 7th operand stage at BN = 256: 55.9 -> 55.0 M cycles at base clock (the QKV GEMM measured 1% slower
// with 7, so every other mode keeps 6; SWF_GEMM_DEEP=0: 6 stages everywhere)
#ifndef SWF_GEMM_DEEP
#define SWF_GEMM_DEEP 1
#endif
constexpr bool uses_stg(int mode) { return mode != EPI_SWIGLU; }

template <int BN, bool STG = true>
struct Cfg {
    static constexpr int kStageA = BM * BK * 2;
    static constexpr int kStageB = (BN / 2) * BK * 2;
    static constexpr int kStage = kStageA + kStageB;
    static constexpr int kStages = (BN == 256) ? ((STG || !SWF_GEMM_DEEP) ? 6 : 7) : 8;
    static constexpr int kTmemCols = 2 * BN;  // two accumulator buffers
    static constexpr int kStageFloats = (STG || !SWF_GEMM_DEEP) ? kEpiWarps * 32 * 33 : 0;  // epilogue transposes
    static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/ + kStageFloats * 4;
    static constexpr uint32_t kIdesc = (1u << 4)                 // D = F32
                                       | (1u << 7) | (1u << 10)  // A, B = BF16
                                       | (uint32_t(BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// arrive on a (possibly remote) barrier of the cluster; CTA-scope release: the data handed over lives
// in TMEM (ordered by tcgen05.wait + tcgen05.fence::before_thread_sync), and a cluster-scope release
// would cost a GPU-wide MEMBAR per arrival
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// release-ordered arrive (cluster scope): publishes shared-memory writes made before it to the
// waiting threads of either CTA (the tile queue, once per tile)
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t bar_cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acquire_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void tma_load_2cta(uint32_t dst, const void* tmap, uint32_t bar_cluster, int c0, int c1,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
// L2 eviction policies: weights stay resident (evict_last); epilogue output streams go first
// (evict_first), so the 19 GB SwiGLU stream does not flush the weights or the A row-blocks.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_ef_v4(void* ptr, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16)  // LBO (unused for swizzled K-major)
           | (uint64_t(1024 >> 4) << 32)                          // SBO: 8 rows x 128 B
           | (uint64_t(1) << 46)                                  // sm100 descriptor version
           | (uint64_t(2) << 61);                                 // SWIZZLE_128B
}
// MN-major SW128 operand (the backward's weight gradients: tokens = K run along the rows of a TMA box
// [K rows][64 MN elements]): 64-element MN chunks LBO = one box (64 rows x 128 B) apart, 8-row K
// groups SBO = 1024 B apart; a K step of 16 advances the start by 16 rows (2048 B)
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((BK * 128) >> 4) << 16)  // LBO: next 64-wide MN chunk
           | (uint64_t(1024 >> 4) << 32)                                        // SBO: next 8 K rows
           | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void umma_2cta(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    tc::ld32(taddr, r);
    tc::wait_ld_dep(r);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- vectorised epilogues (32 columns)
// bf16 copy of 32 residual values (operand A of the next normed GEMM); returns their sum of squares
__device__ __forceinline__ float store_xb32(const EpiParams& ep, const float* xbase, i64 m, int n0, const float* o) {
    uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(const_cast<float*>(xbase) + ep.off_xb) +
                                        m * ep.hp + n0);
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        d[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]), pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                          pack_bf16x2(o[8 * j + 4], o[8 * j + 5]), pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
#pragma unroll
        for (int t = 0; t < 8; ++t) ss = fmaf(o[8 * j + t], o[8 * j + t], ss);
    }
    return ss;
}

template <int MODE>
__device__ __forceinline__ float epi32(const EpiParams& ep, i64 m, int n0, float* v) {
    if (m >= ep.M || n0 >= ep.N) return 0.f;
    const int h = ep.h;
    if constexpr (MODE == EPI_ENCODE) {
        float4* xr = reinterpret_cast<float4*>(ep.x + m * h + n0);
        float o[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 b = reinterpret_cast<const float4*>(ep.bias + n0)[j];
            o[4 * j] = v[4 * j] + b.x;
            o[4 * j + 1] = v[4 * j + 1] + b.y;
            o[4 * j + 2] = v[4 * j + 2] + b.z;
            o[4 * j + 3] = v[4 * j + 3] + b.w;
            xr[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
        return ep.nss ? store_xb32(ep, ep.x, m, n0, o) : 0.f;
    } else if constexpr (MODE == EPI_RESID) {
        float4* xr = reinterpret_cast<float4*>(ep.x + m * h + n0);
        float o[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float4 x4 = xr[j];
            x4.x += v[4 * j];
            x4.y += v[4 * j + 1];
            x4.z += v[4 * j + 2];
            x4.w += v[4 * j + 3];
            xr[j] = x4;
            o[4 * j] = x4.x;
            o[4 * j + 1] = x4.y;
            o[4 * j + 2] = x4.z;
            o[4 * j + 3] = x4.w;
        }
        return ep.nss ? store_xb32(ep, ep.x, m, n0, o) : 0.f;
    } else if constexpr (MODE == EPI_DOWN) {
        int rank;
        const i64 li = ep.nxt.pix_to_loc(ep.cur.loc_to_pix(m), &rank);
        const float4* xs = reinterpret_cast<const float4*>(ep.x + m * h + n0);
        float4* xd = reinterpret_cast<float4*>(ep.xdst[rank] + li * h + n0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 o = xs[j];
            xd[j] = make_float4(o.x + v[4 * j], o.y + v[4 * j + 1], o.z + v[4 * j + 2], o.w + v[4 * j + 3]);
        }
    } else if constexpr (MODE == EPI_QKV) {
        // d >= 32 so the 32 columns lie inside one head of one of q/k/v. The head's planes live on
        // the rank of its head group (Ulysses sequence parallelism, simulator.hpp:464-507): the
        // store goes straight to that rank over NVLink (own buffer when sp == 1).
        const int s = ep.cur.g.w * ep.cur.g.w;
        int gw, tok, lw;
        ep.cur.loc_to_wtok(m, gw, tok, lw);
        const int which = n0 / h;
        const int e = n0 - which * h;
        const int head = e / ep.d;
        const int dd = e - head * ep.d;
        const int hg = head / ep.heads_loc, hl = head - hg * ep.heads_loc;
        __nv_bfloat16* base =
            reinterpret_cast<__nv_bfloat16*>(ep.qkv_dst[ep.wp_rank * ep.cur.sp + hg]) + which * ep.plane;
        if (which < 2) {
            const int w = ep.cur.g.w;
            const int wy = gw / ep.cur.g.nx, wx = gw - wy * ep.cur.g.nx;
            const int prow = wy * w + ep.cur.g.shift + tok / w;
            const int pcol = wx * w + ep.cur.g.shift + tok % w;
#pragma unroll
            for (int j = 0; j < 32; j += 2) rope_pair(ep, prow, pcol, (dd + j) >> 1, v[j], v[j + 1]);
        } else {
            // V is stored transposed ([window][head][d][token]) so the attention's P.V MMA reads a
            // K-major operand; the 32 lanes of a warp hold consecutive tokens -> 64 B per store.
            __nv_bfloat16* vt = base + ((i64(lw) * ep.heads_loc + hl) * ep.d + dd) * s + tok;
#pragma unroll
            for (int j = 0; j < 32; ++j) vt[i64(j) * s] = __float2bfloat16_rn(v[j]);
            return 0.f;
        }
        __nv_bfloat16* dst = base + ((i64(lw) * ep.heads_loc + hl) * s + tok) * ep.d + dd;
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            d4[j] = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                               pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
    } else if constexpr (MODE == EPI_DECODE) {
        float* o = reinterpret_cast<float*>(ep.out) + m * ep.ld_out;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (n0 + j < ep.N) o[n0 + j] = (v[j] + ep.bias[n0 + j]) * ep.out_scale;
    }
    return 0.f;
}

// QKV epilogue with the row's window / token / RoPE positions resolved once per tile (not per
// 32-column chunk): RoPE pairs from the position-major tables (a chunk's 16 pairs are one line, read
// as 8 float4), q / k rows as 16-byte stores, V^T as 64-byte warp-wide rows.
// The column half's pairs are read from the frequency-major table (entry j at rcf[j * ncol]): the 32
// lanes of a warp are consecutive tokens, i.e. mostly consecutive columns, so one load instruction
// touches 2-3 lines instead of 32 (the position-major row of a lane is its own line). The row half
// stays position-major: the lanes share 1-2 image rows. ncu: the q/k tiles' epilogue was bound by
// L1 wavefronts (~12.8 K per tile against 12.3 K cycles of MMA per tile).
#ifndef SWF_QKV_ROPE_FM
#define SWF_QKV_ROPE_FM 1
#endif
struct QkvRow {
    bool ok;
    int lw, tok;
    const float2 *rr, *rc;  // this row's RoPE (cos, sin) for the row / column halves
};
__device__ __forceinline__ QkvRow qkv_row(const EpiParams& ep, i64 m) {
    QkvRow r;
    r.ok = m < ep.M;
    if (!r.ok) return r;
    int gw;
    ep.cur.loc_to_wtok(m, gw, r.tok, r.lw);
    const int w = ep.cur.g.w, q4 = ep.d >> 2;
    const int wy = gw / ep.cur.g.nx, wx = gw - wy * ep.cur.g.nx;
    const int prow = wy * w + ep.cur.g.shift + r.tok / w;  // unwrapped RoPE position (window.hpp:54-56)
    const int pcol = wx * w + ep.cur.g.shift + r.tok % w;
    r.rr = ep.rope_row_pm + i64(prow) * q4;
    r.rc = SWF_QKV_ROPE_FM ? ep.rope_col + pcol : ep.rope_col_pm + i64(pcol) * q4;
    return r;
}
// 32 rows x 64 B of bf16 (lane = row, u = its 4 16-byte pieces) stored through the warp's shared-memory
// staging so that 4 lanes write one row's 64 B and an instruction touches 8 lines instead of 32 (pieces
// XOR-swizzled by row: both shared-memory passes are conflict-free); rows with dst == nullptr and
// pieces >= npieces are skipped.
__device__ __forceinline__ void store_rows_bf16x32(const uint4* u, __nv_bfloat16* dst, int npieces, float* stg,
                                                   int lane) {
    uint4* st4 = reinterpret_cast<uint4*>(stg);  // [32 rows][4 pieces of 16 B]
    __syncwarp();                                // the previous chunk's reads are done
#pragma unroll
    for (int p = 0; p < 4; ++p) st4[lane * 4 + (p ^ ((lane >> 1) & 3))] = u[p];
    __syncwarp();
    const int p = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = 8 * i + (lane >> 2);
        const uint4 val = st4[r * 4 + (p ^ ((r >> 1) & 3))];
        auto* rd = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), r));
        if (rd && p < npieces) rd[p] = val;
    }
}

// q / k rows leave through the warp's shared-memory staging: a lane holds 64 B of its own row (the
// rows are 256 B apart in the destination plane), so a direct 16-byte store touches 32 lines per
// instruction; transposed, 4 lanes write one row's 64 B and an instruction touches 8 lines (pieces
// XOR-swizzled by row so both shared-memory passes are conflict-free).
#ifndef SWF_QKV_STS
#define SWF_QKV_STS 1
#endif
__device__ __forceinline__ void epi_qkv32(const EpiParams& ep, const QkvRow& qr, int n0, float* v, float* stg,
                                          int lane) {
    if (n0 >= ep.N) return;  // warp-uniform
    const int h = ep.h, s = ep.cur.g.w * ep.cur.g.w, q4 = ep.d >> 2;
    const int which = n0 / h;
    const int e = n0 - which * h;
    const int head = e / ep.d;
    const int dd = e - head * ep.d;
    const int hg = head / ep.heads_loc, hl = head - hg * ep.heads_loc;
    __nv_bfloat16* base =
        reinterpret_cast<__nv_bfloat16*>(ep.qkv_dst[ep.wp_rank * ep.cur.sp + hg]) + which * ep.plane;
    if (which == 2) {  // V^T [window][head][d][token]: the warp's 32 lanes are consecutive tokens
        if (!qr.ok) return;
        __nv_bfloat16* vt = base + ((i64(qr.lw) * ep.heads_loc + hl) * ep.d + dd) * s + qr.tok;
#pragma unroll
        for (int j = 0; j < 32; ++j) vt[i64(j) * s] = __float2bfloat16_rn(v[j]);
        return;
    }
    __nv_bfloat16* dst = nullptr;
    if (qr.ok) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // pairs j, j + 1 lie in the same half (q4 is even); warp-uniform branch
            const int j = (dd >> 1) + 2 * k;
            float4 cs;
            if (j < q4) {
                cs = *reinterpret_cast<const float4*>(qr.rr + j);
            } else if (SWF_QKV_ROPE_FM) {
                const float2 a = qr.rc[i64(j - q4) * ep.rope_ncol], b = qr.rc[i64(j + 1 - q4) * ep.rope_ncol];
                cs = make_float4(a.x, a.y, b.x, b.y);
            } else {
                cs = *reinterpret_cast<const float4*>(qr.rc + (j - q4));
            }
            float x = v[4 * k], y = v[4 * k + 1];
            v[4 * k] = cs.x * x - cs.y * y;
            v[4 * k + 1] = cs.y * x + cs.x * y;
            x = v[4 * k + 2];
            y = v[4 * k + 3];
            v[4 * k + 2] = cs.z * x - cs.w * y;
            v[4 * k + 3] = cs.w * x + cs.z * y;
        }
        dst = base + ((i64(qr.lw) * ep.heads_loc + hl) * s + qr.tok) * ep.d + dd;
    }
    uint4 u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        u[j] = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                          pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
#if SWF_QKV_STS
    store_rows_bf16x32(u, dst, 4, stg, lane);
#else
    if (dst)
#pragma unroll
        for (int j = 0; j < 4; ++j) reinterpret_cast<uint4*>(dst)[j] = u[j];
#endif
}

// Attention backward (EPI_SMAX / EPI_DSM): 32 columns of one row of the s x s plane -> bf16 P or dS.
template <int MODE>
__device__ __forceinline__ void epi_attn_rows32(const EpiParams& ep, i64 m, int n0, const float* v, float* stg,
                                                int lane, int bb) {
    if (n0 >= ep.N) return;  // warp-uniform
    const bool ok = m < ep.M;
    uint4 u[4];
    __nv_bfloat16* dst = nullptr;
    if (ok) {
        float o[32];
        const float rv = ep.rowv[i64(bb) * ep.bst_rv + m];
        if constexpr (MODE == EPI_SMAX) {
            const int lo = (ep.masked && m >= ep.split) ? ep.split : 0;
            const int hi = (ep.masked && m < ep.split) ? ep.split : ep.N;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                o[j] = (n0 + j >= lo && n0 + j < hi) ? exp2f(fmaf(v[j], ep.out_scale, -rv)) : 0.f;
        } else {
            const uint4* pr = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.pin) +
                                                             i64(bb) * ep.bst_p + m * ep.ld_out + n0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 pp = n0 + 8 * q < ep.N ? pr[q] : make_uint4(0, 0, 0, 0);
                const uint32_t w[4] = {pp.x, pp.y, pp.z, pp.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[t]));
                    o[8 * q + 2 * t] = f.x * (v[8 * q + 2 * t] - rv) * ep.out_scale;
                    o[8 * q + 2 * t + 1] = f.y * (v[8 * q + 2 * t + 1] - rv) * ep.out_scale;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            u[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]), pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                              pack_bf16x2(o[8 * j + 4], o[8 * j + 5]), pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
        dst = static_cast<__nv_bfloat16*>(ep.out) + i64(bb) * ep.bst_c + m * ep.ld_out + n0;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = make_uint4(0, 0, 0, 0);
    }
    const int npieces = min(4, (ep.N - n0) >> 3);  // 8-column pieces inside N (N % 8 == 0)
    store_rows_bf16x32(u, dst, npieces, stg, lane);
}

__device__ __forceinline__ void epi_swiglu32(const EpiParams& ep, i64 m, int j0, const float* g, const float* u,
                                             uint64_t pol) {
    if (m >= ep.M || j0 >= ep.N) return;
    uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.out) + m * ep.ld_out + j0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float r[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {  // SiLU with ex2.approx + rcp.approx (error far below the bf16 output)
            const float x = g[8 * j + t];
            r[t] = __fdividef(x, 1.0f + __expf(-x)) * u[8 * j + t];
        }
        st_ef_v4(d4 + j, make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]), pack_bf16x2(r[4], r[5]),
                                    pack_bf16x2(r[6], r[7])),
                 pol);
    }
}

// Rasterisation: bands of group_m m-blocks are swept n-block by n-block (m fastest inside a band).
// With the dynamic schedule the concurrently running clusters take consecutive tile indices, i.e.
// group_m row blocks x (clusters / group_m) N tiles: each A slice is shared by fewer clusters at
// the same instant (group_m = 1: every cluster on one row block), while the weights B stay
// L2-resident under the evict_last policy.
__device__ __forceinline__ void tile_coords(i64 t, int n_tiles, i64 m_tiles, int group_m, int& m_blk, int& n_blk) {
    const i64 per_group = i64(group_m) * n_tiles;
    const i64 g = t / per_group;
    const i64 r = t - g * per_group;
    const i64 gm = min(i64(group_m), m_tiles - g * group_m);
    n_blk = int(r / gm);
    m_blk = int(g * group_m + r % gm);
}

// fp32 row-major outputs (encode / residual / down): the 32x32 chunk a warp holds (thread = row)
// is transposed through shared memory so each global access is one contiguous 128-byte row segment.
// The out projection's and the encode's full 32 x 32 chunks (the common case) move through shared
// memory in 16-byte pieces instead: 8 lanes cover one row's 128 B, an instruction 4 rows -- a quarter
// of the scalar path's shared-memory and global instructions (ncu: the out projection's epilogue had
// the L1 data pipe at 65% of peak, ~12 K wavefronts per tile against 12.9 K cycles of MMA). Same
// arithmetic and the same summation order for the row's sum of squares as the scalar path, so the
// results are bitwise equal whichever path a row takes.
#ifndef SWF_RESID_V4
#define SWF_RESID_V4 1
#endif
// the 16-byte path needs 16-byte fp32 rows and 8-byte bf16-copy rows (the general GEMM's accumulate
// mode runs EPI_RESID on any caller matrix, e.g. a 70-column gradient)
template <int MODE>
__device__ __forceinline__ bool v4_aligned(const EpiParams& ep) {
    uintptr_t a = reinterpret_cast<uintptr_t>(ep.x) | (uintptr_t(ep.h) * 4);
    if (MODE == EPI_ENCODE) a |= reinterpret_cast<uintptr_t>(ep.bias);
    uintptr_t b = ep.nss ? reinterpret_cast<uintptr_t>(ep.x + ep.off_xb) | (uintptr_t(ep.hp) * 2) : 0;
    return (a & 15) == 0 && (b & 7) == 0;
}
template <int MODE>  // EPI_RESID: x += acc in place; EPI_ENCODE: x = acc + bias
__device__ __forceinline__ float epi32_v4(const EpiParams& ep, i64 row0, int n0, const float* v, float* stg, int lane) {
    float4* s4 = reinterpret_cast<float4*>(stg);  // [32 rows][8 pieces], piece p of row r at slot p ^ (r & 7)
#pragma unroll
    for (int p = 0; p < 8; ++p)
        s4[lane * 8 + (p ^ (lane & 7))] = make_float4(v[4 * p], v[4 * p + 1], v[4 * p + 2], v[4 * p + 3]);
    __syncwarp();
    const int q = lane & 7, rs = lane >> 3;
    const int h = ep.h;
    float* xs = ep.x + (row0 + rs) * h + n0 + 4 * q;
    float4 xv[8];
    if constexpr (MODE == EPI_RESID) {
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = *reinterpret_cast<const float4*>(xs + i64(4 * i) * h);
    } else {
        const float4 b = *reinterpret_cast<const float4*>(ep.bias + n0 + 4 * q);
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = b;
    }
    __nv_bfloat16* db =
        ep.nss ? reinterpret_cast<__nv_bfloat16*>(ep.x + ep.off_xb) + (row0 + rs) * ep.hp + n0 + 4 * q : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + rs;
        float4& slot = s4[r * 8 + (q ^ (r & 7))];
        const float4 a = slot;
        const float4 o = make_float4(xv[i].x + a.x, xv[i].y + a.y, xv[i].z + a.z, xv[i].w + a.w);
        *reinterpret_cast<float4*>(xs + i64(4 * i) * h) = o;
        if (db) {
            *reinterpret_cast<uint2*>(db + i64(4 * i) * ep.hp) = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
            slot = o;
        }
    }
    __syncwarp();
    float ss = 0.f;
    if (db) {  // this lane's row: sum of squares of the 32 new values, in column order
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const float4 o = s4[lane * 8 + (p ^ (lane & 7))];
            ss = fmaf(o.x, o.x, ss);
            ss = fmaf(o.y, o.y, ss);
            ss = fmaf(o.z, o.z, ss);
            ss = fmaf(o.w, o.w, ss);
        }
    }
    __syncwarp();
    return ss;
}

template <int MODE>
__device__ __forceinline__ float epi32_coalesced(const EpiParams& ep, i64 row, int n0, const float* v, float* stg,
                                                 float* drow, __nv_bfloat16* dbrow, int lane, float* xstore) {
    if constexpr ((MODE == EPI_RESID || MODE == EPI_ENCODE) && SWF_RESID_V4)
        if (ep.M - (row - lane) >= 32 && n0 + 32 <= ep.N && v4_aligned<MODE>(ep))
            return epi32_v4<MODE>(ep, row - lane, n0, v, stg, lane);
#pragma unroll
    for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = v[i];
    __syncwarp();
    const i64 row0 = row - lane;
    const int n = n0 + lane;
    const bool col_ok = n < ep.N;
    const int h = ep.h;
    const i64 mrem = ep.M - row0;  // rows of this 32-row group that exist
    if constexpr (MODE == EPI_ENCODE) {  // x = acc + bias, plus the bf16 copy for the first block's norm
        const float b = col_ok ? ep.bias[n] : 0.f;
        __nv_bfloat16* db = ep.nss ? reinterpret_cast<__nv_bfloat16*>(ep.x + ep.off_xb) + row0 * ep.hp + n : nullptr;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            const float o = stg[rr * 33 + lane] + b;
            if (rr < mrem && col_ok) {
                ep.x[(row0 + rr) * h + n] = o;
                if (ep.nss) db[i64(rr) * ep.hp] = __float2bfloat16_rn(o);
            }
            if (ep.nss) stg[rr * 33 + lane] = col_ok ? o : 0.f;
        }
    } else if constexpr (MODE == EPI_STORE) {  // xstore: this problem's C (plane-batched launches)
#pragma unroll
        for (int rr = 0; rr < 32; ++rr)
            if (rr < mrem && col_ok) xstore[(row0 + rr) * h + n] = stg[rr * 33 + lane];
    } else if (MODE == EPI_RESID && mrem >= 32 && n0 + 32 <= ep.N) {
        // out projection, full 32 x 32 chunk (the common case): in place, so the bf16 copy's rows are
        // addressed directly (no pointer shuffles) and no per-row predicates
        float* xs = ep.x + row0 * h + n;
        float xv[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) xv[rr] = xs[i64(rr) * h];
        if (ep.nss) {
            __nv_bfloat16* db = reinterpret_cast<__nv_bfloat16*>(ep.x + ep.off_xb) + row0 * ep.hp + n;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                const float o = xv[rr] + stg[rr * 33 + lane];
                xs[i64(rr) * h] = o;
                db[i64(rr) * ep.hp] = __float2bfloat16_rn(o);
                stg[rr * 33 + lane] = o;
            }
        } else {
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) xs[i64(rr) * h] = xv[rr] + stg[rr * 33 + lane];
        }
    } else {
        // all 32 row reads in flight before any dependent store (latency hiding with 4 warps)
        float xv[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) xv[rr] = (rr < mrem && col_ok) ? ep.x[(row0 + rr) * h + n] : 0.f;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            float* dst;
            if constexpr (MODE == EPI_DOWN)
                dst = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(drow), rr)) + n;
            else
                dst = ep.x + (row0 + rr) * h + n;
            const float o = xv[rr] + stg[rr * 33 + lane];
            if (rr < mrem && col_ok) *dst = o;
            if (ep.nss) {
                __nv_bfloat16* db = reinterpret_cast<__nv_bfloat16*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dbrow), rr));
                if (rr < mrem && col_ok) db[n] = __float2bfloat16_rn(o);
                stg[rr * 33 + lane] = col_ok ? o : 0.f;
            }
        }
    }
    __syncwarp();
    float ss = 0.f;
    if (ep.nss) {  // this lane's row: sum of squares of the 32 new values
#pragma unroll
        for (int i = 0; i < 32; ++i) ss = fmaf(stg[lane * 33 + i], stg[lane * 33 + i], ss);
        __syncwarp();
    }
    return ss;
}

// Dynamic tile schedule: a scheduler thread of the leader CTA (warp 3) takes tile indices from a
// global counter (atomicAdd, one per tile) and publishes them through a kQ-slot ring in both CTAs'
// shared memory; every consumer role (both producers, the MMA thread, the 16 epilogue warps) reads
// its next tile from the ring, with CTA-scope synchronisation in the scheduler's CTA. Clusters then take tiles in index order as they free up, so the clusters
// sharing an A row block (consecutive indices) start it together and its K slices are fetched from
// HBM once, instead of drifting apart over the static round-robin schedule (which re-read A ~3x).
constexpr int kQ = 4;
#ifndef SWF_GEMM_XPF
#define SWF_GEMM_XPF 1
#endif
constexpr uint32_t kQConsumers = 2 /*producers*/ + 1 /*MMA*/ + 2 * kEpiWarps;
struct TileQueue {
    uint64_t* full;  // [kQ], one arrival (the scheduler) per round, in each CTA
    uint64_t* empty; // [kQ], kQConsumers arrivals per round, leader CTA only
    int* tile;       // [kQ]
    int* counter;    // global; nullptr -> static round-robin schedule
    i64 total;
    int cluster_id, n_clusters;
    bool local;      // this thread runs in the leader CTA (the scheduler's): CTA-scope synchronisation
    // scheduler (leader CTA, its own thread): publish the i-th tile of this cluster; returns it
    __device__ int publish(int i) {
        const int slot = i % kQ;
        const uint32_t round = uint32_t(i / kQ);
        mbar_wait_acquire_cluster(smem_u32(&empty[slot]), (round & 1) ^ 1);
        const i64 t = atomicAdd(counter, 1);
        const int v = t < total ? int(t) : -1;
        tile[slot] = v;
        st_cluster_u32(map_to_rank(smem_u32(&tile[slot]), 1), uint32_t(v));
        mbar_arrive_release_cluster(map_to_rank(smem_u32(&full[slot]), 1));
        mbar_arrive_release_cluster(smem_u32(&full[slot]));
        return v;
    }
    // consumer: the i-th tile (-1: done); arrive = whether this thread signals the slot free
    __device__ i64 next(int i, bool arrive) {
        if (!counter) {
            const i64 t = cluster_id + i64(i) * n_clusters;
            return t < total ? t : -1;
        }
        const int slot = i % kQ;
        if (local) {  // same CTA as the scheduler: CTA-scope acquire / release (no cluster-wide fence)
            mbar_wait(smem_u32(&full[slot]), uint32_t(i / kQ) & 1);
            const int v = *reinterpret_cast<volatile int*>(&tile[slot]);
            if (arrive) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
            return v;
        }
        mbar_wait_acquire_cluster(smem_u32(&full[slot]), uint32_t(i / kQ) & 1);
        const int v = *reinterpret_cast<volatile int*>(&tile[slot]);
        // a relaxed arrive (no cluster-wide fence): the branch on the loaded value orders the slot's
        // read before the arrive that lets the scheduler overwrite it (v is never INT_MIN)
        if (arrive && v != INT_MIN)
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                             map_to_rank(smem_u32(&empty[slot]), 0))
                         : "memory");
        return v;
    }
};

#ifdef SWF_GEMM_TRACE
// development build only: clock64 stamps of cluster 0's MMA thread per tile: [0] before the tile-queue
// read, [1] after it, [2] after the accumulator-free wait, [3] after the tile's last commit, [4] cycles
// spent waiting for operand stages within the tile
constexpr int kGTr = 2048;
__device__ unsigned long long g_gtrace[5][kGTr];
inline void* g_gtrace_ptr() {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_gtrace);
    return p;
}
#endif
// ---------------------------------------------------------------- the kernel
// MN: operand majors, bit 0 = A MN-major (A stored [K][M]), bit 1 = B MN-major (B stored [K][N]); 0 =
// both K-major (the forward's layout)
template <int BN, int MODE, int MN = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, i64 M, int n_tiles,
              int num_k, EpiParams ep, int* sched, int group_m) {
    using C = Cfg<BN, uses_stg(MODE)>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kStageA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + C::kStages;
    uint64_t* tfull_bar = bars + 2 * C::kStages;
    uint64_t* tempty_bar = bars + 2 * C::kStages + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4);
    uint64_t* q_full = bars + 2 * C::kStages + 5;
    uint64_t* q_empty = q_full + kQ;
    int* q_tile = reinterpret_cast<int*>(q_empty + kQ);
    static_assert((2 * C::kStages + 5 + 2 * kQ) * 8 + kQ * 4 <= 256, "barrier region");

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
    const i64 m_tiles = (M + 2 * BM - 1) / (2 * BM);
    // plane-batched products (the attention backward's): tile t of problem t / per_b
    constexpr bool kBatched = MODE == EPI_STORE || MODE == EPI_SMAX || MODE == EPI_DSM;
    const i64 per_b = m_tiles * n_tiles;
    const i64 total = kBatched ? per_b * max(1, ep.nbatch) : per_b;

    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(smem_u32(&full_bar[s]), 1);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&tfull_bar[a]), 1);
            mbar_init(smem_u32(&tempty_bar[a]), 2 * kEpiWarps);
        }
        for (int a = 0; a < kQ; ++a) {
            mbar_init(smem_u32(&q_full[a]), 1);
            mbar_init(smem_u32(&q_empty[a]), kQConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    TileQueue tq{q_full, q_empty, q_tile, sched, total, cluster_id, n_clusters, leader};

    if (warp == 0) {
        // ===== TMA producer (both CTAs; each loads its A half and B half, signalling the leader)
        if (lane == 0) {
            // A row-blocks are re-read by every N tile of the band -> normal priority; weights -> last
            const uint64_t pol_a = policy_evict_normal(), pol_b = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;

            for (int i = 0;; ++i) {
                const i64 t = tq.next(i, true);
                if (t < 0) break;
                int m_blk, n_blk, bb = 0;
                if constexpr (kBatched) bb = int(t / per_b);
                tile_coords(kBatched ? t - i64(bb) * per_b : t, n_tiles, m_tiles, group_m, m_blk, n_blk);
                int row_a = m_blk * 2 * BM + int(crank) * BM, row_b = n_blk * BN + int(crank) * (BN / 2);
                int ka = 0, kbo = 0;  // problem offsets along the operands' K coordinate
                if constexpr (kBatched) {
                    if constexpr (MN & 1) row_a += bb * ep.adx, ka = bb * ep.ady;
                    else row_a += bb * ep.ady, ka = bb * ep.adx;
                    if constexpr (MN & 2) row_b += bb * ep.bdx, kbo = bb * ep.bdy;
                    else row_b += bb * ep.bdy, kbo = bb * ep.bdx;
                }
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                    const uint32_t fb = map_to_rank(smem_u32(&full_bar[stage]), 0);
                    if (leader) mbar_expect_tx(smem_u32(&full_bar[stage]), 2 * C::kStage);
                    if constexpr (MN & 1) {  // [64 K rows][64 M] boxes, BM / 64 of them
#pragma unroll
                        for (int c = 0; c < BM / 64; ++c)
                            tma_load_2cta(smem_u32(sA + stage * C::kStageA + c * BK * 128), &tmA, fb, row_a + 64 * c,
                                          kb * BK + ka, pol_a);
                    } else {
                        tma_load_2cta(smem_u32(sA + stage * C::kStageA), &tmA, fb, kb * BK + ka, row_a, pol_a);
                    }
                    if constexpr (MN & 2) {
#pragma unroll
                        for (int c = 0; c < BN / 128; ++c)
                            tma_load_2cta(smem_u32(sB + stage * C::kStageB + c * BK * 128), &tmB, fb, row_b + 64 * c,
                                          kb * BK + kbo, pol_b);
                    } else {
                        tma_load_2cta(smem_u32(sB + stage * C::kStageB), &tmB, fb, kb * BK + kbo, row_b, pol_b);
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ===== tile scheduler (leader CTA, one thread): takes tile indices from the global counter and
        // publishes them up to kQ tiles ahead, off the producer's path (the atomic's round trip had
        // stalled the operand loads ~2 K cycles per tile)
        if (leader && lane == 0 && sched)
            for (int i = 0;; ++i)
                if (tq.publish(i) < 0) break;
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA, one thread)
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int i = 0;; ++i) {
#ifdef SWF_GEMM_TRACE
                const bool tr = blockIdx.x == 0 && i < kGTr;
                unsigned long long fw = 0;
                if (tr) g_gtrace[0][i] = clock64();
#endif
                if (tq.next(i, true) < 0) break;
#ifdef SWF_GEMM_TRACE
                if (tr) g_gtrace[1][i] = clock64();
#endif
                mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
                tc_fence_after();
#ifdef SWF_GEMM_TRACE
                if (tr) g_gtrace[2][i] = clock64();
#endif
                const uint32_t dtm = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < num_k; ++kb) {
#ifdef SWF_GEMM_TRACE
                    const unsigned long long w0 = clock64();
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
                    fw += clock64() - w0;
#else
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
#endif
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * C::kStageA);
                    const uint32_t b0 = smem_u32(sB + stage * C::kStageB);
                    constexpr uint32_t kIdesc = C::kIdesc | (uint32_t(MN & 1) << 15) | (uint32_t((MN >> 1) & 1) << 16);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_2cta(dtm, (MN & 1) ? umma_desc_sw128_mn(a0 + k * 2048) : umma_desc_sw128(a0 + k * 32),
                                  (MN & 2) ? umma_desc_sw128_mn(b0 + k * 2048) : umma_desc_sw128(b0 + k * 32), kIdesc,
                                  (kb | k) != 0);
                    umma_commit_mc(smem_u32(&empty_bar[stage]), 0x3);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_mc(smem_u32(&tfull_bar[acc]), 0x3);
#ifdef SWF_GEMM_TRACE
                if (tr) {
                    g_gtrace[3][i] = clock64();
                    g_gtrace[4][i] = fw;
                }
#endif
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ===== epilogue: TMEM -> registers -> fused op -> global (8 warps: quadrant x column half)
        const int q = (warp - kEpiWarp0) & 3;     // TMEM lane quadrant (warp % 4)
        const int half = (warp - kEpiWarp0) >> 2;  // column half of the tile
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty_leader = map_to_rank(smem_u32(&tempty_bar[0]), 0);
        float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256) + (warp - kEpiWarp0) * 32 * 33;
        const uint64_t pol_out = policy_evict_first();
        for (int i = 0;; ++i) {
            const i64 t = tq.next(i, lane == 0);
            if (t < 0) break;
            int m_blk, n_blk, bb = 0;
            if constexpr (kBatched) bb = int(t / per_b);
            tile_coords(kBatched ? t - i64(bb) * per_b : t, n_tiles, m_tiles, group_m, m_blk, n_blk);
            const i64 row = i64(m_blk) * 2 * BM + crank * BM + q * 32 + lane;  // row of problem bb
#if SWF_GEMM_XPF
            // out projection (short K): pull this tile's rows of the residual x (this warp's half: BN/2
            // floats per row) into L2 while the accumulator is computed, so the epilogue's loads hit L2
            // (A/B: out GEMM -4%; for the down projection's long K the lines are evicted before use)
            if constexpr (MODE == EPI_RESID)
                if (row < ep.M && n_blk * BN + (half + 1) * (BN / 2) <= ep.N) {
                    const float* xr = ep.x + row * ep.h + n_blk * BN + half * (BN / 2);
#pragma unroll
                    for (int c = 0; c < BN / 64; ++c)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + c * 32) : "memory");
                }
#endif
            // row-only epilogue inputs load while the accumulator is computed: 1 / rms from the producer
            // partials (fused RMSNorm + AdaLN of operand A's rows) and the QKV row's window / RoPE positions
            float inv_r = 1.f;
            if constexpr (MODE == EPI_QKV || MODE == EPI_SWIGLU || MODE == EPI_DECODE)
                if (ep.inv_r && row < ep.M) inv_r = ep.inv_r[row];
            [[maybe_unused]] QkvRow qr;
            if constexpr (MODE == EPI_QKV) qr = qkv_row(ep, row);
            mbar_wait(smem_u32(&tfull_bar[acc]), acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            auto normed = [&](float* v, int col) {
                if constexpr (MODE == EPI_QKV || MODE == EPI_SWIGLU || MODE == EPI_DECODE) {
                    if (ep.inv_r) {
                        if (ep.beta) {
                            const float4* b4 = reinterpret_cast<const float4*>(ep.beta + col);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float4 bb = b4[j];
                                v[4 * j] = fmaf(v[4 * j], inv_r, bb.x);
                                v[4 * j + 1] = fmaf(v[4 * j + 1], inv_r, bb.y);
                                v[4 * j + 2] = fmaf(v[4 * j + 2], inv_r, bb.z);
                                v[4 * j + 3] = fmaf(v[4 * j + 3], inv_r, bb.w);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] *= inv_r;
                        }
                    }
                }
            };
            if constexpr (MODE == EPI_SWIGLU) {
                // interleave G = BN/2: columns [0, BN/2) gate, [BN/2, BN) up of the same ffn units
                constexpr int NCH = BN / 64;
#pragma unroll 1
                for (int ch = half * NCH / 2; ch < (half + 1) * NCH / 2; ++ch) {
                    float g[32], u[32];
                    tmem_ld32(tbase + ch * 32, g);
                    tmem_ld32(tbase + BN / 2 + ch * 32, u);
                    normed(g, n_blk * BN + ch * 32);
                    normed(u, n_blk * BN + BN / 2 + ch * 32);
                    epi_swiglu32(ep, row, n_blk * (BN / 2) + ch * 32, g, u, pol_out);
                }
            } else if constexpr (MODE == EPI_DOWN || MODE == EPI_RESID || MODE == EPI_STORE || MODE == EPI_ENCODE) {
                float* drow = nullptr;
                __nv_bfloat16* dbrow = nullptr;
                float* dsrow = nullptr;
                if (row < ep.M) {
                    // DOWN: destination row in the next block's layout, possibly on a peer GPU
                    // (NVLink); RESID: in place
                    int rank = 0;
                    i64 li = row;
                    float* xb = ep.x;
                    if constexpr (MODE == EPI_DOWN) {
                        li = ep.nxt.pix_to_loc(ep.cur.loc_to_pix(row), &rank);
                        xb = ep.xdst[rank];
                    }
                    drow = xb + li * ep.h;
                    if (ep.nss) {
                        dbrow = reinterpret_cast<__nv_bfloat16*>(xb + ep.off_xb) + li * ep.hp;
                        dsrow = xb + ep.off_ss + li * ep.nss;
                    }
                }
                constexpr int NCH = BN / 32;
                float ssum = 0.f;
#pragma unroll 1
                for (int ch = half * NCH / 2; ch < (half + 1) * NCH / 2; ++ch) {
                    float v[32];
                    tmem_ld32(tbase + ch * 32, v);
                    ssum += epi32_coalesced<MODE>(ep, row, n_blk * BN + ch * 32, v, stg, drow, dbrow, lane,
                                                  MODE == EPI_STORE ? ep.x + i64(bb) * ep.bst_c : ep.x);
                }
                if (dsrow) dsrow[2 * n_blk + half] = ssum;
            } else {
                constexpr int NCH = BN / 32;
                float ssum = 0.f;
#pragma unroll 1
                for (int ch = half * NCH / 2; ch < (half + 1) * NCH / 2; ++ch) {
                    float v[32];
                    tmem_ld32(tbase + ch * 32, v);
                    normed(v, n_blk * BN + ch * 32);
                    if constexpr (MODE == EPI_QKV)
                        epi_qkv32(ep, qr, n_blk * BN + ch * 32, v, stg, lane);
                    else if constexpr (MODE == EPI_SMAX || MODE == EPI_DSM)
                        epi_attn_rows32<MODE>(ep, row, n_blk * BN + ch * 32, v, stg, lane, bb);
                    else
                        ssum += epi32<MODE>(ep, row, n_blk * BN + ch * 32, v);
                }
                if constexpr (MODE == EPI_ENCODE)
                    if (ep.nss && row < ep.M) ep.x[ep.off_ss + row * ep.nss + 2 * n_blk + half] = ssum;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols));
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// per-device tile counter of the dynamic schedule for callers without a context (self-test); a
// context passes its own counter in EpiParams::sched, so contexts on one device may run concurrently
int* sched_counter() {
    static std::mutex mu;
    static int* ctr[64] = {};
    int dev = 0;
    SWF_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!ctr[dev]) SWF_CUDA(cudaMalloc(&ctr[dev], 256));
    return ctr[dev];
}

template <int BN, int MODE, int MN = 0>
void launch(const TmaMap& A, const TmaMap& B, i64 M, int Npad, int K, const EpiParams& ep, cudaStream_t st) {
    using C = Cfg<BN, uses_stg(MODE)>;
    auto kern = k_gemm_tc<BN, MODE, MN>;  // shared-memory limit set per device by preload_gemm_kernels
    const int n_tiles = Npad / BN;
    const i64 m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const i64 total = m_tiles * n_tiles * std::max(1, ep.nbatch);  // plane-batched launches: all problems
    int sms = 148;
    int clusters = int(std::min<i64>(total, sms / 2));
    // Rounds of the static schedule (tile t on cluster t mod clusters) cover whole M blocks when the
    // cluster count is a multiple of the N-tile count: the clusters sharing an A row block then stream
    // it in lock step and it is fetched from DRAM once, instead of straddling two rounds.
    static const bool align = getenv("SWF_GEMM_NOALIGN") == nullptr;
    if (align && n_tiles <= clusters && total > clusters) clusters = (clusters / n_tiles) * n_tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * clusters));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cfg.attrs = nullptr;  // cluster shape (2,1,1) comes from __cluster_dims__
    cfg.numAttrs = 0;
    const CUtensorMap* a = reinterpret_cast<const CUtensorMap*>(&A);
    const CUtensorMap* b = reinterpret_cast<const CUtensorMap*>(&B);
    int* sched = nullptr;
    // SWF_GEMM_STATIC=1: static round-robin schedule for every GEMM; SWF_GEMM_STATIC_MASK=bits: for the
    // epilogue modes whose bit is set (A/B knobs)
    static const bool all_static = getenv("SWF_GEMM_STATIC") != nullptr;
    static const int static_mask = getenv("SWF_GEMM_STATIC_MASK") ? atoi(getenv("SWF_GEMM_STATIC_MASK")) : 0;
    const bool dynamic = !all_static && !((static_mask >> MODE) & 1);
    if (dynamic) {
        sched = ep.sched ? ep.sched : sched_counter();
        SWF_CUDA(cudaMemsetAsync(sched, 0, sizeof(int), st));
    }
    static const int env_gm = getenv("SWF_GEMM_GROUPM") ? std::max(1, atoi(getenv("SWF_GEMM_GROUPM"))) : 0;
    const int group_m = env_gm ? env_gm : 1;
    SWF_CUDA(cudaLaunchKernelEx(&cfg, kern, *a, *b, M, n_tiles, K / BK, ep, sched, group_m));
#ifdef SWF_GEMM_TRACE
    if (const char* path = getenv("SWF_GEMM_TRACE_OUT")) {  // appends: mode, then the five rows
        static unsigned long long h[5][kGTr];
        SWF_CUDA(cudaStreamSynchronize(st));
        SWF_CUDA(cudaMemcpyFromSymbol(h, g_gtrace, sizeof(h)));
        if (FILE* f = fopen(path, "ab")) {
            const unsigned long long tag = (unsigned long long)(MODE * 1000 + BN);
            fwrite(&tag, 8, 1, f);
            fwrite(h, sizeof(h), 1, f);
            fclose(f);
        }
        SWF_CUDA(cudaMemset(g_gtrace_ptr(), 0, sizeof(h)));
    }
#endif
}

template <int BN>
void dispatch(const TmaMap& A, const TmaMap& B, i64 M, int Npad, int K, int mode, const EpiParams& ep,
              cudaStream_t st) {
    switch (mode) {
        case EPI_ENCODE: launch<BN, EPI_ENCODE>(A, B, M, Npad, K, ep, st); break;
        case EPI_QKV: launch<BN, EPI_QKV>(A, B, M, Npad, K, ep, st); break;
        case EPI_RESID: launch<BN, EPI_RESID>(A, B, M, Npad, K, ep, st); break;
        case EPI_SWIGLU: launch<BN, EPI_SWIGLU>(A, B, M, Npad, K, ep, st); break;
        case EPI_DOWN: launch<BN, EPI_DOWN>(A, B, M, Npad, K, ep, st); break;
        case EPI_DECODE: launch<BN, EPI_DECODE>(A, B, M, Npad, K, ep, st); break;
        default: throw CudaError("gemm_bf16_tc: bad epilogue mode");
    }
}

}  // namespace

void make_tma_bf16(TmaMap* m, const void* base, i64 rows, i64 kcols, int box_rows) {
    static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "TmaMap size");
    if (kcols % BK != 0) throw CudaError("make_tma_bf16: K must be a multiple of 64");
    cuuint64_t dims[2] = {cuuint64_t(kcols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(kcols) * 2};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(m), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

void make_tma_bf16_2d(TmaMap* m, const void* base, i64 rows, i64 inner, int box_inner, int box_rows, int swizzle) {
    if ((inner * 2) % 16 != 0) throw CudaError("make_tma_bf16_2d: row pitch must be a multiple of 16 bytes");
    cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(inner) * 2};
    cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                  : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(m), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (2d) failed: " + std::to_string(int(r)));
}

template <int BN>
void preload_bn(cudaFuncAttributes& a) {
    auto set = [&](const void* f, int smem) {
        SWF_CUDA(cudaFuncGetAttributes(&a, f));
        SWF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    };
    constexpr int kS = Cfg<BN, true>::kSmem, kN = Cfg<BN, false>::kSmem;
    set((const void*)k_gemm_tc<BN, EPI_ENCODE>, kS);
    set((const void*)k_gemm_tc<BN, EPI_QKV>, kS);
    set((const void*)k_gemm_tc<BN, EPI_SWIGLU>, kN);
    set((const void*)k_gemm_tc<BN, EPI_DECODE>, kS);
    set((const void*)k_gemm_tc<BN, EPI_RESID>, kS);
    set((const void*)k_gemm_tc<BN, EPI_DOWN>, kS);
    set((const void*)k_gemm_tc<BN, EPI_RESID, 3>, kS);
    set((const void*)k_gemm_tc<BN, EPI_RESID, 2>, kS);
    set((const void*)k_gemm_tc<BN, EPI_STORE, 0>, kS);
    set((const void*)k_gemm_tc<BN, EPI_STORE, 3>, kS);
    set((const void*)k_gemm_tc<BN, EPI_STORE, 2>, kS);
    if constexpr (BN == 256) {
        set((const void*)k_gemm_tc<BN, EPI_SMAX, 0>, kS);
        set((const void*)k_gemm_tc<BN, EPI_DSM, 0>, kS);
    }
}
void preload_gemm_kernels() {
    cudaFuncAttributes a;
    preload_bn<128>(a);
    preload_bn<256>(a);
}

// bf16 [rows][inner] operand with row pitch `pitch` elements, box {64, box_rows}, 128-byte swizzle;
// reads beyond `inner` / `rows` are zero filled (K and MN tails)
void make_tma_bf16_pitch(TmaMap* m, const void* base, i64 rows, i64 inner, i64 pitch, int box_rows) {
    if ((pitch * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        throw CudaError("make_tma_bf16_pitch: row pitch and base must be 16-byte aligned");
    cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(pitch) * 2};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(m), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (pitch) failed: " + std::to_string(int(r)));
}

template <int MODE>
void general_launch(int BN, int mn, const TmaMap& ta, const TmaMap& tb, i64 M, int Np, int Kp, const EpiParams& ep,
                    cudaStream_t st) {
    if (BN == 256) {
        if (mn == 3) launch<256, MODE, 3>(ta, tb, M, Np, Kp, ep, st);
        else if (mn == 2) launch<256, MODE, 2>(ta, tb, M, Np, Kp, ep, st);
        else launch<256, MODE, 0>(ta, tb, M, Np, Kp, ep, st);
    } else {
        if (mn == 3) launch<128, MODE, 3>(ta, tb, M, Np, Kp, ep, st);
        else if (mn == 2) launch<128, MODE, 2>(ta, tb, M, Np, Kp, ep, st);
        else launch<128, MODE, 0>(ta, tb, M, Np, Kp, ep, st);
    }
}

void gemm_bf16_general(const __nv_bfloat16* A, bool a_mn, i64 lda, const __nv_bfloat16* B, bool b_mn, i64 ldb, i64 M,
                       i64 N, i64 K, float* C, i64 ldc, bool accumulate, int* sched, cudaStream_t st) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    if (a_mn && !b_mn) throw CudaError("gemm_bf16_general: A MN-major with B K-major is not instantiated");

    const int BN = N > 128 ? 256 : 128;
    TmaMap ta, tb;
    if (a_mn)
        make_tma_bf16_pitch(&ta, A, K, M, lda, BK);
    else
        make_tma_bf16_pitch(&ta, A, M, K, lda, BM);
    if (b_mn)
        make_tma_bf16_pitch(&tb, B, K, N, ldb, BK);
    else
        make_tma_bf16_pitch(&tb, B, N, K, ldb, BN / 2);
    EpiParams ep;
    std::memset(&ep, 0, sizeof ep);
    ep.M = M;
    ep.N = int(N);
    ep.x = C;
    ep.h = int(ldc);
    ep.out_scale = 1.f;
    ep.sched = sched;
    const int Kp = int((K + BK - 1) / BK * BK);
    const int Np = int((N + BN - 1) / BN * BN);
    const int mn = (a_mn ? 1 : 0) | (b_mn ? 2 : 0);
    if (accumulate)
        general_launch<EPI_RESID>(BN, mn, ta, tb, M, Np, Kp, ep, st);
    else
        general_launch<EPI_STORE>(BN, mn, ta, tb, M, Np, Kp, ep, st);
}

void gemm_bf16_batched(const __nv_bfloat16* A, bool a_mn, i64 lda, i64 a_rows, i64 a_inner, const __nv_bfloat16* B,
                       bool b_mn, i64 ldb, i64 b_rows, i64 b_inner, i64 M, i64 N, i64 K, float* C, i64 ldc, int nbatch,
                       int adx, int ady, int bdx, int bdy, i64 bst_c, int* sched, cudaStream_t st) {
    if (M <= 0 || N <= 0 || K <= 0 || nbatch <= 0) return;
    if (a_mn && !b_mn) throw CudaError("gemm_bf16_batched: A MN-major with B K-major is not instantiated");
    const int BN = N > 128 ? 256 : 128;
    TmaMap ta, tb;
    make_tma_bf16_pitch(&ta, A, a_rows, a_inner, lda, a_mn ? BK : BM);
    make_tma_bf16_pitch(&tb, B, b_rows, b_inner, ldb, b_mn ? BK : BN / 2);
    EpiParams ep;
    std::memset(&ep, 0, sizeof ep);
    ep.M = M;
    ep.N = int(N);
    ep.x = C;
    ep.h = int(ldc);
    ep.out_scale = 1.f;
    ep.sched = sched;
    ep.nbatch = nbatch;
    ep.adx = adx;
    ep.ady = ady;
    ep.bdx = bdx;
    ep.bdy = bdy;
    ep.bst_c = bst_c;
    const int Kp = int((K + BK - 1) / BK * BK);
    const int Np = int((N + BN - 1) / BN * BN);
    general_launch<EPI_STORE>(BN, (a_mn ? 1 : 0) | (b_mn ? 2 : 0), ta, tb, M, Np, Kp, ep, st);
}

void gemm_bf16_attn_rows(int mode, const __nv_bfloat16* A, i64 lda, const __nv_bfloat16* B, i64 ldb, int s, int K,
                         __nv_bfloat16* out, int ldo, const float* rowv, const __nv_bfloat16* pin, int split,
                         int masked, float scale, int* sched, cudaStream_t st, int nbatch, i64 a_rows_b,
                         int a_col_b, i64 b_rows_b, i64 bst_out) {
    if (s <= 0 || K <= 0) return;
    if (s % 8 != 0) throw CudaError("gemm_bf16_attn_rows: s must be a multiple of 8");
    nbatch = std::max(1, nbatch);
    TmaMap ta, tb;
    // K-major operands: A [rows][K (+ a_col_b per problem)], B [rows][K]; maps over all problems
    make_tma_bf16_pitch(&ta, A, nbatch > 1 && a_rows_b ? (nbatch - 1) * a_rows_b + s : s,
                        K + i64(nbatch - 1) * a_col_b, lda, BM);
    make_tma_bf16_pitch(&tb, B, nbatch > 1 ? (nbatch - 1) * b_rows_b + s : s, K, ldb, 128);
    EpiParams ep;
    std::memset(&ep, 0, sizeof ep);
    ep.nbatch = nbatch;
    ep.adx = a_col_b;
    ep.ady = int(a_rows_b);
    ep.bdy = int(b_rows_b);
    ep.bst_c = bst_out;
    ep.bst_p = bst_out;
    ep.bst_rv = s;
    ep.M = s;
    ep.N = s;
    ep.out = out;
    ep.ld_out = ldo;
    ep.out_scale = scale;
    ep.rowv = rowv;
    ep.pin = pin;
    ep.split = split;
    ep.masked = masked;
    ep.sched = sched;
    const int Kp = (K + BK - 1) / BK * BK, Np = (s + 255) / 256 * 256;
    if (mode == EPI_SMAX)
        launch<256, EPI_SMAX, 0>(ta, tb, s, Np, Kp, ep, st);
    else if (mode == EPI_DSM)
        launch<256, EPI_DSM, 0>(ta, tb, s, Np, Kp, ep, st);
    else
        throw CudaError("gemm_bf16_attn_rows: bad mode");
}

void gemm_bf16_tc(const TmaMap& A, const TmaMap& B, i64 M, int Npad, int K, int BN, int mode, const EpiParams& ep,
                  cudaStream_t st) {
    if (K % BK != 0) throw CudaError("gemm_bf16_tc: K must be a multiple of 64");
    if (Npad % BN != 0) throw CudaError("gemm_bf16_tc: N must be a multiple of the N tile");
    if (BN == 256)
        dispatch<256>(A, B, M, Npad, K, mode, ep, st);
    else if (BN == 128)
        dispatch<128>(A, B, M, Npad, K, mode, ep, st);
    else
        throw CudaError("gemm_bf16_tc: BN must be 128 or 256");
}

}  // namespace swf

// ====================================================================== self-test (C-ABI)
namespace {
using swf::i64;
__global__ void k_fill_bf16(__nv_bfloat16* p, i64 n, uint64_t seed, float* f32) {
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
        uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (i + 1);
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        x ^= x >> 31;
        const float v = (float((x >> 40) & 0xFFFF) / 65536.0f - 0.5f) * 2.0f;
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        p[i] = b;
        f32[i] = __bfloat162float(b);
    }
}
__global__ void k_maxdiff(const float* a, const float* b, i64 n, float* out) {
    float md = 0.f, mr = 0.f;
    for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
        md = fmaxf(md, fabsf(a[i] - b[i]));
        mr = fmaxf(mr, fabsf(b[i]));
    }
    atomicMax(reinterpret_cast<int*>(out), __float_as_int(md));
    atomicMax(reinterpret_cast<int*>(out + 1), __float_as_int(mr));
}
}  // namespace

extern "C" int swf_selftest_gemm(int device, long long M, int N, int K, double* max_abs_err, double* max_ref) {
    using namespace swf;
    try {
        SWF_CUDA(cudaSetDevice(device));
        ensure_device(device);
        if (N % 128 != 0 || K % 64 != 0) throw CudaError("selftest: N % 128 and K % 64 required");
        __nv_bfloat16 *A, *B;
        float *Af, *Bf, *C1, *C2, *bias, *res;
        SWF_CUDA(cudaMalloc(&A, size_t(M) * K * 2));
        SWF_CUDA(cudaMalloc(&B, size_t(N) * K * 2));
        SWF_CUDA(cudaMalloc(&Af, size_t(M) * K * 4));
        SWF_CUDA(cudaMalloc(&Bf, size_t(N) * K * 4));
        SWF_CUDA(cudaMalloc(&C1, size_t(M) * N * 4));
        SWF_CUDA(cudaMalloc(&C2, size_t(M) * N * 4));
        SWF_CUDA(cudaMalloc(&bias, size_t(N) * 4));
        SWF_CUDA(cudaMalloc(&res, 8));
        SWF_CUDA(cudaMemset(bias, 0, size_t(N) * 4));
        SWF_CUDA(cudaMemset(res, 0, 8));
        SWF_CUDA(cudaMemset(C1, 0xff, size_t(M) * N * 4));
        k_fill_bf16<<<1024, 256>>>(A, M * K, 1, Af);
        k_fill_bf16<<<1024, 256>>>(B, i64(N) * K, 2, Bf);
        SWF_LAUNCH_CHECK();
        TmaMap ta, tb;
        const int BN = (N % 256 == 0) ? 256 : 128;
        make_tma_bf16(&ta, A, M, K, 128);
        make_tma_bf16(&tb, B, N, K, BN / 2);
        EpiParams ep;
        memset(&ep, 0, sizeof ep);
        ep.M = M;
        ep.N = N;
        ep.h = N;
        ep.x = C1;
        ep.bias = bias;
        gemm_bf16_tc(ta, tb, M, N, K, BN, EPI_ENCODE, ep, 0);
        ep.x = C2;
        gemm_f32(Af, Bf, M, N, K, EPI_ENCODE, ep, 0);
        k_maxdiff<<<1024, 256>>>(C1, C2, M * N, res);
        float h[2];
        SWF_CUDA(cudaMemcpy(h, res, 8, cudaMemcpyDeviceToHost));
        *max_abs_err = h[0];
        *max_ref = h[1];
        for (void* p : {(void*)A, (void*)B, (void*)Af, (void*)Bf, (void*)C1, (void*)C2, (void*)bias, (void*)res})
            cudaFree(p);
        return 0;
    } catch (const std::exception& e) {
        fprintf(stderr, "swf_selftest_gemm: %s\n", e.what());
        return SWF_ERR_CUDA;
    }
}
