// k_attn.cu -- BF16 windowed attention on the 5th-generation tensor cores (sm_100a).
//
// Persistent CTAs; a work item is one 128-query tile of one (window, head). Restates
// head_attention_fwd (swin.hpp:161-188) without materialising the s x s logits:
//   * S = Q K^T : tcgen05.mma (M=128, N=128 keys, K=d), A = Q and B = K, K-major SW128 shared-
//     memory tiles loaded by TMA; FP32 S in TMEM, double-buffered (S0 / S1) so the QK^T of key
//     tile j+1 runs while the softmax warps work on tile j;
//   * softmax: one thread per query row (TMEM lane), base-2 online max/sum with lazy O rescaling
//     (only when the running max grows by > 2^8), packed f32x2 arithmetic for the exponent
//     arguments and the row sum, 3/8 of the exponentials on the FMA pipe (degree-3 polynomial)
//     and 5/8 on MUFU; P is packed to BF16 and written back into its S buffer's columns;
//   * O += P V : tcgen05.mma with A = P read from TMEM and B = V^T (K-major, written transposed by
//     the QKV GEMM epilogue); O accumulates in TMEM;
//   * the latitude-seam mask (window.hpp:107-122) is a per-row key range: the two seam groups are
//     the contiguous token ranges [0, (w-shift)*w) and [(w-shift)*w, w*w); fully-outside key tiles
//     are skipped and only boundary tiles pay per-element masking.
// Warp roles: w0 TMA producer (Q double buffer, 3-stage K ring), w3 TMA producer (2-stage V^T
// ring), w1 MMA issuer, w2 TMEM allocator, w4-w7 softmax + epilogue.
// TMEM: S0 [0,128) S1 [128,256) O [256,256+D).
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace swf {

namespace {

using namespace tc;

constexpr int BQ = 128;   // queries per work item (= UMMA M, = TMEM lanes)
constexpr int BKV = 128;  // keys per tile
constexpr int kThreads = 256;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)

template <int D>
struct ACfg {
    static constexpr int kSw = D >= 64 ? 128 : 2 * D;  // swizzle bytes of Q/K rows (d contiguous)
    static constexpr int kColsPerBox = kSw / 2;         // d elements per TMA box row
    static constexpr int kBoxes = D / kColsPerBox;      // boxes along d
    static constexpr int kQBytes = BQ * D * 2;
    static constexpr int kKBytes = BKV * D * 2;
    static constexpr int kVBytes = D * BKV * 2;         // V^T tile: D rows x 128 keys (two SW128 boxes)
    static constexpr int kNK = 3, kNV = 2;
    static constexpr int kSmem = 2 * kQBytes + kNK * kKBytes + kNV * kVBytes + 1024 + 256;
    static constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV);
    static constexpr uint32_t kIdescO = idesc_bf16(BQ, D);
};

// barrier slots (u64 each)
enum : int {
    B_QF = 0, B_QE = 2, B_KF = 4, B_KE = 7, B_VF = 10, B_VE = 12, B_SF = 14, B_SE = 16, B_PF = 18, B_OD = 20,
    B_OF = 21, B_NUM = 22
};

// Work item -> (q tile, head, local window); items of one (window, head) are consecutive so the
// concurrently running CTAs share K / V^T tiles through L2.
struct Item {
    int q0, head, lw;
};
__device__ __forceinline__ Item item_of(int it, int nqt, int heads) {
    Item r;
    const int qt = it % nqt;
    const int hw = it / nqt;
    r.q0 = qt * BQ;
    r.head = hw % heads;
    r.lw = hw / heads;
    return r;
}

// key range of a work item (seam groups)
struct Range {
    int split, t_lo, ntiles;
    bool masked;
};
__device__ __forceinline__ Range range_of(const AttnParams& p, const Item& it) {
    Range r;
    const int s = p.s;
    const int gw = p.lay.loc2glob[it.lw];
    r.masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;
    r.split = r.masked ? (p.w - p.lay.g.shift) * p.w : s;
    const int qlast = min(it.q0 + BQ, s) - 1;
    const int kv_lo = (r.masked && it.q0 >= r.split) ? r.split : 0;
    const int kv_hi = (r.masked && qlast < r.split) ? r.split : s;
    r.t_lo = kv_lo / BKV;
    r.ntiles = (kv_hi + BKV - 1) / BKV - r.t_lo;
    return r;
}

__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float lo_f(unsigned long long v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float hi_f(unsigned long long v) { return __uint_as_float(uint32_t(v >> 32)); }

// 2^z for two packed values on the FMA pipe (see tc::ex2_poly)
__device__ __forceinline__ unsigned long long ex2_poly2(unsigned long long z) {
    const unsigned long long magic = f2_pack(12582912.0f, 12582912.0f);
    const unsigned long long nmagic = f2_pack(-12582912.0f, -12582912.0f);
    z = f2_pack(fmaxf(lo_f(z), -126.f), fmaxf(hi_f(z), -126.f));
    const unsigned long long t = fadd2(z, magic);
    const unsigned long long fi = fadd2(t, nmagic);
    const unsigned long long f = fadd2(z, fi ^ 0x8000000080000000ull);  // z - fi
    unsigned long long q = ffma2(f2_pack(0.05500815f, 0.05500815f), f, f2_pack(0.24220921f, 0.24220921f));
    q = ffma2(q, f, f2_pack(0.69328305f, 0.69328305f));
    q = ffma2(q, f, f2_pack(1.f, 1.f));
    const uint32_t lo = uint32_t(q) + (uint32_t(t) << 23);
    const uint32_t hi = uint32_t(q >> 32) + (uint32_t(t >> 32) << 23);
    return (unsigned long long)lo | ((unsigned long long)hi << 32);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnParams p, int n_items) {
    using C = ACfg<D>;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                        // [2][BQ x D]
    uint8_t* sK = sm + 2 * C::kQBytes;       // [kNK][BKV x D]
    uint8_t* sV = sK + C::kNK * C::kKBytes;  // [kNV][D x BKV] (V^T)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kNV * C::kVBytes);
    auto bar = [&](int slot) { return smem_u32(&bars[slot]); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[B_NUM]);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int nqt = (s + BQ - 1) / BQ;

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar(B_QF + i), 1);
            mbar_init(bar(B_QE + i), 1);
            mbar_init(bar(B_VF + i), 1);
            mbar_init(bar(B_VE + i), 1);
            mbar_init(bar(B_SF + i), 1);
            mbar_init(bar(B_SE + i), 1);
            mbar_init(bar(B_PF + i), 4);
        }
        for (int i = 0; i < C::kNK; ++i) {
            mbar_init(bar(B_KF + i), 1);
            mbar_init(bar(B_KE + i), 1);
        }
        mbar_init(bar(B_OD), 1);
        mbar_init(bar(B_OF), 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer 1: Q (double-buffered across work items) and the K ring
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
            int g = 0, n = 0;
            for (int itx = blockIdx.x; itx < n_items; itx += gridDim.x, ++n) {
                const Item it = item_of(itx, nqt, p.heads);
                const Range rg = range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                const int qb = n & 1;
                mbar_wait(bar(B_QE + qb), ((n >> 1) & 1) ^ 1);
                mbar_expect_tx(bar(B_QF + qb), C::kQBytes);
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2d(smem_u32(sQ + qb * C::kQBytes + b * BQ * C::kSw), &tmQ, bar(B_QF + qb),
                                b * C::kColsPerBox, plane * s + it.q0);
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g % C::kNK;
                    mbar_wait(bar(B_KE + st), ((g / C::kNK) & 1) ^ 1);
                    mbar_expect_tx(bar(B_KF + st), C::kKBytes);
                    for (int b = 0; b < C::kBoxes; ++b)
                        tma_load_2d(smem_u32(sK + st * C::kKBytes + b * BKV * C::kSw), &tmK, bar(B_KF + st),
                                    b * C::kColsPerBox, plane * s + (rg.t_lo + j) * BKV);
                }
            }
        }
    } else if (warp == 3) {
        // ===== TMA producer 2: the V^T ring (D rows x 64 keys per box)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
            int g = 0;
            for (int itx = blockIdx.x; itx < n_items; itx += gridDim.x) {
                const Item it = item_of(itx, nqt, p.heads);
                const Range rg = range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g & 1;
                    mbar_wait(bar(B_VE + st), ((g >> 1) & 1) ^ 1);
                    mbar_expect_tx(bar(B_VF + st), C::kVBytes);
                    for (int b = 0; b < 2; ++b)
                        tma_load_2d(smem_u32(sV + st * C::kVBytes + b * D * 128), &tmV, bar(B_VF + st),
                                    (rg.t_lo + j) * BKV + b * 64, plane * D);
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: S(g) is issued before PV(g-1), so QK^T of the next key tile overlaps the
        // softmax of the current one; tensor-pipe order guarantees PV(g-2) read P before S(g) lands
        // in the same buffer (s_free is committed after that PV).
        if (lane == 0) {
            int g = 0, n = 0;
            auto issue_pv = [&](int gg, bool first) {
                const int b = gg & 1;
                mbar_wait(bar(B_PF + b), (gg >> 1) & 1);
                mbar_wait(bar(B_VF + b), (gg >> 1) & 1);
                fence_after();
                const uint8_t* vt = sV + b * C::kVBytes;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    const uint64_t bd = desc_kmajor(smem_u32(vt + (kk >> 2) * D * 128 + (kk & 3) * 32), 128);
                    mma_ts(tmem + 256u, tmem + uint32_t(b * 128 + kk * 8), bd, C::kIdescO,
                           (!first || kk > 0) ? 1u : 0u);
                }
                commit(bar(B_OD));
                commit(bar(B_VE + b));
                commit(bar(B_SE + b));
            };
            for (int itx = blockIdx.x; itx < n_items; itx += gridDim.x, ++n) {
                const Item it = item_of(itx, nqt, p.heads);
                const Range rg = range_of(p, it);
                const int qb = n & 1;
                mbar_wait(bar(B_QF + qb), (n >> 1) & 1);
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int b = g & 1, st = g % C::kNK;
                    mbar_wait(bar(B_KF + st), (g / C::kNK) & 1);
                    if (g >= 2) mbar_wait(bar(B_SE + b), ((g >> 1) + 1) & 1);
                    fence_after();
                    const uint8_t* kt = sK + st * C::kKBytes;
                    const uint8_t* qt = sQ + qb * C::kQBytes;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const int box = (kk * 32) / C::kSw, off = (kk * 32) % C::kSw;
                        const uint64_t a = desc_kmajor(smem_u32(qt + box * BQ * C::kSw + off), C::kSw);
                        const uint64_t bd = desc_kmajor(smem_u32(kt + box * BKV * C::kSw + off), C::kSw);
                        mma_ss(tmem + uint32_t(b * 128), a, bd, C::kIdescS, kk > 0 ? 1u : 0u);
                    }
                    commit(bar(B_SF + b));
                    commit(bar(B_KE + st));
                    if (j + 1 == rg.ntiles) commit(bar(B_QE + qb));  // Q of this item no longer read
                    if (j >= 1) {
                        if (j == 1 && n >= 1) mbar_wait(bar(B_OF), (n - 1) & 1);  // O of the last item read out
                        issue_pv(g - 1, j == 1);
                    }
                }
                if (rg.ntiles == 1 && n >= 1) mbar_wait(bar(B_OF), (n - 1) & 1);
                issue_pv(g - 1, rg.ntiles == 1);
            }
        }
    } else if (warp >= 4) {
        // ===== softmax (one thread per query row) + epilogue
        const int wq = warp - 4;  // TMEM lane quadrant (warp % 4)
        const int r = wq * 32 + lane;
        const uint32_t lane_off = uint32_t(wq * 32) << 16;
        const uint32_t tO = tmem + lane_off + 256u;
        const float sl2 = p.scale * 1.4426950408889634f;
        int g = 0;
        for (int itx = blockIdx.x; itx < n_items; itx += gridDim.x) {
            const Item it = item_of(itx, nqt, p.heads);
            const Range rg = range_of(p, it);
            const int q = it.q0 + r;
            const int rlo = (rg.masked && q >= rg.split) ? rg.split : 0;
            const int rhi = (rg.masked && q < rg.split) ? rg.split : s;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int b = g & 1;
                const uint32_t tS = tmem + lane_off + uint32_t(b * 128);
                mbar_wait(bar(B_SF + b), (g >> 1) & 1);
                fence_after();
                uint32_t sr[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) ld32(tS + uint32_t(c * 32), sr + 32 * c);
#pragma unroll
                for (int c = 0; c < 4; ++c) wait_ld_dep(sr + 32 * c);
                const int kb = (rg.t_lo + j) * BKV;
                if (kb < rlo || kb + BKV > rhi) {  // boundary tile: mask keys outside [rlo, rhi)
#pragma unroll
                    for (int i = 0; i < 128; ++i)
                        if (kb + i < rlo || kb + i >= rhi) sr[i] = __float_as_uint(-INFINITY);
                }
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < 128; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sr[i]));
                const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
                if (mx > m + kRescale || (m == -INFINITY && mx != -INFINITY)) {
                    if (m != -INFINITY) {
                        // O *= 2^(m - mx): the PV of the previous key tile must have landed
                        mbar_wait(bar(B_OD), (g - 1) & 1);
                        fence_after();
                        const float f = ex2(m - mx);
#pragma unroll 1
                        for (int c = 0; c < D / 32; ++c) {
                            uint32_t o[32];
                            ld32(tO + uint32_t(c * 32), o);
                            wait_ld_dep(o);
#pragma unroll
                            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                            st32(tO + uint32_t(c * 32), o);
                        }
                        wait_st();
                        l *= f;
                    }
                    m = mx;
                }
                const float nb = m == -INFINITY ? 0.f : -m;
                const unsigned long long sl2x2 = f2_pack(sl2, sl2), nbx2 = f2_pack(nb, nb);
                unsigned long long ls2 = 0ull, ls2b = 0ull;
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed bf16x2 columns per store
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const unsigned long long sv =
                            (unsigned long long)sr[32 * c + 2 * i] | ((unsigned long long)sr[32 * c + 2 * i + 1] << 32);
                        const unsigned long long z = ffma2(sv, sl2x2, nbx2);
                        unsigned long long pv;
                        if ((i & 7) < 3)  // 3/8 of the exponentials on the FMA pipe
                            pv = ex2_poly2(z);
                        else
                            pv = f2_pack(ex2(lo_f(z)), ex2(hi_f(z)));
                        if (i & 1)
                            ls2b = fadd2(ls2b, pv);
                        else
                            ls2 = fadd2(ls2, pv);
                        pk[i] = pack_bf16x2(lo_f(pv), hi_f(pv));
                    }
                    st16(tS + uint32_t(16 * c), pk);
                }
                const unsigned long long lsum = fadd2(ls2, ls2b);
                l += lo_f(lsum) + hi_f(lsum);
                wait_st();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar(B_PF + b));
            }
            // epilogue: O / l -> bf16 rows to the token owner (its SP band; this rank when sp == 1),
            // head columns of the global head index (swin.hpp:319-320 concat)
            mbar_wait(bar(B_OD), (g - 1) & 1);
            fence_after();
            const float inv = 1.f / l;
            int orank = 0;
            const i64 oloc = q < s ? p.lay.wtok_to_loc(p.wp_rank, it.lw, q, &orank) : 0;
            __nv_bfloat16* O =
                reinterpret_cast<__nv_bfloat16*>(p.o_dst[orank]) + oloc * p.ldo + (p.head0 + it.head) * D;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                ld32(tO + uint32_t(c * 32), o);
                wait_ld_dep(o);
                if (q < s) {
                    uint4* d4 = reinterpret_cast<uint4*>(O + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        d4[v] = make_uint4(
                            pack_bf16x2(__uint_as_float(o[8 * v]) * inv, __uint_as_float(o[8 * v + 1]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv));
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(B_OF));  // O may be overwritten by the next item's first PV
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        tmem_free(tmem, 512);
    }
}

template <int D>
void launch(const AttnParams& p, cudaStream_t st) {
    using C = ACfg<D>;
    static bool configured = false;
    if (!configured) {
        SWF_CUDA(cudaFuncSetAttribute(k_attn_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        configured = true;
    }
    const int nqt = (p.s + BQ - 1) / BQ;
    const int n_items = nqt * p.heads * p.nloc;
    const int grid = std::min(n_items, 148);
    k_attn_tc<D><<<grid, kThreads, C::kSmem, st>>>(*reinterpret_cast<const CUtensorMap*>(p.tmq),
                                                  *reinterpret_cast<const CUtensorMap*>(p.tmk),
                                                  *reinterpret_cast<const CUtensorMap*>(p.tmv), p, n_items);
    SWF_LAUNCH_CHECK();
}

}  // namespace

void attention_bf16(const AttnParams& p, cudaStream_t st) {
    if (!p.tmq || !p.tmk || !p.tmv) throw CudaError("attention_bf16: TMA descriptors missing");
    switch (p.d) {
        case 32: launch<32>(p, st); break;
        case 64: launch<64>(p, st); break;
        case 128: launch<128>(p, st); break;
        default: throw CudaError("attention_bf16: head_dim must be 32, 64 or 128");
    }
}

}  // namespace swf
