// k_attn.cu -- BF16 windowed attention on the 5th-generation tensor cores (sm_100a).
//
// One CTA per (window, head, 128-query tile). Restates head_attention_fwd (swin.hpp:161-188)
// without materialising the s x s logits:
//   * S = Q K^T : tcgen05.mma (A = Q, B = K, both K-major SW128 smem tiles loaded by TMA),
//     FP32 accumulator in TMEM, double-buffered so QK^T of tile j+1 overlaps softmax of tile j;
//   * softmax: one thread per query row (TMEM lane), base-2 online max/sum, lazy O rescaling
//     (only when the running max grows by > 2^8), P packed to BF16 and written back to TMEM;
//   * O += P V : tcgen05.mma with the A operand (P) read from TMEM and B = V^T (K-major, written
//     transposed by the QKV GEMM epilogue), FP32 O accumulator in TMEM;
//   * the latitude-seam mask (window.hpp:107-122) is a per-query-tile KV range: the two seam
//     groups are the contiguous token ranges [0, (w-shift)*w) and [(w-shift)*w, w*w).
// Warp roles: w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4-w7 softmax + epilogue.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace swf {

namespace {

using namespace tc;

constexpr int BQ = 128;   // queries per CTA (= UMMA M, = TMEM lanes)
constexpr int BKV = 128;  // keys per tile
constexpr int kThreads = 256;
constexpr int kSoftWarp0 = 4;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)

template <int D>
struct ACfg {
    static constexpr int kSw = D >= 64 ? 128 : 2 * D;    // swizzle bytes of Q/K rows (d contiguous)
    static constexpr int kColsPerBox = kSw / 2;           // d elements per TMA box row
    static constexpr int kBoxes = D / kColsPerBox;        // boxes along d
    static constexpr int kQBytes = BQ * D * 2;
    static constexpr int kKBytes = BKV * D * 2;
    static constexpr int kVBytes = D * BKV * 2;           // V^T tile: D rows x 128 keys (two SW128 boxes)
    static constexpr int kStage = kKBytes + kVBytes;
    static constexpr int kSmem = kQBytes + 2 * kStage + 1024 + 256;
    static constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV);
    static constexpr uint32_t kIdescO = idesc_bf16(BQ, D);
    static constexpr uint32_t kTmemCols = 512;  // S0 [0,128) S1 [128,256) O [256, 256+D)
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    using C = ACfg<D>;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sKV = sm + C::kQBytes;  // [2][K tile | V^T tile]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::kQBytes + 2 * C::kStage);
    const uint32_t q_full = smem_u32(&bars[0]);
    const uint32_t kv_full0 = smem_u32(&bars[1]), kv_empty0 = smem_u32(&bars[3]);
    const uint32_t s_full0 = smem_u32(&bars[5]), s_free0 = smem_u32(&bars[7]);
    const uint32_t p_full0 = smem_u32(&bars[9]), o_done = smem_u32(&bars[11]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[12]);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int q0 = blockIdx.x * BQ;
    const int head = blockIdx.y, lw = blockIdx.z;
    const int plane = lw * p.heads + head;

    // seam groups (window.hpp:58-65): only the last window row of a shifted layout is masked
    const int gw = p.lay.loc2glob[lw];
    const bool masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;
    const int split = masked ? (p.w - p.lay.g.shift) * p.w : s;
    const int qlast = min(q0 + BQ, s) - 1;
    int kv_lo = 0, kv_hi = s;
    bool elementwise = false;
    if (masked) {
        if (qlast < split)
            kv_hi = split;
        else if (q0 >= split)
            kv_lo = split;
        else
            elementwise = true;
    }
    const int t_lo = kv_lo / BKV, t_hi = (kv_hi + BKV - 1) / BKV;
    const int ntiles = t_hi - t_lo;

    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(kv_full0 + 8 * i, 1);
            mbar_init(kv_empty0 + 8 * i, 1);
            mbar_init(s_full0 + 8 * i, 1);
            mbar_init(s_free0 + 8 * i, 1);
            mbar_init(p_full0 + 8 * i, 4);
        }
        mbar_init(o_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tmem_slot), C::kTmemCols);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
            mbar_expect_tx(q_full, C::kQBytes);
            for (int b = 0; b < C::kBoxes; ++b)
                tma_load_2d(smem_u32(sQ + b * BQ * C::kSw), &tmQ, q_full, b * C::kColsPerBox, plane * s + q0);
            for (int j = 0; j < ntiles; ++j) {
                const int st = j & 1;
                const int k0 = (t_lo + j) * BKV;
                mbar_wait(kv_empty0 + 8 * st, ((j >> 1) & 1) ^ 1);
                const uint32_t bar = kv_full0 + 8 * st;
                mbar_expect_tx(bar, C::kStage);
                uint8_t* sK = sKV + st * C::kStage;
                uint8_t* sV = sK + C::kKBytes;
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2d(smem_u32(sK + b * BKV * C::kSw), &tmK, bar, b * C::kColsPerBox, plane * s + k0);
                for (int b = 0; b < 2; ++b)  // V^T: D rows x 64 keys per box
                    tma_load_2d(smem_u32(sV + b * D * 128), &tmV, bar, k0 + b * 64, plane * D);
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer
        if (lane == 0) {
            mbar_wait(q_full, 0);
            auto issue_pv = [&](int i) {
                const int b = i & 1;
                mbar_wait(p_full0 + 8 * b, (i >> 1) & 1);
                fence_after();
                const uint8_t* sV = sKV + b * C::kStage + C::kKBytes;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    const uint32_t bA = tmem + uint32_t(b * 128 + kk * 8);  // P: bf16 pairs in S buffer cols
                    const uint64_t bB = desc_kmajor(smem_u32(sV + (kk >> 2) * D * 128 + (kk & 3) * 32), 128);
                    mma_ts(tmem + 256, bA, bB, C::kIdescO, (i > 0 || kk > 0) ? 1u : 0u);
                }
                commit(o_done);
                commit(kv_empty0 + 8 * b);
                commit(s_free0 + 8 * b);
            };
            for (int j = 0; j < ntiles; ++j) {
                const int b = j & 1;
                mbar_wait(kv_full0 + 8 * b, (j >> 1) & 1);
                if (j >= 2) mbar_wait(s_free0 + 8 * b, ((j >> 1) - 1) & 1);
                fence_after();
                const uint8_t* sK = sKV + b * C::kStage;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const int box = (kk * 32) / C::kSw, off = (kk * 32) % C::kSw;
                    const uint64_t a = desc_kmajor(smem_u32(sQ + box * BQ * C::kSw + off), C::kSw);
                    const uint64_t bb = desc_kmajor(smem_u32(sK + box * BKV * C::kSw + off), C::kSw);
                    mma_ss(tmem + uint32_t(b * 128), a, bb, C::kIdescS, kk > 0 ? 1u : 0u);
                }
                commit(s_full0 + 8 * b);
                if (j >= 1) issue_pv(j - 1);
            }
            issue_pv(ntiles - 1);
        }
    } else if (warp >= kSoftWarp0) {
        // ===== softmax (one thread per query row) + epilogue
        const int r = (warp - kSoftWarp0) * 32 + lane;  // row in tile == TMEM lane
        const int q = q0 + r;
        const uint32_t lane_off = uint32_t((warp - kSoftWarp0) * 32) << 16;
        const int gq = q < split ? 0 : 1;
        const float sl2 = p.scale * 1.4426950408889634f;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < ntiles; ++j) {
            const int b = j & 1;
            mbar_wait(s_full0 + 8 * b, (j >> 1) & 1);
            fence_after();
            uint32_t sr[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) ld32(tmem + lane_off + uint32_t(b * 128 + c * 32), sr + 32 * c);
#pragma unroll
            for (int c = 0; c < 4; ++c) wait_ld_dep(sr + 32 * c);
            const int kb = (t_lo + j) * BKV;
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < 128; ++i) {
                const int key = kb + i;
                bool keep = key < kv_hi && key >= kv_lo;
                if (elementwise) keep = keep && ((key < split ? 0 : 1) == gq);
                const float z = keep ? __uint_as_float(sr[i]) * sl2 : -INFINITY;
                sr[i] = __float_as_uint(z);
                mx = fmaxf(mx, z);
            }
            if (mx > m + kRescale || (m == -INFINITY && mx != -INFINITY)) {
                if (m != -INFINITY && j > 0) {
                    // O *= 2^(m - mx): PV of the previous tile must have landed in TMEM
                    mbar_wait(o_done, (j - 1) & 1);
                    fence_after();
                    const float f = ex2(m - mx);
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        ld32(tmem + lane_off + uint32_t(256 + c * 32), o);
                        wait_ld_dep(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
                        st32(tmem + lane_off + uint32_t(256 + c * 32), o);
                    }
                    wait_st();
                    l *= f;
                }
                m = mx;
            }
            const float base = m == -INFINITY ? 0.f : m;
            uint32_t pk[64];
            float ls = 0.f;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                const float p0 = ex2(__uint_as_float(sr[2 * i]) - base);
                const float p1 = ex2(__uint_as_float(sr[2 * i + 1]) - base);
                ls += p0 + p1;
                pk[i] = pack_bf16x2(p0, p1);
            }
            l += ls;
            st32(tmem + lane_off + uint32_t(b * 128), pk);
            st32(tmem + lane_off + uint32_t(b * 128 + 32), pk + 32);
            wait_st();
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full0 + 8 * b);
        }
        // epilogue: O / l -> bf16, heads concatenated in token rows
        mbar_wait(o_done, (ntiles - 1) & 1);
        fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o) + (i64(lw) * s + q) * p.ldo + head * D;
        for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            ld32(tmem + lane_off + uint32_t(256 + c * 32), o);
            wait_ld_dep(o);
            if (q < s) {
                uint4* d4 = reinterpret_cast<uint4*>(O + c * 32);
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    d4[v] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * v]) * inv, __uint_as_float(o[8 * v + 1]) * inv),
                                       pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv),
                                       pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv),
                                       pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv));
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        tmem_free(tmem, C::kTmemCols);
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
    dim3 grid(unsigned((p.s + BQ - 1) / BQ), unsigned(p.heads), unsigned(p.nloc));
    k_attn_tc<D><<<grid, kThreads, C::kSmem, st>>>(*reinterpret_cast<const CUtensorMap*>(p.tmq),
                                                  *reinterpret_cast<const CUtensorMap*>(p.tmk),
                                                  *reinterpret_cast<const CUtensorMap*>(p.tmv), p);
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
