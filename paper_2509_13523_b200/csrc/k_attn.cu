// k_attn.cu -- BF16 windowed attention on the 5th-generation tensor cores (sm_100a).
//
// One CTA per (window, head, pair of 128-query tiles). Restates head_attention_fwd
// (swin.hpp:161-188) without materialising the s x s logits:
//   * S_h = Q_h K^T for the two query tiles h = 0, 1: tcgen05.mma (M=128, N=128 keys), A = Q_h and
//     B = K both K-major SW128 shared-memory tiles loaded by TMA; FP32 S_h in TMEM;
//   * two softmax warpgroups (one per query tile, one thread per query row = TMEM lane) ping-pong
//     against the single MMA-issuing thread: while warpgroup 0 exponentiates S_0 of key tile j the
//     tensor core runs P_1 V and S_1 of the next tile, and vice versa;
//   * base-2 online softmax with lazy O rescaling (only when the running max grows by > 2^8);
//     P is packed to BF16 and written back into the S_h columns of TMEM;
//   * O_h += P_h V : tcgen05.mma with A = P_h read from TMEM and B = V^T (K-major, written
//     transposed by the QKV GEMM epilogue); O_h accumulates in TMEM; K/V tiles are shared by both
//     query tiles (3-stage K ring freed after QK^T, 2-stage V^T ring freed after PV);
//   * the latitude-seam mask (window.hpp:107-122) is a per-row key range: the two seam groups are
//     the contiguous token ranges [0, (w-shift)*w) and [(w-shift)*w, w*w); fully-outside key tiles
//     are skipped and only boundary tiles pay per-element masking.
// Warp roles: w0 TMA producer (Q, K ring), w3 TMA producer (V^T ring), w1 MMA issuer, w2 TMEM allocator,
// w4-w7 softmax(q-tile 0),
// w8-w11 softmax(q-tile 1). TMEM: S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D).
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace swf {

namespace {

using namespace tc;

constexpr int BQ = 128;   // queries per tile (= UMMA M, = TMEM lanes)
constexpr int BKV = 128;  // keys per tile
constexpr int kThreads = 384;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)

template <int D>
struct ACfg {
    static constexpr int kSw = D >= 64 ? 128 : 2 * D;  // swizzle bytes of Q/K rows (d contiguous)
    static constexpr int kColsPerBox = kSw / 2;         // d elements per TMA box row
    static constexpr int kBoxes = D / kColsPerBox;      // boxes along d
    static constexpr int kQBytes = BQ * D * 2;          // one query tile
    static constexpr int kKBytes = BKV * D * 2;
    static constexpr int kVBytes = D * BKV * 2;         // V^T tile: D rows x 128 keys (two SW128 boxes)
    static constexpr int kNK = 3, kNV = 2;  // K ring (freed after QK^T) deeper than the V ring
    static constexpr int kSmem = 2 * kQBytes + kNK * kKBytes + kNV * kVBytes + 1024 + 256;
    static constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV);
    static constexpr uint32_t kIdescO = idesc_bf16(BQ, D);
};

// barrier slots (u64 each)
enum : int { B_Q = 0, B_KF = 1, B_KE = 4, B_VF = 7, B_VE = 9, B_SF = 11, B_PF = 13, B_OD = 15, B_NUM = 17 };

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    using C = ACfg<D>;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                                // [2][BQ x D]
    uint8_t* sK = sm + 2 * C::kQBytes;               // [kNK][BKV x D]
    uint8_t* sV = sK + C::kNK * C::kKBytes;          // [kNV][D x BKV] (V^T)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kNV * C::kVBytes);
    auto bar = [&](int slot) { return smem_u32(&bars[slot]); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[B_NUM]);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int q0 = blockIdx.x * 2 * BQ;
    const int nq = (q0 + BQ < s) ? 2 : 1;  // second query tile present?
    const int head = blockIdx.y, lw = blockIdx.z;
    const int plane = lw * p.heads + head;

    // seam groups (window.hpp:58-65): only the last window row of a shifted layout is masked
    const int gw = p.lay.loc2glob[lw];
    const bool masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;
    const int split = masked ? (p.w - p.lay.g.shift) * p.w : s;
    const int qlast = min(q0 + nq * BQ, s) - 1;
    const int kv_lo = (masked && q0 >= split) ? split : 0;
    const int kv_hi = (masked && qlast < split) ? split : s;
    const int t_lo = kv_lo / BKV, t_hi = (kv_hi + BKV - 1) / BKV;
    const int ntiles = t_hi - t_lo;

    if (warp == 1 && lane == 0) {
        mbar_init(bar(B_Q), 1);
        for (int i = 0; i < C::kNK; ++i) {
            mbar_init(bar(B_KF + i), 1);
            mbar_init(bar(B_KE + i), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar(B_VF + i), 1);
            mbar_init(bar(B_VE + i), 1);
            mbar_init(bar(B_SF + i), 1);
            mbar_init(bar(B_PF + i), 4);
            mbar_init(bar(B_OD + i), 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // register rebalancing: the producer / MMA / allocator warpgroup needs few registers, the two
    // softmax warpgroups hold a 128-column S row each (64K-register file: 128*40 + 256*232)
    if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {
        // ===== TMA producer 1: both query tiles, then the K ring
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
            mbar_expect_tx(bar(B_Q), nq * C::kQBytes);
            for (int h = 0; h < nq; ++h)
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2d(smem_u32(sQ + h * C::kQBytes + b * BQ * C::kSw), &tmQ, bar(B_Q),
                                b * C::kColsPerBox, plane * s + q0 + h * BQ);
            for (int j = 0; j < ntiles; ++j) {
                const int st = j % C::kNK;
                mbar_wait(bar(B_KE + st), ((j / C::kNK) & 1) ^ 1);
                mbar_expect_tx(bar(B_KF + st), C::kKBytes);
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2d(smem_u32(sK + st * C::kKBytes + b * BKV * C::kSw), &tmK, bar(B_KF + st),
                                b * C::kColsPerBox, plane * s + (t_lo + j) * BKV);
            }
        }
    } else if (warp == 3) {
        // ===== TMA producer 2: the V^T ring (D rows x 64 keys per box)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
            for (int j = 0; j < ntiles; ++j) {
                const int st = j & 1;
                mbar_wait(bar(B_VE + st), ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(bar(B_VF + st), C::kVBytes);
                for (int b = 0; b < 2; ++b)
                    tma_load_2d(smem_u32(sV + st * C::kVBytes + b * D * 128), &tmV, bar(B_VF + st),
                                (t_lo + j) * BKV + b * 64, plane * D);
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer
        if (lane == 0) {
            auto issue_s = [&](int h, int j) {  // S_h = Q_h K_j^T
                const uint8_t* kt = sK + (j % C::kNK) * C::kKBytes;
                const uint8_t* qh = sQ + h * C::kQBytes;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const int box = (kk * 32) / C::kSw, off = (kk * 32) % C::kSw;
                    const uint64_t a = desc_kmajor(smem_u32(qh + box * BQ * C::kSw + off), C::kSw);
                    const uint64_t b = desc_kmajor(smem_u32(kt + box * BKV * C::kSw + off), C::kSw);
                    mma_ss(tmem + uint32_t(h * 128), a, b, C::kIdescS, kk > 0 ? 1u : 0u);
                }
                commit(bar(B_SF + h));
            };
            auto issue_pv = [&](int h, int j) {  // O_h += P_h V_j
                mbar_wait(bar(B_PF + h), j & 1);
                fence_after();
                const uint8_t* vt = sV + (j & 1) * C::kVBytes;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    const uint64_t b = desc_kmajor(smem_u32(vt + (kk >> 2) * D * 128 + (kk & 3) * 32), 128);
                    mma_ts(tmem + uint32_t(256 + h * 128), tmem + uint32_t(h * 128 + kk * 8), b, C::kIdescO,
                           (j > 0 || kk > 0) ? 1u : 0u);
                }
                commit(bar(B_OD + h));
            };
            auto wait_k = [&](int j) {
                mbar_wait(bar(B_KF + j % C::kNK), (j / C::kNK) & 1);
                fence_after();
            };
            mbar_wait(bar(B_Q), 0);
            wait_k(0);
            issue_s(0, 0);
            if (nq == 2) issue_s(1, 0);
            commit(bar(B_KE + 0));  // K_0 consumed once both S MMAs complete
            for (int j = 0; j < ntiles; ++j) {
                const bool more = j + 1 < ntiles;
                mbar_wait(bar(B_VF + (j & 1)), (j >> 1) & 1);
                fence_after();
                // P_0 V_j, then S_0 of the next key tile (in-order tensor pipe: S_0 overwrites P_0 after
                // the P V that reads it)
                issue_pv(0, j);
                if (more) {
                    wait_k(j + 1);
                    issue_s(0, j + 1);
                }
                if (nq == 2) {
                    issue_pv(1, j);
                    if (more) issue_s(1, j + 1);
                }
                commit(bar(B_VE + (j & 1)));  // V_j consumed
                if (more) commit(bar(B_KE + (j + 1) % C::kNK));
            }
        }
    } else if (warp >= 4) {
        // ===== softmax warpgroups (thread per query row) + epilogue
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
        const int h = (warp - 4) >> 2;      // query tile
        const int wq = (warp - 4) & 3;      // TMEM lane quadrant (warp % 4)
        if (h < nq) {
            const int r = wq * 32 + lane;
            const int q = q0 + h * BQ + r;
            const uint32_t lane_off = uint32_t(wq * 32) << 16;
            const uint32_t tS = tmem + lane_off + uint32_t(h * 128);
            const uint32_t tO = tmem + lane_off + uint32_t(256 + h * 128);
            // this row's admissible keys (seam group), intersected with the CTA range
            const int rlo = (masked && q >= split) ? split : 0;
            const int rhi = (masked && q < split) ? split : s;
            const float sl2 = p.scale * 1.4426950408889634f;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < ntiles; ++j) {
                mbar_wait(bar(B_SF + h), j & 1);
                fence_after();
                uint32_t sr[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) ld32(tS + uint32_t(c * 32), sr + 32 * c);
#pragma unroll
                for (int c = 0; c < 4; ++c) wait_ld_dep(sr + 32 * c);
                const int kb = (t_lo + j) * BKV;
                if (kb < rlo || kb + BKV > rhi) {  // boundary tile: mask keys outside [rlo, rhi)
#pragma unroll
                    for (int i = 0; i < 128; ++i)
                        if (kb + i < rlo || kb + i >= rhi) sr[i] = __float_as_uint(-INFINITY);
                }
                // row max of raw scores (scale > 0 commutes with max), 4-way tree
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < 128; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sr[i]));
                const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
                if (mx > m + kRescale || (m == -INFINITY && mx != -INFINITY)) {
                    if (m != -INFINITY) {
                        // O *= 2^(m - mx): the P V of the previous key tile must have landed
                        mbar_wait(bar(B_OD + h), (j - 1) & 1);
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
                float ls4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed bf16x2 columns per store
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        // 1 in 4 exponentials on the FMA pipe, the rest on MUFU (balances the two)
                        const float z0 = fmaf(__uint_as_float(sr[32 * c + 2 * i]), sl2, nb);
                        const float z1 = fmaf(__uint_as_float(sr[32 * c + 2 * i + 1]), sl2, nb);
                        const float p0 = ex2(z0);
                        const float p1 = (i & 1) ? ex2_poly(z1) : ex2(z1);
                        ls4[i & 3] += p0 + p1;
                        pk[i] = pack_bf16x2(p0, p1);
                    }
                    st16(tS + uint32_t(16 * c), pk);
                }
                l += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
                wait_st();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar(B_PF + h));
            }
            // epilogue: O / l -> bf16, heads concatenated in token rows
            mbar_wait(bar(B_OD + h), (ntiles - 1) & 1);
            fence_after();
            const float inv = 1.f / l;
            __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o) + (i64(lw) * s + q) * p.ldo + head * D;
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
    dim3 grid(unsigned((p.s + 2 * BQ - 1) / (2 * BQ)), unsigned(p.heads), unsigned(p.nloc));
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
