// k_attn.cu -- BF16 windowed attention, flash-style: per (window, head, 128-query tile) CTA,
// softmax(Q K^T / sqrt(d) + seam mask) V with an online max/sum (exp2, warp-shuffle row
// reductions), K/V tiles double-buffered through shared memory with cp.async.
// Restates head_attention_fwd (swin.hpp:161-188) without materialising the s x s logits; the
// latitude-seam mask (window.hpp:107-122) becomes per-query KV-range limits, since the two seam
// groups are the contiguous token ranges [0, (w-shift)*w) and [(w-shift)*w, w*w).
#include "kernels.cuh"

namespace swf {

namespace {

constexpr int BQ = 128;  // queries per CTA (8 warps x 16 rows)
constexpr int BKV = 64;  // keys per tile
constexpr int kWarps = 8;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>
struct Smem {
    static constexpr int LD = D + 8;  // padded row (bf16) -> conflict-free ldmatrix
    static constexpr int kQ = BQ * LD;
    static constexpr int kKV = BKV * LD;
    static constexpr int kBytes = (kQ + 4 * kKV) * 2;
};

template <int D>
__device__ __forceinline__ void load_tile(__nv_bfloat16* dst, const __nv_bfloat16* src, int row0, int nrows_total,
                                          int rows) {
    constexpr int LD = Smem<D>::LD;
    constexpr int CH = D / 8;  // 16-byte chunks per row
    for (int c = threadIdx.x; c < rows * CH; c += kWarps * 32) {
        const int r = c / CH, k = c - (c / CH) * CH;
        const int gr = row0 + r;
        const bool ok = gr < nrows_total;
        const __nv_bfloat16* s = src + i64(ok ? gr : 0) * D + k * 8;
        cp_async16(smem_addr(dst + r * LD + k * 8), s, ok ? 16 : 0);
    }
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32, 1) k_attn_bf16(AttnParams p) {
    using S = Smem<D>;
    constexpr int LD = S::LD;
    extern __shared__ __align__(128) uint8_t smraw[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smraw);
    __nv_bfloat16* sK = sQ + S::kQ;          // [2][BKV][LD]
    __nv_bfloat16* sV = sK + 2 * S::kKV;     // [2][BKV][LD]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int q0 = blockIdx.x * BQ;
    const int head = blockIdx.y, lw = blockIdx.z;
    const i64 base = (i64(lw) * p.heads + head) * s;
    const __nv_bfloat16* Q = reinterpret_cast<const __nv_bfloat16*>(p.q) + base * D;
    const __nv_bfloat16* K = reinterpret_cast<const __nv_bfloat16*>(p.k) + base * D;
    const __nv_bfloat16* V = reinterpret_cast<const __nv_bfloat16*>(p.v) + base * D;

    // seam groups (window.hpp:58-65): only the last window row of a shifted layout is masked
    const int gw = p.lay.loc2glob[lw];
    const bool masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;
    const int split = masked ? (p.w - p.lay.g.shift) * p.w : s;
    const int qlast = min(q0 + BQ, s) - 1;
    int kv_lo = 0, kv_hi = s;
    bool elementwise = false;
    if (masked) {
        if (qlast < split) {
            kv_hi = split;
        } else if (q0 >= split) {
            kv_lo = split;
        } else {
            elementwise = true;
        }
    }
    const int t_lo = kv_lo / BKV, t_hi = (kv_hi + BKV - 1) / BKV;

    load_tile<D>(sQ, Q, q0, s, BQ);
    load_tile<D>(sK, K, t_lo * BKV, s, BKV);
    load_tile<D>(sV, V, t_lo * BKV, s, BKV);
    cp_commit();

    const int g = lane >> 2, tq = lane & 3;
    const int r0 = q0 + warp * 16 + g;  // this thread's rows r0 and r0 + 8
    const int grp0 = r0 < split ? 0 : 1, grp1 = (r0 + 8) < split ? 0 : 1;
    const float sl2 = p.scale * 1.4426950408889634f;

    uint32_t qf[D / 16][4];
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int t = t_lo; t < t_hi; ++t) {
        const int buf = (t - t_lo) & 1;
        if (t + 1 < t_hi) {
            load_tile<D>(sK + (buf ^ 1) * S::kKV, K, (t + 1) * BKV, s, BKV);
            load_tile<D>(sV + (buf ^ 1) * S::kKV, V, (t + 1) * BKV, s, BKV);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        if (t == t_lo) {
#pragma unroll
            for (int kc = 0; kc < D / 16; ++kc) {
                const int row = warp * 16 + (lane & 15);
                const int col = kc * 16 + (lane >> 4) * 8;
                ldsm_x4(smem_addr(sQ + row * LD + col), qf[kc][0], qf[kc][1], qf[kc][2], qf[kc][3]);
            }
        }
        const __nv_bfloat16* kt = sK + buf * S::kKV;
        const __nv_bfloat16* vt = sV + buf * S::kKV;
        // S = Q K^T : 16 x 64 per warp
        float sc[BKV / 8][4];
#pragma unroll
        for (int nt = 0; nt < BKV / 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int kc = 0; kc < D / 16; ++kc) {
#pragma unroll
            for (int np = 0; np < BKV / 16; ++np) {
                // two n8 tiles (keys np*16 .. +16) x k16: ldmatrix x4 over K rows
                uint32_t b0, b1, b2, b3;
                const int krow = np * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int kcol = kc * 16 + ((lane >> 3) & 1) * 8;
                ldsm_x4(smem_addr(kt + krow * LD + kcol), b0, b1, b2, b3);
                mma16816(sc[2 * np], qf[kc][0], qf[kc][1], qf[kc][2], qf[kc][3], b0, b1);
                mma16816(sc[2 * np + 1], qf[kc][0], qf[kc][1], qf[kc][2], qf[kc][3], b2, b3);
            }
        }
        // scale, mask (ragged tail + seam), online softmax in base 2
        const int kb = t * BKV;
        float mx0 = m0, mx1 = m1;
#pragma unroll
        for (int nt = 0; nt < BKV / 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = kb + nt * 8 + 2 * tq + (e & 1);
                float v = sc[nt][e] * sl2;
                bool keep = key < kv_hi && key >= kv_lo;
                if (elementwise) keep = keep && ((key < split ? 0 : 1) == ((e < 2) ? grp0 : grp1));
                v = keep ? v : -INFINITY;
                sc[nt][e] = v;
                if (e < 2)
                    mx0 = fmaxf(mx0, v);
                else
                    mx1 = fmaxf(mx1, v);
            }
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float b0s = mx0 == -INFINITY ? 0.f : mx0;
        const float b1s = mx1 == -INFINITY ? 0.f : mx1;
        const float c0 = exp2f(m0 - b0s), c1 = exp2f(m1 - b1s);
        m0 = mx0;
        m1 = mx1;
        l0 *= c0;
        l1 *= c1;
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            o[i][0] *= c0;
            o[i][1] *= c0;
            o[i][2] *= c1;
            o[i][3] *= c1;
        }
        uint32_t pf[BKV / 16][4];
#pragma unroll
        for (int nt = 0; nt < BKV / 8; ++nt) {
            const float p0 = exp2f(sc[nt][0] - b0s), p1 = exp2f(sc[nt][1] - b0s);
            const float p2 = exp2f(sc[nt][2] - b1s), p3 = exp2f(sc[nt][3] - b1s);
            l0 += p0 + p1;
            l1 += p2 + p3;
            pf[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16x2(p0, p1);
            pf[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16x2(p2, p3);
        }
        // O += P V : A = P (16 x 64), B = V (64 x D) via ldmatrix.trans
#pragma unroll
        for (int kc = 0; kc < BKV / 16; ++kc) {
#pragma unroll
            for (int np = 0; np < D / 16; ++np) {
                uint32_t b0, b1, b2, b3;
                const int vrow = kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                const int vcol = np * 16 + (lane >> 4) * 8;
                ldsm_x4_t(smem_addr(vt + vrow * LD + vcol), b0, b1, b2, b3);
                mma16816(o[2 * np], pf[kc][0], pf[kc][1], pf[kc][2], pf[kc][3], b0, b1);
                mma16816(o[2 * np + 1], pf[kc][0], pf[kc][1], pf[kc][2], pf[kc][3], b2, b3);
            }
        }
        __syncthreads();
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o);
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt) {
        const int col = head * D + nt * 8 + 2 * tq;
        if (r0 < s) *reinterpret_cast<uint32_t*>(O + (i64(lw) * s + r0) * p.ldo + col) = pack_bf16x2(o[nt][0] * i0, o[nt][1] * i0);
        if (r0 + 8 < s)
            *reinterpret_cast<uint32_t*>(O + (i64(lw) * s + r0 + 8) * p.ldo + col) = pack_bf16x2(o[nt][2] * i1, o[nt][3] * i1);
    }
}

template <int D>
void launch_attn(const AttnParams& p, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        SWF_CUDA(cudaFuncSetAttribute(k_attn_bf16<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<D>::kBytes));
        configured = true;
    }
    dim3 grid(unsigned((p.s + BQ - 1) / BQ), unsigned(p.heads), unsigned(p.nloc));
    k_attn_bf16<D><<<grid, kWarps * 32, Smem<D>::kBytes, st>>>(p);
    SWF_LAUNCH_CHECK();
}

}  // namespace

void attention_bf16(const AttnParams& p, cudaStream_t st) {
    switch (p.d) {
        case 32: launch_attn<32>(p, st); break;
        case 64: launch_attn<64>(p, st); break;
        case 128: launch_attn<128>(p, st); break;
        default: throw CudaError("attention_bf16: head_dim must be 32, 64 or 128");
    }
}

}  // namespace swf
