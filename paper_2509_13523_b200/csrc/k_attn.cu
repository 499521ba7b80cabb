// k_attn.cu -- BF16 windowed attention on the 5th-generation tensor cores (sm_100a).
//
// Persistent 2-CTA clusters running the pair-wide tensor-core MMA (tcgen05.mma.cta_group::2): a
// work item is a pair of 128-query tiles of one (window, head), one tile per CTA, and every MMA
// covers both (M = 256). Each CTA holds its own query tile and HALF of every K / V^T tile (the MMA's
// B operand is split by N across the pair), so a key tile costs each SM 32 KB of TMA fill and half
// the B-operand shared-memory reads. Restates head_attention_fwd (swin.hpp:161-188) without
// materialising the s x s logits:
//   * S = Q K^T : M=256 (2 x 128 queries), N=128 keys, K=d; A = Q and B = K, K-major SW128 tiles
//     loaded by TMA; FP32 S in each CTA's TMEM, triple-buffered (S0 / S1 / S2): the QK^T issuer runs
//     up to three key tiles ahead of the P V issuer (over the flattened sequence of work items), so
//     the softmax warps find the next S ready when they finish a tile;
//   * softmax (per CTA): 8 warps, each TMEM lane (query row) is shared by two threads that take 64
//     keys each (the row maximum is exchanged through shared memory); base-2 online max/sum with lazy
//     O rescaling (only when the running max grows by > 2^8), packed f32x2 arithmetic, kPoly8/8 of
//     the exponentials on the FMA pipe (degree-3 polynomial) and the rest on MUFU (sm_100 has no
//     packed BF16x2 MUFU: ex2.approx.bf16x2 compiles to two scalar MUFU ops); P is packed to BF16
//     into the first columns of each thread's S slice;
//   * O += P V : M=256, N=d, A = P read from TMEM, B = V^T (K-major, written transposed by the QKV
//     GEMM epilogue); O accumulates in TMEM. S(j+3) is issued only after P(j) V completed;
//   * epilogue: O / l in BF16 is staged in the finished item's Q buffer (SW128) and written by TMA
//     tensor stores (whole tiles, sp == 1); partial tiles and sequence-parallel rows (scattered to
//     the band owners) are stored row by row;
//   * the latitude-seam mask (window.hpp:107-122) is a per-row key range: the two seam groups are
//     the contiguous token ranges [0, (w-shift)*w) and [(w-shift)*w, w*w); fully-outside key tiles
//     are skipped and only boundary tiles pay per-element masking.
// Two leader-CTA warps issue the pair's MMAs (QK^T and P V), each one key tile per asm block with a
// single elect.sync: a tcgen05.mma instruction costs ~45 cycles to issue, so one issuer serialising
// 16 MMAs and its barrier waits per key tile cannot keep the tensor pipe busy. TMA loads of both CTAs and the P-ready / O-free
// arrivals of both CTAs' softmax warps complete on the leader's barriers; MMA commits multicast to
// both CTAs.
// Warp roles (per CTA): w0 TMA (Q double buffer, K-half ring), w3 TMA (V^T-half ring), w1 QK^T
// issuer (leader), w2 TMEM allocator + P V issuer (leader), w4-w7 softmax keys [0,64), w8-w11 keys
// [64,128).
// TMEM (per CTA): S0 [0,128) S1 [128,256) S2 [256,384) O [384,384+D).
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace swf {

namespace {

using namespace tc;

#ifdef SWF_ATTN_TRACE
// development build only (make EXTRA=-DSWF_ATTN_TRACE): clock64 stamps of CTA 0's pipeline events,
// written to $SWF_ATTN_TRACE_OUT after each launch. Per key tile g: 0 S ready, 1 row max exchanged,
// 2 P stores issued, 3 P stored, 4 P seen by the MMA issuer, 5 P V issued; per item n: 6 MMA saw
// Q, 7 MMA saw O free, 8 epilogue start, 9 epilogue end; MMA warp per tile: 10 S issue entry,
// 11 K landed, 12 S issued, 13 P V entry, 14 P seen. The ping-pong kernel (tools/attn_pp_trace.py):
// 1 first global tile of item n, 10/11/12 QK^T issuer entry / K landed / ring slot free, 13/14/15 P V
// issuer entry / P seen / V landed, 7 O free; per softmax warp w (g_trace_w): w S ready, 8 + w S in
// registers, 16 + w P handed over; 8 / 9 item epilogue start / end.
constexpr int kTrN = 1024;
__device__ unsigned long long g_trace[2][16][kTrN];  // [CTA 0 / 1 of the first cluster]
__device__ unsigned long long g_trace_w[2][32][kTrN];  // per softmax warp: [cta][warp-4 (S ready) / 8+warp-4 (P done)]
#define SWF_TR(row, idx)                                                                 \
    do {                                                                                 \
        if (blockIdx.x < 2 && (idx) < kTrN) g_trace[blockIdx.x][row][idx] = clock64(); \
    } while (0)
#define SWF_TRW(row, idx)                                                                    \
    do {                                                                                     \
        if (blockIdx.x < 2 && (idx) < kTrN) g_trace_w[blockIdx.x][row][idx] = clock64();   \
    } while (0)
#else
#define SWF_TR(row, idx) \
    do {                 \
    } while (0)
#define SWF_TRW(row, idx) \
    do {                  \
    } while (0)
#endif

constexpr int BQ = 128;   // queries per CTA tile (= UMMA M, = TMEM lanes)
constexpr int BKV = 128;  // keys per tile
// softmax threads per query row (each takes BKV / kSplit keys of every tile); 4 control warps +
// 4 * kSplit softmax warps. 2 is the default: with 4 (640 threads) the C2 launch is ~5% slower --
// the softmax is bound by its sub-partition's issue / MUFU throughput, not by per-thread latency
// (tools/gpurun/gpu_attn_ab.sh).
#ifndef SWF_ATTN_SPLIT
#define SWF_ATTN_SPLIT 2
#endif
constexpr int kSplit = SWF_ATTN_SPLIT;
#ifndef SWF_ATTN_POLY8
#define SWF_ATTN_POLY8 2
#endif
// exponentials per 8 evaluated by the FMA-pipe polynomial: 0..2 of 8 measured equal within noise and
// ~5% faster / ~25% less energy than 4 of 8 (tools/gpurun/gpu_attn_poly.sh)
constexpr int kPoly8 = SWF_ATTN_POLY8;
constexpr int kKPT = 128 / kSplit;  // keys per thread per tile
constexpr int kThreads = 128 + 128 * kSplit;
constexpr int kNS = 3;       // S buffers in TMEM
#ifndef SWF_ATTN_BACKOFF
#define SWF_ATTN_BACKOFF 40
#endif
constexpr uint32_t kBackoffNs = SWF_ATTN_BACKOFF;  // poll back-off of the control warps' barrier waits
// TMA producers of the ping-pong kernel wait for free ring slots 8 tiles ahead of their consumers: a
// long back-off costs nothing there, while each poll takes an issue slot from the softmax warp sharing
// the sub-partition (ncu: the producers' polling was ~17% of all issued instructions at 40 ns)
#ifndef SWF_ATTN_PBACKOFF
#define SWF_ATTN_PBACKOFF 256
#endif
constexpr uint32_t kTO = 384;  // TMEM column of O
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)

template <int D>
struct ACfg {
    static constexpr int kSw = D >= 64 ? 128 : 2 * D;  // swizzle bytes of Q/K rows (d contiguous)
    static constexpr int kColsPerBox = kSw / 2;         // d elements per TMA box row
    static constexpr int kBoxes = D / kColsPerBox;      // boxes along d
    static constexpr int kQBytes = BQ * D * 2;          // this CTA's query tile
    static constexpr int kKHalf = (BKV / 2) * D * 2;    // this CTA's 64 keys of a K tile
    static constexpr int kVHalf = (D / 2) * BKV * 2;    // this CTA's d/2 rows of a V^T tile
    static constexpr int kNK = 4, kNV = 4;
    static constexpr int kRedBytes = kSplit * BQ * 4;   // row-max / row-sum exchange between key splits
    static constexpr int kSmem = 2 * kQBytes + kNK * kKHalf + kNV * kVHalf + kRedBytes + 256 + 1024;
    static constexpr int kOC = D / kSplit;              // O columns per softmax thread (epilogue / rescale)
    static constexpr uint32_t kIdescS = idesc_bf16(2 * BQ, BKV);
    static constexpr uint32_t kIdescO = idesc_bf16(2 * BQ, D);
};

// barrier slots (u64 each)
enum : int {
    B_QF = 0, B_QE = 2, B_KF = 4, B_KE = 8, B_VF = 12, B_VE = 16, B_SF = 20, B_PF = 23, B_PVD = 26, B_OD = 29,
    B_OF = 30, B_NUM = 31
};

// Work item -> (pair of q tiles, head, local window); the two CTAs of a cluster take the two q tiles
// of a pair (crank 0 / 1). Items of one (window, head) are consecutive so concurrently running
// clusters also share K / V^T tiles through L2.
struct Item {
    int q0, qp0, head, lw;  // q0: this CTA's tile; qp0: first row of the pair
};
__device__ __forceinline__ Item item_of(int it, int npairs, int heads, int crank) {
    Item r;
    const int qp = it % npairs;
    const int hw = it / npairs;
    r.qp0 = qp * 2 * BQ;
    r.q0 = r.qp0 + crank * BQ;
    r.head = hw % heads;
    r.lw = hw / heads;
    return r;
}

// key range of a work item (seam groups), the union over the pair so both CTAs walk the same tiles
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
    const int qlast = min(it.qp0 + 2 * BQ, s) - 1;
    const int kv_lo = (r.masked && it.qp0 >= r.split) ? r.split : 0;
    const int kv_hi = (r.masked && qlast < r.split) ? r.split : s;
    r.t_lo = kv_lo / BKV;
    r.ntiles = (kv_hi + BKV - 1) / BKV - r.t_lo;
    return r;
}

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// arrive on a (possibly remote) barrier of the cluster; CTA-scope release: the data handed over lives
// in TMEM (ordered by tcgen05.wait + tcgen05.fence::before_thread_sync), and a cluster-scope release
// would cost a GPU-wide MEMBAR per arrival
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// TMA 2D tile load into this CTA's shared memory, completing on the leader CTA's mbarrier
__device__ __forceinline__ void tma_load_2cta(uint32_t dst, const void* tmap, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
// mbarrier wait for the control warps: poll with a short nanosleep back-off, so a waiting producer /
// MMA warp leaves the issue slots of its SM sub-partition to the softmax warp pair that shares it
template <uint32_t kNs = kBackoffNs>
__device__ __forceinline__ void mbar_sleep_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) break;
        if constexpr (kNs > 0) __nanosleep(kNs);
    }
}
// named barrier of the kSplit warps sharing a TMEM lane quadrant (one per key split)
__device__ __forceinline__ void pair_sync(int quadrant) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + quadrant), "r"(32 * kSplit) : "memory");
}

// TMA tensor store of a 2D box from shared memory (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(src),
                 "r"(c0), "r"(c1)
                 : "memory");
}
// all 256 softmax threads
__device__ __forceinline__ void softmax_sync() { asm volatile("bar.sync 5, %0;" ::"r"(128 * kSplit) : "memory"); }

// commit of the pair's MMAs arriving on this CTA's barrier
__device__ __forceinline__ void commit2(uint32_t bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
        "}\n" ::"r"(bar)
        : "memory");
}
// commit of the pair's MMAs arriving on the barrier at the same offset in both CTAs
__device__ __forceinline__ void commit2_mc(uint32_t bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        ".reg .b16 m;\n"
        "mov.b16 m, 3;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
        "}\n" ::"r"(bar)
        : "memory");
}

// Tile-level pair-wide MMA issue: ONE asm block per tile with one elect.sync, descriptor start
// addresses advanced by immediates inside the block. Issuing MMA by MMA costs a register-to-uniform
// broadcast chain per instruction (~50 cycles each), which starves the tensor pipe at N = 128.
template <int OA1, int OB1>
__device__ __forceinline__ void mma2_ss_x2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 pf, %3, %3;\n"
        "setp.eq.b32 pt, %3, %3;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, pf;\n"
        "add.s64 a, %1, %4;\n"
        "add.s64 b, %2, %5;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(idesc), "n"(OA1), "n"(OB1));
}
template <int OA1, int OA2, int OA3, int OB1, int OB2, int OB3>
__device__ __forceinline__ void mma2_ss_x4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 pf, %3, %3;\n"
        "setp.eq.b32 pt, %3, %3;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, pf;\n"
        "add.s64 a, %1, %4;\n"
        "add.s64 b, %2, %7;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %5;\n"
        "add.s64 b, %2, %8;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %6;\n"
        "add.s64 b, %2, %9;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(idesc), "n"(OA1), "n"(OA2), "n"(OA3), "n"(OB1), "n"(OB2), "n"(OB3));
}
template <int OA1, int OA2, int OA3, int OA4, int OA5, int OA6, int OA7, int OB1, int OB2, int OB3, int OB4, int OB5, int OB6, int OB7>
__device__ __forceinline__ void mma2_ss_x8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b64 a, b;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 pf, %3, %3;\n"
        "setp.eq.b32 pt, %3, %3;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, pf;\n"
        "add.s64 a, %1, %4;\n"
        "add.s64 b, %2, %11;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %5;\n"
        "add.s64 b, %2, %12;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %6;\n"
        "add.s64 b, %2, %13;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %7;\n"
        "add.s64 b, %2, %14;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %8;\n"
        "add.s64 b, %2, %15;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %9;\n"
        "add.s64 b, %2, %16;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, %10;\n"
        "add.s64 b, %2, %17;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, pt;\n"
        "}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(idesc), "n"(OA1), "n"(OA2), "n"(OA3), "n"(OA4), "n"(OA5), "n"(OA6), "n"(OA7), "n"(OB1), "n"(OB2), "n"(OB3), "n"(OB4), "n"(OB5), "n"(OB6), "n"(OB7));
}
// 8 pair-wide TS MMAs of one P V tile: A = P at TMEM columns a + TA_k, B start address + OB_k
template <int TA1, int TA2, int TA3, int TA4, int TA5, int TA6, int TA7, int OB1, int OB2, int OB3, int OB4, int OB5, int OB6, int OB7>
__device__ __forceinline__ void mma2_ts_x8(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n"
        ".reg .pred e, p0, pt;\n"
        ".reg .b64 b;\n"
        ".reg .b32 a;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p0, %4, 0;\n"
        "setp.eq.b32 pt, %3, %3;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p0;\n"
        "add.u32 a, %1, %5;\n"
        "add.s64 b, %2, %12;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %6;\n"
        "add.s64 b, %2, %13;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %7;\n"
        "add.s64 b, %2, %14;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %8;\n"
        "add.s64 b, %2, %15;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %9;\n"
        "add.s64 b, %2, %16;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %10;\n"
        "add.s64 b, %2, %17;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, %11;\n"
        "add.s64 b, %2, %18;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "}\n"
        ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc0), "n"(TA1), "n"(TA2), "n"(TA3), "n"(TA4), "n"(TA5), "n"(TA6), "n"(TA7), "n"(OB1), "n"(OB2), "n"(OB3), "n"(OB4), "n"(OB5), "n"(OB6), "n"(OB7));
}
// all QK^T MMAs of one key tile (D/16 k-steps): A = Q rows (BQ x kSw boxes), B = this CTA's 64 keys
template <int D>
__device__ __forceinline__ void issue_s_tile(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if constexpr (D == 128)
        mma2_ss_x8<2, 4, 6, 1024, 1026, 1028, 1030, 2, 4, 6, 512, 514, 516, 518>(d, a, b, idesc);
    else if constexpr (D == 64)
        mma2_ss_x4<2, 4, 6, 2, 4, 6>(d, a, b, idesc);
    else
        mma2_ss_x2<2, 2>(d, a, b, idesc);
}
// all P V MMAs of one key tile: P of keys [64h, 64h+64) at S columns [64h, 64h+32); V^T half in
// two 64-key SW128 boxes of D/2 rows
// P of keys [KPT s, KPT s + KPT) sits at S columns [KPT s, KPT s + KPT/2): key block kk of 16 keys
// starts at column KPT * (16 kk / KPT) + (16 kk % KPT) / 2
__host__ __device__ constexpr int p_col(int kk) { return kKPT * ((16 * kk) / kKPT) + ((16 * kk) % kKPT) / 2; }
template <int D>
__device__ __forceinline__ void issue_pv_tile(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    constexpr int BX = (D / 2) * 128 / 16;  // 16-byte units per V^T box
    mma2_ts_x8<p_col(1), p_col(2), p_col(3), p_col(4), p_col(5), p_col(6), p_col(7), 2, 4, 6, BX, BX + 2, BX + 4,
               BX + 6>(d, a, b, idesc, acc0);
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

// this thread's OC = D/2 O columns (TMEM address t): scale in place / read out
template <int OC>
__device__ __forceinline__ void o_scale(uint32_t t, float f) {
    if constexpr (OC == 8) {
        uint32_t o[8];
        ld8(t, o);
        wait_ld_dep8(o);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
        st8(t, o);
    } else if constexpr (OC == 16) {
        uint32_t o[16];
        ld16(t, o);
        wait_ld_dep16(o);
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
        st16(t, o);
    } else {
#pragma unroll 1
        for (int c = 0; c < OC / 32; ++c) {
            uint32_t o[32];
            ld32(t + uint32_t(c * 32), o);
            wait_ld_dep(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            st32(t + uint32_t(c * 32), o);
        }
    }
    wait_st();
}
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const uint32_t* o, float inv) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int v = 0; v < 2; ++v)
        d4[v] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * v]) * inv, __uint_as_float(o[8 * v + 1]) * inv),
                           pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv),
                           pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv),
                           pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv));
}
template <int OC>
__device__ __forceinline__ void o_store(uint32_t t, __nv_bfloat16* dst, float inv, bool valid) {
    if constexpr (OC == 8) {
        uint32_t o[8];
        ld8(t, o);
        wait_ld_dep8(o);
        if (valid)
            *reinterpret_cast<uint4*>(dst) =
                make_uint4(pack_bf16x2(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv),
                           pack_bf16x2(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv),
                           pack_bf16x2(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv),
                           pack_bf16x2(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv));
    } else if constexpr (OC == 16) {
        uint32_t o[16];
        ld16(t, o);
        wait_ld_dep16(o);
        if (valid) store_bf16x16(dst, o, inv);
    } else {
#pragma unroll 1
        for (int c = 0; c < OC / 32; ++c) {
            uint32_t o[32];
            ld32(t + uint32_t(c * 32), o);
            wait_ld_dep(o);
            if (valid) {
                store_bf16x16(dst + c * 32, o, inv);
                store_bf16x16(dst + c * 32 + 16, o + 16, inv);
            }
        }
    }
}

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, AttnParams p,
              int n_items) {
    using C = ACfg<D>;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                        // [2][BQ x D]
    uint8_t* sK = sm + 2 * C::kQBytes;       // [kNK][BKV/2 x D]: keys [64 crank, 64 crank + 64)
    uint8_t* sV = sK + C::kNK * C::kKHalf;   // [kNV][D/2 x BKV]: V^T rows [D/2 crank, D/2 crank + D/2)
    float* red = reinterpret_cast<float*>(sV + C::kNV * C::kVHalf);  // [2 key halves][BQ rows]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kNV * C::kVHalf + C::kRedBytes);
    auto bar = [&](int slot) { return smem_u32(&bars[slot]); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[B_NUM]);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int npairs = (s + 2 * BQ - 1) / (2 * BQ);
    const int crank = int(cta_rank());
    const bool lead = crank == 0;
    auto lbar = [&](int slot) { return map_to_rank(bar(slot), 0); };  // the leader CTA's barrier
    const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar(B_QF + i), 1);
            mbar_init(bar(B_QE + i), 1);  // released by the epilogue (its TMA store reads the buffer)
        }
        for (int i = 0; i < kNS; ++i) {
            mbar_init(bar(B_SF + i), 1);
            mbar_init(bar(B_PF + i), 2 * 4 * kSplit);  // leader's: the softmax warps of both CTAs
            mbar_init(bar(B_PVD + i), 1);   // leader's: P V of this buffer complete
        }
        for (int i = 0; i < C::kNK; ++i) {
            mbar_init(bar(B_KF + i), 1);
            mbar_init(bar(B_KE + i), 1);
        }
        for (int i = 0; i < C::kNV; ++i) {
            mbar_init(bar(B_VF + i), 1);
            mbar_init(bar(B_VE + i), 1);
        }
        mbar_init(bar(B_OD), 1);
        mbar_init(bar(B_OF), 2 * 4 * kSplit);  // leader's: the epilogue warps of both CTAs
        fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();  // barrier inits visible to the peer's TMA completions / commits / arrivals
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // register rebalancing within the 168 x 384 launch allocation: the control warpgroup drops to 72,
    // the softmax warpgroups rise to 216 (128 x (168 - 72) >= 256 x (216 - 168), else the increase blocks)
    if constexpr (kSplit == 2)
        if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");

    if (warp == 0) {
        // ===== TMA producer 1: Q (double-buffered across work items) and the K ring
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
            int g = 0, n = 0;
            for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
                const Item it = item_of(itx, npairs, p.heads, crank);
                const Range rg = range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                const int qb = n & 1;
                mbar_sleep_wait(bar(B_QE + qb), ((n >> 1) & 1) ^ 1);
                if (lead) mbar_expect_tx(bar(B_QF + qb), 2 * C::kQBytes);  // both query tiles
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2cta(smem_u32(sQ + qb * C::kQBytes + b * BQ * C::kSw), &tmQ, lbar(B_QF + qb),
                                  b * C::kColsPerBox, plane * s + it.q0);
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g % C::kNK;
                    mbar_sleep_wait(bar(B_KE + st), ((g / C::kNK) & 1) ^ 1);
                    if (lead) mbar_expect_tx(bar(B_KF + st), 2 * C::kKHalf);  // both key halves
                    for (int b = 0; b < C::kBoxes; ++b)
                        tma_load_2cta(smem_u32(sK + st * C::kKHalf + b * (BKV / 2) * C::kSw), &tmK, lbar(B_KF + st),
                                      b * C::kColsPerBox, plane * s + (rg.t_lo + j) * BKV + crank * (BKV / 2));
                }
            }
        }
    } else if (warp == 3) {
        // ===== TMA producer 2: the V^T ring (D rows x 64 keys per box)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
            int g = 0;
            for (int itx = cluster_id; itx < n_items; itx += n_clusters) {
                const Item it = item_of(itx, npairs, p.heads, crank);
                const Range rg = range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g % C::kNV;
                    mbar_sleep_wait(bar(B_VE + st), ((g / C::kNV) & 1) ^ 1);
                    if (lead) mbar_expect_tx(bar(B_VF + st), 2 * C::kVHalf);  // both d halves
                    // this CTA's d rows [D/2 crank, D/2 crank + D/2), keys in two 64-key boxes
                    for (int b = 0; b < 2; ++b)
                        tma_load_2cta(smem_u32(sV + st * C::kVHalf + b * (D / 2) * 128), &tmV, lbar(B_VF + st),
                                      (rg.t_lo + j) * BKV + b * 64, plane * D + crank * (D / 2));
                }
            }
        }
    } else if (warp == 1 && lead) {
        // ===== QK^T issuer for the pair (leader CTA; whole warp, converged; one elected lane issues),
        // running over the flattened (item, key tile) sequence up to three tiles ahead of P V
        // a CTA holding all 512 columns owns TMEM from address 0 (checked)
        if (tmem != 0) __trap();
        const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK);
        int g = 0, n = 0;
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Range rg = range_of(p, item_of(itx, npairs, p.heads, crank));
            const int qb = n & 1;
            mbar_sleep_wait(bar(B_QF + qb), (n >> 1) & 1);
            if (lane == 0) SWF_TR(6, n);
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int st = g % C::kNK, b = g % kNS;
                if (lane == 0) SWF_TR(10, g);
                mbar_sleep_wait(bar(B_KF + st), (g / C::kNK) & 1);
                // S buffer b last held P(g-3): its P V must have completed
                mbar_sleep_wait(bar(B_PVD + b), ((g / kNS) & 1) ^ 1);
                if (lane == 0) SWF_TR(11, g);
                fence_after();
                const uint64_t a0 = desc_kmajor(sQa + uint32_t(qb * C::kQBytes), C::kSw);
                const uint64_t b0 = desc_kmajor(sKa + uint32_t(st * C::kKHalf), C::kSw);
                issue_s_tile<D>(uint32_t(b * 128), a0, b0, C::kIdescS);
                commit2_mc(bar(B_SF + b));
                commit2_mc(bar(B_KE + st));  // K halves consumed in both CTAs
                if (lane == 0) SWF_TR(12, g);
#ifdef SWF_ATTN_SWAIT  // development only: measure the QK^T completion latency
                mbar_wait(bar(B_SF + b), (g / kNS) & 1);
                if (lane == 0) SWF_TR(15, g);
#endif
            }
        }
    } else if (warp == 2 && lead) {
        // ===== P V issuer for the pair (leader CTA), in key-tile order
        const uint32_t sVa = smem_u32(sV);
        int g = 0, n = 0;
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Range rg = range_of(p, item_of(itx, npairs, p.heads, crank));
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int b = g % kNS, vs = g % C::kNV;
                if (j == 0 && n >= 1) {
                    mbar_sleep_wait(bar(B_OF), (n - 1) & 1);  // O of the previous item read out
                    if (lane == 0) SWF_TR(7, n);
                }
                if (lane == 0) SWF_TR(13, g);
                mbar_sleep_wait(bar(B_PF + b), (g / kNS) & 1);
                if (lane == 0) SWF_TR(14, g);
                mbar_sleep_wait(bar(B_VF + vs), (g / C::kNV) & 1);
                fence_after();
                if (lane == 0) SWF_TR(4, g);
                const uint64_t b0 = desc_kmajor(sVa + uint32_t(vs * C::kVHalf), 128);
                issue_pv_tile<D>(kTO, uint32_t(b * 128), b0, C::kIdescO, j == 0 ? 0u : 1u);
                commit2_mc(bar(B_OD));
                commit2_mc(bar(B_VE + vs));  // V^T halves consumed in both CTAs
                commit2(bar(B_PVD + b));     // S buffer b free for S(g+3)
                if (lane == 0) SWF_TR(5, g);
            }
        }
    } else if (warp >= 4) {
        // ===== softmax (kSplit threads per query row, kKPT keys each) + epilogue
        if constexpr (kSplit == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        const int hk = (warp - 4) >> 2;  // key split of every tile
        const int wq = warp & 3;         // TMEM lane quadrant
        const int r = wq * 32 + lane;
        const uint32_t lane_off = uint32_t(wq * 32) << 16;
        const uint32_t tO = lane_off + kTO + uint32_t(hk * C::kOC);
        const float sl2 = p.scale * 1.4426950408889634f;
        const bool tr = threadIdx.x == 128;
        const bool leader = threadIdx.x == 128;  // issues the O TMA stores, releases Q buffers
        int qe_pending = -1;                     // Q buffer whose TMA-store read is still in flight
        auto release_q = [&]() {
            if (qe_pending >= 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_arrive(bar(B_QE + qe_pending));
                qe_pending = -1;
            }
        };
        int g = 0, n = 0;
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Item it = item_of(itx, npairs, p.heads, crank);
            const Range rg = range_of(p, it);
            const int q = it.q0 + r;
            const int rlo = (rg.masked && q >= rg.split) ? rg.split : 0;
            const int rhi = (rg.masked && q < rg.split) ? rg.split : s;
            // destination row (token owner's SP band; this rank when sp == 1), resolved early
            int orank = 0;
            const i64 oloc = q < s ? p.lay.wtok_to_loc(p.wp_rank, it.lw, q, &orank) : 0;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int b = g % kNS;
                const uint32_t tS = lane_off + uint32_t(b * 128 + hk * kKPT);
                mbar_wait(bar(B_SF + b), (g / kNS) & 1);
                fence_after();
                if (tr) SWF_TR(0, g);
#ifdef SWF_ATTN_TRACE
                if (lane == 0 && blockIdx.x < 2 && g < kTrN) g_trace_w[blockIdx.x][warp - 4][g] = clock64();
#endif
#ifdef SWF_ATTN_NOSOFTMAX  // development only: pipeline rate without the softmax
                if (tr) SWF_TR(3, g);
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(lbar(B_PF + b));
                if (leader) release_q();
                l = 1.f;
                continue;
#endif
                uint32_t sa[kKPT];
#pragma unroll
                for (int c = 0; c < kKPT / 32; ++c) ld32(tS + uint32_t(32 * c), sa + 32 * c);
#pragma unroll
                for (int c = 0; c < kKPT / 32; ++c) wait_ld_dep(sa + 32 * c);
                const int kb = (rg.t_lo + j) * BKV + hk * kKPT;
                if (kb < rlo || kb + kKPT > rhi) {  // boundary tile: mask keys outside [rlo, rhi)
#pragma unroll
                    for (int i = 0; i < kKPT; ++i)
                        if (kb + i < rlo || kb + i >= rhi) sa[i] = __float_as_uint(-INFINITY);
                }
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < kKPT; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sa[i]));
                const float pm = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                red[hk * BQ + r] = pm;
                pair_sync(wq);
                float mxr = red[r];
#pragma unroll
                for (int k2 = 1; k2 < kSplit; ++k2) mxr = fmaxf(mxr, red[k2 * BQ + r]);
                const float mx = mxr * sl2;
                pair_sync(wq);  // every split read before the next exchange overwrites
                if (tr) SWF_TR(1, g);
                // Lazy rescale, decided per WARP: the O rescale is a tcgen05.ld / st pair, warp-collective
                // (.sync.aligned), so a row that needs it (running max grew by > 2^kRescale) takes its
                // whole warp along; every lane then moves to max(m, mx). Both key halves of a row sit in
                // warps holding the same 32 rows, so they take the same decision and factor.
                const bool grow = m != -INFINITY && mx > m + kRescale;
                if (__any_sync(0xffffffffu, grow)) {
                    // O *= 2^(m - m_new): P(g-1) V must have landed
                    mbar_wait(bar(B_OD), (g - 1) & 1);
                    fence_after();
                    const float mn = fmaxf(m, mx);
                    const float f = m == -INFINITY ? 0.f : ex2(m - mn);  // m = -inf: O and l are still 0
                    if (!(p.dbg & 1)) o_scale<C::kOC>(tO, f);
                    l *= f;
                    m = mn;
                } else if (m == -INFINITY && mx != -INFINITY) {
                    m = mx;  // first unmasked keys of this row: O and l are still 0, nothing to scale
                }
                const float nb = m == -INFINITY ? 0.f : -m;
                const unsigned long long sl2x2 = f2_pack(sl2, sl2), nbx2 = f2_pack(nb, nb);
                unsigned long long ls2 = 0ull, ls2b = 0ull;
#pragma unroll
                for (int c = 0; c < kKPT / 32; ++c) {  // 32 keys -> 16 packed bf16x2 columns per store
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const unsigned long long sv =
                            (unsigned long long)sa[32 * c + 2 * i] | ((unsigned long long)sa[32 * c + 2 * i + 1] << 32);
                        const unsigned long long z = ffma2(sv, sl2x2, nbx2);
                        unsigned long long pv;
                        if ((i & 7) < kPoly8)  // kPoly8/8 of the exponentials on the FMA pipe
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
                if (tr) SWF_TR(2, g);
                const unsigned long long lsum = fadd2(ls2, ls2b);
                l += lo_f(lsum) + hi_f(lsum);
                wait_st();
                fence_before();
                __syncwarp();
                if (tr) SWF_TR(3, g);
#ifdef SWF_ATTN_TRACE
                if (lane == 0 && blockIdx.x < 2 && g < kTrN) g_trace_w[blockIdx.x][16 + warp - 4][g] = clock64();
#endif
                if (lane == 0) mbar_arrive_cluster(lbar(B_PF + b));
                if (leader) release_q();  // the previous item's O store has long finished reading
            }
            // epilogue: O / l -> bf16 (swin.hpp:319-320 head concat); l is the sum of both halves
            mbar_wait(bar(B_OD), (g - 1) & 1);  // every MMA of this item (incl. its QK^T) complete
            fence_after();
            if (tr) SWF_TR(8, n);
            red[hk * BQ + r] = l;
            pair_sync(wq);
            float lt = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < kSplit; ++k2) lt += red[k2 * BQ + r];  // fixed order: deterministic
            const float inv = 1.f / lt;
            pair_sync(wq);
            const int qb = n & 1;
            if (D >= 64 && p.tmo != nullptr && it.q0 + BQ <= s) {  // (p.tmo: host flag; the map is tmO)
                // whole tile, own rows lw*s + q0 ..: stage in this item's Q buffer (SW128, the TMA
                // box layout) and store with TMA
                uint8_t* stg = sQ + qb * C::kQBytes;
                constexpr int CW = C::kOC < 32 ? C::kOC : 32;  // columns per TMEM load
#pragma unroll 1
                for (int c = 0; c < C::kOC / CW; ++c) {
                    uint32_t o[32];
                    if constexpr (CW == 32) {
                        ld32(tO + uint32_t(c * 32), o);
                        wait_ld_dep(o);
                    } else {
                        ld16(tO + uint32_t(c * 16), o);
                        wait_ld_dep16(o);
                    }
#pragma unroll
                    for (int v = 0; v < CW / 8; ++v) {
                        const int col = hk * C::kOC + c * CW + v * 8;  // first of 8 bf16 = one 16-byte chunk
                        const int ch = (col & 63) >> 3;
                        uint4* dst = reinterpret_cast<uint4*>(stg + (col >> 6) * (BQ * 128) + r * 128 +
                                                              ((ch ^ (r & 7)) << 4));
                        *dst = make_uint4(
                            pack_bf16x2(__uint_as_float(o[8 * v]) * inv, __uint_as_float(o[8 * v + 1]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv),
                            pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv));
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                fence_before();
                softmax_sync();
                if (leader) {
                    // this thread holds row 0 of the tile: its destination row starts the box
                    for (int bx = 0; bx < D / 64; ++bx)
                        tma_store_2d(&tmO, smem_u32(stg + bx * (BQ * 128)), (p.head0 + it.head) * D + bx * 64,
                                     int(oloc));
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    qe_pending = qb;
                }
            } else {
                __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o_dst[orank]) + oloc * p.ldo +
                                   (p.head0 + it.head) * D + hk * C::kOC;
                o_store<C::kOC>(tO, O, inv, q < s);
                fence_before();
                if (leader) mbar_arrive(bar(B_QE + qb));
            }
            __syncwarp();
            if (tr) SWF_TR(9, n);
            if (lane == 0) mbar_arrive_cluster(lbar(B_OF));  // O may be overwritten by the next item's first PV
        }
        if (leader && qe_pending >= 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    fence_before();
    cluster_sync_all();  // the peer may still arrive on / commit to this CTA until here
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// ============================================================================================
// Ping-pong kernel (default). The 8 softmax warps of a CTA form two groups that take alternate
// 64-key tiles of an item -- group 0 the even tiles, group 1 the odd ones -- each thread owning a
// whole query row of its tile, with its own running max / sum and its own O accumulator in TMEM
// (O0 / O1). The groups run out of phase: while one loads S and reduces its row maximum, the other's
// exponentials keep the sub-partition's MUFU and FMA pipes busy; there is no per-tile max exchange
// and no named barrier between warps. S is a ring of four 64-column buffers, so QK^T runs two tiles
// ahead of each group (QK^T(g) waits only for P(g-4) V), which takes the tensor-core round trip
// (P V of a tile, QK^T of the group's next tile) off the softmax critical path. The two partial
// outputs are merged once per item in the epilogue:
//   O = (O0 2^(m0-M) + O1 2^(m1-M)) / (l0 2^(m0-M) + l1 2^(m1-M)),  M = max(m0, m1)
// (each group writes half of the head's columns).
// TMEM (per CTA): S ring [0, 256) (buffer b at 64 b), O0 [256, 256+D), O1 [256+D, 256+2D).
// Operands per 64-key tile: each CTA loads its 32 keys of K (QK^T: M = 256 pair-wide, N = 64 split
// 32 / 32 across the pair) and its D/2 rows of V^T (P V: N = D split across the pair, K = 64 keys).
namespace pp {
constexpr int KT = 64;  // keys per tile
constexpr int kNS = 4;  // S buffers
enum : int {
    QF = 0, QE = 2, KF = 4, KE = 12, VF = 20, VE = 28, SF = 36, PF = 40, SFREE = 44, OD = 48, OF = 50, NUM = 51
};
constexpr uint32_t kTO = 256;
constexpr int kThreads = 384;
template <int D>
struct Cfg {
    static constexpr int kSw = D >= 64 ? 128 : 2 * D;
    static constexpr int kColsPerBox = kSw / 2;
    static constexpr int kBoxes = D / kColsPerBox;
    static constexpr int kQBytes = BQ * D * 2;
    static constexpr int kKHalf = (KT / 2) * D * 2;  // this CTA's 32 keys of a K tile
    static constexpr int kVHalf = (D / 2) * KT * 2;  // this CTA's D/2 rows of a V^T tile
    static constexpr int kNK = 8, kNV = 8;
    static constexpr int kRedBytes = 4 * BQ * 4;  // (m, l) x 2 groups x BQ rows
    static constexpr int kSmem = 2 * kQBytes + kNK * kKHalf + kNV * kVHalf + kRedBytes + 512 + 1024;
    static constexpr int kOC = D / 2;  // O columns per thread in the epilogue (its group's half)
    static constexpr uint32_t kIdescS = idesc_bf16(2 * BQ, KT);
    static constexpr uint32_t kIdescO = idesc_bf16(2 * BQ, D);
};
// QK^T of one 64-key tile: D/16 k-steps; A = Q (BQ rows per box), B = this CTA's 32 keys per box
template <int D>
__device__ __forceinline__ void issue_s(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if constexpr (D == 128)
        mma2_ss_x8<2, 4, 6, 1024, 1026, 1028, 1030, 2, 4, 6, 256, 258, 260, 262>(d, a, b, idesc);
    else if constexpr (D == 64)
        mma2_ss_x4<2, 4, 6, 2, 4, 6>(d, a, b, idesc);
    else
        mma2_ss_x2<2, 2>(d, a, b, idesc);
}
// P V of one tile: 4 pair-wide TS MMAs (K = 16 keys each); P of keys [16 kk, 16 kk + 16) at S
// columns [8 kk, 8 kk + 8) (bf16 pairs in key order), B = the V^T half (one SW128 box, 64 keys)
__device__ __forceinline__ void issue_pv(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n"
        ".reg .pred e, p0, pt;\n"
        ".reg .b64 b;\n"
        ".reg .b32 a;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p0, %4, 0;\n"
        "setp.eq.b32 pt, %3, %3;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p0;\n"
        "add.u32 a, %1, 8;\n"
        "add.s64 b, %2, 2;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, 16;\n"
        "add.s64 b, %2, 4;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.u32 a, %1, 24;\n"
        "add.s64 b, %2, 6;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, pt;\n"
        "}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc0));
}
__device__ __forceinline__ void quad_sync(int quadrant) {  // the two warps (one per group) of a lane quadrant
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quadrant) : "memory");
}
__device__ __forceinline__ void all_softmax_sync() { asm volatile("bar.sync 5, 256;" ::: "memory"); }
__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// key range of a work item (seam groups) in 64-key tiles, the union over the pair
__device__ __forceinline__ Range range_of(const AttnParams& p, const Item& it) {
    Range r;
    const int s = p.s;
    const int gw = p.lay.loc2glob[it.lw];
    r.masked = p.lay.g.shift > 0 && (gw / p.lay.g.nx) == p.lay.g.ny - 1;
    r.split = r.masked ? (p.w - p.lay.g.shift) * p.w : s;
    const int qlast = min(it.qp0 + 2 * BQ, s) - 1;
    const int kv_lo = (r.masked && it.qp0 >= r.split) ? r.split : 0;
    const int kv_hi = (r.masked && qlast < r.split) ? r.split : s;
    r.t_lo = kv_lo / KT;
    r.ntiles = (kv_hi + KT - 1) / KT - r.t_lo;
    return r;
}
}  // namespace pp

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pp::kThreads, 1)
    k_attn_pp(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, AttnParams p,
              int n_items) {
    using C = pp::Cfg<D>;
    constexpr int KT = pp::KT;
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sK = sm + 2 * C::kQBytes;
    uint8_t* sV = sK + C::kNK * C::kKHalf;
    float* red = reinterpret_cast<float*>(sV + C::kNV * C::kVHalf);  // [m0 | m1 | l0 | l1][BQ]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kNV * C::kVHalf + C::kRedBytes);
    auto bar = [&](int slot) { return smem_u32(&bars[slot]); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[pp::NUM]);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = p.s;
    const int npairs = (s + 2 * BQ - 1) / (2 * BQ);
    const int crank = int(cta_rank());
    const bool lead = crank == 0;
    auto lbar = [&](int slot) { return map_to_rank(bar(slot), 0); };
    const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar(pp::QF + i), 1);
            mbar_init(bar(pp::QE + i), 1);
            mbar_init(bar(pp::OD + i), 1);
        }
        for (int i = 0; i < pp::kNS; ++i) {
            mbar_init(bar(pp::SF + i), 1);
            mbar_init(bar(pp::PF + i), 2 * 4);
            mbar_init(bar(pp::SFREE + i), 1);
        }
        for (int i = 0; i < C::kNK; ++i) {
            mbar_init(bar(pp::KF + i), 1);
            mbar_init(bar(pp::KE + i), 1);
        }
        for (int i = 0; i < C::kNV; ++i) {
            mbar_init(bar(pp::VF + i), 1);
            mbar_init(bar(pp::VE + i), 1);
        }
        mbar_init(bar(pp::OF), 2 * 8);
        fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");

    if (warp == 0) {
        // ===== TMA: Q (double-buffered across items) and the K ring (this CTA's 32 keys of a tile)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
            int g = 0, n = 0;
            for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
                const Item it = item_of(itx, npairs, p.heads, crank);
                const Range rg = pp::range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                const int qb = n & 1;
                mbar_sleep_wait<SWF_ATTN_PBACKOFF>(bar(pp::QE + qb), ((n >> 1) & 1) ^ 1);
                if (lead) mbar_expect_tx(bar(pp::QF + qb), 2 * C::kQBytes);
                for (int b = 0; b < C::kBoxes; ++b)
                    tma_load_2cta(smem_u32(sQ + qb * C::kQBytes + b * BQ * C::kSw), &tmQ, lbar(pp::QF + qb),
                                  b * C::kColsPerBox, plane * s + it.q0);
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g % C::kNK;
                    mbar_sleep_wait<SWF_ATTN_PBACKOFF>(bar(pp::KE + st), ((g / C::kNK) & 1) ^ 1);
                    if (lead) mbar_expect_tx(bar(pp::KF + st), 2 * C::kKHalf);
                    for (int b = 0; b < C::kBoxes; ++b)
                        tma_load_2cta(smem_u32(sK + st * C::kKHalf + b * (KT / 2) * C::kSw), &tmK, lbar(pp::KF + st),
                                      b * C::kColsPerBox, plane * s + (rg.t_lo + j) * KT + crank * (KT / 2));
                }
            }
        }
    } else if (warp == 3) {
        // ===== TMA: the V^T ring (this CTA's D/2 rows x 64 keys, one SW128 box)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
            int g = 0;
            for (int itx = cluster_id; itx < n_items; itx += n_clusters) {
                const Item it = item_of(itx, npairs, p.heads, crank);
                const Range rg = pp::range_of(p, it);
                const int plane = it.lw * p.heads + it.head;
                for (int j = 0; j < rg.ntiles; ++j, ++g) {
                    const int st = g % C::kNV;
                    mbar_sleep_wait<SWF_ATTN_PBACKOFF>(bar(pp::VE + st), ((g / C::kNV) & 1) ^ 1);
                    if (lead) mbar_expect_tx(bar(pp::VF + st), 2 * C::kVHalf);
                    tma_load_2cta(smem_u32(sV + st * C::kVHalf), &tmV, lbar(pp::VF + st), (rg.t_lo + j) * KT,
                                  plane * D + crank * (D / 2));
                }
            }
        }
    } else if (warp == 1 && lead) {
        // ===== QK^T issuer for the pair: S(g) into ring buffer g % 4 once P(g-4) V has completed
        if (tmem != 0) __trap();
        const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK);
        int g = 0, n = 0;
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Range rg = pp::range_of(p, item_of(itx, npairs, p.heads, crank));
            const int qb = n & 1;
            mbar_sleep_wait(bar(pp::QF + qb), (n >> 1) & 1);
            if (lane == 0) SWF_TR(6, n);
#ifdef SWF_ATTN_TRACE
            if (lane == 0 && blockIdx.x < 2 && n < kTrN) g_trace[blockIdx.x][1][n] = (unsigned long long)g;
#endif
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int st = g % C::kNK, b = g % pp::kNS;
                if (lane == 0) SWF_TR(10, g);
                mbar_sleep_wait(bar(pp::KF + st), (g / C::kNK) & 1);
                if (lane == 0) SWF_TR(11, g);
                mbar_sleep_wait(bar(pp::SFREE + b), ((g / pp::kNS) & 1) ^ 1);
                if (lane == 0) SWF_TR(12, g);
                fence_after();
                const uint64_t a0 = desc_kmajor(sQa + uint32_t(qb * C::kQBytes), C::kSw);
                const uint64_t b0 = desc_kmajor(sKa + uint32_t(st * C::kKHalf), C::kSw);
                pp::issue_s<D>(uint32_t(b * KT), a0, b0, C::kIdescS);
                commit2_mc(bar(pp::SF + b));
                commit2_mc(bar(pp::KE + st));
            }
        }
    } else if (warp == 2 && lead) {
        // ===== P V issuer: tile j of an item accumulates into O[j % 2]
        const uint32_t sVa = smem_u32(sV);
        int g = 0, n = 0;
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Range rg = pp::range_of(p, item_of(itx, npairs, p.heads, crank));
            for (int j = 0; j < rg.ntiles; ++j, ++g) {
                const int b = g % pp::kNS, vs = g % C::kNV, par = j & 1;
                if (j == 0 && n >= 1) mbar_sleep_wait(bar(pp::OF), (n - 1) & 1);  // O0 / O1 of the last item read
                if (j == 0 && lane == 0) SWF_TR(7, n);
                if (lane == 0) SWF_TR(13, g);
                mbar_sleep_wait(bar(pp::PF + b), (g / pp::kNS) & 1);
                if (lane == 0) SWF_TR(14, g);
                mbar_sleep_wait(bar(pp::VF + vs), (g / C::kNV) & 1);
                if (lane == 0) SWF_TR(15, g);
                fence_after();
                const uint64_t b0 = desc_kmajor(sVa + uint32_t(vs * C::kVHalf), 128);
                pp::issue_pv(pp::kTO + uint32_t(par * D), uint32_t(b * KT), b0, C::kIdescO, j >= 2 ? 1u : 0u);
                commit2_mc(bar(pp::OD + par));
                commit2_mc(bar(pp::VE + vs));
                commit2(bar(pp::SFREE + b));
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: group grp takes the tiles j % 2 == grp, one query row per thread
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        const int grp = (warp - 4) >> 2;
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lane_off = uint32_t(wq * 32) << 16;
        const float sl2 = p.scale * 1.4426950408889634f;
        const bool leader = threadIdx.x == 128;  // issues the O TMA stores, releases Q buffers
        int qe_pending = -1;
        auto release_q = [&]() {
            if (qe_pending >= 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_arrive(bar(pp::QE + qe_pending));
                qe_pending = -1;
            }
        };
        int g = 0, n = 0;
        int cnt0 = 0, cnt1 = 0;  // P V products issued into O0 / O1 so far (all items); scalars, not an
                                 // array: indexed by the group it would live in local memory
        const unsigned long long sl2x2 = f2_pack(sl2, sl2);
        // P = 2^(s sl2 - m) of this thread's 64 keys into 32 packed bf16x2 registers; returns the sum
        auto exps = [&](const uint32_t* sa, float m, uint32_t* pk) {
            const float nb = m == -INFINITY ? 0.f : -m;
            const unsigned long long nbx2 = f2_pack(nb, nb);
            unsigned long long ls2 = 0ull, ls2b = 0ull;
#pragma unroll
            for (int i = 0; i < KT / 2; ++i) {
                const unsigned long long sv = (unsigned long long)sa[2 * i] | ((unsigned long long)sa[2 * i + 1] << 32);
                const unsigned long long z = ffma2(sv, sl2x2, nbx2);
                unsigned long long pv;
                if ((i & 7) < kPoly8)  // kPoly8 / 8 of the exponentials on the FMA pipe
                    pv = ex2_poly2(z);
                else
                    pv = f2_pack(ex2(lo_f(z)), ex2(hi_f(z)));
                if (i & 1)
                    ls2b = fadd2(ls2b, pv);
                else
                    ls2 = fadd2(ls2, pv);
                pk[i] = pack_bf16x2(lo_f(pv), hi_f(pv));
            }
            const unsigned long long lsum = fadd2(ls2, ls2b);
            return lo_f(lsum) + hi_f(lsum);
        };
        auto tile_max = [&](const uint32_t* sa) {  // 3-input max (FMNMX3), 4 chains of 16 keys
            float mx4[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
                mx4[c] = pp::max3(__uint_as_float(sa[16 * c]), __uint_as_float(sa[16 * c + 1]),
                                  __uint_as_float(sa[16 * c + 2]));
#pragma unroll
            for (int i = 3; i < 16; i += 2)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    mx4[c] = i + 1 < 16 ? pp::max3(mx4[c], __uint_as_float(sa[16 * c + i]),
                                                   __uint_as_float(sa[16 * c + i + 1]))
                                        : fmaxf(mx4[c], __uint_as_float(sa[16 * c + i]));
            return fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
        };
        for (int itx = cluster_id; itx < n_items; itx += n_clusters, ++n) {
            const Item it = item_of(itx, npairs, p.heads, crank);
            const Range rg = pp::range_of(p, it);
            const int q = it.q0 + r;
            const int rlo = (rg.masked && q >= rg.split) ? rg.split : 0;
            const int rhi = (rg.masked && q < rg.split) ? rg.split : s;
            int orank = 0;
            const i64 oloc = q < s ? p.lay.wtok_to_loc(p.wp_rank, it.lw, q, &orank) : 0;
            float m = -INFINITY, l = 0.f;
            const int g0 = g;
            auto s_col = [&](int jj) { return lane_off + uint32_t(((g0 + jj) % pp::kNS) * KT); };
            auto s_bar = [&](int jj) { return bar(pp::SF + (g0 + jj) % pp::kNS); };
            auto s_par = [&](int jj) { return uint32_t(((g0 + jj) / pp::kNS) & 1); };
            auto s_load = [&](int jj, uint32_t* s) {  // wait for S of tile jj, start its TMEM load
                mbar_wait(s_bar(jj), s_par(jj));
                if (lane == 0) SWF_TRW(warp - 4, g0 + jj);
                fence_after();
                ld32(s_col(jj), s);
                ld32(s_col(jj) + 32u, s + 32);
            };
            // one tile whose S is in registers: seam mask, row max, lazy rescale, P, hand-off to P V
            auto tile = [&](int j, uint32_t* sa) {
                const int b = (g0 + j) % pp::kNS;
                const int k = (grp ? cnt1 : cnt0) + (j >> 1) + 1;  // P V products into O[grp] incl. this tile's
                const uint32_t tS = s_col(j);
                const int kb = (rg.t_lo + j) * KT;
                if (kb < rlo || kb + KT > rhi) {  // boundary tile: keys outside [rlo, rhi) get -inf
#pragma unroll
                    for (int i = 0; i < KT; ++i)
                        if (kb + i < rlo || kb + i >= rhi) sa[i] = __float_as_uint(-INFINITY);
                }
                const float mx = tile_max(sa);
                if (__any_sync(0xffffffffu, m != -INFINITY && mx > m + kRescale)) {
                    // lazy rescale, warp-uniform (tcgen05.ld / st are warp-collective): O[grp] *= 2^(m - m_new)
                    // once this group's previous P V into O[grp] has landed
                    mbar_wait(bar(pp::OD + grp), (k - 2) & 1);
                    fence_after();
                    const float mn = fmaxf(m, mx);
                    const float f = m == -INFINITY ? 0.f : ex2(m - mn);
                    if (!(p.dbg & 1)) o_scale<D>(lane_off + pp::kTO + uint32_t(grp * D), f);
                    l *= f;
                    m = mn;
                } else if (m == -INFINITY) {
                    m = mx;  // first unmasked keys of this row: O and l are still 0
                }
                l += exps(sa, m, sa);  // P packed in place: pair i reads sa[2i], sa[2i+1], writes sa[i]
                st16(tS, sa);
                st16(tS + 16u, sa + 16);
                wait_st();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(lbar(pp::PF + b));
                if (lane == 0) SWF_TRW(16 + warp - 4, g0 + j);
                if (leader) release_q();
            };
            // this group's tiles j = grp, grp + 2, ... (prefetching the next S from TMEM during a tile
            // measured +21% cycles per launch: register pressure; dropped)
            for (int j = grp; j < rg.ntiles; j += 2) {
                uint32_t sa[KT];
                s_load(j, sa);
                wait_ld_dep(sa);
                wait_ld_dep(sa + 32);
                if (lane == 0) SWF_TRW(8 + warp - 4, g0 + j);
                tile(j, sa);
            }
            cnt0 += (rg.ntiles + 1) >> 1;
            cnt1 += rg.ntiles >> 1;
            g = g0 + rg.ntiles;
            if (warp == 4 && lane == 0) SWF_TR(8, n);
            // ---- epilogue: merge the two groups' partial softmax states, O / l -> bf16
            red[grp * BQ + r] = m;
            red[(2 + grp) * BQ + r] = l;
            pp::quad_sync(wq);
            const float m0 = red[r], m1 = red[BQ + r], l0 = red[2 * BQ + r], l1 = red[3 * BQ + r];
            pp::quad_sync(wq);  // both read before the next item's epilogue overwrites
            if (warp == 4 && lane == 0) SWF_TR(2, n);
            const float M = fmaxf(m0, m1);
            const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - M), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - M);
            const float inv = 1.f / (l0 * f0 + l1 * f1);
            if (p.lse && grp == 0 && q < s)  // BF16 training mode: the row's log2-sum-exp for the backward
                p.lse[(i64(it.lw) * p.heads + it.head) * s + q] = M + __log2f(l0 * f0 + l1 * f1);
            const bool has1 = rg.ntiles >= 2;  // item-uniform: O1 holds this item's odd tiles
            mbar_wait(bar(pp::OD + 0), (cnt0 - 1) & 1);
            if (has1) mbar_wait(bar(pp::OD + 1), (cnt1 - 1) & 1);
            if (warp == 4 && lane == 0) SWF_TR(3, n);
            fence_after();
            const uint32_t tO0 = lane_off + pp::kTO + uint32_t(grp * C::kOC), tO1 = tO0 + uint32_t(D);
            const int qb = n & 1;
            constexpr int CW = C::kOC < 16 ? C::kOC : 16;  // columns per TMEM load
            auto combined = [&](int c, uint32_t* o) {      // this thread's columns [c CW, c CW + CW), merged
                uint32_t o1[CW];
                if constexpr (CW == 16) {
                    ld16(tO0 + uint32_t(c * CW), o);
                    if (has1) ld16(tO1 + uint32_t(c * CW), o1);
                    wait_ld_dep16(o);
                    if (has1) wait_ld_dep16(o1);
                } else {
                    ld8(tO0 + uint32_t(c * CW), o);
                    if (has1) ld8(tO1 + uint32_t(c * CW), o1);
                    wait_ld_dep8(o);
                    if (has1) wait_ld_dep8(o1);
                }
#pragma unroll
                for (int i = 0; i < CW; ++i) {
                    float v = __uint_as_float(o[i]) * f0;
                    if (has1) v = fmaf(__uint_as_float(o1[i]), f1, v);
                    o[i] = __float_as_uint(v * inv);
                }
            };
            if (D >= 64 && p.tmo != nullptr && it.q0 + BQ <= s) {
                uint8_t* stg = sQ + qb * C::kQBytes;  // SW128 staging in this item's Q buffer (TMA box layout)
#pragma unroll 1
                for (int c = 0; c < C::kOC / CW; ++c) {
                    uint32_t o[CW];
                    combined(c, o);
#pragma unroll
                    for (int v = 0; v < CW / 8; ++v) {
                        const int col = grp * C::kOC + c * CW + v * 8;
                        const int ch = (col & 63) >> 3;
                        uint4* dst = reinterpret_cast<uint4*>(stg + (col >> 6) * (BQ * 128) + r * 128 +
                                                              ((ch ^ (r & 7)) << 4));
                        *dst = make_uint4(pack_bf16x2(__uint_as_float(o[8 * v]), __uint_as_float(o[8 * v + 1])),
                                          pack_bf16x2(__uint_as_float(o[8 * v + 2]), __uint_as_float(o[8 * v + 3])),
                                          pack_bf16x2(__uint_as_float(o[8 * v + 4]), __uint_as_float(o[8 * v + 5])),
                                          pack_bf16x2(__uint_as_float(o[8 * v + 6]), __uint_as_float(o[8 * v + 7])));
                    }
                }
                if (warp == 4 && lane == 0) SWF_TR(4, n);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                fence_before();
                pp::all_softmax_sync();
                if (warp == 4 && lane == 0) SWF_TR(5, n);
                if (leader) {
                    for (int bx = 0; bx < D / 64; ++bx)
                        tma_store_2d(&tmO, smem_u32(stg + bx * (BQ * 128)), (p.head0 + it.head) * D + bx * 64,
                                     int(oloc));
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    qe_pending = qb;
                }
            } else {
                __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o_dst[orank]) + oloc * p.ldo +
                                   (p.head0 + it.head) * D + grp * C::kOC;
#pragma unroll 1
                for (int c = 0; c < C::kOC / CW; ++c) {
                    uint32_t o[CW];
                    combined(c, o);
                    if (q < s) {
                        uint4* d4 = reinterpret_cast<uint4*>(O + c * CW);
#pragma unroll
                        for (int v = 0; v < CW / 8; ++v)
                            d4[v] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * v]), __uint_as_float(o[8 * v + 1])),
                                               pack_bf16x2(__uint_as_float(o[8 * v + 2]), __uint_as_float(o[8 * v + 3])),
                                               pack_bf16x2(__uint_as_float(o[8 * v + 4]), __uint_as_float(o[8 * v + 5])),
                                               pack_bf16x2(__uint_as_float(o[8 * v + 6]), __uint_as_float(o[8 * v + 7])));
                    }
                }
                fence_before();
                pp::all_softmax_sync();  // both groups done with this item's Q buffer and O columns
                if (leader) mbar_arrive(bar(pp::QE + qb));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lbar(pp::OF));  // O0 / O1 may be overwritten
            if (warp == 4 && lane == 0) SWF_TR(9, n);
        }
        if (leader && qe_pending >= 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    fence_before();
    cluster_sync_all();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// SWF_ATTN=split selects the key-split kernel (two threads per query row, one shared O); the default
// is the ping-pong kernel.
inline bool use_split_kernel() {
    static const bool v = [] {
        const char* e = std::getenv("SWF_ATTN");
        return e && std::string(e) == "split";
    }();
    return v;
}

inline int pp_grid(const AttnParams& p) {
    const int npairs = (p.s + 2 * BQ - 1) / (2 * BQ);
    return 2 * std::min(npairs * p.heads * p.nloc, 74);
}

template <int D>
void launch(const AttnParams& p, cudaStream_t st) {
    using C = ACfg<D>;
    const int npairs = (p.s + 2 * BQ - 1) / (2 * BQ);
    const int n_items = npairs * p.heads * p.nloc;
    const int grid = 2 * std::min(n_items, 74);  // 2-CTA clusters, one CTA per SM
    const CUtensorMap& tq = *reinterpret_cast<const CUtensorMap*>(p.tmq);
    const CUtensorMap& tk = *reinterpret_cast<const CUtensorMap*>(p.tmk);
    const CUtensorMap& tk2 = *reinterpret_cast<const CUtensorMap*>(p.tmk2 ? p.tmk2 : p.tmk);
    const CUtensorMap& tv = *reinterpret_cast<const CUtensorMap*>(p.tmv);
    const CUtensorMap& to = *reinterpret_cast<const CUtensorMap*>(p.tmo ? p.tmo : p.tmv);
    if (use_split_kernel())
        k_attn_tc<D><<<grid, kThreads, C::kSmem, st>>>(tq, tk, tv, to, p, n_items);
    else
        k_attn_pp<D><<<pp_grid(p), pp::kThreads, pp::Cfg<D>::kSmem, st>>>(tq, tk2, tv, to, p, n_items);
    SWF_LAUNCH_CHECK();
#ifdef SWF_ATTN_TRACE
    if (const char* path = getenv("SWF_ATTN_TRACE_OUT")) {
        static unsigned long long h[2][16][kTrN];
        SWF_CUDA(cudaStreamSynchronize(st));
        SWF_CUDA(cudaMemcpyFromSymbol(h, g_trace, sizeof(h)));
        if (FILE* f = fopen(path, "wb")) {
            fwrite(h, sizeof(h), 1, f);
            static unsigned long long hw[2][32][kTrN];
            SWF_CUDA(cudaMemcpyFromSymbol(hw, g_trace_w, sizeof(hw)));
            fwrite(hw, sizeof(hw), 1, f);
            fclose(f);
        }
    }
#endif
}

}  // namespace

template <int D>
void configure_attn() {  // dynamic shared memory limits of this head size's kernels (current device)
    SWF_CUDA(cudaFuncSetAttribute(k_attn_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<D>::kSmem));
    SWF_CUDA(cudaFuncSetAttribute(k_attn_pp<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, pp::Cfg<D>::kSmem));
}
void preload_attn_kernels() {
    cudaFuncAttributes a;
    const void* k[] = {(const void*)k_attn_tc<32>, (const void*)k_attn_tc<64>, (const void*)k_attn_tc<128>,
                       (const void*)k_attn_pp<32>, (const void*)k_attn_pp<64>, (const void*)k_attn_pp<128>};
    for (const void* f : k) SWF_CUDA(cudaFuncGetAttributes(&a, f));
    configure_attn<32>();
    configure_attn<64>();
    configure_attn<128>();
}

void attention_bf16(const AttnParams& p, cudaStream_t st) {
    if (!p.tmq || !p.tmk || !p.tmv) throw CudaError("attention_bf16: TMA descriptors missing");
    if (!use_split_kernel() && !p.tmk2) throw CudaError("attention_bf16: the K map with 32-row boxes is missing");
    if (use_split_kernel() && p.lse) throw CudaError("attention_bf16: the row statistics need the ping-pong kernel");
    switch (p.d) {
        case 32: launch<32>(p, st); break;
        case 64: launch<64>(p, st); break;
        case 128: launch<128>(p, st); break;
        default: throw CudaError("attention_bf16: head_dim must be 32, 64 or 128");
    }
}

}  // namespace swf
