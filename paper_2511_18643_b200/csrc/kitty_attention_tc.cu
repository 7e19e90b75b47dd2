// Fused dequant-attention decode on the 5th-generation tensor cores (tcgen05).
//
// Semantics: KittyCacheState.attend (cache.py:217-252) per (sequence, KV head)
// unit -- logits q.k / sqrt(d) over sink | key pages | key q-buffer, fp32
// max-subtracted softmax, probabilities times values over sink | value pages |
// value q-buffer | local -- with the 2-bit pages dequantised inside the loop
// (Alg. 1) instead of from cached f32 rows.
//
// Design.  One persistent CTA per SM, warp-specialised,
// one page pair (key page i, value page i of a unit) flowing through:
//
//   TMA warp      cp.async.bulk of the KTYP key + value bodies (+ the unit's q
//                 rows on an item's first page) into a 6-stage ring;
//   WG-A (4 w)    key page -> u8 operand tile: one LOP3 per 4 codes, no
//                 transposes -- byte j-code of a packed byte becomes a byte of
//                 value code * 4^j, which is the tensor core's MN-major layout
//                 with the token order permuted inside 16-token chunks; the
//                 boosted channels' high bits are 16 more K rows.  The scale
//                 fold puts the per-channel scale into B: B[d] = q_d alpha s_d
//                 (4 q alpha s for boosted rows), B_z[d] = q_d alpha z_d, as
//                 15-bit fixed point split into two int8 columns (lo, hi);
//   MMA thread    tcgen05.mma.kind::i8 (u8 x s8 -> s32 in TMEM, M = 128 tokens,
//                 N = 16): S = A_K x B, and a constant "ones" tile x B for
//                 sum_d q alpha z_d; then O = A_V x P for the previous page;
//   WG-B (4 w)    softmax: thread = token (TMEM lane), logits from the two
//                 integer accumulators, page max over 128 lanes (f16x2 shuffles
//                 + one named barrier), p = 2^(logit - m), P * s_token as int8
//                 (lo, hi) -> B operand of the value MMA; running l, l_z;
//   WG-C (4 w)    value page -> u8 operand tile (same LOP3 expansion, channels
//                 permuted); then the output correction of the previous page:
//                 thread = channel, o = o * corr + O / 4^j * step;
//   FP warps (2)  full-precision tokens (sink, q-buffers, local window) on CUDA
//                 cores, 32 tokens per item, from their own queue.
//
// Every item writes a partial (acc, m, l) per query row; combine_kernel merges
// a unit's partials (log-sum-exp) and writes the bf16 / f32 output.
#include "kitty_attention.cuh"
#include "kitty_codec.cuh"

namespace kitty {
namespace tcattn {

constexpr int D = 128;
constexpr int G = 128;
constexpr int NST = 6;             // TMA ring stages
constexpr int kKeySlotMax = 5760;  // d_boost = 32
constexpr int kValueSlot = 4608;
constexpr int kFpChunk = 32;       // fp tokens per fp item
constexpr int kFpWarps = 2;
constexpr int kThreads = (14 + kFpWarps) * 32;  // WG-A 0-3, WG-B 4-7, WG-C 8-11, TMA 12, MMA 13, FP 14-15
constexpr float kAlpha = 0.12751743074f;        // log2(e) / sqrt(128)
constexpr int kQuant = 16000;                   // fixed-point range of the int8 (lo, hi) pairs (< 2^14)
constexpr int kTileA = 1024 * 16;               // 128 x 128 u8 operand tile
constexpr int kTileAK = 1024 * 20;              // + 32 boosted rows

constexpr uint32_t FL_FIRST = 1, FL_LAST = 2, FL_END = 4;

struct StageInfo {
    int unit, page, flags, slot;
};
struct KInfo {
    float stepx, stepz;
    int flags, unit, slot, pad[3];
};
struct RingEntry {
    float corr[8];
    float lz[8];
    int tag;
    int pad[15];
};

// Shared-memory layout of one CTA (dynamic, 1024-aligned regions).
template <int GROUP>
struct Smem {
    static constexpr int NX = GROUP * 2 > 8 ? GROUP * 2 : 8;  // bytes of the q*s columns in a B row
    static constexpr int NQK = 2 * NX;                          // B row: (q s | q z) columns
    static constexpr int NCH = NQK / 16;                        // 16-byte MN chunks per B row
    static constexpr int NP = 16;                               // value-MMA B row (p s lo/hi, padded)
    static constexpr int kStage = kKeySlotMax + kValueSlot + GROUP * D * 2;
    static constexpr int kStageAl = (kStage + 127) / 128 * 128;
    static constexpr int kBQK = 160 * NQK;
    // offsets
    static constexpr int o_ring = 0;
    static constexpr int o_ak = (o_ring + NST * kStageAl + 1023) / 1024 * 1024;
    static constexpr int o_av = o_ak + 2 * kTileAK;
    static constexpr int o_ones = o_av + 2 * kTileA;
    static constexpr int o_bqk = o_ones + 4096;
    static constexpr int o_bp = o_bqk + 2 * kBQK;
    static constexpr int o_vmeta = o_bp + 2 * 128 * NP;          // [2][128] float2 (s, z)
    static constexpr int o_fp = o_vmeta + 2 * 128 * 8;           // per fp warp scratch
    static constexpr int kFpBytes = kKeySlotMax + GROUP * D * 2 + GROUP * kFpChunk * 4;
    static constexpr int kFpAl = (kFpBytes + 127) / 128 * 128;
    static constexpr int o_ring4 = o_fp + kFpWarps * kFpAl;      // RingEntry[4]
    static constexpr int o_misc = o_ring4 + 4 * sizeof(RingEntry);
    // misc: stage info [NST], kinfo [2], vinfo [2] (float invp), xch [3][4][16] floats, barriers
    static constexpr int o_sinfo = o_misc;
    static constexpr int o_kinfo = o_sinfo + NST * 16;
    static constexpr int o_vinfo = o_kinfo + 2 * 32;
    static constexpr int o_xch = o_vinfo + 16;
    static constexpr int o_bar = o_xch + 3 * 64 * 4;  // two page-max buffers + one item-end sum buffer
    static constexpr int kBars = 2 * NST + 9 * 2;
    static constexpr int o_tmem = o_bar + kBars * 8;
    static constexpr int kBytes = o_tmem + 16;
    // TMEM columns: S[b] = (D1 | D2) at b * 2 NQK, O[b] at 4 NQK + b * NP
    static constexpr int kTmemCols = (4 * NQK + 2 * NP) <= 128 ? 128 : 256;
};

struct Params {
    KittyCacheDesc c;
    const uint16_t* q;
    void* out;
    int out_dtype;
    int cs[3];   // page-chunk size of schedule level 0 / 1 / 2
    int cmx[3];  // chunks per unit bound of each level
    int fmax;    // fp items per unit bound
    int nslot;   // partial slots per unit: fmax + cmx[0] + cmx[1] + cmx[2]
    int units;
    int* ctr;    // [0] next page item, [1] finished CTAs, [2] next fp item
    float* part;
};

// ---- PTX helpers -------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// UMMA shared-memory descriptor, no swizzle (canonical interleaved layout):
// 16-byte MN chunks of 8 K rows = 128-byte core matrices; LBO = stride between
// K groups of 8, SBO = stride between MN chunks (tools/probe_umma_i8.cu).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// kind::i8 instruction descriptor: D s32, A u8 MN-major, B s8 MN-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[N]);
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t a, uint32_t (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a) : "memory");
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t a, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(a)
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t a, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(a)
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t a, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(a)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t x) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
}

__device__ __forceinline__ float h2f(uint32_t h) { return __half2float(__ushort_as_half((unsigned short)h)); }
__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ int f2i(float x) {
    int r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// X = 128 h + l (l in [0, 127], h = X >> 7 in [-128, 127]) -> 16-bit (l | h << 8)
__device__ __forceinline__ uint32_t enc16(int x) { return (uint32_t)(x + (x & ~127)); }
// bytes (l0, h0, l1, h1)
__device__ __forceinline__ uint32_t enc_pair(int x0, int x1) { return prmt(enc16(x0), enc16(x1), 0x5410); }

// Byte j-code of every byte of a packed word, kept in place: value code * 4^j.
constexpr uint32_t M0 = 0x03030303u, M1 = 0x0C0C0C0Cu, M2 = 0x30303030u, M3 = 0xC0C0C0C0u;
// Operand tile address of (16-row MN chunk, K row): 128-byte core matrices,
// MN chunks 128 B apart, K groups of 8 rows 1024 B apart.
__device__ __forceinline__ uint32_t a_off(int mchunk, int k) { return 16 * (k & 7) + 128 * mchunk + 1024 * (k >> 3); }
// TMEM lane m of a permuted tile <-> token (or channel) index and its 4^-j weight
__device__ __forceinline__ int perm_index(int m) { return 16 * (m >> 4) + 4 * (m & 3) + ((m >> 2) & 3); }
__device__ __forceinline__ float perm_weight(int m) {
    const int j = (m >> 2) & 3;
    return j == 0 ? 1.f : (j == 1 ? 0.25f : (j == 2 ? 0.0625f : 0.015625f));
}

// ---- work schedule -----------------------------------------------------------------

struct UnitGeom {
    int n, kp, vp, nfp;
};
__device__ __forceinline__ UnitGeom unit_geom(const KittyCacheDesc& c, int u) {
    UnitGeom g;
    g.n = c.unit_len[u];
    const int S = c.cfg.s;
    const int past = g.n > S ? g.n - S : 0;
    g.kp = past / G;
    g.vp = (past - min(c.cfg.r, past)) / G;
    g.nfp = g.n > S ? S + (past - g.vp * G) : g.n;  // sink + value fp tokens
    return g;
}
// Pages of a unit in three levels of decreasing chunk size: [0, 3vp/5) in
// chunks of cs[0], [3vp/5, 9vp/10) in cs[1], the rest page by page; the queue
// serves level 0 of every unit first, so it drains in small pieces.
__host__ __device__ __forceinline__ int level_begin(int lv, int vp) {
    return lv == 0 ? 0 : (lv == 1 ? (vp * 3) / 5 : (lv == 2 ? (vp * 9) / 10 : vp));
}

// ---- the full-precision tokens of a unit (CUDA cores), one 32-token chunk ----------
// Tokens: sink, then the value q-buffer + local window (cache.py:196-208); the
// keys of those tokens come from the key sink, a key page (dequantised from a
// shared-memory copy, Alg. 1) or the key q-buffer.  Lane = token for QK, lane
// = 4 channels for PV.
template <int GROUP>
__device__ void fp_chunk(const Params& P, uint8_t* scratch, int u, int fc, int lane) {
    const KittyCacheDesc& c = P.c;
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g, d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    uint8_t* kbuf = scratch;
    __half2* qf = reinterpret_cast<__half2*>(scratch + kKeySlotMax);           // [GROUP][D/2]
    float* ps = reinterpret_cast<float*>(scratch + kKeySlotMax + GROUP * D * 2);  // [GROUP][32]
    const UnitGeom gm = unit_geom(c, u);
    const int s_len = min(gm.n, S);
    const int c0 = fc * kFpChunk;
    const int cnt = min(kFpChunk, gm.nfp - c0);
    const int vbase = S + gm.vp * G;
    auto token_of = [&](int j) { return j < s_len ? j : vbase + (j - s_len); };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const uint16_t* qbase = P.q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D;
#pragma unroll
    for (int g = 0; g < GROUP; ++g) {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(qbase + g * D) + lane);
        qf[g * (D / 2) + 2 * lane] = __floats2half2_rn(__uint_as_float(w.x << 16) * kAlpha, __uint_as_float(w.x & 0xffff0000u) * kAlpha);
        qf[g * (D / 2) + 2 * lane + 1] = __floats2half2_rn(__uint_as_float(w.y << 16) * kAlpha, __uint_as_float(w.y & 0xffff0000u) * kAlpha);
    }
    __syncwarp();
    const bool valid = lane < cnt;
    const int t = token_of(c0 + (valid ? lane : 0));
    const int pc = t - S;
    const bool in_page = t >= S && pc < gm.kp * G;
    float lg[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) lg[g] = 0.f;
    if (!in_page) {
        const uint16_t* krow = t < S ? c.k_sink + ((int64_t)u * S + t) * D : c.k_qbuf + ((int64_t)u * G + pc % G) * D;
#pragma unroll 2
        for (int i = 0; i < 16; ++i) {
            const uint4 w = reinterpret_cast<const uint4*>(krow)[i];
            const float k8[8] = {__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                                 __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u),
                                 __uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u),
                                 __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u)};
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 qq = __half22float2(qf[g * (D / 2) + 4 * i + e]);
                    lg[g] = fmaf(qq.x, k8[2 * e], lg[g]);
                    lg[g] = fmaf(qq.y, k8[2 * e + 1], lg[g]);
                }
            }
        }
    }
    // keys that sit in key pages: stage each such page in the warp's key buffer
    unsigned need = __ballot_sync(0xffffffffu, valid && in_page);
    while (need) {
        const int src = __ffs(need) - 1;
        const int page = __shfl_sync(0xffffffffu, pc / G, src);
        const uint4* gsrc = reinterpret_cast<const uint4*>(c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + page] * kslot);
        for (int i = lane; i < kslot / 16; i += 32) reinterpret_cast<uint4*>(kbuf)[i] = gsrc[i];
        __syncwarp();
        const bool mine = valid && in_page && pc / G == page;
        if (mine) {
            const int tl = pc % G, sh = 2 * (tl & 3), byte = tl >> 2;
            const uint8_t* hb = kbuf + D * G / 4;
            const uint8_t* ib = kbuf + D * G / 4 + d_boost * G / 4;
#pragma unroll 4
            for (int d = 0; d < D; ++d) {
                uint32_t code = (kbuf[d * (G / 4) + byte] >> sh) & 3u;
                const uint32_t r = ib[d];
                if (r != kSentinel) code |= ((hb[r * (G / 4) + byte] >> sh) & 3u) << 2;
                const float s_ = half_bits_to_f32(ld_u16(kbuf + scale_off + 2 * d));
                const float z_ = half_bits_to_f32(ld_u16(kbuf + zero_off + 2 * d));
                const float kv = fmaf(static_cast<float>(code), s_, z_);
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    const __half2 qq = qf[g * (D / 2) + (d >> 1)];
                    lg[g] = fmaf((d & 1) ? __high2float(qq) : __low2float(qq), kv, lg[g]);
                }
            }
        }
        __syncwarp();
        need &= ~__ballot_sync(0xffffffffu, mine);
    }
    float m[GROUP], l[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) {
        const float x = valid ? lg[g] : -INFINITY;
        float mc = x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        const float p = valid ? ex2(x - mc) : 0.f;
        float s = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        m[g] = mc;
        l[g] = s;
        ps[g * kFpChunk + lane] = p;
    }
    __syncwarp();
    float acc[GROUP][4];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
    const uint16_t* vsink = c.v_sink + (int64_t)u * S * D;
    const uint16_t* vr = c.v_ring + (int64_t)u * W * D;
#pragma unroll 1
    for (int j0 = 0; j0 < cnt; j0 += 8) {
        uint2 vv[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int tt = token_of(c0 + min(j0 + jj, cnt - 1));
            const uint16_t* vrow = tt < S ? vsink + (int64_t)tt * D : vr + (int64_t)((tt - S) % W) * D;
            vv[jj] = reinterpret_cast<const uint2*>(vrow)[lane];
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const float v0 = __uint_as_float(vv[jj].x << 16), v1 = __uint_as_float(vv[jj].x & 0xffff0000u);
            const float v2 = __uint_as_float(vv[jj].y << 16), v3 = __uint_as_float(vv[jj].y & 0xffff0000u);
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const float pg = (j0 + jj < cnt) ? ps[g * kFpChunk + j0 + jj] : 0.f;
                acc[g][0] = fmaf(pg, v0, acc[g][0]);
                acc[g][1] = fmaf(pg, v1, acc[g][1]);
                acc[g][2] = fmaf(pg, v2, acc[g][2]);
                acc[g][3] = fmaf(pg, v3, acc[g][3]);
            }
        }
    }
    __syncwarp();
    float* base = P.part + ((int64_t)u * P.nslot + fc) * GROUP * (D + 2);
#pragma unroll
    for (int g = 0; g < GROUP; ++g) {
        reinterpret_cast<float4*>(base + g * D)[lane] = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
        if (lane == 0) {
            base[GROUP * D + 2 * g] = m[g];
            base[GROUP * D + 2 * g + 1] = l[g];
        }
    }
    __syncwarp();
}

// ---- the kernel --------------------------------------------------------------------

template <int GROUP>
__global__ void __launch_bounds__(kThreads, 1) tc_attention_kernel(Params P) {
    using L = Smem<GROUP>;
    constexpr int NX = L::NX, NQK = L::NQK, NCH = L::NCH, NP = L::NP;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(smem);
    const KittyCacheDesc& c = P.c;
    const int d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int vslot = static_cast<int>(c.value_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D;
    const int zero_off = scale_off + 2 * D;
    const int idx_off = D * G / 4 + d_boost * G / 4;

    auto stage_k = [&](int s) { return sbase + L::o_ring + s * L::kStageAl; };
    auto stage_v = [&](int s) { return stage_k(s) + kKeySlotMax; };
    auto stage_q = [&](int s) { return stage_k(s) + kKeySlotMax + kValueSlot; };
    StageInfo* sinfo = reinterpret_cast<StageInfo*>(smem + L::o_sinfo);
    KInfo* kinfo = reinterpret_cast<KInfo*>(smem + L::o_kinfo);
    float* vinfo = reinterpret_cast<float*>(smem + L::o_vinfo);
    float* xch = reinterpret_cast<float*>(smem + L::o_xch);
    RingEntry* ring = reinterpret_cast<RingEntry*>(smem + L::o_ring4);
    const uint32_t bar0 = sbase + L::o_bar;
    auto b_full = [&](int s) { return bar0 + 8 * s; };
    auto b_empty = [&](int s) { return bar0 + 8 * (NST + s); };
    auto b_kready = [&](int b) { return bar0 + 8 * (2 * NST + b); };
    auto b_sfull = [&](int b) { return bar0 + 8 * (2 * NST + 2 + b); };
    auto b_sfree = [&](int b) { return bar0 + 8 * (2 * NST + 4 + b); };
    auto b_vready = [&](int b) { return bar0 + 8 * (2 * NST + 6 + b); };
    auto b_pready = [&](int b) { return bar0 + 8 * (2 * NST + 8 + b); };
    auto b_vfree = [&](int b) { return bar0 + 8 * (2 * NST + 10 + b); };
    auto b_ofull = [&](int b) { return bar0 + 8 * (2 * NST + 12 + b); };
    auto b_ofree = [&](int b) { return bar0 + 8 * (2 * NST + 14 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::o_tmem);

    // ---- setup: TMEM, barriers, constant tiles ----
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(L::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(b_full(s), 1);
            mbar_init(b_empty(s), 8);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(b_kready(b), 4);
            mbar_init(b_sfull(b), 1);
            mbar_init(b_sfree(b), 4);
            mbar_init(b_vready(b), 4);
            mbar_init(b_pready(b), 4);
            mbar_init(b_vfree(b), 1);
            mbar_init(b_ofull(b), 1);
            mbar_init(b_ofree(b), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // A_ones (K = 32 rows of 4^j per permuted token row) and zeroed B tiles
    for (int i = tid; i < 4096 / 16; i += kThreads) {
        // byte (mchunk, k, r) at a_off(mchunk, k) + r; weight 4^(r / 4)
        sts128(sbase + L::o_ones + 16 * i, 0x01010101u, 0x04040404u, 0x10101010u, 0x40404040u);
    }
    for (int i = tid; i < 2 * L::kBQK / 16; i += kThreads) sts128(sbase + L::o_bqk + 16 * i, 0u, 0u, 0u, 0u);
    for (int i = tid; i < 2 * 128 * NP / 16; i += kThreads) sts128(sbase + L::o_bp + 16 * i, 0u, 0u, 0u, 0u);
    if (tid < 4) ring[tid].tag = -1;
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ===================== WG-A: key pages -> operand tiles, B = q * (s | z) =====================
        const int d = tid;  // channel
        float qa[GROUP];
        float qmax = 0.f;
        for (int i = 0;; ++i) {
            const int s = i % NST, b = i & 1;
            mbar_wait(b_full(s), (i / NST) & 1);
            const StageInfo si = sinfo[s];
            if (i >= 2) mbar_wait(b_sfree(b), ((i >> 1) - 1) & 1);
            if (si.flags & FL_END) {
                if (d == 0) kinfo[b].flags = FL_END;
                __syncwarp();
                if (lane == 0) mbar_arrive(b_kready(b));
                break;
            }
            const uint32_t kp = stage_k(s);
            if (si.flags & FL_FIRST) {
                const uint32_t qs = stage_q(s);
                float mx = 0.f;
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    qa[g] = bf16_to_f32(lds16(qs + 2 * (g * D + d))) * kAlpha;
                    const uint2 w = lds64(qs + 2 * (g * D + 4 * lane));
                    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(__uint_as_float(w.x << 16)), fabsf(__uint_as_float(w.x & 0xffff0000u))),
                                         fmaxf(fabsf(__uint_as_float(w.y << 16)), fabsf(__uint_as_float(w.y & 0xffff0000u)))));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                qmax = mx * kAlpha;
            }
            // per-page bounds: max scale, max |zero| over the 128 channels (every warp redundantly)
            float smax, zmax;
            {
                const uint2 sv = lds64(kp + scale_off + 8 * lane);
                const uint2 zv = lds64(kp + zero_off + 8 * lane);
                const __half2 s2 = __hmax2(*reinterpret_cast<const __half2*>(&sv.x), *reinterpret_cast<const __half2*>(&sv.y));
                const __half2 z2 = __hmax2(__habs2(*reinterpret_cast<const __half2*>(&zv.x)), __habs2(*reinterpret_cast<const __half2*>(&zv.y)));
                __half2 m2 = __halves2half2(__hmax(__low2half(s2), __high2half(s2)), __hmax(__low2half(z2), __high2half(z2)));
                uint32_t mu = *reinterpret_cast<uint32_t*>(&m2);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mu = hmax2(mu, __shfl_xor_sync(0xffffffffu, mu, o));
                m2 = *reinterpret_cast<__half2*>(&mu);
                smax = __low2float(m2);
                zmax = __high2float(m2);
            }
            const float bx = 4.f * qmax * smax, bz = qmax * zmax;
            const float invx = bx > 0.f ? kQuant / bx : 0.f, invz = bz > 0.f ? kQuant / bz : 0.f;
            const uint32_t ak = sbase + L::o_ak + b * kTileAK;
            const uint32_t bq = sbase + L::o_bqk + b * L::kBQK;
            // dense_low row d: 32 bytes = 128 tokens -> 128 u8 (code * 4^j), 8 MN chunks
            {
                const uint4 wa = lds128(kp + 32 * d), wb = lds128(kp + 32 * d + 16);
                const uint32_t w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
                const uint32_t dst = ak + a_off(0, d);
#pragma unroll
                for (int i8 = 0; i8 < 8; ++i8) sts128(dst + 128 * i8, w[i8] & M0, w[i8] & M1, w[i8] & M2, w[i8] & M3);
            }
            // high_bits rows (boosted channels) -> K rows 128 + r
            for (int r = d >> 3; r < d_boost; r += 16) {
                const uint32_t w = lds32(kp + D * G / 4 + 32 * r + 4 * (d & 7));
                sts128(ak + a_off(d & 7, 128 + r), w & M0, w & M1, w & M2, w & M3);
            }
            // B rows: (lo, hi) of q alpha s_d per query, then of q alpha z_d
            {
                const float s_d = h2f(lds16(kp + scale_off + 2 * d));
                const float z_d = h2f(lds16(kp + zero_off + 2 * d));
                const float sx = s_d * invx, sz = z_d * invz;
                uint32_t xw[GROUP > 1 ? GROUP / 2 : 1], zw[GROUP > 1 ? GROUP / 2 : 1];
#pragma unroll
                for (int g = 0; g < GROUP; g += 2) {
                    const int x0 = f2i(qa[g] * sx), z0 = f2i(qa[g] * sz);
                    const int x1 = GROUP > 1 ? f2i(qa[g + 1 < GROUP ? g + 1 : g] * sx) : 0;
                    const int z1 = GROUP > 1 ? f2i(qa[g + 1 < GROUP ? g + 1 : g] * sz) : 0;
                    xw[g / 2] = GROUP > 1 ? enc_pair(x0, x1) : (enc16(x0) & 0xffffu);
                    zw[g / 2] = GROUP > 1 ? enc_pair(z0, z1) : (enc16(z0) & 0xffffu);
                }
                const uint32_t row = bq + 16 * (d & 7) + 128 * NCH * (d >> 3);
                if (GROUP == 8) {
                    sts128(row, xw[0], xw[GROUP > 4 ? 1 : 0], xw[GROUP > 4 ? 2 : 0], xw[GROUP > 4 ? 3 : 0]);
                    sts128(row + 128, zw[0], zw[GROUP > 4 ? 1 : 0], zw[GROUP > 4 ? 2 : 0], zw[GROUP > 4 ? 3 : 0]);
                } else if (GROUP == 4) {
                    sts128(row, xw[0], xw[GROUP > 2 ? 1 : 0], zw[0], zw[GROUP > 2 ? 1 : 0]);
                } else {
                    sts128(row, xw[0], 0u, zw[0], 0u);
                }
                const uint32_t bi = lds8(kp + idx_off + d);
                if ((int)bi < d_boost) {
                    const float s4 = 4.f * sx;
                    uint32_t bw[GROUP > 1 ? GROUP / 2 : 1];
#pragma unroll
                    for (int g = 0; g < GROUP; g += 2) {
                        const int x0 = f2i(qa[g] * s4);
                        const int x1 = GROUP > 1 ? f2i(qa[g + 1 < GROUP ? g + 1 : g] * s4) : 0;
                        bw[g / 2] = GROUP > 1 ? enc_pair(x0, x1) : (enc16(x0) & 0xffffu);
                    }
                    const int k = 128 + (int)bi;
                    const uint32_t brow = bq + 16 * (k & 7) + 128 * NCH * (k >> 3);
                    if (GROUP == 8)
                        sts128(brow, bw[0], bw[GROUP > 4 ? 1 : 0], bw[GROUP > 4 ? 2 : 0], bw[GROUP > 4 ? 3 : 0]);
                    else if (GROUP == 4)
                        sts64(brow, bw[0], bw[GROUP > 2 ? 1 : 0]);
                    else
                        sts32(brow, bw[0]);
                }
            }
            if (d == 0) {
                KInfo ki;
                ki.stepx = bx / kQuant;
                ki.stepz = bz / kQuant;
                ki.flags = si.flags;
                ki.unit = si.unit;
                ki.slot = si.slot;
                kinfo[b] = ki;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_kready(b));
                mbar_arrive(b_empty(s));
            }
        }
    } else if (warp < 8) {
        // ===================== WG-B: softmax (thread = TMEM lane = token) =====================
        const int m = tid - 128;
        const int wq = warp - 4;
        const int t = perm_index(m);
        const float wj = perm_weight(m);
        const uint32_t lane_base = tmem + ((uint32_t)(32 * wq) << 16);
        float mrun[GROUP], l[GROUP], lz[GROUP];
        for (int i = 0;; ++i) {
            const int b = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            mbar_wait(b_sfull(b), ph);
            mbar_wait(b_kready(b), ph);
            const KInfo ki = kinfo[b];
            if (ki.flags & FL_END) break;
            if (ki.flags & FL_FIRST) {
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    mrun[g] = -INFINITY;
                    l[g] = 0.f;
                    lz[g] = 0.f;
                }
            }
            tc_fence_after();
            uint32_t xs[2 * GROUP], zs[2 * GROUP];
            tmem_ld<2 * GROUP>(lane_base + b * 2 * NQK, xs);
            tmem_ld<2 * GROUP>(lane_base + b * 2 * NQK + NQK + NX, zs);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_sfree(b));
            const float fx = ki.stepx * wj, fz = ki.stepz * wj;
            float lg[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const int sx = (int)xs[2 * g] + 128 * (int)xs[2 * g + 1];
                const int sz = (int)zs[2 * g] + 128 * (int)zs[2 * g + 1];
                lg[g] = (float)sx * fx + (float)sz * fz;
            }
            // page max over the 128 tokens (f16x2 pairs), one named barrier
            constexpr int NPAIR = GROUP > 1 ? GROUP / 2 : 1;
            uint32_t hm[NPAIR];
#pragma unroll
            for (int k = 0; k < NPAIR; ++k) hm[k] = pack_f16x2(lg[2 * k < GROUP ? 2 * k : 0], lg[2 * k + 1 < GROUP ? 2 * k + 1 : 0]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int k = 0; k < NPAIR; ++k) hm[k] = hmax2(hm[k], __shfl_xor_sync(0xffffffffu, hm[k], o));
            float* xb = xch + (i & 1) * 4 * 16;
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < NPAIR; ++k) reinterpret_cast<uint32_t*>(xb)[wq * 4 + k] = hm[k];
            named_sync(1, 128);
#pragma unroll
            for (int k = 0; k < NPAIR; ++k) {
                const uint32_t* xu = reinterpret_cast<const uint32_t*>(xb);
                hm[k] = hmax2(hmax2(xu[k], xu[4 + k]), hmax2(xu[8 + k], xu[12 + k]));
            }
            float pm[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const __half2 h2 = *reinterpret_cast<const __half2*>(&hm[g / 2]);
                pm[g] = (g & 1) ? __high2float(h2) : __low2float(h2);
            }
            // vmeta of this page (s_t, z_t) + the P scale; B_P of page i - 2 consumed
            mbar_wait(b_vready(b), ph);
            if (i >= 2) mbar_wait(b_vfree(b), ((i >> 1) - 1) & 1);
            const float2 sz = *reinterpret_cast<const float2*>(smem + L::o_vmeta + b * 1024 + 8 * t);
            const float invp = vinfo[b];
            const float sc = sz.x * invp;
            float corr[GROUP];
            int xp[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const float mn = fmaxf(mrun[g], pm[g]);
                corr[g] = ex2(mrun[g] - mn);
                const float p = ex2(lg[g] - mn);
                l[g] = fmaf(l[g], corr[g], p);
                lz[g] = fmaf(lz[g], corr[g], p * sz.y);
                mrun[g] = mn;
                xp[g] = min(f2i(p * sc), 16383);
            }
            const uint32_t prow = sbase + L::o_bp + b * 128 * NP + NP * t;
            if (GROUP == 8) {
                sts128(prow, enc_pair(xp[0], xp[1 % GROUP]), enc_pair(xp[2 % GROUP], xp[3 % GROUP]),
                       enc_pair(xp[4 % GROUP], xp[5 % GROUP]), enc_pair(xp[6 % GROUP], xp[7 % GROUP]));
            } else if (GROUP == 4) {
                sts64(prow, enc_pair(xp[0], xp[1 % GROUP]), enc_pair(xp[2 % GROUP], xp[3 % GROUP]));
            } else if (GROUP == 2) {
                sts32(prow, enc_pair(xp[0], xp[1 % GROUP]));
            } else {
                sts32(prow, enc16(xp[0]) & 0xffffu);
            }
            RingEntry& re = ring[i & 3];
            if (ki.flags & FL_LAST) {
                // item done: sum l, l_z over the 128 tokens; (m, l) -> partial, l_z -> correction warps
                float red[2 * GROUP];
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    red[g] = l[g];
                    red[GROUP + g] = lz[g];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int k = 0; k < 2 * GROUP; ++k) red[k] += __shfl_xor_sync(0xffffffffu, red[k], o);
                float* xs2 = xch + 128;  // [4 warps][16]
                if (lane == 0)
#pragma unroll
                    for (int k = 0; k < 2 * GROUP; ++k) xs2[wq * 16 + k] = red[k];
                named_sync(1, 128);
                if (m == 0) {
                    const int u = ki.unit;
                    float* base = P.part + ((int64_t)u * P.nslot + ki.slot) * GROUP * (D + 2);
#pragma unroll
                    for (int g = 0; g < GROUP; ++g) {
                        const float lt = xs2[g] + xs2[16 + g] + xs2[32 + g] + xs2[48 + g];
                        const float lzt = xs2[GROUP + g] + xs2[16 + GROUP + g] + xs2[32 + GROUP + g] + xs2[48 + GROUP + g];
                        base[GROUP * D + 2 * g] = mrun[g];
                        base[GROUP * D + 2 * g + 1] = lt;
                        re.lz[g] = lzt;
                    }
                }
                named_sync(1, 128);  // xs2 reusable
            }
            if (m == 0) {
#pragma unroll
                for (int g = 0; g < GROUP; ++g) re.corr[g] = corr[g];
                __threadfence_block();
                *reinterpret_cast<volatile int*>(&re.tag) = i;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_pready(b));
        }
    } else if (warp < 12) {
        // ===================== WG-C: value pages -> operand tiles; output correction =====================
        const int r = tid - 256;  // token row for the conversion, TMEM lane for the correction
        const int wq = warp - 8;
        const int ch = perm_index(r);
        const float wch = perm_weight(r);
        const uint32_t lane_base = tmem + ((uint32_t)(32 * wq) << 16);
        float o[GROUP];
#pragma unroll
        for (int g = 0; g < GROUP; ++g) o[g] = 0.f;
        StageInfo prev;
        prev.flags = 0;
        float prev_step = 0.f;
        auto correct = [&](int j) {
            const int b = j & 1;
            mbar_wait(b_ofull(b), (j >> 1) & 1);
            tc_fence_after();
            uint32_t ov[2 * GROUP];
            tmem_ld<2 * GROUP>(lane_base + 4 * NQK + b * NP, ov);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_ofree(b));
            RingEntry& re = ring[j & 3];
            while (*reinterpret_cast<volatile int*>(&re.tag) != j) {
            }
            __threadfence_block();
            const float f = prev_step * wch;
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const int v = (int)ov[2 * g] + 128 * (int)ov[2 * g + 1];
                o[g] = fmaf(o[g], re.corr[g], (float)v * f);
            }
            if (prev.flags & FL_LAST) {
                float* base = P.part + ((int64_t)prev.unit * P.nslot + prev.slot) * GROUP * (D + 2);
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    base[g * D + ch] = o[g] + re.lz[g];
                    o[g] = 0.f;
                }
            }
        };
        int i = 0;
        for (;; ++i) {
            const int s = i % NST, b = i & 1;
            mbar_wait(b_full(s), (i / NST) & 1);
            const StageInfo si = sinfo[s];
            if (si.flags & FL_END) break;
            if (i >= 2) mbar_wait(b_vfree(b), ((i >> 1) - 1) & 1);
            const uint32_t vp = stage_v(s);
            const uint32_t av = sbase + L::o_av + b * kTileA;
            {
                const uint4 wa = lds128(vp + 32 * r), wb = lds128(vp + 32 * r + 16);
                const uint32_t w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
                const uint32_t dst = av + a_off(0, r);
#pragma unroll
                for (int i8 = 0; i8 < 8; ++i8) sts128(dst + 128 * i8, w[i8] & M0, w[i8] & M1, w[i8] & M2, w[i8] & M3);
            }
            const float s_t = h2f(lds16(vp + G * D / 4 + 2 * r));
            const float z_t = h2f(lds16(vp + G * D / 4 + 2 * G + 2 * r));
            *reinterpret_cast<float2*>(smem + L::o_vmeta + b * 1024 + 8 * r) = make_float2(s_t, z_t);
            float smax;
            {
                const uint2 sv = lds64(vp + G * D / 4 + 8 * lane);
                const __half2 s2 = __hmax2(*reinterpret_cast<const __half2*>(&sv.x), *reinterpret_cast<const __half2*>(&sv.y));
                __half2 m2 = __halves2half2(__hmax(__low2half(s2), __high2half(s2)), __low2half(s2));
                uint32_t mu = *reinterpret_cast<uint32_t*>(&m2);
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) mu = hmax2(mu, __shfl_xor_sync(0xffffffffu, mu, o2));
                m2 = *reinterpret_cast<__half2*>(&mu);
                smax = __low2float(m2) * 1.125f;  // p <= 2^(f16 max rounding) < 1.125
            }
            const float invp = smax > 0.f ? kQuant / smax : 0.f;
            if (r == 0) vinfo[b] = invp;
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_vready(b));
                mbar_arrive(b_empty(s));
            }
            if (i >= 1) correct(i - 1);
            prev = si;
            prev_step = smax / kQuant;
        }
        if (i >= 1) correct(i - 1);
    } else if (warp == 12) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const int units = P.units;
            const int nq0 = units * P.cmx[0], nq1 = units * P.cmx[1], nq2 = units * P.cmx[2];
            int tk = atomicAdd(P.ctr, 1);
            int it = 0;
            for (;;) {
                // next non-empty page item
                int u = 0, p0 = 0, p1 = 0, slot = 0;
                bool have = false;
                while (!have) {
                    const int t = tk;
                    if (t >= nq0 + nq1 + nq2) break;
                    tk = atomicAdd(P.ctr, 1);
                    int sect, idx;
                    if (t < nq0) {
                        sect = 0;
                        idx = t;
                    } else if (t < nq0 + nq1) {
                        sect = 1;
                        idx = t - nq0;
                    } else {
                        sect = 2;
                        idx = t - nq0 - nq1;
                    }
                    const int chn = idx / units;
                    u = idx - chn * units;
                    const UnitGeom gm = unit_geom(c, u);
                    const int lb = level_begin(sect, gm.vp), le = level_begin(sect + 1, gm.vp);
                    p0 = lb + chn * P.cs[sect];
                    p1 = min(le, p0 + P.cs[sect]);
                    if (p0 < p1 && gm.n > 0) {
                        have = true;
                        slot = P.fmax + chn;
                        for (int l2 = 0; l2 < sect; ++l2) slot += P.cmx[l2];
                    }
                }
                const int s = it % NST;
                if (it >= NST) mbar_wait(b_empty(s), ((it / NST) - 1) & 1);
                if (!have) {
                    sinfo[s].flags = FL_END;
                    mbar_arrive(b_full(s));
                    break;
                }
                const int b_ = u / c.cfg.h_kv, h_ = u - b_ * c.cfg.h_kv;
                const uint16_t* qsrc = P.q + ((int64_t)b_ * c.cfg.h_q + (int64_t)h_ * GROUP) * D;
                for (int p = p0; p < p1; ++p) {
                    const int st = it % NST;
                    if (p > p0 && it >= NST) mbar_wait(b_empty(st), ((it / NST) - 1) & 1);
                    StageInfo si;
                    si.unit = u;
                    si.page = p;
                    si.flags = (p == p0 ? FL_FIRST : 0) | (p == p1 - 1 ? FL_LAST : 0);
                    si.slot = slot;
                    sinfo[st] = si;
                    const uint8_t* ks = c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + p] * kslot;
                    const uint8_t* vs = c.value_pool + (int64_t)c.value_block_table[(int64_t)u * c.max_pages + p] * vslot;
                    const uint32_t qbytes = p == p0 ? GROUP * D * 2 : 0;
                    mbar_expect_tx(b_full(st), kslot + vslot + qbytes);
                    bulk_g2s(stage_k(st), ks, kslot, b_full(st));
                    bulk_g2s(stage_v(st), vs, vslot, b_full(st));
                    if (qbytes) bulk_g2s(stage_q(st), qsrc, qbytes, b_full(st));
                    ++it;
                }
            }
        }
    } else if (warp == 13) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t id_qk = idesc_i8(NQK), id_pv = idesc_i8(NP);
            const uint32_t ones = sbase + L::o_ones;
            const int nkb = d_boost > 0 ? 1 : 0;
            auto issue_pv = [&](int j) {
                const int b = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(b_pready(b), ph);
                mbar_wait(b_vready(b), ph);
                if (j >= 2) mbar_wait(b_ofree(b), ((j >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t av = sbase + L::o_av + b * kTileA;
                const uint32_t bp = sbase + L::o_bp + b * 128 * NP;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_i8(tmem + 4 * NQK + b * NP, sdesc(av + 4096 * k, 1024, 128), sdesc(bp + 512 * k, 128, 128), id_pv, k > 0);
                umma_commit(b_ofull(b));
                umma_commit(b_vfree(b));
            };
            int i = 0;
            for (;; ++i) {
                const int b = i & 1;
                mbar_wait(b_kready(b), (i >> 1) & 1);
                if (kinfo[b].flags & FL_END) break;
                tc_fence_after();
                const uint32_t ak = sbase + L::o_ak + b * kTileAK;
                const uint32_t bq = sbase + L::o_bqk + b * L::kBQK;
                const uint32_t d1 = tmem + b * 2 * NQK, d2 = d1 + NQK;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_i8(d1, sdesc(ak + 4096 * k, 1024, 128), sdesc(bq + 4 * 128 * NCH * k, 128 * NCH, 128), id_qk, k > 0);
                if (nkb)
                    umma_i8(d1, sdesc(ak + 4096 * 4, 1024, 128), sdesc(bq + 4 * 128 * NCH * 4, 128 * NCH, 128), id_qk, 1);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_i8(d2, sdesc(ones, 1024, 128), sdesc(bq + 4 * 128 * NCH * k, 128 * NCH, 128), id_qk, k > 0);
                umma_commit(b_sfull(b));
                if (i >= 1) issue_pv(i - 1);
            }
            if (i >= 1) issue_pv(i - 1);
            mbar_arrive(b_sfull(i & 1));  // end marker for the softmax warps
        }
    } else {
        // ===================== FP warps: full-precision tokens =====================
        const int fw = warp - 14;
        uint8_t* scratch = smem + L::o_fp + fw * L::kFpAl;
        const int nf = P.units * P.fmax;
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(&P.ctr[2], 1);
            it = __shfl_sync(0xffffffffu, it, 0);
            if (it >= nf) break;
            const int fc = it / P.units, u = it - fc * P.units;
            const UnitGeom gm = unit_geom(c, u);
            if (gm.n == 0 || fc * kFpChunk >= gm.nfp) continue;
            fp_chunk<GROUP>(P, scratch, u, fc, lane);
        }
    }

    // ---- teardown ----
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(L::kTmemCols));
    }
    if (tid == 0) {
        __threadfence();
        const int done = atomicAdd(&P.ctr[1], 1);
        if (done == static_cast<int>(gridDim.x) - 1) {
            P.ctr[0] = 0;
            P.ctr[1] = 0;
            P.ctr[2] = 0;
        }
    }
}

// Log-sum-exp merge of a unit's partials (fp chunks + page chunks).  One CTA
// per unit, 4 warps per query row, each warp over a quarter of the parts.
template <int GROUP>
__global__ void __launch_bounds__(GROUP * 128) combine_kernel(Params P) {
    constexpr int kSub = 4;
    __shared__ float sm_l[GROUP][kSub];
    __shared__ float4 sm_acc[GROUP][kSub][32];
    const int u = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp / kSub, sub = warp % kSub;
    const KittyCacheDesc& c = P.c;
    const UnitGeom gm = unit_geom(c, u);
    if (gm.n == 0) return;
    const int nfc = (gm.nfp + kFpChunk - 1) / kFpChunk;
    int nch[3];
    for (int lv = 0; lv < 3; ++lv) {
        const int n = level_begin(lv + 1, gm.vp) - level_begin(lv, gm.vp);
        nch[lv] = (n + P.cs[lv] - 1) / P.cs[lv];
    }
    const int nparts = nfc + nch[0] + nch[1] + nch[2];
    constexpr int kStride = GROUP * (D + 2);
    const float* pb = P.part + (int64_t)u * P.nslot * kStride;
    auto part_ptr = [&](int i) {
        int slot;
        if (i < nfc) slot = i;
        else if (i < nfc + nch[0]) slot = P.fmax + (i - nfc);
        else if (i < nfc + nch[0] + nch[1]) slot = P.fmax + P.cmx[0] + (i - nfc - nch[0]);
        else slot = P.fmax + P.cmx[0] + P.cmx[1] + (i - nfc - nch[0] - nch[1]);
        return pb + (int64_t)slot * kStride;
    };
    float M = -INFINITY;
    for (int i = lane; i < nparts; i += 32) M = fmaxf(M, __ldcg(part_ptr(i) + GROUP * D + 2 * g));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i0 = sub; i0 < nparts; i0 += kSub * 8) {
        float4 a[8];
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = i0 + kSub * j;
            if (i < nparts) {
                const float* pi = part_ptr(i);
                a[j] = __ldcg(reinterpret_cast<const float4*>(pi + g * D) + lane);
                const float mi = __ldcg(pi + GROUP * D + 2 * g);
                const float li = __ldcg(pi + GROUP * D + 2 * g + 1);
                w[j] = mi == -INFINITY ? 0.f : ex2(mi - M);
                L = fmaf(w[j], li, L);
            } else {
                a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                w[j] = 0.f;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc.x = fmaf(w[j], a[j].x, acc.x);
            acc.y = fmaf(w[j], a[j].y, acc.y);
            acc.z = fmaf(w[j], a[j].z, acc.z);
            acc.w = fmaf(w[j], a[j].w, acc.w);
        }
    }
    sm_acc[g][sub][lane] = acc;
    if (lane == 0) sm_l[g][sub] = L;
    __syncthreads();
    if (sub == 0) {
        float4 o = sm_acc[g][0][lane];
        float Lt = sm_l[g][0];
#pragma unroll
        for (int k = 1; k < kSub; ++k) {
            const float4 x = sm_acc[g][k][lane];
            o.x += x.x;
            o.y += x.y;
            o.z += x.z;
            o.w += x.w;
            Lt += sm_l[g][k];
        }
        const float inv = 1.f / Lt;
        const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
        const int64_t row = (int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + g;
        if (P.out_dtype == KITTY_F32) {
            reinterpret_cast<float4*>(static_cast<float*>(P.out) + row * D)[lane] = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
        } else {
            uint2 v;
            v.x = f32_to_bf16_bits(o.x * inv) | (f32_to_bf16_bits(o.y * inv) << 16);
            v.y = f32_to_bf16_bits(o.z * inv) | (f32_to_bf16_bits(o.w * inv) << 16);
            reinterpret_cast<uint2*>(static_cast<uint16_t*>(P.out) + row * D)[lane] = v;
        }
    }
}

}  // namespace tcattn

// ---- host side ---------------------------------------------------------------------

using namespace tcattn;

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

bool fast_attention_supported(const KittyCacheDesc& c) {
    const int group = c.cfg.h_q / c.cfg.h_kv;
    return c.cfg.d == D && c.cfg.g == G && c.cfg.key_bits == 2 && c.cfg.value_bits == 2 &&
           (group == 1 || group == 2 || group == 4 || group == 8) && c.cfg.d_boost <= 32 &&
           c.key_slot_bytes <= kKeySlotMax && c.value_slot_bytes == kValueSlot;
}

struct TcPlan {
    int units, group, cs[3], cmx[3], fmax, nslot;
    size_t ctr_bytes, part_bytes;
};

static TcPlan plan(const KittyCacheDesc& c, int max_tokens) {
    TcPlan p;
    p.units = c.num_seqs * c.cfg.h_kv;
    p.group = c.cfg.h_q / c.cfg.h_kv;
    const int past = max_tokens > c.cfg.s ? max_tokens - c.cfg.s : 0;
    const int maxp = past / G + 1;
    const long long pages = (long long)p.units * maxp;
    int ppc = static_cast<int>(pages / (4LL * num_sms()));
    ppc = ppc < 1 ? 1 : (ppc > 16 ? 16 : ppc);
    p.cs[0] = ppc;
    p.cs[1] = ppc / 4 > 1 ? ppc / 4 : 1;
    p.cs[2] = 1;
    for (int lv = 0; lv < 3; ++lv) {
        const int n = level_begin(lv + 1, maxp) - level_begin(lv, maxp) + 2;
        p.cmx[lv] = (n + p.cs[lv] - 1) / p.cs[lv];
    }
    const int nfp_max = min(max_tokens, c.cfg.s + c.cfg.r + c.cfg.g - 1);
    p.fmax = (nfp_max + kFpChunk - 1) / kFpChunk;
    if (p.fmax < 1) p.fmax = 1;
    p.nslot = p.fmax + p.cmx[0] + p.cmx[1] + p.cmx[2];
    p.ctr_bytes = 256;
    p.part_bytes = (size_t)p.units * p.nslot * p.group * (D + 2) * sizeof(float);
    return p;
}

size_t fast_attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens) {
    if (!fast_attention_supported(c)) return 0;
    const TcPlan p = plan(c, max_tokens);
    return p.ctr_bytes + p.part_bytes;
}

template <int GROUP>
static cudaError_t launch_t(const Params& prm, cudaStream_t st) {
    auto kfn = tc_attention_kernel<GROUP>;
    const int sm = Smem<GROUP>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    kfn<<<num_sms(), kThreads, sm, st>>>(prm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    combine_kernel<GROUP><<<prm.units, GROUP * 128, 0, st>>>(prm);
    return cudaGetLastError();
}

cudaError_t launch_fast_attention(const KittyCacheDesc& c, const uint16_t* q, void* out, int out_dtype,
                                  int max_tokens, void* ws, size_t ws_bytes, cudaStream_t st) {
    const TcPlan p = plan(c, max_tokens);
    if (ws_bytes < p.ctr_bytes + p.part_bytes) return cudaErrorInvalidValue;
    Params prm;
    prm.c = c;
    prm.q = q;
    prm.out = out;
    prm.out_dtype = out_dtype;
    for (int lv = 0; lv < 3; ++lv) {
        prm.cs[lv] = p.cs[lv];
        prm.cmx[lv] = p.cmx[lv];
    }
    prm.fmax = p.fmax;
    prm.nslot = p.nslot;
    prm.units = p.units;
    prm.ctr = static_cast<int*>(ws);
    prm.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + p.ctr_bytes);
    switch (p.group) {
        case 1: return launch_t<1>(prm, st);
        case 2: return launch_t<2>(prm, st);
        case 4: return launch_t<4>(prm, st);
        default: return launch_t<8>(prm, st);
    }
}

cudaError_t fast_attention_trace(int, long long*, int) { return cudaSuccess; }

}  // namespace kitty
