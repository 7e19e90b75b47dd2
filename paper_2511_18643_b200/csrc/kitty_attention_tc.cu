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
#include "kitty_combine.cuh"
#include "kitty_fp.cuh"
#include "kitty_codec.cuh"

namespace kitty {
namespace tcattn {

constexpr int D = 128;
constexpr int G = 128;
// floats per partial record (acc[group][D], then (m, l) per row), padded to 16 B
__host__ __device__ constexpr int part_stride(int group) { return (group * (D + 2) + 3) & ~3; }
constexpr int NDESC = 8;           // page-descriptor ring (scheduler -> converters)
constexpr int kKeySlotMax = 5760;  // d_boost = 32
constexpr int kValueSlot = 4608;
constexpr int kFpChunk = 32;       // fp tokens per fp item
constexpr int kFpWarps = 2;
constexpr int kCtasPerSm = 1;    // independent page pipelines per SM
constexpr int kThreads = (14 + kFpWarps) * 32;  // WG-A 0-3, WG-B 4-7, WG-C 8-11, scheduler 12, MMA 13, FP 14-15
constexpr float kAlpha = 0.12751743074f;        // log2(e) / sqrt(128)
constexpr int kQuant = 16000;                   // fixed-point range of the int8 (lo, hi) pairs (< 2^14)
constexpr int kTileA = 1024 * 16;               // 128 x 128 u8 operand tile
constexpr int kTileAK = 1024 * 20;              // + 32 boosted rows
constexpr int NB = 16;                          // B row bytes of both MMAs: (lo, hi) per query, padded

constexpr uint32_t FL_FIRST = 1, FL_LAST = 2, FL_END = 4;

// One page pair of an item, written by the scheduler; q rows of the unit follow
// (bulk-copied) on an item's first page.
struct PageDesc {
    const uint8_t* kp;
    const uint8_t* vp;
    int unit, flags, slot, pad;
};
struct KInfo {
    float stepx;
    int flags, unit, slot;
};
struct RingEntry {
    float corr[8];
    float lz[8];
    int tag;
    int pad[15];
};

// Shared-memory layout of one CTA (dynamic, 1024-aligned operand tiles).
template <int GROUP>
struct Smem {
    static constexpr int kDesc = (32 + GROUP * D * 2 + 127) / 128 * 128;
    static constexpr int o_desc = 0;
    static constexpr int o_ak = (NDESC * kDesc + 1023) / 1024 * 1024;
    static constexpr int o_av = o_ak + 2 * kTileAK;
    static constexpr int o_bqk = o_av + 2 * kTileA;
    static constexpr int o_bp = o_bqk + 2 * 160 * NB;
    static constexpr int o_vmeta = o_bp + 2 * 128 * NB;          // [2][128] float2 (s, z)
    static constexpr int o_zx = o_vmeta + 2 * 128 * 8;            // [2][4 warps][8] partial sum_d q alpha z_d
    static constexpr int o_fp = o_zx + 2 * 4 * 8 * 4;             // per fp warp scratch
    static constexpr int kFpBytes = fptok::scratch_bytes<GROUP>();
    static constexpr int kFpAl = (kFpBytes + 127) / 128 * 128;
    static constexpr int o_ring4 = o_fp + kFpWarps * kFpAl;      // RingEntry[4]
    static constexpr int o_kinfo = o_ring4 + 4 * sizeof(RingEntry);
    static constexpr int o_vinfo = o_kinfo + 2 * 16;
    static constexpr int o_xch = o_vinfo + 16;                    // [3][64] floats: page-max x2, item sums
    static constexpr int o_bar = o_xch + 3 * 64 * 4;
    static constexpr int kBars = 2 * NDESC + 8 * 2;
    static constexpr int o_tmem = o_bar + kBars * 8;
    static constexpr int kBytes = o_tmem + 16;
    // TMEM columns: S[b] at 16 b, O[b] at 32 + 16 b
    static constexpr int kTmemCols = 64;
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

// ---- optional event trace of CTA 0 (kitty_debug_attention_trace) ----
constexpr int kTrPages = 512;
constexpr int kTrFields = 24;
__device__ long long g_tr[kTrPages * kTrFields];
__device__ int g_tr_on;
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

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
// try_wait with a suspend-time hint: the waiting warp sleeps until the phase
// completes instead of polling the barrier (polling competes with the
// converters for issue slots and the shared-memory pipe).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(phase), "r"(1000000)
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

// ---- the kernel --------------------------------------------------------------------

__device__ __forceinline__ uint4 ldg_na128(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ldg64(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg16(const void* p) {
    unsigned short v;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg8(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// max of the 4 f16 of (x, y) as float
__device__ __forceinline__ float hmax4(uint2 v) {
    const uint32_t m = hmax2(v.x, v.y);
    return fmaxf(h2f(m & 0xffffu), h2f(m >> 16));
}

// Sum of v[g] over the 32 lanes for every g: reduce-scatter over the top
// log2(N) lane bits, then a butterfly; lane l ends with the sum for query
// scatter_query<N>(l) in v[0].
template <int N>
__device__ __forceinline__ void warp_sum_scatter(float (&v)[N], int lane) {
    int n = N;
    int m = 16;
#pragma unroll
    for (int lv = 0; lv < 3; ++lv) {
        if (n > 1) {
            const int half = n / 2;
            const bool hi = (lane & m) != 0;
#pragma unroll
            for (int k = 0; k < N / 2; ++k) {
                if (k < half) {
                    const float keep = hi ? v[half + k] : v[k];
                    const float send = hi ? v[k] : v[half + k];
                    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            }
            n = half;
            m >>= 1;
        }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if (m > 0) {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
            m >>= 1;
        }
    }
}
template <int N>
__device__ __forceinline__ int scatter_query(int lane) {
    return N == 1 ? 0 : (N == 2 ? (lane >> 4) & 1 : (N == 4 ? (lane >> 3) & 3 : (lane >> 2) & 7));
}
template <int N>
__device__ __forceinline__ bool scatter_owner(int lane) {
    return (lane & (32 / N - 1)) == 0;
}

template <int GROUP>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) tc_attention_kernel(Params P) {
    using L = Smem<GROUP>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(smem);
    const KittyCacheDesc& c = P.c;
    const int d_boost = c.cfg.d_boost;
    const int scale_off = D * G / 4 + d_boost * G / 4 + D;
    const int zero_off = scale_off + 2 * D;
    const int idx_off = D * G / 4 + d_boost * G / 4;

    auto desc_ptr = [&](int i) { return reinterpret_cast<const PageDesc*>(smem + L::o_desc + (i % NDESC) * L::kDesc); };
    auto desc_q = [&](int i) { return sbase + L::o_desc + (i % NDESC) * L::kDesc + 32; };
    KInfo* kinfo = reinterpret_cast<KInfo*>(smem + L::o_kinfo);
    float* vinfo = reinterpret_cast<float*>(smem + L::o_vinfo);
    float* xch = reinterpret_cast<float*>(smem + L::o_xch);
    float* zx = reinterpret_cast<float*>(smem + L::o_zx);
    RingEntry* ring = reinterpret_cast<RingEntry*>(smem + L::o_ring4);
    const uint32_t bar0 = sbase + L::o_bar;
    auto b_dfull = [&](int s) { return bar0 + 8 * s; };
    auto b_dempty = [&](int s) { return bar0 + 8 * (NDESC + s); };
    auto b_kready = [&](int b) { return bar0 + 8 * (2 * NDESC + b); };
    auto b_sfull = [&](int b) { return bar0 + 8 * (2 * NDESC + 2 + b); };
    auto b_sfree = [&](int b) { return bar0 + 8 * (2 * NDESC + 4 + b); };
    auto b_vready = [&](int b) { return bar0 + 8 * (2 * NDESC + 6 + b); };
    auto b_pready = [&](int b) { return bar0 + 8 * (2 * NDESC + 8 + b); };
    auto b_vfree = [&](int b) { return bar0 + 8 * (2 * NDESC + 10 + b); };
    auto b_ofull = [&](int b) { return bar0 + 8 * (2 * NDESC + 12 + b); };
    auto b_ofree = [&](int b) { return bar0 + 8 * (2 * NDESC + 14 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::o_tmem);
    const bool tr = g_tr_on != 0 && blockIdx.x == 0;
    auto TR = [&](int i, int f) {
        if (tr && (threadIdx.x & 31) == 0 && i < kTrPages) g_tr[i * kTrFields + f] = gtimer();
    };

    // ---- setup: TMEM, barriers, zeroed B tiles ----
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(L::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < NDESC; ++s) {
            mbar_init(b_dfull(s), 1);
            mbar_init(b_dempty(s), 8);
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
    for (int i = tid; i < 2 * 160 * NB / 16; i += kThreads) sts128(sbase + L::o_bqk + 16 * i, 0u, 0u, 0u, 0u);
    for (int i = tid; i < 2 * 128 * NB / 16; i += kThreads) sts128(sbase + L::o_bp + 16 * i, 0u, 0u, 0u, 0u);
    if (tid < 4) ring[tid].tag = -1;
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ============ WG-A: key pages (global -> registers) -> u8 operand tile, B = q alpha s ============
        const int d = tid;  // channel
        float qa[GROUP];
#pragma unroll
        for (int g = 0; g < GROUP; ++g) qa[g] = 0.f;
        float qmax = 0.f;
        int end_at = 0x7fffffff;
        struct KR {
            uint4 c0, c1;
            uint32_t hb0, hb1, s16, z16, idx;
            uint2 s4;
            int unit, flags, slot;
        };
        // packed page -> registers, PF pages ahead of its conversion
        auto kload = [&](KR& r, int i) {
            if (i > end_at) {
                r.flags = FL_END;
                return;
            }
            mbar_wait(b_dfull(i % NDESC), (i / NDESC) & 1);
            const PageDesc pd = *desc_ptr(i);
            r.unit = pd.unit;
            r.flags = pd.flags;
            r.slot = pd.slot;
            if (pd.flags & FL_END) {
                end_at = i;
                return;
            }
            const uint8_t* kp = pd.kp;
            r.c0 = ldg_na128(kp + 32 * d);
            r.c1 = ldg_na128(kp + 32 * d + 16);
            r.hb0 = (d >> 3) < d_boost ? ldg32(kp + D * G / 4 + 32 * (d >> 3) + 4 * (d & 7)) : 0u;
            r.hb1 = (d >> 3) + 16 < d_boost ? ldg32(kp + D * G / 4 + 32 * ((d >> 3) + 16) + 4 * (d & 7)) : 0u;
            r.s4 = ldg64(kp + scale_off + 8 * lane);
            r.s16 = ldg16(kp + scale_off + 2 * d);  // combined only at use: keeps the load in flight
            r.z16 = ldg16(kp + zero_off + 2 * d);
            r.idx = ldg8(kp + idx_off + d);
        };
        auto kproc = [&](KR& r, int i) -> bool {
            const int b = i & 1;
            if (i >= 2) mbar_wait(b_sfree(b), ((i >> 1) - 1) & 1);
            if (warp == 0) TR(i, 2);
            if (r.flags & FL_END) {
                if (d == 0) kinfo[b].flags = FL_END;
                __syncwarp();
                if (lane == 0) mbar_arrive(b_kready(b));
                return false;
            }
            if (r.flags & FL_FIRST) {
                const uint32_t qs = desc_q(i);
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
            // page bound: max scale over the 128 channels (every warp redundantly)
            float smax = hmax4(r.s4);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
            const float bx = 4.f * qmax * smax;
            const float invx = bx > 0.f ? __fdividef((float)kQuant, bx) : 0.f;
            if (warp == 0) TR(i, 10);
            const uint32_t ak = sbase + L::o_ak + b * kTileAK;
            const uint32_t bq = sbase + L::o_bqk + b * 160 * NB;
            {
                const uint32_t w[8] = {r.c0.x, r.c0.y, r.c0.z, r.c0.w, r.c1.x, r.c1.y, r.c1.z, r.c1.w};
                const uint32_t dst = ak + a_off(0, d);
#pragma unroll
                for (int i8 = 0; i8 < 8; ++i8) sts128(dst + 128 * i8, w[i8] & M0, w[i8] & M1, w[i8] & M2, w[i8] & M3);
            }
            if ((d >> 3) < d_boost)
                sts128(ak + a_off(d & 7, 128 + (d >> 3)), r.hb0 & M0, r.hb0 & M1, r.hb0 & M2, r.hb0 & M3);
            if ((d >> 3) + 16 < d_boost)
                sts128(ak + a_off(d & 7, 144 + (d >> 3)), r.hb1 & M0, r.hb1 & M1, r.hb1 & M2, r.hb1 & M3);
            if (warp == 0) TR(i, 11);
            const float s_d = h2f(r.s16), z_d = h2f(r.z16);
            const float sx = s_d * invx;
            auto brow = [&](uint32_t addr, float f) {
                int x[GROUP];
#pragma unroll
                for (int g = 0; g < GROUP; ++g) x[g] = f2i(qa[g] * f);
                if (GROUP == 8)
                    sts128(addr, enc_pair(x[0], x[1 % GROUP]), enc_pair(x[2 % GROUP], x[3 % GROUP]),
                           enc_pair(x[4 % GROUP], x[5 % GROUP]), enc_pair(x[6 % GROUP], x[7 % GROUP]));
                else if (GROUP == 4)
                    sts64(addr, enc_pair(x[0], x[1 % GROUP]), enc_pair(x[2 % GROUP], x[3 % GROUP]));
                else if (GROUP == 2)
                    sts32(addr, enc_pair(x[0], x[1 % GROUP]));
                else
                    sts32(addr, enc16(x[0]) & 0xffffu);
            };
            brow(bq + NB * d, sx);
            if ((int)r.idx < d_boost) brow(bq + NB * (128 + (int)r.idx), 4.f * sx);
            if (warp == 0) TR(i, 12);
            // sum_d q alpha z_d in fp32: per-warp partials for the softmax warps
            float zz[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) zz[g] = qa[g] * z_d;
            warp_sum_scatter<GROUP>(zz, lane);
            if (scatter_owner<GROUP>(lane)) zx[(b * 4 + warp) * 8 + scatter_query<GROUP>(lane)] = zz[0];
            if (warp == 0) TR(i, 13);
            if (d == 0) {
                KInfo ki;
                ki.stepx = bx / kQuant;
                ki.flags = r.flags;
                ki.unit = r.unit;
                ki.slot = r.slot;
                kinfo[b] = ki;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_kready(b));
                mbar_arrive(b_dempty(i % NDESC));
            }
            if (warp == 0) TR(i, 3);
            return true;
        };
        KR r0, r1, r2, r3;
        kload(r0, 0);
        kload(r1, 1);
        kload(r2, 2);
        for (int i = 0;; i += 4) {
            kload(r3, i + 3);
            if (!kproc(r0, i)) break;
            kload(r0, i + 4);
            if (!kproc(r1, i + 1)) break;
            kload(r1, i + 5);
            if (!kproc(r2, i + 2)) break;
            kload(r2, i + 6);
            if (!kproc(r3, i + 3)) break;
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
            if (warp == 4) TR(i, 5);
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
            float zg[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g)
                zg[g] = zx[(b * 4 + 0) * 8 + g] + zx[(b * 4 + 1) * 8 + g] + zx[(b * 4 + 2) * 8 + g] + zx[(b * 4 + 3) * 8 + g];
            tc_fence_after();
            uint32_t xs[2 * GROUP];
            tmem_ld<2 * GROUP>(lane_base + b * 16, xs);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_sfree(b));
            if (warp == 4) TR(i, 14);
            const float fx = ki.stepx * wj;
            float lg[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) lg[g] = fmaf((float)((int)xs[2 * g] + 128 * (int)xs[2 * g + 1]), fx, zg[g]);
            // page max over the 128 tokens (f16x2 pairs), one named barrier
            constexpr int NPAIR = GROUP > 1 ? GROUP / 2 : 1;
            uint32_t hm[NPAIR];
#pragma unroll
            for (int k = 0; k < NPAIR; ++k) hm[k] = pack_f16x2(lg[2 * k < GROUP ? 2 * k : 0], lg[2 * k + 1 < GROUP ? 2 * k + 1 : 0]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int k = 0; k < NPAIR; ++k) hm[k] = hmax2(hm[k], __shfl_xor_sync(0xffffffffu, hm[k], o));
            float* xb = xch + (i & 1) * 64;
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < NPAIR; ++k) reinterpret_cast<uint32_t*>(xb)[wq * 4 + k] = hm[k];
            named_sync(1, 128);
#pragma unroll
            for (int k = 0; k < NPAIR; ++k) {
                const uint32_t* xu = reinterpret_cast<const uint32_t*>(xb);
                hm[k] = hmax2(hmax2(xu[k], xu[4 + k]), hmax2(xu[8 + k], xu[12 + k]));
            }
            if (warp == 4) TR(i, 15);
            float pm[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                const __half2 h2 = *reinterpret_cast<const __half2*>(&hm[g / 2]);
                pm[g] = (g & 1) ? __high2float(h2) : __low2float(h2);
            }
            mbar_wait(b_vready(b), ph);
            if (warp == 4) TR(i, 16);
            if (i >= 2) mbar_wait(b_vfree(b), ((i >> 1) - 1) & 1);
            if (warp == 4) TR(i, 17);
            const float2 sz = *reinterpret_cast<const float2*>(smem + L::o_vmeta + b * 1024 + 8 * t);
            const float sc = sz.x * vinfo[b];
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
            const uint32_t prow = sbase + L::o_bp + b * 128 * NB + NB * t;
            if (GROUP == 8)
                sts128(prow, enc_pair(xp[0], xp[1 % GROUP]), enc_pair(xp[2 % GROUP], xp[3 % GROUP]),
                       enc_pair(xp[4 % GROUP], xp[5 % GROUP]), enc_pair(xp[6 % GROUP], xp[7 % GROUP]));
            else if (GROUP == 4)
                sts64(prow, enc_pair(xp[0], xp[1 % GROUP]), enc_pair(xp[2 % GROUP], xp[3 % GROUP]));
            else if (GROUP == 2)
                sts32(prow, enc_pair(xp[0], xp[1 % GROUP]));
            else
                sts32(prow, enc16(xp[0]) & 0xffffu);
            if (warp == 4) TR(i, 18);
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
                float* xs2 = xch + 128;
                if (lane == 0)
#pragma unroll
                    for (int k = 0; k < 2 * GROUP; ++k) xs2[wq * 16 + k] = red[k];
                named_sync(1, 128);
                if (m == 0) {
                    float* base = P.part + ((int64_t)ki.unit * P.nslot + ki.slot) * part_stride(GROUP);
#pragma unroll
                    for (int g = 0; g < GROUP; ++g) {
                        base[GROUP * D + 2 * g] = mrun[g];
                        base[GROUP * D + 2 * g + 1] = xs2[g] + xs2[16 + g] + xs2[32 + g] + xs2[48 + g];
                        re.lz[g] = xs2[GROUP + g] + xs2[16 + GROUP + g] + xs2[32 + GROUP + g] + xs2[48 + GROUP + g];
                    }
                }
                named_sync(1, 128);
            }
            if (m == 0) {
#pragma unroll
                for (int g = 0; g < GROUP; ++g) re.corr[g] = corr[g];
                __threadfence_block();
                *reinterpret_cast<volatile int*>(&re.tag) = i;
            }
            if (warp == 4) TR(i, 19);
            fence_async_smem();
            __syncwarp();
            if (warp == 4) TR(i, 20);
            if (lane == 0) mbar_arrive(b_pready(b));
            if (warp == 4) TR(i, 6);
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
        int end_at = 0x7fffffff;
        struct VR {
            uint4 c0, c1;
            uint32_t s16, z16;
            uint2 s4;
            int unit, flags, slot;
        };
        int pflags = 0, punit = 0, pslot = 0;
        float pstep = 0.f;
        auto correct = [&](int j) {
            const int b = j & 1;
            mbar_wait(b_ofull(b), (j >> 1) & 1);
            if (warp == 8) TR(j, 9);
            tc_fence_after();
            uint32_t ov[2 * GROUP];
            tmem_ld<2 * GROUP>(lane_base + 32 + b * 16, ov);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_ofree(b));
            RingEntry& re = ring[j & 3];
            while (*reinterpret_cast<volatile int*>(&re.tag) != j) {
            }
            __threadfence_block();
            const float f = pstep * wch;
#pragma unroll
            for (int g = 0; g < GROUP; ++g) o[g] = fmaf(o[g], re.corr[g], (float)((int)ov[2 * g] + 128 * (int)ov[2 * g + 1]) * f);
            if (pflags & FL_LAST) {
                float* base = P.part + ((int64_t)punit * P.nslot + pslot) * part_stride(GROUP);
#pragma unroll
                for (int g = 0; g < GROUP; ++g) {
                    base[g * D + ch] = o[g] + re.lz[g];
                    o[g] = 0.f;
                }
            }
        };
        auto vload = [&](VR& v, int i) {
            if (i > end_at) {
                v.flags = FL_END;
                return;
            }
            mbar_wait(b_dfull(i % NDESC), (i / NDESC) & 1);
            const PageDesc pd = *desc_ptr(i);
            v.unit = pd.unit;
            v.flags = pd.flags;
            v.slot = pd.slot;
            if (pd.flags & FL_END) {
                end_at = i;
                return;
            }
            const uint8_t* vp = pd.vp;
            v.c0 = ldg_na128(vp + 32 * r);
            v.c1 = ldg_na128(vp + 32 * r + 16);
            v.s16 = ldg16(vp + G * D / 4 + 2 * r);
            v.z16 = ldg16(vp + G * D / 4 + 2 * G + 2 * r);
            v.s4 = ldg64(vp + G * D / 4 + 8 * lane);
        };
        auto vproc = [&](VR& v, int i) -> bool {
            const int b = i & 1;
            if (v.flags & FL_END) {
                if (i >= 1) correct(i - 1);
                return false;
            }
            if (i >= 2) mbar_wait(b_vfree(b), ((i >> 1) - 1) & 1);
            const uint32_t av = sbase + L::o_av + b * kTileA;
            {
                const uint32_t w[8] = {v.c0.x, v.c0.y, v.c0.z, v.c0.w, v.c1.x, v.c1.y, v.c1.z, v.c1.w};
                const uint32_t dst = av + a_off(0, r);
#pragma unroll
                for (int i8 = 0; i8 < 8; ++i8) sts128(dst + 128 * i8, w[i8] & M0, w[i8] & M1, w[i8] & M2, w[i8] & M3);
            }
            *reinterpret_cast<float2*>(smem + L::o_vmeta + b * 1024 + 8 * r) = make_float2(h2f(v.s16), h2f(v.z16));
            float smax = hmax4(v.s4);
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o2));
            smax *= 1.125f;  // p <= 2^(f16 max rounding) < 1.125
            const float invp = smax > 0.f ? __fdividef((float)kQuant, smax) : 0.f;
            if (r == 0) vinfo[b] = invp;
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_vready(b));
                mbar_arrive(b_dempty(i % NDESC));
            }
            if (warp == 8) TR(i, 8);
            if (i >= 1) correct(i - 1);
            pflags = v.flags;
            punit = v.unit;
            pslot = v.slot;
            pstep = smax / kQuant;
            return true;
        };
        VR v0, v1, v2, v3;
        vload(v0, 0);
        vload(v1, 1);
        vload(v2, 2);
        for (int i = 0;; i += 4) {
            vload(v3, i + 3);
            if (!vproc(v0, i)) break;
            vload(v0, i + 4);
            if (!vproc(v1, i + 1)) break;
            vload(v1, i + 5);
            if (!vproc(v2, i + 2)) break;
            vload(v2, i + 6);
            if (!vproc(v3, i + 3)) break;
        }
    } else if (warp == 12) {
        // ===================== scheduler: work items -> page descriptors =====================
        if (lane == 0) {
            const int units = P.units;
            const int nq0 = units * P.cmx[0], nq1 = units * P.cmx[1], nq2 = units * P.cmx[2];
            int tk = atomicAdd(P.ctr, 1);
            int it = 0;
            for (;;) {
                int u = 0, p0 = 0, p1 = 0, slot = 0;
                bool have = false;
                while (!have) {
                    const int tt = tk;
                    if (tt >= nq0 + nq1 + nq2) break;
                    tk = atomicAdd(P.ctr, 1);
                    int sect, idx;
                    if (tt < nq0) {
                        sect = 0;
                        idx = tt;
                    } else if (tt < nq0 + nq1) {
                        sect = 1;
                        idx = tt - nq0;
                    } else {
                        sect = 2;
                        idx = tt - nq0 - nq1;
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
                const int b_ = u / c.cfg.h_kv, h_ = u - b_ * c.cfg.h_kv;
                const uint16_t* qsrc = P.q + ((int64_t)b_ * c.cfg.h_q + (int64_t)h_ * GROUP) * D;
                const int n_pages = have ? p1 - p0 : 1;
                for (int k = 0; k < n_pages; ++k) {
                    const int s = it % NDESC;
                    if (it >= NDESC) mbar_wait(b_dempty(s), ((it / NDESC) - 1) & 1);
                    PageDesc* pd = reinterpret_cast<PageDesc*>(smem + L::o_desc + s * L::kDesc);
                    if (!have) {
                        pd->flags = FL_END;
                        mbar_arrive(b_dfull(s));
                        break;
                    }
                    const int p = p0 + k;
                    pd->kp = c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + p] * c.key_slot_bytes;
                    pd->vp = c.value_pool + (int64_t)c.value_block_table[(int64_t)u * c.max_pages + p] * c.value_slot_bytes;
                    pd->unit = u;
                    pd->flags = (p == p0 ? FL_FIRST : 0) | (p == p1 - 1 ? FL_LAST : 0);
                    pd->slot = slot;
                    if (p == p0) {
                        mbar_expect_tx(b_dfull(s), GROUP * D * 2);
                        bulk_g2s(desc_q(s), qsrc, GROUP * D * 2, b_dfull(s));
                    } else {
                        mbar_arrive(b_dfull(s));
                    }
                    TR(it, 0);
                    ++it;
                }
                if (!have) break;
            }
        }
    } else if (warp == 13) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t id = idesc_i8(NB);
            const int nkb = d_boost > 0 ? 1 : 0;
            auto issue_pv = [&](int j) {
                const int b = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                mbar_wait(b_pready(b), ph);
                mbar_wait(b_vready(b), ph);
                if (j >= 2) mbar_wait(b_ofree(b), ((j >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t av = sbase + L::o_av + b * kTileA;
                const uint32_t bp = sbase + L::o_bp + b * 128 * NB;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_i8(tmem + 32 + b * 16, sdesc(av + 4096 * k, 1024, 128), sdesc(bp + 512 * k, 128, 128), id, k > 0);
                umma_commit(b_ofull(b));
                umma_commit(b_vfree(b));
                TR(j, 7);
            };
            int i = 0;
            for (;; ++i) {
                const int b = i & 1;
                mbar_wait(b_kready(b), (i >> 1) & 1);
                if (kinfo[b].flags & FL_END) break;
                tc_fence_after();
                const uint32_t ak = sbase + L::o_ak + b * kTileAK;
                const uint32_t bq = sbase + L::o_bqk + b * 160 * NB;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_i8(tmem + b * 16, sdesc(ak + 4096 * k, 1024, 128), sdesc(bq + 512 * k, 128, 128), id, k > 0);
                if (nkb) umma_i8(tmem + b * 16, sdesc(ak + 4096 * 4, 1024, 128), sdesc(bq + 512 * 4, 128, 128), id, 1);
                umma_commit(b_sfull(b));
                TR(i, 4);
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
            fptok::chunk<GROUP>(P.c, P.q, P.part, P.nslot, part_stride(GROUP), scratch, u, fc, lane);
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
__global__ void __launch_bounds__(kMergeWarps * 32) combine_kernel(Params P) {
    const int u = blockIdx.x / GROUP, g = blockIdx.x - (blockIdx.x / GROUP) * GROUP;
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
    constexpr int kStride = part_stride(GROUP);
    auto slot_of = [&](int i) {
        if (i < nfc) return i;
        if (i < nfc + nch[0]) return P.fmax + (i - nfc);
        if (i < nfc + nch[0] + nch[1]) return P.fmax + P.cmx[0] + (i - nfc - nch[0]);
        return P.fmax + P.cmx[0] + P.cmx[1] + (i - nfc - nch[0] - nch[1]);
    };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const int64_t row = (int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + g;
    lse_merge_row<GROUP>(P.part + (int64_t)u * P.nslot * kStride, kStride, nparts, slot_of, g, P.out, P.out_dtype, row);
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

bool tc_attention_supported(const KittyCacheDesc& c) {
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
    p.part_bytes = (size_t)p.units * p.nslot * part_stride(p.group) * sizeof(float);
    return p;
}

size_t tc_attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens) {
    if (!tc_attention_supported(c)) return 0;
    const TcPlan p = plan(c, max_tokens);
    return p.ctr_bytes + p.part_bytes;
}

template <int GROUP>
static cudaError_t launch_t(const Params& prm, cudaStream_t st) {
    auto kfn = tc_attention_kernel<GROUP>;
    const int sm = Smem<GROUP>::kBytes;
    static cudaError_t attr = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);  // once per instantiation
    if (attr != cudaSuccess) return attr;
    cudaError_t e;
    kfn<<<num_sms() * kCtasPerSm, kThreads, sm, st>>>(prm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    combine_kernel<GROUP><<<prm.units * GROUP, kMergeWarps * 32, 0, st>>>(prm);
    return cudaGetLastError();
}

cudaError_t launch_tc_attention(const KittyCacheDesc& c, const uint16_t* q, void* out, int out_dtype,
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

cudaError_t tc_attention_trace(int enable, long long* host_out, int max_rows) {
    cudaError_t e = cudaMemcpyToSymbol(tcattn::g_tr_on, &enable, sizeof(int));
    if (e != cudaSuccess || host_out == nullptr) return e;
    const int n = max_rows < tcattn::kTrPages ? max_rows : tcattn::kTrPages;
    return cudaMemcpyFromSymbol(host_out, tcattn::g_tr, sizeof(long long) * n * tcattn::kTrFields);
}

}  // namespace kitty
