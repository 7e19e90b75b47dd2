// Fused dequant-attention decode kernel for d = g = 128 (K4 + K5 in one launch).
//
// Semantics: KittyCacheState.attend (cache.py:217-252) -- per (sequence, KV
// head) unit, logits q.k / sqrt(d) over sink | key pages | key q-buffer, fp32
// max-subtracted softmax, probabilities times values over sink | value pages |
// value q-buffer | local -- with pages dequantised inside the loop (Alg. 1,
// PAPER.md:425-446) instead of from cached f32 rows.
//
// Design:
//  * persistent CTAs (2 per SM x 4 warps); every warp pulls work items from
//    an atomic queue: FP items (the unit's full-precision tokens, CUDA cores)
//    first, then chunks of `ppc` quantized K/V page pairs (tensor cores);
//  * each warp streams page pairs through a private 2-stage shared-memory ring
//    with cp.async.bulk (1-D TMA) + mbarrier, so the next pair is in flight
//    while the current one is computed;
//  * 2-bit codes become fp16 MMA operands with one PRMT (pair two channels)
//    plus one LOP3 per 2 codes: (x & mask) | 0x6400 = 1024 + w*c, w in {16, 64};
//    the 1024 offset and w are removed per row after the MMA;
//  * per-channel key scale is folded into q (B = q*alpha*s, fp16), per-token
//    value scale into p (B = p*s); zero points and the offset sums come out of
//    one auxiliary MMA tile (row 0 = ones, row 8 = zeros) whose B columns 4-7
//    carry the unscaled q / p (GQA group <= 4 leaves them free);
//  * mma.sync.m16n8k16 f16 x f16 -> f32, swap-AB: M = 16 tokens (QK) or 16
//    channels (PV), N = the GQA group, K = 16 channels (QK) or tokens (PV);
//  * warp-shuffle online softmax in the log2 domain; partials (m, l, acc) per
//    item go to the workspace and the last item of a unit merges them (LSE)
//    and writes the bf16/f32 output -- no separate combine launch.
#include <cstdio>
#include <cstdlib>

#include "kitty_attention.cuh"
#include "kitty_combine.cuh"
#include "kitty_fp.cuh"
#include "kitty_codec.cuh"

namespace kitty {
namespace fastattn {

constexpr int D = 128;
constexpr int G = 128;
// floats per partial record (acc[group][D], then (m, l) per row), padded to 16 B
__host__ __device__ constexpr int part_stride(int group) { return (group * (D + 2) + 3) & ~3; }
#ifndef KITTY_FAST_WARPS
#define KITTY_FAST_WARPS 4
#endif
constexpr int kWarps = KITTY_FAST_WARPS;  // warps per CTA (a fifth warp shares lane quarter 0 at TMEM column 64)
#ifndef KITTY_FAST_SINGLE
#define KITTY_FAST_SINGLE 0
#endif
#ifndef KITTY_FAST_CTAS
#define KITTY_FAST_CTAS 3
#endif
#ifndef KITTY_FAST_HALF
#define KITTY_FAST_HALF 0
#endif
// Staging: 2-stage (key, value) page-pair ring per warp at 8 warps / SM; or
// (KITTY_FAST_HALF) two key slots + one value slot per warp at 12 warps / SM,
// the next value page loaded while the next key page's QK runs; or one key
// slot + one value slot per warp, each refilled as soon as it is consumed, at
// 4 * KITTY_FAST_CTAS warps / SM.
constexpr bool kSingle = KITTY_FAST_SINGLE != 0;
constexpr bool kHalf = !kSingle && KITTY_FAST_HALF != 0;
constexpr int kStages = kSingle ? 1 : 2;  // key slots per warp
constexpr int kVStages = (kSingle || kHalf) ? 1 : 2;
#ifndef KITTY_HALF_CTAS
#define KITTY_HALF_CTAS 3
#endif
constexpr int kCtasPerSm = kSingle ? KITTY_FAST_CTAS : (kHalf ? KITTY_HALF_CTAS : 2);
constexpr int kTmemCols = kWarps > 4 ? 128 : 64;  // per CTA; per warp (its TMEM lane quarter, + 64 columns for warps 4-7): [0,32) output accumulators, [32,48) q fragments
constexpr int kKeySlotMax = 5760;  // d_boost = 32
constexpr int kValueSlot = 4608;
constexpr int kPtStride = 136;     // f16 per row of the transposed-P buffer
constexpr int kFpChunk = 32;       // fp tokens per online-softmax step
constexpr int kMaxTableUnits = 2048;  // units whose lengths the kernel caches in shared memory
constexpr float kAlpha = 0.12751743074f;  // log2(e) / sqrt(128)
constexpr uint32_t kMagic = 0x64006400u;  // f16x2 (1024, 1024)
constexpr uint32_t kOnes = 0x3C003C00u;   // f16x2 (1, 1)

// Per-warp shared memory: this fixed part, then the page slots -- kStages key
// slots and kVStages value slots, sized by the cache's slot bytes at launch
// (warp_bytes), so that a 5 248-byte key page costs no more than that.
template <int PT_ROWS>
struct __align__(16) WarpFixedT {
    struct {
        uint32_t pt[PT_ROWS][kPtStride / 2];  // P^T as f16x2: p*s per query, then p (rows 4-7 / 8-15 for group 4 / 8)
    } u;
    uint32_t ones[64];            // f16x2 (1, 1): scale operand of the aux B columns
    uint8_t inv[32];              // boosted channel of high_bits row j
    unsigned long long mbar[3];   // 2-stage: one per stage; single / half: key slot(s), value slot
};
template <int GROUP>
__host__ __device__ constexpr int warp_fixed_bytes() {
    return static_cast<int>((sizeof(WarpFixedT<GROUP == 8 ? 16 : 8>) + 127) & ~size_t(127));
}
template <int GROUP>
__host__ __device__ inline int warp_smem_bytes(int kslot, int vslot) {
    return (warp_fixed_bytes<GROUP>() + kStages * kslot + kVStages * vslot + 127) & ~127;
}

struct Params {
    KittyCacheDesc c;
    const uint16_t* q;
    void* out;
    int out_dtype;
    int ppc;    // page pairs per quantized item
    int cmax;   // quantized items per unit (grid bound)
    int fmax;   // fp-token chunk items per unit (grid bound)
    int cs[3];    // page-chunk size of schedule level 0 / 1 / 2
    int cmx[3];   // chunks per unit bound of each level
    int lvl[4];   // level 1 / 2 starts in per mille of vp: units < 512 pages, >= 512 pages
    int nslot;    // partial slots per unit: fmax + cmx[0] + cmx[1] + cmx[2]
    int units;
    int max_tokens;  // the caller's bound on the unit lengths (longer units: clamped + KITTY_STATUS_LENGTH)
    uint32_t units_mul, units_shift;  // fast division by units (quotient = (umulhi(n, mul) + n) >> shift)
    int* ctr;   // [0] next item, [1] finished warps
    float* part;
};

// ---- optional per-warp trace (kitty_attention_trace): where does the time go ----
constexpr int kTraceWarps = 16384;
constexpr int kTraceFields = 10;
__device__ long long g_trace[kTraceWarps * kTraceFields];
__device__ int g_trace_on;   // bit 0: record the trace; bit 1: skip page loads (compute-only timing)

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- small PTX helpers --------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Pages are read once per step: stream them through L2 with evict_first so the
// split-KV partials (re-read by the combine right after) stay resident.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first())
        : "memory");
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Tensor memory as an extension of the register file: the running output
// accumulators (32 fp32 per lane) live in TMEM between pages, so the QK phase
// runs with 32 more free registers (16 warps / SM instead of 12).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[8][4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0][0]), "f"(v[0][1]), "f"(v[0][2]), "f"(v[0][3]), "f"(v[1][0]), "f"(v[1][1]), "f"(v[1][2]), "f"(v[1][3]),
        "f"(v[2][0]), "f"(v[2][1]), "f"(v[2][2]), "f"(v[2][3]), "f"(v[3][0]), "f"(v[3][1]), "f"(v[3][2]), "f"(v[3][3]),
        "f"(v[4][0]), "f"(v[4][1]), "f"(v[4][2]), "f"(v[4][3]), "f"(v[5][0]), "f"(v[5][1]), "f"(v[5][2]), "f"(v[5][3]),
        "f"(v[6][0]), "f"(v[6][1]), "f"(v[6][2]), "f"(v[6][3]), "f"(v[7][0]), "f"(v[7][1]), "f"(v[7][2]), "f"(v[7][3])
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[8][4]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=f"(v[0][0]), "=f"(v[0][1]), "=f"(v[0][2]), "=f"(v[0][3]), "=f"(v[1][0]), "=f"(v[1][1]), "=f"(v[1][2]),
          "=f"(v[1][3]), "=f"(v[2][0]), "=f"(v[2][1]), "=f"(v[2][2]), "=f"(v[2][3]), "=f"(v[3][0]), "=f"(v[3][1]),
          "=f"(v[3][2]), "=f"(v[3][3]), "=f"(v[4][0]), "=f"(v[4][1]), "=f"(v[4][2]), "=f"(v[4][3]), "=f"(v[5][0]),
          "=f"(v[5][1]), "=f"(v[5][2]), "=f"(v[5][3]), "=f"(v[6][0]), "=f"(v[6][1]), "=f"(v[6][2]), "=f"(v[6][3]),
          "=f"(v[7][0]), "=f"(v[7][1]), "=f"(v[7][2]), "=f"(v[7][3])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[8][2]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0][0]), "r"(v[0][1]), "r"(v[1][0]), "r"(v[1][1]), "r"(v[2][0]), "r"(v[2][1]), "r"(v[3][0]), "r"(v[3][1]),
        "r"(v[4][0]), "r"(v[4][1]), "r"(v[5][0]), "r"(v[5][1]), "r"(v[6][0]), "r"(v[6][1]), "r"(v[7][0]), "r"(v[7][1])
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[8][2]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[3][0]),
          "=r"(v[3][1]), "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[5][0]), "=r"(v[5][1]), "=r"(v[6][0]), "=r"(v[6][1]),
          "=r"(v[7][0]), "=r"(v[7][1])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D = A x B (C = 0): lets ptxas feed RZ instead of zeroing accumulators.
__device__ __forceinline__ void mma16816_z(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
    uint32_t r;
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}

__device__ __forceinline__ uint32_t lds32(const void* p) { return *reinterpret_cast<const uint32_t*>(p); }

// Two 32-bit words = 16 tokens (K: one channel row) or 16 channels (V: one
// token row) each; byte b of both -> the fp16x2 A operands of 4 tokens x 2
// rows.  Values are 1024 + 16 c (rows gid) and 1024 + 64 c (rows gid + 8).
//   e_lo / e_hi: codes 0 / 1 of the byte, o_lo / o_hi: codes 2 / 3.
// (a & b) | c in ONE LOP3: with two immediates ptxas splits it into two, so
// the masks / magic are kept in registers (Consts, made opaque once per warp).
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

struct Consts {
    uint32_t m0, m1, m2, m3, magic;
    __device__ __forceinline__ Consts() {
        m0 = 0x03000300u;  // code 0 of the byte, from its copy in bits 8-15: weight 256
        m1 = 0x000C000Cu;  // code 1, bits 2-3: weight 4
        m2 = 0x00300030u;  // code 2, bits 4-5: weight 16
        m3 = 0x00C000C0u;  // code 3, bits 6-7: weight 64
        magic = kMagic;
        asm volatile("" : "+r"(m0), "+r"(m1), "+r"(m2), "+r"(m3), "+r"(magic));
    }
};

// Byte b of two rows -> the fp16x2 A operands of its 4 codes: one PRMT puts
// byte b of w0 in bytes 0 and 1 and byte b of w1 in bytes 2 and 3, then one
// LOP3 per code keeps that code's two bits inside the mantissa and ORs the
// exponent of 1024: f16 = 1024 + w * code with w = 256 / 4 / 16 / 64 for
// codes 0 / 1 / 2 / 3 (the weight and the 1024 are removed per row after the
// MMA; w >= 4 keeps the offset cancellation far below fp16 operand rounding).
template <int B>
__device__ __forceinline__ void conv_byte(const Consts& k, uint32_t w0, uint32_t w1, uint32_t& c0,
                                          uint32_t& c1, uint32_t& c2, uint32_t& c3) {
    constexpr uint32_t sel = B | (B << 4) | ((4 + B) << 8) | ((4 + B) << 12);
    const uint32_t x = prmt(w0, w1, sel);
    c0 = and_or(x, k.m0, k.magic);
    c1 = and_or(x, k.m1, k.magic);
    c2 = and_or(x, k.m2, k.magic);
    c3 = and_or(x, k.m3, k.magic);
}

// acc[8][4] += A(2-bit codes of rows r0..r3, word gid) x B for one k-step.
// rows = (w0, w1) pair P0 and (w2, w3) pair P1.
template <bool FIRST = false>
__device__ __forceinline__ void mma_codes(const Consts& k, float (&acc)[8][4], uint32_t w0, uint32_t w1,
                                          uint32_t w2, uint32_t w3, uint32_t b0, uint32_t b1) {
    // all 8 tiles' A fragments first (32 registers): distinct registers let the
    // HMMAs issue back to back instead of waiting on operand-read WAR hazards
    uint32_t a[8][4];
    conv_byte<0>(k, w0, w1, a[0][0], a[0][1], a[1][0], a[1][1]);
    conv_byte<0>(k, w2, w3, a[0][2], a[0][3], a[1][2], a[1][3]);
    conv_byte<1>(k, w0, w1, a[2][0], a[2][1], a[3][0], a[3][1]);
    conv_byte<1>(k, w2, w3, a[2][2], a[2][3], a[3][2], a[3][3]);
    conv_byte<2>(k, w0, w1, a[4][0], a[4][1], a[5][0], a[5][1]);
    conv_byte<2>(k, w2, w3, a[4][2], a[4][3], a[5][2], a[5][3]);
    conv_byte<3>(k, w0, w1, a[6][0], a[6][1], a[7][0], a[7][1]);
    conv_byte<3>(k, w2, w3, a[6][2], a[6][3], a[7][2], a[7][3]);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        if (FIRST)
            mma16816_z(acc[m], a[m][0], a[m][1], a[m][2], a[m][3], b0, b1);
        else
            mma16816(acc[m], a[m][0], a[m][1], a[m][2], a[m][3], b0, b1);
    }
}

struct UnitGeom {
    int n, kp, vp, nfp;
};

// Pages of a unit are scheduled in three levels of decreasing chunk size:
// [0, 0.85 vp) in chunks of cs[0] (<= 8 pages), [0.85 vp, 0.95 vp) in cs[0] / 4,
// the rest page by page; the queue serves level 0, 1, 2, so it drains in small
// pieces and no SM idles behind a long item (swept on B200 with
// tools/sweep_sched.sh).  Level boundaries are per-mille of vp (tuning knobs,
// set once by the host plan; KITTY_SCHED overrides them for sweeps).
// Level starts per mille of vp, one pair for units below 512 pages and one
// from 512 pages on (128K-token contexts have tails long enough that a larger
// level 0 wins: C4 45.9 -> 44.0 us per layer).  The host plan passes them per
// launch (Params::lvl), after quantising level 0 to whole rounds of the warps.
static int h_lvl[4] = {850, 950, 880, 960};
__host__ __device__ __forceinline__ int level_begin(int lv, int vp, const int* lvl4) {
    const int* lvl = lvl4 + (vp >= 512 ? 2 : 0);
    return lv == 0 ? 0 : (lv == 1 ? (vp * lvl[0]) / 1000 : (lv == 2 ? (vp * lvl[1]) / 1000 : vp));
}

__device__ __forceinline__ UnitGeom unit_geom(const KittyCacheDesc& c, int u, int max_tokens) {
    UnitGeom g;
    g.n = min(c.unit_len[u], max_tokens);
    const int S = c.cfg.s;
    const int past = g.n > S ? g.n - S : 0;
    g.kp = past / G;
    g.vp = (past - min(c.cfg.r, past)) / G;
    g.nfp = g.n > S ? S + (past - g.vp * G) : g.n;  // sink + value fp tokens
    return g;
}

// ---- the kernel ------------------------------------------------------------------

template <int GROUP, int NKH>
__global__ void __launch_bounds__(kWarps * 32, kCtasPerSm) fast_attention_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    using WarpFixed = WarpFixedT<GROUP == 8 ? 16 : 8>;
    const int wbytes = warp_smem_bytes<GROUP>(static_cast<int>(P.c.key_slot_bytes), static_cast<int>(P.c.value_slot_bytes));
    uint8_t* wbase = smem_raw + warp * wbytes;
    WarpFixed& sm = *reinterpret_cast<WarpFixed*>(wbase);
    uint8_t* const kslots = wbase + warp_fixed_bytes<GROUP>();
    uint8_t* const vslots = kslots + kStages * static_cast<int>(P.c.key_slot_bytes);
    const KittyCacheDesc& c = P.c;
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g;
    const int d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int vslot = static_cast<int>(c.value_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D;  // KTYP key scales
    const int zero_off = scale_off + 2 * D;
    const int hkv = c.cfg.h_kv;
    // group <= 4: B columns 0-3 are the queries, 4-7 auxiliary (unscaled q / p);
    // group 8: all eight are queries and the auxiliary sums take a second MMA
    constexpr bool kFull = GROUP == 8;
    const bool main_col = kFull || gid < 4;
    const bool row0 = gid == 0;

    __shared__ uint32_t tmem_base_sh;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (lane == 0) {
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        mbar_init(&sm.mbar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tmem_base_sh + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + 64u * (warp >> 2);
    sm.inv[lane] = 0;
    sm.ones[lane] = kOnes;
    sm.ones[lane + 32] = kOnes;
    __syncwarp();
    const Consts kc;
    // launched as a programmatic dependent of the preceding kernel (the append):
    // the prologue above overlaps its tail; nothing of the cache is read before this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the fp-token grid (our programmatic dependent) may be scheduled from now on
    asm volatile("griddepcontrol.launch_dependents;");
    // per-CTA copy of the unit lengths: the queue decode reads them from shared
    // memory instead of paying a global round trip per work item
    int* s_ulen = reinterpret_cast<int*>(smem_raw + wbytes * kWarps);  // dynamic, units entries
    const bool len_table = P.units <= kMaxTableUnits;
    if (len_table) {
        for (int i = threadIdx.x; i < P.units; i += blockDim.x) s_ulen[i] = min(c.unit_len[i], P.max_tokens);
    }
    __syncthreads();
    auto geom = [&](int u) {
        UnitGeom g;
        g.n = len_table ? s_ulen[u] : min(c.unit_len[u], P.max_tokens);
        const int S = c.cfg.s;
        const int past = g.n > S ? g.n - S : 0;
        g.kp = past / G;
        g.vp = (past - min(c.cfg.r, past)) / G;
        g.nfp = g.n > S ? S + (past - g.vp * G) : g.n;
        return g;
    };
    auto div_units = [&](int n) {
        return static_cast<int>((__umulhi(static_cast<uint32_t>(n), P.units_mul) + static_cast<uint32_t>(n)) >> P.units_shift);
    };
#ifndef KITTY_TRACE
#define KITTY_TRACE 0
#endif
    // tracing is compiled in only with -DKITTY_TRACE=1 (the timer reads cost ~30 instructions / page)
    const bool trace = KITTY_TRACE && (g_trace_on & 1) != 0;
    const bool noload = KITTY_TRACE && (g_trace_on & 2) != 0;
    long long tr_t0 = trace ? gtimer() : 0, tr_fp = 0, tr_merge = 0, tr_wait = 0;
    int tr_nfp = 0, tr_npages = 0, tr_nmerge = 0;

    uint32_t issued = 0, consumed = 0;  // page pairs put in flight / consumed (stage = count & 1)

    // work tickets are fetched one pull ahead so the atomic's round trip overlaps
    // the current item (lane 0 holds the outstanding ticket)
    int tk = 0;
    if (lane == 0) tk = atomicAdd(P.ctr, 1);
    auto pull = [&]() -> int {
        const int i = __shfl_sync(0xffffffffu, tk, 0);
        if (lane == 0) tk = atomicAdd(P.ctr, 1);
        return i;
    };
    // item -> (kind, unit, a, b); kind 0 = end, 1 = fp chunk a, 2 = pages [a, b), 3 = empty.
    // Queue: all fp chunks first (latency-bound CUDA-core work, one wave across
    // every warp while the first page loads are in flight; measured 148 -> 140 us
    // per C2 layer against interleaving them with level 0), then level-0, level-1
    // and level-2 page chunks.
    const int nf = 0, nq0 = P.units * P.cmx[0];  // fp chunks run in fp_tokens_kernel
    const int nq1 = P.units * P.cmx[1], nq2 = P.units * P.cmx[2];
    const int n2 = 2 * min(nf, nq0);
    auto decode = [&](int it, int& kind, int& u, int& p0, int& p1) {
        int sect, idx;  // -1 fp, 0..2 page level
        if (it < nf) {  // the fp chunks first: latency-bound, they overlap on all warps at once
            sect = -1;
            idx = it;
        } else if (it < nf + nq0) {
            sect = 0;
            idx = it - nf;
        } else if (it < nf + nq0 + nq1) {
            sect = 1;
            idx = it - nf - nq0;
        } else if (it < nf + nq0 + nq1 + nq2) {
            sect = 2;
            idx = it - nf - nq0 - nq1;
        } else {
            kind = 0;
            return;
        }
        const int ch = div_units(idx);
        u = idx - ch * P.units;
        const UnitGeom gm = geom(u);
        if (sect < 0) {
            p0 = ch;
            p1 = 0;
            kind = (gm.n > 0 && ch * kFpChunk < gm.nfp) ? 1 : 3;
        } else {
            const int lb = level_begin(sect, gm.vp, P.lvl), le = level_begin(sect + 1, gm.vp, P.lvl);
            p0 = lb + ch * P.cs[sect];
            p1 = min(le, p0 + P.cs[sect]);
            kind = (p0 < p1 && gm.n > 0) ? 2 : 3;
        }
    };
    // partial slot of the page chunk starting at p0, and the chunk count of a unit
    auto page_slot = [&](int p0_, int vp) {
        const int lv = p0_ < level_begin(1, vp, P.lvl) ? 0 : (p0_ < level_begin(2, vp, P.lvl) ? 1 : 2);
        int slot = P.fmax + (p0_ - level_begin(lv, vp, P.lvl)) / P.cs[lv];
        for (int l = 0; l < lv; ++l) slot += P.cmx[l];
        return slot;
    };
    auto page_chunks = [&](int lv, int vp) {
        const int n = level_begin(lv + 1, vp, P.lvl) - level_begin(lv, vp, P.lvl);
        return (n + P.cs[lv] - 1) / P.cs[lv];
    };
    auto next_item = [&](int& kind, int& u, int& p0, int& p1) {
        for (;;) {
            decode(pull(), kind, u, p0, p1);
            if (kind != 3) return;
        }
    };
    auto issue = [&](int u, int p) {
        const int st = issued & 1;
        if (lane == 0 && noload) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.mbar[st])) : "memory");
        } else if (lane == 0) {
            const uint8_t* ks = c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + p] * kslot;
            const uint8_t* vs = c.value_pool + (int64_t)c.value_block_table[(int64_t)u * c.max_pages + p] * vslot;
            mbar_expect_tx(&sm.mbar[st], kslot + vslot);
            bulk_g2s(kslots + st * kslot, ks, kslot, &sm.mbar[st]);
            bulk_g2s(vslots + st * vslot, vs, vslot, &sm.mbar[st]);
        }
        __syncwarp();
        ++issued;
    };

    // per-unit query state: B fragments of q*alpha (f16x2) for this lane's column
    int cur_unit = -1;
    const uint16_t* q_cur = P.q;  // q rows of cur_unit (no per-page division)
    auto q_row = [&](int u, int g) {
        const int b = u / hkv, h = u - b * hkv;
        return P.q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + g) * D;
    };
    auto load_unit = [&](int u) {
        if (u == cur_unit) return;
        cur_unit = u;
        q_cur = q_row(u, 0);
        const int col = kFull ? gid : (gid & 3);
        const uint16_t* qg = q_row(u, col < GROUP ? col : 0);
        uint32_t qa[8][2];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int d = 16 * ks + 2 * tig + 8 * hh;
                const uint32_t w = col < GROUP ? __ldg(reinterpret_cast<const unsigned int*>(qg + d)) : 0u;
                qa[ks][hh] = pack_f16x2(__uint_as_float(w << 16) * kAlpha, __uint_as_float(w & 0xffff0000u) * kAlpha);
            }
        }
        tmem_wait_st();
        tmem_st16(taddr + 32, qa);
    };

    // ---- quantized pages: QK^T on the key slot, then P V on the value slot ----
    float om[2], ol[2], ob[4][2];  // running max / sum; per-weight-class row constants
    bool ofresh = true;  // output accumulators in TMEM not yet written for this item
    float acc[8][4];     // logits of the current page
    uint32_t pu[8][2];   // its probabilities, f16x2 (token pairs)
    float mnew[2], corr[2], bw[4][2];

    auto qk_page = [&](int st) {
        const uint8_t* kp = kslots + st * kslot;
        const uint32_t* kw = reinterpret_cast<const uint32_t*>(kp);
        // boosted rows -> channels (inverse of boost_idx)
        if (NKH > 0) {
            const uint32_t bw = lds32(kp + D * G / 4 + d_boost * G / 4 + 4 * lane);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t bi = (bw >> (8 * i)) & 0xffu;
                if (bi < 32u) sm.inv[bi] = static_cast<uint8_t>(4 * lane + i);
            }
            __syncwarp();
        }
        float aux[4], aux2[4];
        // aux lanes (B columns 4-7) read their "scale" from a ones buffer
        const uint8_t* sbase = main_col ? kp + scale_off : reinterpret_cast<const uint8_t*>(sm.ones);
        uint32_t qa[8][2];
        tmem_wait_st();
        tmem_ld16(taddr + 32, qa);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int c0 = 16 * ks + 2 * tig;
            const uint32_t b0 = hmul2(qa[ks][0], lds32(sbase + 2 * c0));
            const uint32_t b1 = hmul2(qa[ks][1], lds32(sbase + 2 * (c0 + 8)));
            const uint32_t w0 = kw[8 * c0 + gid], w1 = kw[8 * (c0 + 1) + gid];
            const uint32_t w2 = kw[8 * (c0 + 8) + gid], w3 = kw[8 * (c0 + 9) + gid];
            // aux tile: only rows 0 (ones) and 8 (zero points) are read back, so
            // every lane may load (rows 1-7 / 9-15 carry harmless copies)
            const uint32_t z0 = lds32(kp + zero_off + 2 * c0);
            const uint32_t z1 = lds32(kp + zero_off + 2 * (c0 + 8));
            if (ks == 0) {
                mma_codes<true>(kc, acc, w0, w1, w2, w3, b0, b1);
                mma16816_z(aux, kOnes, z0, kOnes, z1, b0, b1);
                if (kFull) mma16816_z(aux2, kOnes, z0, kOnes, z1, qa[ks][0], qa[ks][1]);
            } else {
                mma_codes(kc, acc, w0, w1, w2, w3, b0, b1);
                mma16816(aux, kOnes, z0, kOnes, z1, b0, b1);
                if (kFull) mma16816(aux2, kOnes, z0, kOnes, z1, qa[ks][0], qa[ks][1]);
            }
        }
        if (NKH > 0) {
            const int col = kFull ? gid : (gid & 3);
            const uint16_t* qg = q_cur + (col < GROUP ? col : 0) * D;
#pragma unroll
            for (int hk = 0; hk < NKH; ++hk) {
                const int j0 = 16 * hk + 2 * tig;
                const int jj[4] = {j0, j0 + 1, j0 + 8, j0 + 9};
                float hv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = sm.inv[jj[i]];
                    const float q4 = 4.f * kAlpha * bf16_to_f32(__ldg(reinterpret_cast<const unsigned short*>(qg) + ch));
                    const float sc = half_bits_to_f32(ld_u16(kp + scale_off + 2 * ch));
                    hv[i] = (main_col && col < GROUP && jj[i] < d_boost) ? q4 * sc : 0.f;
                }
                const uint32_t b0 = pack_f16x2(hv[0], hv[1]);
                const uint32_t b1 = pack_f16x2(hv[2], hv[3]);
                const uint32_t* hw = reinterpret_cast<const uint32_t*>(kp + D * G / 4);
                mma_codes(kc, acc, hw[8 * j0 + gid], hw[8 * (j0 + 1) + gid], hw[8 * (j0 + 8) + gid],
                          hw[8 * (j0 + 9) + gid], b0, b1);
                mma16816(aux, kOnes, 0u, kOnes, 0u, b0, b1);
            }
        }
        // aux row 0 (lanes 0-3): sum of B per column; row 8, columns 4-7: sum(z * q * alpha).
        // Row weights: even tiles hold codes 0 / 1 of a byte (w 256 / 4), odd tiles 2 / 3 (w 16 / 64).
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float sumB = __shfl_sync(0xffffffffu, aux[j], kFull ? tig : (tig & 1));
            const float cst = kFull ? __shfl_sync(0xffffffffu, aux2[2 + j], tig)
                                    : __shfl_sync(0xffffffffu, aux[2 + j], 2 + (tig & 1));
            bw[0][j] = cst - 4.f * sumB;    // w 256
            bw[1][j] = cst - 256.f * sumB;  // w 4
            bw[2][j] = cst - 64.f * sumB;   // w 16
            bw[3][j] = cst - 16.f * sumB;   // w 64
            float x0 = acc[0][j], x1 = acc[0][2 + j], x2 = acc[1][j], x3 = acc[1][2 + j];
#pragma unroll
            for (int m = 2; m < 8; m += 2) {
                x0 = fmaxf(x0, acc[m][j]);
                x1 = fmaxf(x1, acc[m][2 + j]);
                x2 = fmaxf(x2, acc[m + 1][j]);
                x3 = fmaxf(x3, acc[m + 1][2 + j]);
            }
            float pm = fmaxf(fmaxf(fmaf(x0, 1.f / 256.f, bw[0][j]), fmaf(x1, 1.f / 4.f, bw[1][j])),
                             fmaxf(fmaf(x2, 1.f / 16.f, bw[2][j]), fmaf(x3, 1.f / 64.f, bw[3][j])));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 4));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 8));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 16));
            mnew[j] = fmaxf(om[j], pm);
            corr[j] = ex2(om[j] - mnew[j]);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) bw[c4][j] -= mnew[j];
        }
        // probabilities (log2 domain), two tokens per f16x2 ex2: pu[m][j] = (p(tok), p(tok + 1))
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float wlo = (m & 1) ? 1.f / 16.f : 1.f / 256.f, whi = (m & 1) ? 1.f / 64.f : 1.f / 4.f;
            const int clo = (m & 1) ? 2 : 0, chi = (m & 1) ? 3 : 1;
#pragma unroll
            for (int j = 0; j < 2; ++j)
                pu[m][j] = ex2_h2(pack_f16x2(fmaf(acc[m][j], wlo, bw[clo][j]), fmaf(acc[m][2 + j], whi, bw[chi][j])));
        }
    };

    auto pv_page = [&](int st) {
        const uint8_t* vp = vslots + st * vslot;
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(vp);
        const uint8_t* vscale = vp + G * D / 4;
        // P^T -> shared (rows 0-3: p * s_token, rows 4-7: p), tokens 16 gid + 2m (+1)
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int tok = 16 * gid + 2 * m;
            const uint32_t sv = lds32(vscale + 2 * tok);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (kFull || tig < 2) {
                    const int g = 2 * tig + j;
                    const int w = 8 * gid + (m ^ gid);  // XOR swizzle: conflict-free stores and loads
                    sm.u.pt[g][w] = hmul2(pu[m][j], sv);
                    sm.u.pt[(kFull ? 8 : 4) + g][w] = pu[m][j];
                }
            }
        }
        __syncwarp();
        // the output accumulators (TMEM-parked, unweighted: a row's weight class
        // is the same on every page, so it is applied once at the flush) are
        // rescaled first when a real column's running max moved (warp vote),
        // then the P V MMAs accumulate straight into them
        const bool real0 = kFull || (tig < 2 && 2 * tig < GROUP), real1 = kFull || (tig < 2 && 2 * tig + 1 < GROUP);
        const bool rescale = __any_sync(0xffffffffu, (real0 && corr[0] != 1.f) || (real1 && corr[1] != 1.f));
        float oacc[8][4];
        if (ofresh) {
#pragma unroll
            for (int m = 0; m < 8; ++m) oacc[m][0] = oacc[m][1] = oacc[m][2] = oacc[m][3] = 0.f;
        } else {
            tmem_wait_st();
            tmem_ld32(taddr, oacc);
            if (rescale) {
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    oacc[m][0] *= corr[0];
                    oacc[m][2] *= corr[0];
                    oacc[m][1] *= corr[1];
                    oacc[m][3] *= corr[1];
                }
            }
        }
        float vaux[4], vaux2[4];
        const uint8_t* vzero = vscale + 2 * G;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int t0 = 16 * ks + 2 * tig;
            const uint32_t b0 = sm.u.pt[gid][8 * ks + (tig ^ ks)];
            const uint32_t b1 = sm.u.pt[gid][8 * ks + ((tig + 4) ^ ks)];
            const uint32_t w0 = vw[8 * t0 + gid], w1 = vw[8 * (t0 + 1) + gid];
            const uint32_t w2 = vw[8 * (t0 + 8) + gid], w3 = vw[8 * (t0 + 9) + gid];
            const uint32_t z0 = lds32(vzero + 2 * t0);
            const uint32_t z1 = lds32(vzero + 2 * (t0 + 8));
            mma_codes(kc, oacc, w0, w1, w2, w3, b0, b1);
            if (ks == 0)
                mma16816_z(vaux, kOnes, z0, kOnes, z1, b0, b1);
            else
                mma16816(vaux, kOnes, z0, kOnes, z1, b0, b1);
            if (kFull) {  // the unscaled p (rows 8-15 of P^T): sum p and sum p z
                const uint32_t c0u = sm.u.pt[8 + gid][8 * ks + (tig ^ ks)];
                const uint32_t c1u = sm.u.pt[8 + gid][8 * ks + ((tig + 4) ^ ks)];
                if (ks == 0)
                    mma16816_z(vaux2, kOnes, z0, kOnes, z1, c0u, c1u);
                else
                    mma16816(vaux2, kOnes, z0, kOnes, z1, c0u, c1u);
            }
        }
        // vaux lanes 0-1: sum(p s) per column; lanes 2-3: sum(p) and sum(p z).
        // Row constants (zero points, the 1024 offset) accumulate per column in
        // ob[weight class] and are added at the flush.
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float sBv = __shfl_sync(0xffffffffu, vaux[j], kFull ? tig : (tig & 1));
            const float lp = kFull ? __shfl_sync(0xffffffffu, vaux2[j], tig) : __shfl_sync(0xffffffffu, vaux[j], 2 + (tig & 1));
            const float zz = kFull ? __shfl_sync(0xffffffffu, vaux2[2 + j], tig)
                                   : __shfl_sync(0xffffffffu, vaux[2 + j], 2 + (tig & 1));
            ol[j] = fmaf(ol[j], corr[j], lp);
            ob[0][j] = fmaf(ob[0][j], corr[j], zz - 4.f * sBv);
            ob[1][j] = fmaf(ob[1][j], corr[j], zz - 256.f * sBv);
            ob[2][j] = fmaf(ob[2][j], corr[j], zz - 64.f * sBv);
            ob[3][j] = fmaf(ob[3][j], corr[j], zz - 16.f * sBv);
            om[j] = mnew[j];
        }
        tmem_st32(taddr, oacc);
        ofresh = false;
    };

    // single-stage mode: key slot (mbar[0]) and value slot (mbar[1]) refilled separately
    uint32_t kcon = 0, vcon = 0;
    auto issue_k = [&](int u_, int p_) {
        if (lane == 0) {
            const uint8_t* ks = c.key_pool + (int64_t)c.key_block_table[(int64_t)u_ * c.max_pages + p_] * kslot;
            mbar_expect_tx(&sm.mbar[0], kslot);
            bulk_g2s(kslots, ks, kslot, &sm.mbar[0]);
        }
        __syncwarp();
    };
    auto issue_v = [&](int u_, int p_) {
        if (lane == 0) {
            const uint8_t* vs = c.value_pool + (int64_t)c.value_block_table[(int64_t)u_ * c.max_pages + p_] * vslot;
            mbar_expect_tx(&sm.mbar[1], vslot);
            bulk_g2s(vslots, vs, vslot, &sm.mbar[1]);
        }
        __syncwarp();
    };
    // ---- work loop -------------------------------------------------------------------
    int kind, u, p0, p1;
    next_item(kind, u, p0, p1);
    int nkind = 0, nu = 0, np0 = 0, np1 = 0;
    if (kind != 0) next_item(nkind, nu, np0, np1);
    bool pending = false;  // the current item's first page pair is already in flight
    bool kpend = false, vpend = false;  // single-stage: next item's first key / value page in flight
    int p = p0;
#pragma unroll 1
    while (kSingle && kind != 0) {
        bool item_done;
        {
            if (p == p0) {
                if (!kpend) issue_k(u, p0);
                if (!vpend) issue_v(u, p0);
                kpend = vpend = false;
                load_unit(u);
                om[0] = om[1] = -INFINITY;
                ol[0] = ol[1] = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) ob[c4][0] = ob[c4][1] = 0.f;
                ofresh = true;
            }
            const bool more = p + 1 < p1;
            const bool chain = !more && nkind == 2;
            mbar_wait(&sm.mbar[0], kcon & 1);
            ++kcon;
            qk_page(0);
            __syncwarp();
            if (more) issue_k(u, p + 1);
            if (chain) {
                issue_k(nu, np0);
                kpend = true;
            }
            mbar_wait(&sm.mbar[1], vcon & 1);
            ++vcon;
            pv_page(0);
            __syncwarp();
            if (more) issue_v(u, p + 1);
            if (chain) {
                issue_v(nu, np0);
                vpend = true;
            }
            ++p;
            item_done = p == p1;
            if (item_done) {
                const int slot = page_slot(p0, geom(u).vp);
                float* base = P.part + ((int64_t)u * P.nslot + slot) * part_stride(GROUP);
                float oacc[8][4];
                tmem_wait_st();
                tmem_ld32(taddr, oacc);
                if (kFull || tig < 2) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int g = 2 * tig + j;
                        if (g < GROUP) {
#pragma unroll
                            for (int m = 0; m < 8; ++m)
                                *reinterpret_cast<float2*>(base + g * D + 16 * gid + 2 * m) =
                                    make_float2(fmaf(oacc[m][j], (m & 1) ? 1.f / 16.f : 1.f / 256.f, ob[(m & 1) ? 2 : 0][j]),
                                                fmaf(oacc[m][2 + j], (m & 1) ? 1.f / 64.f : 1.f / 4.f, ob[(m & 1) ? 3 : 1][j]));
                            if (gid == 0) {
                                base[GROUP * D + 2 * g] = om[j];
                                base[GROUP * D + 2 * g + 1] = ol[j];
                            }
                        }
                    }
                }
            }
        }
        if (item_done) {
            kind = nkind;
            u = nu;
            p0 = np0;
            p1 = np1;
            p = p0;
            if (kind != 0) next_item(nkind, nu, np0, np1);
        }
    }
    // half mode: key slots ring on mbar[0..1] (kiss / kcon), the value slot on mbar[2]
    uint32_t kiss = 0;
    auto issue_kh = [&](int u_, int p_) {
        const int ks_ = kiss & 1;
        if (lane == 0) {
            const uint8_t* src = c.key_pool + (int64_t)c.key_block_table[(int64_t)u_ * c.max_pages + p_] * kslot;
            mbar_expect_tx(&sm.mbar[ks_], kslot);
            bulk_g2s(kslots + ks_ * kslot, src, kslot, &sm.mbar[ks_]);
        }
        __syncwarp();
        ++kiss;
    };
    auto issue_vh = [&](int u_, int p_) {
        if (lane == 0) {
            const uint8_t* src = c.value_pool + (int64_t)c.value_block_table[(int64_t)u_ * c.max_pages + p_] * vslot;
            mbar_expect_tx(&sm.mbar[2], vslot);
            bulk_g2s(vslots, src, vslot, &sm.mbar[2]);
        }
        __syncwarp();
    };
#pragma unroll 1
    while (kHalf && kind != 0) {
        bool item_done;
        {
            if (p == p0) {
                if (!kpend) issue_kh(u, p0);
                if (!vpend) issue_vh(u, p0);
                kpend = vpend = false;
                load_unit(u);
                om[0] = om[1] = -INFINITY;
                ol[0] = ol[1] = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) ob[c4][0] = ob[c4][1] = 0.f;
                ofresh = true;
            }
            // the next key page into the other key slot right away; the next
            // value page once this one is consumed (it lands during the next QK)
            const bool more = p + 1 < p1;
            const bool chain = !more && nkind == 2;
            if (more) issue_kh(u, p + 1);
            if (chain) {
                issue_kh(nu, np0);
                kpend = true;
            }
            const int ks_ = kcon & 1;
            mbar_wait(&sm.mbar[ks_], (kcon >> 1) & 1);
            ++kcon;
            qk_page(ks_);
            mbar_wait(&sm.mbar[2], vcon & 1);
            ++vcon;
            pv_page(0);
            __syncwarp();
            if (more) issue_vh(u, p + 1);
            if (chain) {
                issue_vh(nu, np0);
                vpend = true;
            }
            ++p;
            item_done = p == p1;
            if (item_done) {
                const int slot = page_slot(p0, geom(u).vp);
                float* base = P.part + ((int64_t)u * P.nslot + slot) * part_stride(GROUP);
                float oacc[8][4];
                tmem_wait_st();
                tmem_ld32(taddr, oacc);
                if (kFull || tig < 2) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int g = 2 * tig + j;
                        if (g < GROUP) {
#pragma unroll
                            for (int m = 0; m < 8; ++m)
                                *reinterpret_cast<float2*>(base + g * D + 16 * gid + 2 * m) =
                                    make_float2(fmaf(oacc[m][j], (m & 1) ? 1.f / 16.f : 1.f / 256.f, ob[(m & 1) ? 2 : 0][j]),
                                                fmaf(oacc[m][2 + j], (m & 1) ? 1.f / 64.f : 1.f / 4.f, ob[(m & 1) ? 3 : 1][j]));
                            if (gid == 0) {
                                base[GROUP * D + 2 * g] = om[j];
                                base[GROUP * D + 2 * g + 1] = ol[j];
                            }
                        }
                    }
                }
            }
        }
        if (item_done) {
            kind = nkind;
            u = nu;
            p0 = np0;
            p1 = np1;
            p = p0;
            if (kind != 0) next_item(nkind, nu, np0, np1);
        }
    }
#pragma unroll 1
    while (!kSingle && !kHalf && kind != 0) {
        bool item_done;
        {
            if (p == p0) {
                if (!pending) issue(u, p0);
                pending = false;
                load_unit(u);
                om[0] = om[1] = -INFINITY;
                ol[0] = ol[1] = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) ob[c4][0] = ob[c4][1] = 0.f;
                ofresh = true;
            }
            // next page pair into the other stage: this item's next page, or the
            // next item's first page
            const bool more = p + 1 < p1;
            const bool chain = !more && nkind == 2;
            if (more) issue(u, p + 1);
            if (chain) {
                issue(nu, np0);
                pending = true;
            }
            const int st = consumed & 1;
            const long long tw0 = trace ? gtimer() : 0;
            mbar_wait(&sm.mbar[st], (consumed >> 1) & 1);
            if (trace) tr_wait += gtimer() - tw0;
            ++tr_npages;
            qk_page(st);
            pv_page(st);
            __syncwarp();
            ++consumed;
            ++p;
            item_done = p == p1;
            if (item_done) {
                const int slot = page_slot(p0, geom(u).vp);
                float* base = P.part + ((int64_t)u * P.nslot + slot) * part_stride(GROUP);
                float oacc[8][4];
                tmem_wait_st();
                tmem_ld32(taddr, oacc);
                if (kFull || tig < 2) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int g = 2 * tig + j;
                        if (g < GROUP) {
#pragma unroll
                            for (int m = 0; m < 8; ++m)
                                *reinterpret_cast<float2*>(base + g * D + 16 * gid + 2 * m) =
                                    make_float2(fmaf(oacc[m][j], (m & 1) ? 1.f / 16.f : 1.f / 256.f, ob[(m & 1) ? 2 : 0][j]),
                                                fmaf(oacc[m][2 + j], (m & 1) ? 1.f / 64.f : 1.f / 4.f, ob[(m & 1) ? 3 : 1][j]));
                            if (gid == 0) {
                                base[GROUP * D + 2 * g] = om[j];
                                base[GROUP * D + 2 * g + 1] = ol[j];
                            }
                        }
                    }
                }
            }
        }
        if (item_done) {
            kind = nkind;
            u = nu;
            p0 = np0;
            p1 = np1;
            p = p0;
            if (kind != 0) next_item(nkind, nu, np0, np1);
        }
    }
    if (trace && lane == 0) {
        const int wid = blockIdx.x * kWarps + warp;
        if (wid < kTraceWarps) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            long long* r = g_trace + (int64_t)wid * kTraceFields;
            r[0] = smid;
            r[1] = tr_t0;
            r[2] = gtimer();
            r[3] = tr_nfp;
            r[4] = tr_npages;
            r[5] = tr_fp;
            r[6] = tr_merge;
            r[7] = tr_wait;
            r[8] = warp;
            r[9] = 0;
        }
    }
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(kTmemCols));
    }
    // the last warp out resets the work queue for the next launch (after this
    // warp's outstanding ticket returned: using its value orders the atomics)
    __syncwarp();
    if (lane == 0) {
        asm volatile("" ::"r"(tk) : "memory");  // wait for the outstanding ticket
        const int done = atomicAdd(&P.ctr[1], 1);
        if (done == static_cast<int>(gridDim.x) * kWarps - 1) {
            P.ctr[0] = 0;
            P.ctr[1] = 0;
        }
    }
}

// K5: log-sum-exp merge of a unit's partials (fp chunks + page chunks).  One
// CTA per unit, 4 warps per query row, each warp over a quarter of the parts;
// loads are independent so the merge is one or two L2 round trips deep.
// The full-precision tokens: one 128-thread CTA per 32-token chunk
// (kitty_fp.cuh), run as its own launch before the page kernel so neither
// code path's register allocation or instruction footprint burdens the other.
template <int GROUP>
__global__ void __launch_bounds__(128) fp_tokens_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t fsm[];
    const int it = blockIdx.x;
    const int fc = it / P.units, u = it - fc * P.units;
    const fptok::Geom gm = fptok::geom(P.c, u, P.max_tokens);
    asm volatile("griddepcontrol.launch_dependents;");  // the merge may pre-launch
    if (gm.n > 0 && fc * kFpChunk < gm.nfp) fptok::chunk_tc<GROUP>(P.c, P.q, P.part, P.nslot, part_stride(GROUP), fsm, u, fc, P.max_tokens);
    // launched as a programmatic dependent of the page grid: finish only after it
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// WARPS warps merge one (unit, query row): 2 when a unit has <= 32 partial
// slots (short contexts: many small CTAs, one wave); 4 when 8-warp CTAs would
// need more than one wave and a unit has <= 128 slots; 16 above 128 slots
// (long contexts); else 8
template <int GROUP, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) combine_parts_kernel(Params P) {
    const int u = blockIdx.x / GROUP, g = blockIdx.x - (blockIdx.x / GROUP) * GROUP;
    const KittyCacheDesc& c = P.c;
    // the unit's part list depends only on its length (written by the append,
    // before the page grid): computed before waiting on the fp grid
    const UnitGeom gm = unit_geom(c, u, P.max_tokens);
    // a unit longer than the caller's bound was attended over its first
    // max_tokens tokens only: make the caller's check() raise
    if (g == 0 && threadIdx.x == 0 && c.unit_len[u] > P.max_tokens) set_status(c.status, KITTY_STATUS_LENGTH);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the fp grid (KITTY_PDL bit 2)
    if (gm.n == 0) return;
    const int nfc = (gm.nfp + kFpChunk - 1) / kFpChunk;
    int nch[3];
    for (int lv = 0; lv < 3; ++lv) {
        const int n = level_begin(lv + 1, gm.vp, P.lvl) - level_begin(lv, gm.vp, P.lvl);
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
    lse_merge_row<GROUP, decltype(slot_of), WARPS>(P.part + (int64_t)u * P.nslot * kStride, kStride, nparts, slot_of, g,
                                                  P.out, P.out_dtype, row);
}

}  // namespace fastattn

// ---- host side ---------------------------------------------------------------------

using namespace fastattn;

static int num_sms() { return device_sms(); }

bool fast_attention_supported(const KittyCacheDesc& c) {
    const int group = c.cfg.h_q / c.cfg.h_kv;
    return c.cfg.d == D && c.cfg.g == G && c.cfg.key_bits == 2 && c.cfg.value_bits == 2 &&
           (group == 1 || group == 2 || group == 4 || group == 8) && c.cfg.d_boost <= 32 &&
           c.key_slot_bytes <= kKeySlotMax && c.value_slot_bytes == 4608;
}

struct FastPlan {
    int ppc, cmax, fmax, units, group, cs[3], cmx[3], lvl[4], nslot;
    size_t ctr_bytes, part_bytes;
};

static FastPlan plan(const KittyCacheDesc& c, int max_tokens) {
    FastPlan p;
    p.units = c.num_seqs * c.cfg.h_kv;
    p.group = c.cfg.h_q / c.cfg.h_kv;
    const int past = max_tokens > c.cfg.s ? max_tokens - c.cfg.s : 0;
    const int maxp = past / G + 1;
    const long long pages = (long long)p.units * maxp;
    const long long warps = (long long)num_sms() * kCtasPerSm * kWarps;
    static int ppc_max = 8, cs1_div = 4, inited = 0;
    if (!inited) {
        inited = 1;
        if (const char* e = getenv("KITTY_SCHED")) {  // experiments: "l1,l2,ppc_max,cs1_div"
            sscanf(e, "%d,%d,%d,%d", &h_lvl[0], &h_lvl[1], &ppc_max, &cs1_div);
            h_lvl[2] = h_lvl[0];  // a sweep sets one pair for every unit length
            h_lvl[3] = h_lvl[1];
        }
    }
    int ppc = static_cast<int>(pages / (2 * warps));
    ppc = ppc < 1 ? 1 : (ppc > ppc_max ? ppc_max : ppc);
    p.ppc = ppc;
    p.cmax = (maxp + ppc - 1) / ppc;
    p.cs[0] = ppc;
    p.cs[1] = ppc / cs1_div > 1 ? ppc / cs1_div : 1;
    p.cs[2] = 1;
    // Level 0 in whole rounds: its items (ppc pages each, for units at the
    // longest length) are pulled round by round by the `warps` warps; when
    // there are only 1-2 whole rounds and the last would be nearly empty
    // (< 35 %), a few warps would start one more long item -- a large share of
    // a warp's work -- as everyone else runs out, so level 0 shrinks to the
    // whole rounds (C4: 2.03 rounds; with 3+ rounds, C3 / C5, the cut costs
    // more than the tail it removes).
    for (int i = 0; i < 4; ++i) p.lvl[i] = h_lvl[i];
    {
        const int past_m = max_tokens > c.cfg.s ? max_tokens - c.cfg.s : 0;
        const int vpm = (past_m - min(c.cfg.r, past_m)) / G;
        const int rule = vpm >= 512 ? 2 : 0;
        const int l0 = (vpm * p.lvl[rule]) / 1000;
        const long long items0 = (long long)p.units * ((l0 + ppc - 1) / ppc);
        const long long rounds = items0 / warps, rest = items0 - rounds * warps;
        if (vpm > 0 && rounds >= 1 && rounds < 3 && rest * 100 < 35 * warps) {
            const int l0n = static_cast<int>((rounds * warps) / p.units) * ppc;
            if (l0n > 0 && l0n < l0) p.lvl[rule] = static_cast<int>((long long)l0n * 1000 / vpm);
        }
    }
    // chunk bound per level over every unit length up to maxp: level sizes grow
    // with vp within one split rule (+2 absorbs the floor rounding), and the
    // rule switches at 512 pages, so both sides of the switch are evaluated
    for (int lv = 0; lv < 3; ++lv) {
        int n = level_begin(lv + 1, maxp, p.lvl) - level_begin(lv, maxp, p.lvl) + 2;
        if (maxp >= 512) {
            const int n2 = level_begin(lv + 1, 511, p.lvl) - level_begin(lv, 511, p.lvl) + 2;
            n = n2 > n ? n2 : n;
        }
        p.cmx[lv] = (n + p.cs[lv] - 1) / p.cs[lv];
    }
    const int nfp_max = min(max_tokens, c.cfg.s + c.cfg.r + c.cfg.g - 1);
    p.fmax = (nfp_max + kFpChunk - 1) / kFpChunk;
    if (p.fmax < 1) p.fmax = 1;
    p.ctr_bytes = 256;
    p.nslot = p.fmax + p.cmx[0] + p.cmx[1] + p.cmx[2];
    p.part_bytes = (size_t)p.units * p.nslot * part_stride(p.group) * sizeof(float);
    return p;
}

size_t fast_attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens) {
    if (!fast_attention_supported(c)) return 0;
    const FastPlan p = plan(c, max_tokens);
    return p.ctr_bytes + p.part_bytes;
}

// programmatic dependent launch per edge, a bit mask (A/B knob KITTY_PDL):
// 1 = page grid behind the preceding kernel, 2 = fp grid behind the page grid,
// 4 = merge grid behind the fp grid
static const int g_pdl = [] {
    const char* e = std::getenv("KITTY_PDL");
    return e ? std::atoi(e) : 3;
}();

template <int GROUP, int NKH>
static cudaError_t launch_t(const Params& prm, int grid, cudaStream_t st) {
    auto kfn = fast_attention_kernel<GROUP, NKH>;
    const size_t sm = (size_t)warp_smem_bytes<GROUP>((int)prm.c.key_slot_bytes, (int)prm.c.value_slot_bytes) * kWarps +
                      (prm.units <= kMaxTableUnits ? 4 * prm.units : 0);
    cudaError_t e = set_kernel_smem((const void*)kfn, (int)(warp_smem_bytes<GROUP>(kKeySlotMax, kValueSlot) * kWarps +
                                                          4 * kMaxTableUnits), true);
    if (e != cudaSuccess) return e;
    // persistent grid: kCtasPerSm CTAs per SM must be co-resident (their shared
    // memory, the 1 KB per-CTA reservation and the static part fit the SM), else
    // one fewer per SM.  (cudaOccupancyMaxActiveBlocksPerMultiprocessor reports
    // 1 for this kernel on B200 at any shared-memory size, so it is not used.)
    const int smpm = device_smem_per_sm();
    int per_sm = kCtasPerSm;
    while (per_sm > 1 && (size_t)per_sm * (sm + 128 + 1024) > (size_t)smpm) --per_sm;
    if (grid > num_sms() * per_sm) grid = num_sms() * per_sm;
    // the pages first; the fp-token chunks as a programmatic dependent of the
    // page grid, so their CTAs backfill SMs as persistent page CTAs retire (the
    // fp grid waits on the page grid only before it exits); then the merge
    cudaLaunchAttribute at[3];
    for (int i = 0; i < 3; ++i) {
        at[i].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[i].val.programmaticStreamSerializationAllowed = (g_pdl >> i) & 1;
    }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kWarps * 32);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cfg.attrs = at + 0;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kfn, prm);
        if (e != cudaSuccess) return e;
    }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(prm.units * prm.fmax);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = fptok::tc_scratch_bytes((int)prm.c.key_slot_bytes);
        cfg.stream = st;
        cfg.attrs = at + 1;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, fp_tokens_kernel<GROUP>, prm);
        if (e != cudaSuccess) return e;
    }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(prm.units * GROUP);
        cfg.stream = st;
        cfg.attrs = at + 2;
        cfg.numAttrs = 1;
        if (prm.nslot <= 32) {
            cfg.blockDim = dim3(2 * 32);
            return cudaLaunchKernelEx(&cfg, combine_parts_kernel<GROUP, 2>, prm);
        }
        // 4 warps when 8-warp CTAs would not be resident in one wave (~48 warps / SM)
        if (prm.nslot <= 128 && (long long)prm.units * GROUP * kMergeWarps > 48LL * num_sms()) {
            cfg.blockDim = dim3(4 * 32);
            return cudaLaunchKernelEx(&cfg, combine_parts_kernel<GROUP, 4>, prm);
        }
        if (prm.nslot > 128) {  // long contexts: few rows, hundreds of parts each
            cfg.blockDim = dim3(16 * 32);
            return cudaLaunchKernelEx(&cfg, combine_parts_kernel<GROUP, 16>, prm);
        }
        cfg.blockDim = dim3(kMergeWarps * 32);
        return cudaLaunchKernelEx(&cfg, combine_parts_kernel<GROUP, kMergeWarps>, prm);
    }
}

template <int GROUP>
static cudaError_t launch_g(const Params& prm, int nkh, int grid, cudaStream_t st) {
    if (nkh == 0) return launch_t<GROUP, 0>(prm, grid, st);
    if (nkh == 1) return launch_t<GROUP, 1>(prm, grid, st);
    return launch_t<GROUP, 2>(prm, grid, st);
}

cudaError_t launch_fast_attention(const KittyCacheDesc& c, const uint16_t* q, void* out, int out_dtype,
                                  int max_tokens, void* ws, size_t ws_bytes, cudaStream_t st) {
    const FastPlan p = plan(c, max_tokens);
    if (ws_bytes < p.ctr_bytes + p.part_bytes) return cudaErrorInvalidValue;
    Params prm;
    prm.c = c;
    prm.q = q;
    prm.out = out;
    prm.out_dtype = out_dtype;
    prm.ppc = p.ppc;
    prm.cmax = p.cmax;
    prm.fmax = p.fmax;
    for (int lv = 0; lv < 3; ++lv) {
        prm.cs[lv] = p.cs[lv];
        prm.cmx[lv] = p.cmx[lv];
    }
    for (int i = 0; i < 4; ++i) prm.lvl[i] = p.lvl[i];
    prm.nslot = p.nslot;
    prm.units = p.units;
    prm.max_tokens = max_tokens;
    {
        // fast division by units: q = (umulhi(n, mul) + n) >> shift, n < 2^31
        uint32_t sh = 0;
        while ((1u << sh) < static_cast<uint32_t>(p.units)) ++sh;
        prm.units_shift = sh;
        prm.units_mul = static_cast<uint32_t>((((1ull << 32) * ((1ull << sh) - static_cast<uint64_t>(p.units))) / p.units) + 1);
    }
    prm.ctr = static_cast<int*>(ws);
    prm.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + p.ctr_bytes);
    const long long items = (long long)p.units * p.nslot;
    long long ctas = (items + kWarps - 1) / kWarps;
    const long long cap = (long long)num_sms() * kCtasPerSm;
    const int grid = static_cast<int>(ctas < cap ? ctas : cap);
    const int nkh = (c.cfg.d_boost + 15) / 16;
    switch (p.group) {
        case 1: return launch_g<1>(prm, nkh, grid, st);
        case 2: return launch_g<2>(prm, nkh, grid, st);
        case 4: return launch_g<4>(prm, nkh, grid, st);
        default: return launch_g<8>(prm, nkh, grid, st);
    }
}

cudaError_t fast_attention_trace(int enable, long long* host_out, int max_warps) {
    cudaError_t e = cudaMemcpyToSymbol(fastattn::g_trace_on, &enable, sizeof(int));
    if (e != cudaSuccess || host_out == nullptr) return e;
    const int n = max_warps < fastattn::kTraceWarps ? max_warps : fastattn::kTraceWarps;
    return cudaMemcpyFromSymbol(host_out, fastattn::g_trace, sizeof(long long) * n * fastattn::kTraceFields);
}

}  // namespace kitty
