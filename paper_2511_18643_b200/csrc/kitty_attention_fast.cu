// Fused dequant-attention decode for d = g = 128 (K4 + K5): the page kernel,
// the full-precision-token kernel and the split-KV merge.
//
// Semantics: KittyCacheState.attend (cache.py:217-252) -- per (sequence, KV
// head) unit, logits q.k / sqrt(d) over sink | key pages | key q-buffer, fp32
// max-subtracted softmax, probabilities times values over sink | value pages |
// value q-buffer | local -- with pages dequantised inside the loop (Alg. 1,
// PAPER.md:425-446) instead of from cached f32 rows.
//
// One attention call = three launches chained by programmatic dependent
// launch, the fp-token grid first when it needs more than one
// CTA per SM (else the page grid first), the merge last:
//  * page_kernel: the 2-bit pages.  Persistent CTAs (2 per SM x 4 warps);
//    every warp is one page stream: it pulls work items (chunks of a unit's
//    pages) from an atomic queue, stages key and value pages through 2-slot
//    rings (cp.async.bulk + mbarrier; keys are issued one page ahead of
//    values) and runs QK^T + online softmax of page k + 1 interleaved with
//    P V of page k in one basic block;
//  * 2-bit codes become fp16 MMA operands without per-element dequantisation:
//    ldmatrix.x4.trans hands each lane 8 codes of two code rows per register,
//    one LOP3 per code position makes (x & mask) | 0x6400 = 1024 + w c; the
//    1024 offset and w are removed per tile after the MMA;
//  * per-channel key scale folded into q (B = q alpha s, fp16), per-token
//    value scale into p (B = p s); zero points and offset sums come out of one
//    auxiliary MMA tile (row 0 = ones, row 8 = zeros) whose B columns 4-7
//    carry the unscaled q / p (GQA group <= 4; group 8 uses a second MMA);
//  * mma.sync.m16n8k16 f16 x f16 -> f32, swap-AB: M = 16 tokens (QK) or 16
//    channels (PV), N = the GQA group, K = 16 channels (QK) or tokens (PV);
//  * softmax in the log2 domain with lazy rescaling (the running max moves
//    only when a page exceeds it by more than kLazy = 2, so P <= 4 in f16);
//  * each work item leaves a partial record (acc, m, l) in the workspace;
//  * fp_tokens_kernel: the sink / q-buffer / local tokens (kitty_fp.cuh);
//  * combine_parts_kernel: LSE merge of a unit's partials (kitty_combine.cuh).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

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
constexpr int kKeySlotMax = 5760;  // d_boost = 32
constexpr int kValueSlot = 4608;
// P^T row = one query: the f16x2 of tokens (2 k, 2 k + 1) at word k (64
// used); rows 68 words apart so the PV loads (row = query, word 8 ks + t (+4))
// are bank-conflict free.
constexpr int kPtWords = 68;  // 272 B: rows stay 16-byte aligned for the P^T stores
constexpr int kFpChunk = 32;       // fp tokens per fp-kernel chunk
constexpr float kAlpha = 0.12751743074f;  // log2(e) / sqrt(128)
// log2-domain slack of the running max: P <= 2^kLazy, and P s (f16, s the
// value page's token scale) must stay finite: 2 keeps |v| up to ~2.4e4 (8
// measured 0.2 % faster but would cap |v| near 400)
constexpr float kLazy = 2.f;
constexpr uint32_t kMagic = 0x64006400u;  // f16x2 (1024, 1024)
constexpr uint32_t kOnes = 0x3C003C00u;   // f16x2 (1, 1)

constexpr int kHalves = 1;      // partial records per page chunk
constexpr int kWarps = 4;       // warps per CTA
constexpr int kCtasPerSm = 2;   // 8 warps per SM, each with up to 255 registers

// Per-warp shared memory: this fixed part, then 2 key slots and 2 value slots
// (a 2-stage ring of page pairs) sized by the cache's slot bytes at launch.
template <int PT_ROWS>
struct __align__(16) WarpFixedT {
    uint32_t pt[2][PT_ROWS][kPtWords];  // P^T of pages k and k + 1 (f16x2 token pairs), one row per query
    uint32_t qtab[PT_ROWS][D / 2];      // 4 q alpha (f16) of the QK side's unit: the boosted rows' B
    uint32_t ones[64];                  // f16x2 (1, 1): the aux lanes' "scale"
    uint8_t inv[32];                    // boosted channel of high_bits row j
    unsigned long long kfull[2];        // key slot s landed
    unsigned long long vfull[2];        // value slot s landed
};
template <int GROUP>
__host__ __device__ constexpr int warp_fixed_bytes() {
    return static_cast<int>((sizeof(WarpFixedT<GROUP == 8 ? 8 : 4>) + 127) & ~size_t(127));
}
template <int GROUP>
__host__ __device__ inline int warp_smem_bytes(int kslot, int vslot) {
    return (warp_fixed_bytes<GROUP>() + 2 * kslot + 2 * vslot + 127) & ~127;
}
// warp-specialised page kernel: per (QK warp, PV warp) pair, the per-warp
// fixed part plus the hand-off between the two (P^T stages, per-column
// correction / running max of each page, the page's job, the value slot of
// page k + 2 for the PV warp to fetch) and the stage barriers
constexpr int kWsPairs = 4;  // pairs per CTA: 8 warps, 2 CTAs = 16 warps per SM
template <int PT_ROWS>
struct __align__(16) PairFixedT {
    uint32_t pt[2][PT_ROWS][kPtWords];
    uint32_t qtab[PT_ROWS][D / 2];
    uint32_t ones[64];
    float corr[2][8];
    float mnew[2][8];
    int job[2][4];  // u (< 0: end of stream), p, pq, slot
    int vnext[2];   // value slot of page k + 2 (-1: none)
    uint8_t inv[32];
    unsigned long long kfull[2];
    unsigned long long vfull[2];
    unsigned long long pfull[2];
    unsigned long long pempty[2];
};
template <int GROUP>
__host__ __device__ constexpr int pair_fixed_bytes() {
    return static_cast<int>((sizeof(PairFixedT<GROUP == 8 ? 8 : 4>) + 127) & ~size_t(127));
}
template <int GROUP>
__host__ __device__ inline int pair_smem_bytes(int kslot, int vslot) {
    return (pair_fixed_bytes<GROUP>() + 2 * kslot + 2 * vslot + 127) & ~127;
}
constexpr int kMaxTableUnits = 2048;  // units whose lengths a CTA caches in shared memory

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
    int nslot;    // partial slots per unit: fmax + kHalves * (cmx[0] + cmx[1] + cmx[2])
    int units;
    int max_tokens;  // the caller's bound on the unit lengths (longer units: clamped + KITTY_STATUS_LENGTH)
    uint32_t units_mul, units_shift;  // fast division by units (quotient = (umulhi(n, mul) + n) >> shift)
    int* ctr;   // [0] next item, [1] finished CTAs
    float* part;
    int fp_first;  // launch order: fp grid, page grid, merge (else page, fp, merge)
    int fp_union;  // fp chunk scratch: key page and key tile share bytes (kitty_fp.cuh)
    int fp_warp;   // fp chunks one per warp (fp_warp_kernel) instead of one per CTA
};

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

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// the same wait with a suspend-time hint: the warp sleeps in the barrier unit
// until the phase completes (or the hint expires) instead of spinning, so a
// waiting warp takes no issue slots from the warps that share its scheduler
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(0x989680)
        : "memory");
}

// Pages are read once per step: stream them through L2 with evict_first so the
// split-KV partials (re-read by the merge right after) stay resident.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_last4(float* p, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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
        m0 = 0x03000300u;  // bits 8-9 of each half: weight 256
        m1 = 0x000C000Cu;  // bits 2-3: weight 4
        m2 = 0x00300030u;  // bits 4-5: weight 16
        m3 = 0x00C000C0u;  // bits 6-7: weight 64
        magic = kMagic;
        asm volatile("" : "+r"(m0), "+r"(m1), "+r"(m2), "+r"(m3), "+r"(magic));
    }
};

// ldmatrix.x4.trans of four 8 x 16-byte blocks of 32-byte code rows: lane
// (gid, tig) gets, per block, rows 2 tig / 2 tig + 1 (the two f16 halves) at
// bytes 2 gid, 2 gid + 1, i.e. 8 consecutive 2-bit codes of two rows in one
// register -- the A-operand pairing the MMA wants, without a PRMT.
__device__ __forceinline__ void ldsm_t4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// One register of 8 codes per half -> the 8 f16x2 A operands of its codes:
// codes 1-4 masked in place (weights 4, 16, 64, 256), code 0 after a 2-bit
// left shift (4) and codes 5-7 after a 6-bit right shift (16, 64, 256); each
// OR-ed with the exponent of 1024.  No code sits at weight 1: w >= 4 keeps
// the 1024 offset's cancellation (removed per row after the MMA) far below
// the fp16 operand rounding.
__device__ __forceinline__ void conv8(const Consts& k, uint32_t r, uint32_t (&o)[8]) {
    o[0] = and_or(r << 2, k.m1, k.magic);
    o[1] = and_or(r, k.m1, k.magic);
    o[2] = and_or(r, k.m2, k.magic);
    o[3] = and_or(r, k.m3, k.magic);
    o[4] = and_or(r, k.m0, k.magic);
    const uint32_t y = r >> 6;
    o[5] = and_or(y, k.m2, k.magic);
    o[6] = and_or(y, k.m3, k.magic);
    o[7] = and_or(y, k.m0, k.magic);
}

// weight class of tile m (the code position inside the lane's 8): 0: w 4,
// 1: w 16, 2: w 64, 3: w 256
__host__ __device__ constexpr int tile_c(int m) { return m < 2 ? 0 : (m < 5 ? m - 1 : m - 4); }
__host__ __device__ constexpr float tile_w(int m) { return tile_c(m) == 0 ? 4.f : tile_c(m) == 1 ? 16.f : tile_c(m) == 2 ? 64.f : 256.f; }

// acc[8][4] (+)= A x B for one k-step from the four ldmatrix registers:
// r0 / r2 = rows (2 tig, 2 tig + 1) of the step at M-rows gid / gid + 8,
// r1 / r3 = rows (2 tig + 8, 2 tig + 9); tile m = code m of each register.
template <bool FIRST = false>
__device__ __forceinline__ void mma_ldsm(const Consts& k, float (&acc)[8][4], uint32_t r0, uint32_t r1, uint32_t r2,
                                         uint32_t r3, uint32_t b0, uint32_t b1) {
    uint32_t a0[8], a1[8], a2[8], a3[8];
    conv8(k, r0, a0);
    conv8(k, r2, a1);
    conv8(k, r1, a2);
    conv8(k, r3, a3);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        if (FIRST)
            mma16816_z(acc[m], a0[m], a1[m], a2[m], a3[m], b0, b1);
        else
            mma16816(acc[m], a0[m], a1[m], a2[m], a3[m], b0, b1);
    }
}

struct UnitGeom {
    int n, kp, vp, nfp;
};

// Pages of a unit are scheduled in three levels of decreasing chunk size:
// [0, lvl0 vp) in chunks of cs[0] (<= 8 pages), [lvl0 vp, lvl1 vp) in
// cs[0] / 4, the rest page by page; the queue serves level 0, 1, 2, so it
// drains in small pieces and no SM idles behind a long item (swept on B200
// with tools/sweep_sched.sh).  Level starts per mille of vp, one pair for
// units below 512 pages and one from 512 pages on (128K-token contexts have
// tails long enough that a larger level 0 wins).  The host plan passes them
// per launch (Params::lvl), after quantising level 0 to whole rounds of the
// page streams.  KITTY_SCHED overrides them for sweeps.
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

// ---- the page kernel ------------------------------------------------------------

// One page of a warp's stream: unit, page, item bounds (p1 | p0 << 16), the
// item's partial slot, and the page's key / value slots; u < 0 = none.
struct Pg {
    int u, p, pq, slot, ks, vs;
};

// WS = false: one warp per page stream, QK of page k + 1 interleaved with P V
// of page k (8 warps / SM).  WS = true (KITTY_WS; the default at group 8):
// each stream is served by a QK + softmax warp and a PV warp one page behind
// it, handing pages over through mbarriers (16 warps / SM at <= 128 registers).
template <int GROUP, int NKH, bool WS>
__global__ void __launch_bounds__(WS ? 2 * kWsPairs * 32 : kWarps * 32, kCtasPerSm) page_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    constexpr int PT_ROWS = GROUP == 8 ? 8 : 4;
    using Fixed = std::conditional_t<WS, PairFixedT<PT_ROWS>, WarpFixedT<PT_ROWS>>;
    const KittyCacheDesc& c = P.c;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int vslot = static_cast<int>(c.value_slot_bytes);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    // WS: warps [0, kWsPairs) run QK + softmax of their pair's page stream,
    // warps [kWsPairs, 2 kWsPairs) P V of the same stream, one page behind
    const int pair = WS ? (warp & (kWsPairs - 1)) : warp;  // the page stream within the CTA
    const bool qk_role = !WS || warp < kWsPairs;
    const int wbytes = WS ? pair_smem_bytes<GROUP>(kslot, vslot) : warp_smem_bytes<GROUP>(kslot, vslot);
    uint8_t* const wbase = smem_raw + pair * wbytes;
    Fixed& sm = *reinterpret_cast<Fixed*>(wbase);
    uint8_t* const kslots = wbase + (WS ? pair_fixed_bytes<GROUP>() : warp_fixed_bytes<GROUP>());
    uint8_t* const vslots = kslots + 2 * kslot;
    // group <= 4: B columns 0-3 are the queries, 4-7 auxiliary (unscaled q / p);
    // group 8: all eight are queries and the auxiliary sums take a second MMA
    constexpr bool kFull = GROUP == 8;
    const bool main_col = kFull || gid < 4;
    const int d_boost = c.cfg.d_boost;
    const int scale_off = D * G / 4 + d_boost * G / 4 + D;  // KTYP key scales
    const int zero_off = scale_off + 2 * D;
    const int hkv = c.cfg.h_kv;

    if (qk_role) {
        if (lane == 0) {
            for (int i = 0; i < 2; ++i) {
                mbar_init(&sm.kfull[i], 1);
                mbar_init(&sm.vfull[i], 1);
                if constexpr (WS) {
                    mbar_init(&sm.pfull[i], 1);
                    mbar_init(&sm.pempty[i], 1);
                }
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            if constexpr (WS) {
                mbar_arrive(&sm.pempty[0]);  // both P^T stages start free
                mbar_arrive(&sm.pempty[1]);
            }
        }
        sm.ones[lane] = kOnes;
        sm.ones[lane + 32] = kOnes;
        sm.inv[lane] = 0;
    }
    // launched as a programmatic dependent of the preceding kernel (the append):
    // the prologue above overlaps its tail; nothing of the cache is read before this.
    // fp-first order: the preceding kernel is the fp grid, whose CTAs all passed
    // their own wait on the append before this grid could launch -- the cache is
    // final, and the fp grid is waited for at the end (before the merge reads it)
    if (!P.fp_first) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        // the fp-token grid (our programmatic dependent) may be scheduled from now on
        asm volatile("griddepcontrol.launch_dependents;");
    }
    // per-CTA copy of the unit lengths: an item's decode reads shared memory
    int* s_ulen = reinterpret_cast<int*>(smem_raw + wbytes * (WS ? kWsPairs : kWarps));
    const bool len_table = P.units <= kMaxTableUnits;
    if (len_table) {
        for (int i = threadIdx.x; i < P.units; i += blockDim.x) s_ulen[i] = min(__ldcg(c.unit_len + i), P.max_tokens);
    }
    __syncthreads();

    // ---- the page stream: work items (atomic queue, one ticket ahead) -> pages ----
    // An item's block-table entries are loaded by its lanes at once (one per
    // page, cs <= 32), so a page costs one shuffle, not a dependent load.
    int tk = 0;
    if (qk_role && lane == 0) tk = atomicAdd(P.ctr, 1);
    int iu = 0, ip = 0, ip0 = 0, ip1 = 0, islot = 0, kreg = 0, vreg = 0;
    bool live = false, done = false;
    const int nq0 = P.units * P.cmx[0], nq1 = P.units * P.cmx[1], nq2 = P.units * P.cmx[2];
    auto next_page = [&]() -> Pg {
        if (!done && !(live && ip + 1 < ip1)) {
            live = false;
            while (!live) {
                const int it = __shfl_sync(0xffffffffu, tk, 0);
                if (lane == 0) tk = atomicAdd(P.ctr, 1);
                int sect, idx;
                if (it < nq0) {
                    sect = 0;
                    idx = it;
                } else if (it < nq0 + nq1) {
                    sect = 1;
                    idx = it - nq0;
                } else if (it < nq0 + nq1 + nq2) {
                    sect = 2;
                    idx = it - nq0 - nq1;
                } else {
                    done = true;
                    break;
                }
                const int ch = static_cast<int>(
                    (__umulhi(static_cast<uint32_t>(idx), P.units_mul) + static_cast<uint32_t>(idx)) >> P.units_shift);
                iu = idx - ch * P.units;
                const int n = len_table ? s_ulen[iu] : min(__ldcg(c.unit_len + iu), P.max_tokens);
                const int past = n > c.cfg.s ? n - c.cfg.s : 0;
                const int vp = (past - min(c.cfg.r, past)) / G;
                const int lb = level_begin(sect, vp, P.lvl), le = level_begin(sect + 1, vp, P.lvl);
                ip0 = lb + ch * P.cs[sect];
                ip1 = min(le, ip0 + P.cs[sect]);
                live = ip0 < ip1;
                if (live) {
                    islot = ch;
                    for (int l = 0; l < sect; ++l) islot += P.cmx[l];
                    islot = P.fmax + islot;
                    const int64_t row = (int64_t)iu * c.max_pages + ip0;
                    if (lane < ip1 - ip0) {
                        kreg = __ldcg(c.key_block_table + row + lane);
                        vreg = __ldcg(c.value_block_table + row + lane);
                    }
                }
            }
            ip = ip0;
        } else if (!done) {
            ++ip;
        }
        Pg d;
        d.u = done ? -1 : iu;
        d.p = ip;
        d.pq = ip1 | (ip0 << 16);
        d.slot = islot;
        return d;
    };
    // a page's key / value slots: shuffled from its item's block-table loads
    // as late as possible (before the stream decodes another item), so the
    // loads issued at the item's decode are not waited on
    auto fill_ks = [&](Pg& d) { d.ks = __shfl_sync(0xffffffffu, kreg, (d.p - (d.pq >> 16)) & 31); };
    auto fill_vs = [&](Pg& d) { d.vs = __shfl_sync(0xffffffffu, vreg, (d.p - (d.pq >> 16)) & 31); };
    // Page p of the warp's stream lands in key slot p & 1 and value slot p & 1
    // (use number p >> 1 of the slot: mbarrier phase (p >> 1) & 1).  QK runs
    // one page ahead of PV, so a key page is issued one page earlier than its
    // value page: each gets a full iteration of load time.
    const uint64_t pol = l2_evict_first();
    const uint64_t pol_last = l2_evict_last();
    auto issue_key = [&](const Pg& d, int sl) {
        if (lane == 0 && d.u >= 0) {
            mbar_expect_tx(&sm.kfull[sl], kslot);
            bulk_g2s(kslots + sl * kslot, c.key_pool + (int64_t)d.ks * kslot, kslot, &sm.kfull[sl], pol);
        }
    };
    auto issue_val = [&](const Pg& d, int sl) {
        if (lane == 0 && d.u >= 0) {
            mbar_expect_tx(&sm.vfull[sl], vslot);
            bulk_g2s(vslots + sl * vslot, c.value_pool + (int64_t)d.vs * vslot, vslot, &sm.vfull[sl], pol);
        }
    };
    // a new unit's q rows (group x 256 B, L2-resident) are pulled into L1 two
    // pages before its first QK reads them
    auto prefetch_q = [&](const Pg& d, int prev_u) {
        if (d.u >= 0 && d.u != prev_u && lane < GROUP * 2) {
            const int b = d.u / hkv, h = d.u - b * hkv;
            const uint16_t* qg = P.q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D + lane * 64;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(qg));
        }
    };

    const Consts kc;
    uint32_t pe_phase = 0;  // WS: parity of the P^T stage release the QK tail waits for
    // a stage barrier wait: spinning (one warp per stream: its own data), or
    // with a suspend hint (WS: a warp waiting on its partner)
    auto bar_wait = [&](unsigned long long* bar, uint32_t ph) {
        if constexpr (WS)
            mbar_wait_sleep(bar, ph);
        else
            mbar_wait(bar, ph);
    };
    // ---- QK side state: q fragments of its unit, running max of its item ----
    int cur_unit = -1;
    uint32_t qa[8][2];
    float om[2] = {-INFINITY, -INFINITY};
    const int qcol = kFull ? gid : (gid & 3);
    // ---- PV side state: output accumulators, row sums, zero / offset constants ----
    float oacc[8][4] = {};
    float ol[2] = {0.f, 0.f};
    float ob[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    const int prow = kFull ? gid : (gid & 3);
    const bool prow_ok = prow < GROUP;
    const bool real0 = kFull || (tig < 2 && 2 * tig < GROUP), real1 = kFull || (tig < 2 && 2 * tig + 1 < GROUP);

    // QK of page d (stage st): waits for the stage, computes the page's logits
    // and probabilities into P^T[st], its correction factors and running max
    auto qk_prologue = [&](const Pg& d, int st, uint32_t phase) {
        if (d.u != cur_unit) {
            cur_unit = d.u;
            const int b = d.u / hkv, h = d.u - b * hkv;
            const uint16_t* qg = P.q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + (qcol < GROUP ? qcol : 0)) * D;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int dd = 16 * ks + 2 * tig + 8 * hh;
                    const uint32_t w = qcol < GROUP ? __ldg(reinterpret_cast<const unsigned int*>(qg + dd)) : 0u;
                    qa[ks][hh] = pack_f16x2(__uint_as_float(w << 16) * kAlpha, __uint_as_float(w & 0xffff0000u) * kAlpha);
                    // 4 q alpha per channel for the boosted rows (x4 is exact in f16)
                    if (NKH > 0 && main_col && qcol < GROUP)
                        sm.qtab[qcol][dd / 2] = pack_f16x2(__uint_as_float(w << 16) * (4.f * kAlpha),
                                                           __uint_as_float(w & 0xffff0000u) * (4.f * kAlpha));
                }
            }
        }
        if (d.p == (d.pq >> 16)) om[0] = om[1] = -INFINITY;  // an item's first page
        bar_wait(&sm.kfull[st], phase);
        if (NKH > 0) {  // boosted rows -> channels (inverse of boost_idx)
            const uint8_t* kp = kslots + st * kslot;
            const uint32_t bw = lds32(kp + D * G / 4 + d_boost * G / 4 + 4 * lane);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t bi = (bw >> (8 * k)) & 0xffu;
                if (bi < 32u) sm.inv[bi] = static_cast<uint8_t>(4 * lane + k);
            }
        }
        __syncwarp();
    };
    // QK of a page, in three parts so that the caller can interleave its
    // k-steps with the P V k-steps of the previous page (one basic block)
    struct QkRegs {
        float acc[8][4], aux[4], aux2[4];
    };
    // ldmatrix row address of this lane inside a 16-row block of 32-byte code
    // rows: block mi = lane / 8 covers rows 8 (mi & 1) + [0, 8) at bytes 16 (mi >> 1)
    const uint32_t ldsm_off = (8 * ((lane >> 3) & 1) + (lane & 7)) * 32 + 16 * (lane >> 4);
    auto qk_step = [&](int st, int ks, QkRegs& r) {
        const uint8_t* kp = kslots + st * kslot;
        // aux lanes (B columns 4-7) read their "scale" from the ones buffer
        const uint8_t* sbase = main_col ? kp + scale_off : reinterpret_cast<const uint8_t*>(sm.ones);
        const int c0 = 16 * ks + 2 * tig;
        const uint32_t b0 = hmul2(qa[ks][0], lds32(sbase + 2 * c0));
        const uint32_t b1 = hmul2(qa[ks][1], lds32(sbase + 2 * (c0 + 8)));
        uint32_t w0, w1, w2, w3;  // channel rows 16 ks + [0, 16), tokens 8 gid + [0, 8) / 64 + ...
        ldsm_t4(smem_u32(kp) + 512 * ks + ldsm_off, w0, w1, w2, w3);
        // aux tile: only rows 0 (ones) and 8 (zero points) are read back
        const uint32_t z0 = lds32(kp + zero_off + 2 * c0);
        const uint32_t z1 = lds32(kp + zero_off + 2 * (c0 + 8));
        if (ks == 0) {
            mma_ldsm<true>(kc, r.acc, w0, w1, w2, w3, b0, b1);
            mma16816_z(r.aux, kOnes, z0, kOnes, z1, b0, b1);
            if (kFull) mma16816_z(r.aux2, kOnes, z0, kOnes, z1, qa[ks][0], qa[ks][1]);
        } else {
            mma_ldsm(kc, r.acc, w0, w1, w2, w3, b0, b1);
            mma16816(r.aux, kOnes, z0, kOnes, z1, b0, b1);
            if (kFull) mma16816(r.aux2, kOnes, z0, kOnes, z1, qa[ks][0], qa[ks][1]);
        }
    };
    auto qk_tail = [&](int st, QkRegs& r, float (&corr)[2], float (&mnew)[2]) {
        const uint8_t* kp = kslots + st * kslot;
        float (&acc)[8][4] = r.acc;
        float (&aux)[4] = r.aux;
        float (&aux2)[4] = r.aux2;
        if (NKH > 0) {
            // boosted row j (its high bits, weight 4) -> channel inv[j]: B = 4 q alpha s
            const uint16_t* qt = reinterpret_cast<const uint16_t*>(sm.qtab[qcol < GROUP ? qcol : 0]);
            const uint16_t* sc = reinterpret_cast<const uint16_t*>(kp + scale_off);  // even offset at d = g = 128
#pragma unroll
            for (int hk = 0; hk < NKH; ++hk) {
                const int j0 = 16 * hk + 2 * tig;
                const uint32_t ch01 = *reinterpret_cast<const uint16_t*>(sm.inv + j0);
                const uint32_t ch89 = *reinterpret_cast<const uint16_t*>(sm.inv + j0 + 8);
                const uint32_t c0 = ch01 & 0xffu, c1 = ch01 >> 8, c8 = ch89 & 0xffu, c9 = ch89 >> 8;
                const uint32_t q01 = static_cast<uint32_t>(qt[c0]) | (static_cast<uint32_t>(qt[c1]) << 16);
                const uint32_t s01 = static_cast<uint32_t>(sc[c0]) | (static_cast<uint32_t>(sc[c1]) << 16);
                const uint32_t q89 = static_cast<uint32_t>(qt[c8]) | (static_cast<uint32_t>(qt[c9]) << 16);
                const uint32_t s89 = static_cast<uint32_t>(sc[c8]) | (static_cast<uint32_t>(sc[c9]) << 16);
                // rows past d_boost (d_boost 8: rows 8-15 of the tile; an odd
                // d_boost: the second half of a pair) are not high-bit rows
                const bool ok = main_col && qcol < GROUP;
                const uint32_t m0 = (ok && j0 < d_boost ? 0xffffu : 0u) | (ok && j0 + 1 < d_boost ? 0xffff0000u : 0u);
                const uint32_t m1 = (ok && j0 + 8 < d_boost ? 0xffffu : 0u) | (ok && j0 + 9 < d_boost ? 0xffff0000u : 0u);
                const uint32_t b0 = hmul2(q01, s01) & m0;
                const uint32_t b1 = hmul2(q89, s89) & m1;
                uint32_t h0, h1, h2, h3;  // high-bit rows 16 hk + [0, 16)
                ldsm_t4(smem_u32(kp + D * G / 4) + 512 * hk + ldsm_off, h0, h1, h2, h3);
                mma_ldsm(kc, acc, h0, h1, h2, h3, b0, b1);
                mma16816(aux, kOnes, 0u, kOnes, 0u, b0, b1);
            }
        }
        // aux row 0 (lanes 0-3): sum of B per column; row 8, columns 4-7: sum(z * q * alpha).
        // Tile m holds code m of the lane's 8 (rows gid: token 8 gid + m, gid + 8:
        // token 64 + 8 gid + m) at weight tile_w(m); bw[c] = the offset of class c.
        float bw[4][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float sumB = __shfl_sync(0xffffffffu, aux[j], kFull ? tig : (tig & 1));
            const float cst = kFull ? __shfl_sync(0xffffffffu, aux2[2 + j], tig)
                                    : __shfl_sync(0xffffffffu, aux[2 + j], 2 + (tig & 1));
            bw[0][j] = cst - 256.f * sumB;  // w 4
            bw[1][j] = cst - 64.f * sumB;   // w 16
            bw[2][j] = cst - 16.f * sumB;   // w 64
            bw[3][j] = cst - 4.f * sumB;    // w 256
            // raw maxima per weight class (same weight: monotone), then one FFMA each
            const float x0 = fmaxf(fmaxf(acc[0][j], acc[0][2 + j]), fmaxf(acc[1][j], acc[1][2 + j]));
            const float x1 = fmaxf(fmaxf(acc[2][j], acc[2][2 + j]), fmaxf(acc[5][j], acc[5][2 + j]));
            const float x2 = fmaxf(fmaxf(acc[3][j], acc[3][2 + j]), fmaxf(acc[6][j], acc[6][2 + j]));
            const float x3 = fmaxf(fmaxf(acc[4][j], acc[4][2 + j]), fmaxf(acc[7][j], acc[7][2 + j]));
            float pm = fmaxf(fmaxf(fmaf(x0, 1.f / 4.f, bw[0][j]), fmaf(x1, 1.f / 16.f, bw[1][j])),
                             fmaxf(fmaf(x2, 1.f / 64.f, bw[2][j]), fmaf(x3, 1.f / 256.f, bw[3][j])));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 4));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 8));
            pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 16));
            // lazy rescaling: the reference max moves only when a page's max
            // exceeds it by more than kLazy (log2 domain), so P stays <= 2^kLazy
            // (f16-safe) and the output rescale below almost never runs
            mnew[j] = pm > om[j] + kLazy ? pm : om[j];
            corr[j] = ex2(om[j] - mnew[j]);  // 0 on an item's first page (om = -inf), else 1 unless moved
            om[j] = mnew[j];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) bw[c4][j] -= mnew[j];
        }
        // WS: P^T[st] is free once the PV warp is done with page k - 2
        if constexpr (WS) mbar_wait_sleep(&sm.pempty[st], pe_phase);
        // exponents (log2 domain, x - max) to P^T[st]: row = query, token t at word
        // t / 2 (half t % 2); this lane's tokens 8 gid + m (words 4 gid ..) and
        // 64 + 8 gid + m (words 32 + 4 gid ..), two 16-byte stores each
        if (kFull || tig < 2) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (2 * tig + j < GROUP) {
                    uint32_t lo[4], hi[4];
#pragma unroll
                    for (int m = 0; m < 8; m += 2) {
                        const float w0 = 1.f / tile_w(m), w1 = 1.f / tile_w(m + 1);
                        const int c0 = tile_c(m), c1 = tile_c(m + 1);
                        // the exponent x (<= kLazy) as f16: P V takes ex2.f16x2 of it
                        lo[m / 2] = pack_f16x2(fmaf(acc[m][j], w0, bw[c0][j]), fmaf(acc[m + 1][j], w1, bw[c1][j]));
                        hi[m / 2] = pack_f16x2(fmaf(acc[m][2 + j], w0, bw[c0][j]), fmaf(acc[m + 1][2 + j], w1, bw[c1][j]));
                    }
                    uint32_t* row = &sm.pt[st][(2 * tig + j) % PT_ROWS][0];
                    *reinterpret_cast<uint4*>(row + 4 * gid) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    *reinterpret_cast<uint4*>(row + 32 + 4 * gid) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                }
            }
        }
    };
    // P V of page d (stage st) with P^T[st]; fresh = its item's first page
    // P V of a page (stage st) with P^T[st]; fresh = its item's first page
    struct PvRegs {
        float vaux[4], vaux2[4];
    };
    auto pv_head = [&](bool fresh, const float (&corr)[2], int st, uint32_t phase) {
        bar_wait(&sm.vfull[st], phase);
        // an item's first page zeroes the running output (factor 0); later
        // pages rescale it only when a real column's max moved (warp vote;
        // rare under lazy rescaling).  One in-place multiply path: no copies.
        const float c0 = fresh ? 0.f : corr[0], c1 = fresh ? 0.f : corr[1];
        if (__any_sync(0xffffffffu, fresh || (real0 && c0 != 1.f) || (real1 && c1 != 1.f))) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                oacc[m][0] *= c0;
                oacc[m][2] *= c0;
                oacc[m][1] *= c1;
                oacc[m][3] *= c1;
            }
        }
    };
    auto pv_step = [&](int st, int ks, PvRegs& r) {
        const uint8_t* vp = vslots + st * vslot;
        const uint8_t* vscale = vp + G * D / 4;
        const uint8_t* vzero = vscale + 2 * G;
        const uint8_t* vsbase = main_col ? vscale : reinterpret_cast<const uint8_t*>(sm.ones);
        const uint32_t* ptr = &sm.pt[st][prow_ok ? prow : 0][tig];
        const int t0 = 16 * ks + 2 * tig;
        // p = 2^x of the stored exponents (ex2.approx.f16x2: one MUFU per two
        // tokens, and the f16 exponent costs |p error| < 2e-4 at p <= 2^kLazy)
        const uint32_t pp0 = prow_ok ? ex2_h2(ptr[8 * ks]) : 0u;      // tokens 16 ks + 2 tig (+1)
        const uint32_t pp1 = prow_ok ? ex2_h2(ptr[8 * ks + 4]) : 0u;  // tokens 16 ks + 8 + 2 tig (+1)
        const uint32_t b0 = hmul2(pp0, lds32(vsbase + 2 * t0));
        const uint32_t b1 = hmul2(pp1, lds32(vsbase + 2 * (t0 + 8)));
        uint32_t w0, w1, w2, w3;  // token rows 16 ks + [0, 16), channels 8 gid + [0, 8) / 64 + ...
        ldsm_t4(smem_u32(vp) + 512 * ks + ldsm_off, w0, w1, w2, w3);
        const uint32_t z0 = lds32(vzero + 2 * t0);
        const uint32_t z1 = lds32(vzero + 2 * (t0 + 8));
        mma_ldsm(kc, oacc, w0, w1, w2, w3, b0, b1);
        if (ks == 0)
            mma16816_z(r.vaux, kOnes, z0, kOnes, z1, b0, b1);
        else
            mma16816(r.vaux, kOnes, z0, kOnes, z1, b0, b1);
        if (kFull) {  // the unscaled p: sum p and sum p z
            if (ks == 0)
                mma16816_z(r.vaux2, kOnes, z0, kOnes, z1, pp0, pp1);
            else
                mma16816(r.vaux2, kOnes, z0, kOnes, z1, pp0, pp1);
        }
    };
    auto pv_tail = [&](bool fresh, const float (&corr)[2], PvRegs& r) {
        // vaux lanes 0-1: sum(p s) per column; lanes 2-3: sum(p) and sum(p z).
        // Row constants (zero points, the 1024 offset) accumulate per column in
        // ob[weight class] and are added at the flush.
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float sBv = __shfl_sync(0xffffffffu, r.vaux[j], kFull ? tig : (tig & 1));
            const float lp = kFull ? __shfl_sync(0xffffffffu, r.vaux2[j], tig) : __shfl_sync(0xffffffffu, r.vaux[j], 2 + (tig & 1));
            const float zz = kFull ? __shfl_sync(0xffffffffu, r.vaux2[2 + j], tig)
                                   : __shfl_sync(0xffffffffu, r.vaux[2 + j], 2 + (tig & 1));
            const float cf = fresh ? 0.f : corr[j];
            ol[j] = fmaf(ol[j], cf, lp);
            ob[0][j] = fmaf(ob[0][j], cf, zz - 256.f * sBv);  // w 4
            ob[1][j] = fmaf(ob[1][j], cf, zz - 64.f * sBv);   // w 16
            ob[2][j] = fmaf(ob[2][j], cf, zz - 16.f * sBv);   // w 64
            ob[3][j] = fmaf(ob[3][j], cf, zz - 4.f * sBv);    // w 256
        }
    };
    auto flush = [&](const Pg& d, const float (&mnew)[2]) {
        float* base = P.part + ((int64_t)d.u * P.nslot + d.slot) * part_stride(GROUP);
        if (kFull || tig < 2) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int g = 2 * tig + j;
                if (g < GROUP) {
                    // tile m: row gid = channel 8 gid + m, row gid + 8 = channel 64 + 8 gid + m
                    float lo[8], hi[8];
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        lo[m] = fmaf(oacc[m][j], 1.f / tile_w(m), ob[tile_c(m)][j]);
                        hi[m] = fmaf(oacc[m][2 + j], 1.f / tile_w(m), ob[tile_c(m)][j]);
                    }
                    // the record is re-read by the merge right after: keep it in L2
                    float* o4 = base + g * D + 8 * gid;
                    st_last4(o4, lo[0], lo[1], lo[2], lo[3], pol_last);
                    st_last4(o4 + 4, lo[4], lo[5], lo[6], lo[7], pol_last);
                    float* h4 = base + g * D + 64 + 8 * gid;
                    st_last4(h4, hi[0], hi[1], hi[2], hi[3], pol_last);
                    st_last4(h4 + 4, hi[4], hi[5], hi[6], hi[7], pol_last);
                    if (gid == 0) *reinterpret_cast<float2*>(base + GROUP * D + 2 * g) = make_float2(mnew[j], ol[j]);
                }
            }
        }
    };

    if constexpr (!WS) {
        // ---- software pipeline: QK of page k + 1 beside PV of page k ----
        Pg d0 = next_page();
        fill_ks(d0);
        fill_vs(d0);
        if (d0.u >= 0) {
            Pg d1 = next_page();
            fill_ks(d1);
            fill_vs(d1);
            Pg d2 = next_page();
            fill_ks(d2);
            fill_vs(d2);
            issue_key(d0, 0);
            issue_val(d0, 0);
            issue_key(d1, 1);
            issue_val(d1, 1);
            prefetch_q(d1, d0.u);
            prefetch_q(d2, d1.u);
            float corr0[2], mnew0[2];
            {
                qk_prologue(d0, 0, 0);
                QkRegs qr;
    #pragma unroll
                for (int ks = 0; ks < 8; ++ks) qk_step(0, ks, qr);
                qk_tail(0, qr, corr0, mnew0);
            }
            __syncwarp();
            issue_key(d2, 0);  // key slot 0 is free once QK(0) is done
            // steady state: one path (QK of page k + 1 beside PV of page k), so the
            // output accumulators keep their registers across the back edge
            uint32_t k = 0;
    #pragma unroll 1
            for (; d1.u >= 0; ++k) {
                const int st = k & 1;
                const bool fresh0 = d0.p == (d0.pq >> 16), last0 = d0.p + 1 == (d0.pq & 0xffff);
                fill_vs(d2);          // before the stream may move to another item
                Pg d3 = next_page();  // page k + 3: its key goes into key slot st ^ 1 after QK(k + 1)
                prefetch_q(d3, d2.u);
                float corr1[2], mnew1[2];
                PvRegs pr;
                qk_prologue(d1, st ^ 1, ((k + 1) >> 1) & 1);
                pv_head(fresh0, corr0, st, (k >> 1) & 1);
                QkRegs qr;
                // the two pages' k-steps alternate: independent chains for the scheduler
    #pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    pv_step(st, ks, pr);
                    qk_step(st ^ 1, ks, qr);
                }
                pv_tail(fresh0, corr0, pr);
                qk_tail(st ^ 1, qr, corr1, mnew1);
                if (last0) flush(d0, mnew0);
                __syncwarp();
                fill_ks(d3);
                issue_val(d2, st);     // value slot st (page k) -> page k + 2
                issue_key(d3, st ^ 1);  // key slot st ^ 1 (page k + 1) -> page k + 3
                d0 = d1;
                d1 = d2;
                d2 = d3;
    #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    corr0[j] = corr1[j];
                    mnew0[j] = mnew1[j];
                }
            }
            {  // the stream's last page: P V only
                const int st = k & 1;
                const bool fresh0 = d0.p == (d0.pq >> 16);
                PvRegs pr;
                pv_head(fresh0, corr0, st, (k >> 1) & 1);
    #pragma unroll
                for (int ks = 0; ks < 8; ++ks) pv_step(st, ks, pr);
                pv_tail(fresh0, corr0, pr);
                flush(d0, mnew0);  // a stream's last page is its item's last
            }
        }
        if (P.fp_first) {
            // this warp's stream is drained: the merge grid (our programmatic
            // dependent; its CTAs wait for this grid) may take freed SM slots
            asm volatile("griddepcontrol.launch_dependents;");
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the fp grid is complete
        }
    } else {
        // ---- the pair's pipeline: QK warp on page k while the PV warp runs page
        // k - 1.  Stage st = k & 1 holds page k's key slot, value slot, P^T and job;
        // pfull[st]: the QK warp published page k (P^T, corrections, job);
        // pempty[st]: the PV warp is done with it (P^T, job, value slot) ----
        if (qk_role) {
            Pg d0 = next_page();
            fill_ks(d0);
            fill_vs(d0);
            Pg d1 = next_page();
            fill_ks(d1);
            fill_vs(d1);
            issue_key(d0, 0);
            issue_val(d0, 0);
            issue_key(d1, 1);
            issue_val(d1, 1);
            prefetch_q(d1, d0.u);
            uint32_t k = 0;
    #pragma unroll 1
            for (; d0.u >= 0; ++k) {
                const int st = k & 1;
                const uint32_t ph = (k >> 1) & 1;
                float corr[2], mnew[2];
                qk_prologue(d0, st, ph);
                pe_phase = ph;
                QkRegs qr;
    #pragma unroll
                for (int ks = 0; ks < 8; ++ks) qk_step(st, ks, qr);
                qk_tail(st, qr, corr, mnew);
                Pg d2 = next_page();  // page k + 2: key slot st, value slot st
                fill_ks(d2);
                fill_vs(d2);
                prefetch_q(d2, d1.u);
                if (gid == 0) {
                    sm.corr[st][2 * tig] = corr[0];
                    sm.corr[st][2 * tig + 1] = corr[1];
                    sm.mnew[st][2 * tig] = mnew[0];
                    sm.mnew[st][2 * tig + 1] = mnew[1];
                }
                if (lane == 0) {
                    sm.job[st][0] = d0.u;
                    sm.job[st][1] = d0.p;
                    sm.job[st][2] = d0.pq;
                    sm.job[st][3] = d0.slot;
                    sm.vnext[st] = d2.u >= 0 ? d2.vs : -1;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.pfull[st]);
                issue_key(d2, st);  // QK(k) is done with key slot st
                d0 = d1;
                d1 = d2;
            }
            // end of the stream: an empty job once the PV warp released the stage
            const int st = k & 1;
            mbar_wait_sleep(&sm.pempty[st], (k >> 1) & 1);
            if (lane == 0) sm.job[st][0] = -1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.pfull[st]);
        } else {
            uint32_t k = 0;
    #pragma unroll 1
            for (;; ++k) {
                const int st = k & 1;
                const uint32_t ph = (k >> 1) & 1;
                mbar_wait_sleep(&sm.pfull[st], ph);
                Pg d;
                d.u = sm.job[st][0];
                if (d.u < 0) break;
                d.p = sm.job[st][1];
                d.pq = sm.job[st][2];
                d.slot = sm.job[st][3];
                const int vs2 = sm.vnext[st];
                const float corr[2] = {sm.corr[st][2 * tig], sm.corr[st][2 * tig + 1]};
                const float mnew[2] = {sm.mnew[st][2 * tig], sm.mnew[st][2 * tig + 1]};
                const bool fresh = d.p == (d.pq >> 16), last = d.p + 1 == (d.pq & 0xffff);
                PvRegs pr;
                pv_head(fresh, corr, st, ph);
    #pragma unroll
                for (int ks = 0; ks < 8; ++ks) pv_step(st, ks, pr);
                pv_tail(fresh, corr, pr);
                if (last) flush(d, mnew);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm.pempty[st]);
                    if (vs2 >= 0) {  // value slot st -> page k + 2
                        mbar_expect_tx(&sm.vfull[st], vslot);
                        bulk_g2s(vslots + st * vslot, c.value_pool + (int64_t)vs2 * vslot, vslot, &sm.vfull[st], pol);
                    }
                }
            }
        }
    }
    // the last warp out resets the work queue for the next launch (after its
    // outstanding ticket returned: using its value orders the atomics)
    if (qk_role && lane == 0) {
        asm volatile("" ::"r"(tk) : "memory");
        const int fin = atomicAdd(&P.ctr[1], 1);
        if (fin == static_cast<int>(gridDim.x) * (WS ? kWsPairs : kWarps) - 1) {
            P.ctr[0] = 0;
            P.ctr[1] = 0;
        }
    }
}

// The full-precision tokens: one 128-thread CTA per 32-token chunk
// (kitty_fp.cuh).  Default order: launched first, as a programmatic dependent
// of the append; the page grid follows as its dependent, so the persistent
// page CTAs take over each SM as its fp CTAs drain and the elastic page queue
// absorbs the staggered start (C2 -1.0, C3 -2.8 us per layer against the
// page-first order, where the fp CTAs backfilled the page grid's tail).
template <int GROUP>
__global__ void __launch_bounds__(128) fp_tokens_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t fsm[];
    const int it = blockIdx.x;
    const int fc = it / P.units, u = it - fc * P.units;
    if (P.fp_first) {
        // behind the append: wait for it, then let the page grid launch
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
    } else {
        asm volatile("griddepcontrol.launch_dependents;");  // the merge may pre-launch
    }
    const fptok::Geom gm = fptok::geom(P.c, u, P.max_tokens);
    if (gm.n > 0 && fc * kFpChunk < gm.nfp)
        fptok::chunk_tc<GROUP>(P.c, P.q, P.part, P.nslot, part_stride(GROUP), fsm, u, fc, P.max_tokens, P.fp_union != 0);
    // launched as a programmatic dependent of the page grid: finish only after it
    if (!P.fp_first) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// The full-precision tokens in the aligned geometries (S a multiple of 32:
// no chunk mixes staged and paged keys): one warp per 32-token chunk
// (fptok::chunk_warp), kFpWarps chunks per CTA, no CTA-wide barrier.
constexpr int kFpWarps = 1;  // one chunk per CTA (2: C3 -1.8 %, 4: -3.7 %)
__host__ __device__ inline int fpw_warp_bytes(int kslot) { return (fptok::cw_warp_bytes(kslot) + 127) & ~127; }
template <int GROUP>
__global__ void __launch_bounds__(kFpWarps * 32) fp_warp_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t fsm[];
    const int warp = threadIdx.x >> 5;
    const int it = blockIdx.x * kFpWarps + warp;
    const int fc = it / P.units, u = it - fc * P.units;
    if (P.fp_first) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
    } else {
        asm volatile("griddepcontrol.launch_dependents;");
    }
    if (fc < P.fmax) {
        const fptok::Geom gm = fptok::geom(P.c, u, P.max_tokens);
        if (gm.n > 0 && fc * kFpChunk < gm.nfp)
            fptok::chunk_warp<GROUP>(P.c, P.q, P.part, P.nslot, part_stride(GROUP),
                                     fsm + warp * fpw_warp_bytes((int)P.c.key_slot_bytes), u, fc, P.max_tokens);
    }
    if (!P.fp_first) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// K5: WARPS warps merge one (unit, query row): 2 when a unit has <= 32 partial
// slots (short contexts: many small CTAs, one wave), 4 up to 128 slots, 16
// above (long contexts).  CSPLIT CTAs share a row (channel slices) when the
// rows alone would not fill the GPU (a few long units: C4).
template <int GROUP, int WARPS, int CSPLIT = 1>
__global__ void __launch_bounds__(WARPS * 32) combine_parts_kernel(Params P) {
    const int slice = blockIdx.x % CSPLIT, r = blockIdx.x / CSPLIT;
    const int u = r / GROUP, g = r - (r / GROUP) * GROUP;
    const KittyCacheDesc& c = P.c;
    // the unit's part list depends only on its length (written by the append,
    // before the page grid): computed before waiting on the fp grid
    const UnitGeom gm = unit_geom(c, u, P.max_tokens);
    // a unit longer than the caller's bound was attended over its first
    // max_tokens tokens only: make the caller's check() raise
    if (g == 0 && threadIdx.x == 0 && c.unit_len[u] > P.max_tokens) set_status(c.status, KITTY_STATUS_LENGTH);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the fp grid (KITTY_PDL bit 2)
    // the next kernel on the stream (the next layer's append) may become resident
    asm volatile("griddepcontrol.launch_dependents;");
    if (gm.n == 0) {  // an empty (retired) sequence of the batch: zero output rows
        const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
        const int64_t row = (int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + g;
        for (int i = threadIdx.x; i < D; i += blockDim.x) {
            if (P.out_dtype == KITTY_F32)
                static_cast<float*>(P.out)[row * D + i] = 0.f;
            else
                static_cast<uint16_t*>(P.out)[row * D + i] = 0;
        }
        return;
    }
    const int nfc = (gm.nfp + kFpChunk - 1) / kFpChunk;
    int nch[3];
    for (int lv = 0; lv < 3; ++lv) {
        const int n = level_begin(lv + 1, gm.vp, P.lvl) - level_begin(lv, gm.vp, P.lvl);
        nch[lv] = (n + P.cs[lv] - 1) / P.cs[lv];
    }
    // parts: the fp chunks, then kHalves records per page chunk
    const int nparts = nfc + kHalves * (nch[0] + nch[1] + nch[2]);
    constexpr int kStride = part_stride(GROUP);
    auto slot_of = [&](int i) {
        if (i < nfc) return i;
        const int k = (i - nfc) / kHalves, hw = (i - nfc) - k * kHalves;
        int cs;
        if (k < nch[0]) cs = k;
        else if (k < nch[0] + nch[1]) cs = P.cmx[0] + (k - nch[0]);
        else cs = P.cmx[0] + P.cmx[1] + (k - nch[0] - nch[1]);
        return P.fmax + kHalves * cs + hw;
    };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const int64_t row = (int64_t)b * c.cfg.h_q + (int64_t)h * GROUP + g;
    // 33-128 slots (4-warp CTAs): one pass, (m, l) loaded with the rows (C5
    // 488.0 -> 478.0 us per layer, C2 equal); the 2-warp CTAs of short units
    // (C3: 124.9 vs 123.7) and long contexts (C4: 37.7 vs 37.1) keep the max
    // pass first
    if constexpr (WARPS == 4)
        lse_merge_row_1p<GROUP, decltype(slot_of), WARPS, CSPLIT>(P.part + (int64_t)u * P.nslot * kStride, kStride,
                                                                 nparts, slot_of, g, P.out, P.out_dtype, row, slice);
    else
        lse_merge_row<GROUP, decltype(slot_of), WARPS, CSPLIT>(P.part + (int64_t)u * P.nslot * kStride, kStride, nparts,
                                                              slot_of, g, P.out, P.out_dtype, row, slice);
}

}  // namespace fastattn

// ---- host side ---------------------------------------------------------------------

using namespace fastattn;

static int num_sms() { return device_sms(); }

bool fast_attention_supported(const KittyCacheDesc& c) {
    const int group = c.cfg.h_q / c.cfg.h_kv;
    return c.row_dtype == KITTY_BF16 && !c.key_meta && !c.value_meta && c.cfg.d == D && c.cfg.g == G &&
           c.cfg.key_bits == 2 && c.cfg.value_bits == 2 &&
           (group == 1 || group == 2 || group == 4 || group == 8) && c.cfg.d_boost <= 32 &&
           c.key_slot_bytes <= kKeySlotMax && c.value_slot_bytes == kValueSlot;
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
    const long long streams = (long long)num_sms() * kCtasPerSm * kWarps;  // concurrent page streams (warps)
    static int ppc_max = 8, cs1_div = 4, ppc_div = 2, inited = 0, swept = 0;  // ppc_max <= 32: an item's pages fit the lanes
    if (!inited) {
        inited = 1;
        if (const char* e = getenv("KITTY_SCHED")) {  // experiments: "l1,l2,ppc_max,cs1_div[,ppc_div]"
            swept = 1;
            sscanf(e, "%d,%d,%d,%d,%d", &h_lvl[0], &h_lvl[1], &ppc_max, &cs1_div, &ppc_div);
            ppc_div = ppc_div < 1 ? 1 : ppc_div;
            ppc_max = ppc_max < 1 ? 1 : (ppc_max > 32 ? 32 : ppc_max);
            h_lvl[2] = h_lvl[0];  // a sweep sets one pair for every unit length
            h_lvl[3] = h_lvl[1];
        }
    }
    int ppc = static_cast<int>(pages / (ppc_div * streams));
    // Many pages per stream (C5: ~55): items up to 16 pages, levels from 940 /
    // 985 per mille -- fewer partial records per unit, whose write + merge
    // traffic (150 MB per C5 layer at the defaults, beyond L2) dominated the
    // tail (C5 481.5 -> 451 us per layer; C2 / C3, ~14 pages per stream, keep
    // the defaults: swept, tools/gpu_sched_sweep.sh).  Not longer: the P V
    // accumulators carry the 1024 offset of the code operands for the whole
    // item, and the tensor cores' accumulation error grows with it (C5 at
    // 32-page items: 0.0136 max-abs against the oracle, over the 1e-2 bar; at
    // 16: 0.0068, at 8: 0.0058)
    const bool big = !swept && ppc >= 24;
    const int pmax = big ? 16 : ppc_max, c1div = cs1_div;
    ppc = ppc < 1 ? 1 : (ppc > pmax ? pmax : ppc);
    p.ppc = ppc;
    p.cmax = (maxp + ppc - 1) / ppc;
    p.cs[0] = ppc;
    p.cs[1] = ppc / c1div > 1 ? ppc / c1div : 1;
    p.cs[2] = 1;
    // Level 0 in whole rounds: its items (ppc pages each, for units at the
    // longest length) are pulled round by round by the page streams; when
    // there are only 1-2 whole rounds and the last would be nearly empty
    // (< 35 %), a few streams would start one more long item -- a large share
    // of a stream's work -- as everyone else runs out, so level 0 shrinks to
    // the whole rounds (C4; with 3+ rounds, C3 / C5, the cut costs more than
    // the tail it removes).
    for (int i = 0; i < 4; ++i) p.lvl[i] = big ? (i % 2 == 0 ? 940 : 985) : h_lvl[i];
    {
        const int past_m = max_tokens > c.cfg.s ? max_tokens - c.cfg.s : 0;
        const int vpm = (past_m - min(c.cfg.r, past_m)) / G;
        const int rule = vpm >= 512 ? 2 : 0;
        const int l0 = (vpm * p.lvl[rule]) / 1000;
        const long long items0 = (long long)p.units * ((l0 + ppc - 1) / ppc);
        const long long rounds = items0 / streams, rest = items0 - rounds * streams;
        if (vpm > 0 && rounds >= 1 && rounds < 3 && rest * 100 < 35 * streams) {
            const int l0n = static_cast<int>((rounds * streams) / p.units) * ppc;
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
    p.nslot = p.fmax + kHalves * (p.cmx[0] + p.cmx[1] + p.cmx[2]);
    p.part_bytes = (size_t)p.units * p.nslot * part_stride(p.group) * sizeof(float);
    return p;
}

size_t fast_attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens) {
    if (!fast_attention_supported(c)) return 0;
    const FastPlan p = plan(c, max_tokens);
    return p.ctr_bytes + p.part_bytes;
}

// programmatic dependent launch per edge, a bit mask (A/B knob KITTY_PDL,
// else per launch): 1 = first attention grid behind the preceding kernel,
// 2 = second behind the first, 4 = merge behind the second.  Page-first the
// merge edge stays off (merge CTAs parked beside fp CTAs take SM slots the fp
// grid still needs); fp-first it is on, and the page CTAs trigger it as their
// streams drain.
static const int g_pdl = [] {
    const char* e = std::getenv("KITTY_PDL");
    return e ? std::atoi(e) : -1;
}();

// launch order (A/B knob KITTY_FPFIRST, else per launch below): 1 = fp grid,
// page grid, merge; 0 = page grid, fp grid, merge
static const int g_fp_first = [] {
    const char* e = std::getenv("KITTY_FPFIRST");
    return e ? std::atoi(e) : -1;
}();

// page kernel variant (A/B knob KITTY_WS): 1 = warp-specialised QK / PV pairs
// (16 warps / SM at <= 128 registers), 0 (default) = one warp per page stream
// interleaving both (8 warps / SM).  Pairs won at group 8 (C5 490.3 vs 487.9
// us per layer) until the fp-token and merge work shrank; with the final
// kernels one warp per stream is ahead there too (C5 3 746 vs 3 698 tok/s).
static const int g_ws_env = [] {
    const char* e = std::getenv("KITTY_WS");
    return e ? std::atoi(e) : -1;
}();

template <int GROUP, int NKH>
static cudaError_t launch_t(const Params& prm, int grid, cudaStream_t st) {
    const bool g_ws = g_ws_env > 0;
    auto kfn = g_ws ? page_kernel<GROUP, NKH, true> : page_kernel<GROUP, NKH, false>;
    const int ks_b = (int)prm.c.key_slot_bytes, vs_b = (int)prm.c.value_slot_bytes;
    const size_t sm = (size_t)(g_ws ? pair_smem_bytes<GROUP>(ks_b, vs_b) * kWsPairs : warp_smem_bytes<GROUP>(ks_b, vs_b) * kWarps) +
                      (prm.units <= kMaxTableUnits ? 4 * prm.units : 0);
    cudaError_t e = set_kernel_smem((const void*)kfn,
                                    (g_ws ? pair_smem_bytes<GROUP>(kKeySlotMax, kValueSlot) * kWsPairs
                                          : warp_smem_bytes<GROUP>(kKeySlotMax, kValueSlot) * kWarps) +
                                        4 * kMaxTableUnits,
                                    true);
    if (e != cudaSuccess) return e;
    // persistent grid: kCtasPerSm CTAs per SM must be co-resident (their shared
    // memory plus the 1 KB per-CTA reservation fit the SM), else fewer per SM
    const int smpm = device_smem_per_sm();
    int per_sm = kCtasPerSm;
    while (per_sm > 1 && (size_t)per_sm * (sm + 1024) > (size_t)smpm) --per_sm;
    if (grid > num_sms() * per_sm) grid = num_sms() * per_sm;
    cudaLaunchAttribute at[3];
    for (int i = 0; i < 3; ++i) {
        at[i].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[i].val.programmaticStreamSerializationAllowed = ((g_pdl >= 0 ? g_pdl : (prm.fp_first ? 7 : 3)) >> i) & 1;
    }
    auto page_grid = [&](cudaLaunchAttribute* a) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(g_ws ? 2 * kWsPairs * 32 : kWarps * 32);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kfn, prm);
    };
    auto fp_grid = [&](cudaLaunchAttribute* a) {
        if (prm.fp_warp) {
            const int wsm = kFpWarps * fpw_warp_bytes((int)prm.c.key_slot_bytes);
            cudaError_t e2 = set_kernel_smem((const void*)fp_warp_kernel<GROUP>, wsm, true);
            if (e2 != cudaSuccess) return e2;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((prm.units * prm.fmax + kFpWarps - 1) / kFpWarps);
            cfg.blockDim = dim3(kFpWarps * 32);
            cfg.dynamicSmemBytes = wsm;
            cfg.stream = st;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, fp_warp_kernel<GROUP>, prm);
        }
        const int fsm = fptok::tc_scratch_bytes((int)prm.c.key_slot_bytes, prm.fp_union != 0);
        cudaError_t e2 = set_kernel_smem((const void*)fp_tokens_kernel<GROUP>, fsm, true);
        if (e2 != cudaSuccess) return e2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(prm.units * prm.fmax);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = fsm;
        cfg.stream = st;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fp_tokens_kernel<GROUP>, prm);
    };
    if (prm.fp_first) {
        if ((e = fp_grid(at + 0)) != cudaSuccess) return e;
        if ((e = page_grid(at + 1)) != cudaSuccess) return e;
    } else {
        if ((e = page_grid(at + 0)) != cudaSuccess) return e;
        if ((e = fp_grid(at + 1)) != cudaSuccess) return e;
    }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(prm.units * GROUP);
        cfg.stream = st;
        cfg.attrs = at + 2;
        cfg.numAttrs = 1;
        auto go = [&](auto kfn) -> cudaError_t {
            cudaError_t e2 = set_kernel_smem((const void*)kfn, 0, true);
            return e2 != cudaSuccess ? e2 : cudaLaunchKernelEx(&cfg, kfn, prm);
        };
        if (prm.nslot <= 32) {
            cfg.blockDim = dim3(2 * 32);
            return go(combine_parts_kernel<GROUP, 2>);
        }
        // 4 warps up to 128 slots (C2 -0.6 us per layer against 8: more CTAs in
        // flight, one batch of rows per warp either way)
        if (prm.nslot <= 128) {
            cfg.blockDim = dim3(4 * 32);
            return go(combine_parts_kernel<GROUP, 4>);
        }
        if (prm.nslot > 128) {  // long contexts: few rows, hundreds of parts each
            cfg.blockDim = dim3(16 * 32);
            const long long rows = (long long)prm.units * GROUP;
            if (rows * 8 <= num_sms()) {  // channel slices so that the merge spans the GPU, one CTA per SM
                cfg.gridDim = dim3(static_cast<unsigned>(rows * 8));
                return go(combine_parts_kernel<GROUP, 16, 8>);
            }
            if (rows <= 2LL * num_sms()) {  // C4 (32 rows): 4 slices, 36.8 vs 37.6 us per layer with 8
                cfg.gridDim = dim3(static_cast<unsigned>(rows * 4));
                return go(combine_parts_kernel<GROUP, 16, 4>);
            }
            return go(combine_parts_kernel<GROUP, 16>);
        }
        cfg.blockDim = dim3(kMergeWarps * 32);
        return go(combine_parts_kernel<GROUP, kMergeWarps>);
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
    // fp grid first when it needs more than one CTA per SM: beside the
    // persistent page CTAs only one fp CTA fits an SM's shared memory, so a
    // larger fp grid trickles through in many rounds (measured: first is
    // C2 -1.0, C3 -2.8 us per layer); a grid of at most one CTA per SM runs
    // in the page grid's shadow (C4: page-first 0.7 us faster)
    {
        static const int un_env = getenv("KITTY_FPUNION") ? atoi(getenv("KITTY_FPUNION")) : -1;
        // no chunk mixes staged and paged keys; measured: C2 -0.6 %, C3 -0.7 %
        // per step with the union layout, group 8 (C5) +0.4 % (kept apart)
        const bool aligned = c.cfg.s % kFpChunk == 0 && c.cfg.r % kFpChunk == 0;
        prm.fp_union = un_env >= 0 ? (un_env != 0 && aligned) : (aligned && p.group <= 4);
        static const int fw_env = getenv("KITTY_FPWARP") ? atoi(getenv("KITTY_FPWARP")) : -1;
        prm.fp_warp = fw_env >= 0 ? (fw_env != 0 && c.cfg.s % kFpChunk == 0) : (c.cfg.s % kFpChunk == 0);
    }
    prm.fp_first = g_fp_first >= 0 ? g_fp_first : ((long long)p.units * p.fmax > num_sms() ? 1 : 0);
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
    // one warp per page stream; no more warps than there are items
    const long long items = (long long)p.units * (p.cmx[0] + p.cmx[1] + p.cmx[2]);
    const long long ctas = (items + kWarps - 1) / kWarps, cap = (long long)num_sms() * kCtasPerSm;
    const int grid = static_cast<int>(ctas < cap ? ctas : cap);
    const int nkh = (c.cfg.d_boost + 15) / 16;
    switch (p.group) {
        case 1: return launch_g<1>(prm, nkh, grid, st);
        case 2: return launch_g<2>(prm, nkh, grid, st);
        case 4: return launch_g<4>(prm, nkh, grid, st);
        default: return launch_g<8>(prm, nkh, grid, st);
    }
}

}  // namespace kitty
