// Bulk page packer for the common geometry (d = g = 128, bf16 rows): the
// prefill path.  Same bytes as pack_key_tile / pack_value_tile
// (and so as pages.py:81-118 / 146-162), restructured for throughput:
//  * the page's 128 rows (32 KB, contiguous in the prefill input) arrive in
//    shared memory by one 1-D TMA copy;
//  * keys: thread = channel pair.  One pass over the tile keeps NaN-propagating
//    bf16x2 min / max and the two sequential fp64 score sums (quant.py:72: the
//    same token order, so the same rounding); a non-finite input shows up as a
//    non-finite score, so the NONFINITE check costs nothing extra.  The boost
//    selection (quant.py:93, stable top-k of the scores) is d_boost rounds of
//    redux.sync max / min over 64-bit keys in one warp, not an O(d^2) rank;
//  * quantiser: rint by the 1.5 * 2^23 magic add (round-half-even, as
//    np.rint), the IEEE quotient only when the reciprocal product lies within
//    1e-5 of a half-integer (the same rule as LaneQuant::code); codes are
//    accumulated by one IMAD each (the magic's constant part is subtracted per
//    word) and the page bytes go from registers straight to the slot.
// Channels whose scale is 0 or non-finite take LaneQuant::code element by
// element, so every edge case keeps the reference's bytes.
#pragma once
#include "kitty_common.cuh"

namespace kitty {
namespace fastpack {

constexpr int kD = 128, kG = 128;
constexpr int kThreads = 128;  // keys: thread = (channel pair, half); pass 1 scores one channel each, pass 2 a token half
constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
constexpr uint32_t kMagicBits = 0x4B400000u;

struct Smem {
    uint32_t tile[kG * kD / 2];  // [token][channel pair] bf16x2
    double score[kD];
    uint8_t row[kD];             // boost row of each channel, kSentinel if not boosted
    float lim[kD][2];            // per-channel (min, max) from pass 1
    unsigned long long bar[2];   // key page, value page (an append may pack both)
};

__device__ __forceinline__ uint32_t bmin2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float lo_f(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Quantiser of one lane (channel or token row); `plain` = the fast path holds.
struct FastQuant {
    LaneQuant q;
    bool plain;
    __device__ __forceinline__ FastQuant(float mn, float mx, float qmax) : q(mn, mx, qmax) {
        plain = q.scale >= 0x1p-90f && q.scale <= 0x1p100f;
    }
    // kMagicBits + rint((x - mn) / safe)
    __device__ __forceinline__ uint32_t biased(float x) const {
        const float dlt = __fsub_rn(x, q.mn);
        const float q0 = __fmul_rn(dlt, q.inv);
        const float q1 = __fmaf_rn(__fmaf_rn(-q0, q.safe, dlt), q.inv, q0);
        return __float_as_uint(__fadd_rn(q1, kMagic));
    }
};

// Sum over k of (kMagicBits << (s * k)) mod 2^32 for k < n: the constant part
// of a word accumulated by acc += biased << (s * k).
__host__ __device__ constexpr uint32_t magic_sum(int s, int n) {
    uint32_t r = 0;
    for (int k = 0; k < n; ++k) r += kMagicBits << (s * k);
    return r;
}

// 8 nibbles (code < 16 each) -> (2-bit low plane, 2-bit high plane), 16 bits each
__device__ __forceinline__ void split_nibbles(uint32_t x, uint32_t& lo, uint32_t& hi) {
    uint32_t l = x & 0x33333333u, h = (x >> 2) & 0x33333333u;
    l = (l | (l >> 2)) & 0x0f0f0f0fu;
    h = (h | (h >> 2)) & 0x0f0f0f0fu;
    l = (l | (l >> 4)) & 0x00ff00ffu;
    h = (h | (h >> 4)) & 0x00ff00ffu;
    lo = (l | (l >> 8)) & 0x0000ffffu;
    hi = (h | (h >> 8)) & 0x0000ffffu;
}

// The page's kG rows, rows [start, start + kG) of a ring of `wrap` rows at
// `base` (prefill: wrap >= start + kG, one copy; the value ring of an
// append may wrap, two copies), into s.tile by 1-D TMA on barrier `which`.
__device__ __forceinline__ void fetch_tile(Smem& s, const uint16_t* base, int start, int wrap, int which) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&s.bar[which]));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kG * kD * 2) : "memory");
        const int n1 = min(kG, wrap - start);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(s.tile))),
            "l"(base + (int64_t)start * kD), "r"(n1 * kD * 2), "r"(b)
            : "memory");
        if (n1 < kG)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    static_cast<uint32_t>(__cvta_generic_to_shared(s.tile + n1 * (kD / 2)))),
                "l"(base), "r"((kG - n1) * kD * 2), "r"(b)
                : "memory");
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "FT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra FT_%=;\n}" ::"r"(b)
        : "memory");
}

// Rows of channel c = 2 tp + col by the reference rule element by element
// (lanes the fast quotient does not cover), written to the slot.
__device__ __noinline__ void slow_key_rows(const uint32_t* tile, int tp, int half, int col, LaneQuant q, uint8_t r,
                                           uint8_t* gslot, int d_boost) {
    const KeyLayout L{kD, kG, d_boost};
    const int c = 2 * tp + col;
    for (int b = 16 * half; b < 16 * half + 16; ++b) {
        uint32_t lo = 0, hi = 0;
        for (int j = 0; j < 4; ++j) {
            const uint32_t w = tile[(4 * b + j) * 64 + tp];
            const uint32_t code = q.code(col ? hi_f(w) : lo_f(w));
            lo |= (code & 3u) << (2 * j);
            hi |= (code >> 2) << (2 * j);
        }
        gslot[L.dense_off() + c * (kG / 4) + b] = static_cast<uint8_t>(lo);
        if (r != kSentinel) gslot[L.high_off() + r * (kG / 4) + b] = static_cast<uint8_t>(hi);
    }
}

// Quantise channels c = 2 tp (low bf16 of each tile word) and c + 1 (high)
// into their dense rows and, when boosted (row != kSentinel), high_bits
// rows; word wd of a row = tokens 16 wd .. 16 wd + 15.
__device__ __forceinline__ void key_pair(const Smem& s, int tp, int half, const FastQuant& qa, const FastQuant& qb,
                                         uint8_t ra, uint8_t rb, uint8_t* gslot, const KeyLayout& L) {
    uint32_t* da = reinterpret_cast<uint32_t*>(gslot + L.dense_off() + 2 * tp * (kG / 4));
    uint32_t* db = da + kG / 16;
    uint32_t* ha = reinterpret_cast<uint32_t*>(gslot + L.high_off() + ra * (kG / 4));
    uint32_t* hb = reinterpret_cast<uint32_t*>(gslot + L.high_off() + rb * (kG / 4));
#pragma unroll 1
    for (int wd = 4 * half; wd < 4 * half + 4; ++wd) {
        // codes as nibbles, tokens 0-7 / 8-15 of the word
        uint32_t a0 = 0, a1 = 0, b0 = 0, b1 = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t w0 = s.tile[(16 * wd + k) * 64 + tp], w1 = s.tile[(16 * wd + 8 + k) * 64 + tp];
            a0 += qa.biased(lo_f(w0)) << (4 * k);
            a1 += qa.biased(lo_f(w1)) << (4 * k);
            b0 += qb.biased(hi_f(w0)) << (4 * k);
            b1 += qb.biased(hi_f(w1)) << (4 * k);
        }
        a0 -= magic_sum(4, 8);
        a1 -= magic_sum(4, 8);
        b0 -= magic_sum(4, 8);
        b1 -= magic_sum(4, 8);
        uint32_t l0, h0, l1, h1;
        split_nibbles(a0, l0, h0);
        split_nibbles(a1, l1, h1);
        da[wd] = l0 | (l1 << 16);
        if (ra != kSentinel) ha[wd] = h0 | (h1 << 16);
        split_nibbles(b0, l0, h0);
        split_nibbles(b1, l1, h1);
        db[wd] = l0 | (l1 << 16);
        if (rb != kSentinel) hb[wd] = h0 | (h1 << 16);
    }
}

// A zero min / max of channel `col` takes the sign of its last zero token
// (np.minimum.reduce / np.maximum.reduce keep the later operand of a tie).
__device__ __noinline__ float last_zero_key(const uint32_t* tile, int tp, int col) {
    for (int t = kG - 1; t >= 0; --t) {
        const float v = col ? hi_f(tile[t * 64 + tp]) : lo_f(tile[t * 64 + tp]);
        if (v == 0.f) return v;
    }
    return 0.f;
}

// pack_key_page (pages.py:81-118) of the page of rows [start, start + kG) of the ring at `base`.
__device__ void key_page(Smem& s, const uint16_t* base, int start, int wrap, int d_boost, uint8_t* gslot,
                         uint32_t* status) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tp = tid & 63, half = tid >> 6;
    fetch_tile(s, base, start, wrap, 0);
    // pass 1: the fp64 score of channel 2 tp + half (each chain sequential in
    // token order, quant.py:72), and on warps 0-1 the bf16x2 min / max of both
    // channels of the pair
    uint32_t mn2 = s.tile[tp], mx2 = mn2;
    double a = 0.0;
    if (half == 0) {
#pragma unroll 8
        for (int t = 0; t < kG; ++t) {
            const uint32_t w = s.tile[t * 64 + tp];
            mn2 = bmin2(mn2, w);
            mx2 = bmax2(mx2, w);
            a += static_cast<double>(fabsf(lo_f(w)));
        }
    } else {
#pragma unroll 8
        for (int t = 0; t < kG; ++t) a += static_cast<double>(fabsf(hi_f(s.tile[t * 64 + tp])));
    }
    s.score[2 * tp + half] = a / static_cast<double>(kG);
    const bool bad = !(fabs(a) < INFINITY);
    if (half == 0) {
        float mn0 = lo_f(mn2), mx0 = lo_f(mx2), mn1 = hi_f(mn2), mx1 = hi_f(mx2);
        if (mn0 == 0.f || mx0 == 0.f) {
            const float z = last_zero_key(s.tile, tp, 0);
            mn0 = mn0 == 0.f ? z : mn0;
            mx0 = mx0 == 0.f ? z : mx0;
        }
        if (mn1 == 0.f || mx1 == 0.f) {
            const float z = last_zero_key(s.tile, tp, 1);
            mn1 = mn1 == 0.f ? z : mn1;
            mx1 = mx1 == 0.f ? z : mx1;
        }
        s.lim[2 * tp][0] = mn0;
        s.lim[2 * tp][1] = mx0;
        s.lim[2 * tp + 1][0] = mn1;
        s.lim[2 * tp + 1][1] = mx1;
    }
    __syncthreads();
    // boost selection (quant.py:93): d_boost rounds of (max score, then lowest
    // channel) over 64-bit keys; channel l + 32 j lives in lane l, slot j
    if (warp == 0) {
        unsigned long long key[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) key[j] = static_cast<unsigned long long>(__double_as_longlong(s.score[lane + 32 * j]));
        uint32_t taken = 0;
        for (int it = 0; it < d_boost; ++it) {
            unsigned long long best = 0;
            uint32_t bidx = 0xffffu;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool free_ = !((taken >> j) & 1u);
                if (free_ && (bidx == 0xffffu || key[j] > best)) {
                    best = key[j];
                    bidx = lane + 32 * j;
                }
            }
            const uint32_t hi = static_cast<uint32_t>(best >> 32), lo = static_cast<uint32_t>(best);
            const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
            const bool c1 = hi == mh;
            const uint32_t ml = __reduce_max_sync(0xffffffffu, c1 ? lo : 0u);
            const bool c2 = c1 && lo == ml;
            const uint32_t sel = __reduce_min_sync(0xffffffffu, c2 ? bidx : 0xffffu);
            if ((sel & 31u) == static_cast<uint32_t>(lane)) taken |= 1u << (sel >> 5);
        }
        // high_bits row = rank among the boosted channels in channel order (pages.py:103)
        int before = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned bal = __ballot_sync(0xffffffffu, (taken >> j) & 1u);
            const int pos = before + __popc(bal & ((1u << lane) - 1u));
            s.row[lane + 32 * j] = ((taken >> j) & 1u) ? static_cast<uint8_t>(pos) : kSentinel;
            before += __popc(bal);
        }
    }
    if (__syncthreads_or(bad) && tid == 0) set_status(status, KITTY_STATUS_NONFINITE);
    // pass 2: quantise both channels over this thread's token half, bytes
    // straight to the slot
    const KeyLayout L{kD, kG, d_boost};
    const int c0 = 2 * tp;
    const uint8_t r0 = s.row[c0], r1 = s.row[c0 + 1];
    const FastQuant q0(s.lim[c0][0], s.lim[c0][1], r0 != kSentinel ? 15.f : 3.f);
    const FastQuant q1(s.lim[c0 + 1][0], s.lim[c0 + 1][1], r1 != kSentinel ? 15.f : 3.f);
    if (q0.plain && q1.plain) {
        key_pair(s, tp, half, q0, q1, r0, r1, gslot, L);
    } else {
        slow_key_rows(s.tile, tp, half, 0, q0.q, r0, gslot, d_boost);
        slow_key_rows(s.tile, tp, half, 1, q1.q, r1, gslot, d_boost);
    }
    if (half == 0) {
        // boost_idx bytes, f16 scales and zero points (2-byte aligned offsets)
        reinterpret_cast<uint16_t*>(gslot + L.idx_off())[tp] = static_cast<uint16_t>(r0 | (r1 << 8));
        uint16_t* s16 = reinterpret_cast<uint16_t*>(gslot + L.scale_off());
        uint16_t* z16 = reinterpret_cast<uint16_t*>(gslot + L.zero_off());
        s16[c0] = static_cast<uint16_t>(f32_to_half_bits(q0.q.scale));
        s16[c0 + 1] = static_cast<uint16_t>(f32_to_half_bits(q1.q.scale));
        z16[c0] = static_cast<uint16_t>(f32_to_half_bits(q0.q.mn));
        z16[c0 + 1] = static_cast<uint16_t>(f32_to_half_bits(q1.q.mn));
    }
}

// Sign of the last zero channel of row r (channels 32 q .. 32 q + 31 in this
// lane, the other three in the row's lanes).
__device__ __noinline__ float last_zero_value(const uint32_t* tile, int r, int q) {
    int best = -1;
    for (int j = 31; j >= 0 && best < 0; --j) {
        const int ch = 32 * q + j;
        const uint32_t w = tile[r * 64 + (ch >> 1)];
        const float v = (ch & 1) ? hi_f(w) : lo_f(w);
        if (v == 0.f) best = (ch << 1) | (signbit(v) ? 1 : 0);
    }
    const unsigned grp = 0xfu << (threadIdx.x & 28);
    best = max(best, __shfl_xor_sync(grp, best, 1));
    best = max(best, __shfl_xor_sync(grp, best, 2));
    return (best & 1) ? -0.f : 0.f;
}

// Codes of channels 32 q .. 32 q + 31 of row r by the reference rule.
__device__ __noinline__ uint2 slow_value_codes(const uint32_t* tile, int r, int q, LaneQuant lq) {
    uint32_t c[2] = {0u, 0u};
    for (int j = 0; j < 32; ++j) {
        const uint32_t w = tile[r * 64 + 16 * q + (j >> 1)];
        c[j >> 4] |= lq.code((j & 1) ? hi_f(w) : lo_f(w)) << (2 * (j & 15));
    }
    return make_uint2(c[0], c[1]);
}

// pack_value_page (pages.py:146-162): per-token quantisation.  Four lanes per
// token row (32 channels each, 16-byte chunks read in a row-rotated order so a
// warp's 8 rows hit distinct banks), 32 rows per pass.
__device__ void value_page(Smem& s, const uint16_t* base, int start, int wrap, uint8_t* gslot, uint32_t* status) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    fetch_tile(s, base, start, wrap, 1);
    const ValueLayout L{kD, kG};
    const int q = lane & 3;
    bool bad = false;
#pragma unroll 1
    for (int pass = 0; pass < kG / (kThreads / 4); ++pass) {
        const int r = (kThreads / 4) * pass + 8 * warp + (lane >> 2);
        // w[4 k ..] = chunk (k + r) & 3 of the lane's 32 channels (8 channels per chunk)
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 x = reinterpret_cast<const uint4*>(s.tile + r * 64 + 16 * q)[(k + r) & 3];
            w[4 * k] = x.x;
            w[4 * k + 1] = x.y;
            w[4 * k + 2] = x.z;
            w[4 * k + 3] = x.w;
        }
        uint32_t mn2 = w[0], mx2 = w[0];
#pragma unroll
        for (int i = 1; i < 16; ++i) {
            mn2 = bmin2(mn2, w[i]);
            mx2 = bmax2(mx2, w[i]);
        }
        float mn = fmin_nan(lo_f(mn2), hi_f(mn2)), mx = fmax_nan(lo_f(mx2), hi_f(mx2));
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            mn = fmin_nan(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        bad |= !(fabsf(mn) < INFINITY) || !(fabsf(mx) < INFINITY);
        if (mn == 0.f || mx == 0.f) {  // uniform over the row's 4 lanes
            const float z = last_zero_value(s.tile, r, q);
            mn = mn == 0.f ? z : mn;
            mx = mx == 0.f ? z : mx;
        }
        const FastQuant fq(mn, mx, 3.f);
        // a chunk's 8 channels -> 16 code bits; chunk kk lands in bits 16 (kk & 1) of word kk >> 1
        uint32_t part[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t a = 0;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                a += fq.biased(lo_f(w[4 * k + m])) << (4 * m);
                a += fq.biased(hi_f(w[4 * k + m])) << (4 * m + 2);
            }
            part[k] = a - magic_sum(2, 8);
        }
        uint32_t c0 = 0, c1 = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int kk = (k + r) & 3;
            const uint32_t v = (part[k] & 0xffffu) << (16 * (kk & 1));
            if (kk < 2) c0 |= v; else c1 |= v;
        }
        if (!fq.plain) {
            const uint2 sc = slow_value_codes(s.tile, r, q, fq.q);
            c0 = sc.x;
            c1 = sc.y;
        }
        reinterpret_cast<uint2*>(gslot + L.codes_off() + r * (kD / 4))[q] = make_uint2(c0, c1);
        if (q == 0) {
            reinterpret_cast<uint16_t*>(gslot + L.scale_off())[r] = static_cast<uint16_t>(f32_to_half_bits(fq.q.scale));
            reinterpret_cast<uint16_t*>(gslot + L.zero_off())[r] = static_cast<uint16_t>(f32_to_half_bits(mn));
        }
    }
    if (__syncthreads_or(bad) && tid == 0) set_status(status, KITTY_STATUS_NONFINITE);
}

}  // namespace fastpack
}  // namespace kitty
