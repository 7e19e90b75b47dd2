// The full-precision tokens of a unit -- the sink and the value q-buffer +
// local window (cache.py:196-208) -- in 32-token chunks, one 128-thread CTA
// per chunk (fp_tokens_kernel).  The keys of those tokens come from the key
// sink, the key q-buffer, or (for the local window, whose keys are already
// packed) key pages dequantised from a shared-memory copy (Alg. 1,
// PAPER.md:425-446).  QK and PV run on mma.sync over f16 tiles.  Every chunk
// writes one partial record (acc, m, l) like a page item does.
//
// Range: the rows are staged as f16 (bf16 -> f16 is exact for
// 2^-14 <= |x| <= 65504; smaller magnitudes round to f16 subnormals), so a
// full-precision key or value row above 65504 in magnitude is outside this
// kernel's range (the reference accepts any finite f32).
#pragma once

#include "kitty_common.cuh"

namespace kitty {
namespace fptok {

constexpr int D = 128;
constexpr int G = 128;
constexpr int kChunk = 32;
constexpr int kKeySlotMax = 5760;               // d_boost = 32
constexpr float kAlpha = 0.12751743074f;        // log2(e) / sqrt(128)


struct Geom {
    int n, kp, vp, nfp;
};
__device__ __forceinline__ Geom geom(const KittyCacheDesc& c, int u, int max_tokens) {
    Geom g;
    g.n = min(c.unit_len[u], max_tokens);
    const int S = c.cfg.s;
    const int past = g.n > S ? g.n - S : 0;
    g.kp = past / G;
    g.vp = (past - min(c.cfg.r, past)) / G;
    g.nfp = g.n > S ? S + (past - g.vp * G) : g.n;  // sink + value fp tokens
    return g;
}

__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---- the chunk's key and value rows staged as f16 tiles, QK and PV on
// mma.sync.m16n8k16 with ldmatrix operands.  One 128-thread CTA per chunk. ----
constexpr int kRowH = D + 8;  // f16 per staged row (272 B: conflict-free ldmatrix)

// Scratch of one chunk CTA: the key page (key_slot_bytes, 16-aligned; the
// logits and P^T reuse it once the page is dequantised), the f16 key and
// value tiles and the page barrier -- ~22 KB at d_boost 16, so two chunk CTAs
// fit beside the page kernel's two CTAs on an SM.
__host__ __device__ inline int tc_kbuf_bytes(int kslot) { return (kslot + 127) & ~127; }
constexpr int kTileBytes = kChunk * kRowH * 2;  // one f16 row tile
// Union layout (un): when no chunk mixes staged and paged keys (S and R
// multiples of 32 at G = 128: every chunk is all-sink / all-q-buffer, or lies
// in one key page), the key page and the key tile share their bytes, and the
// boost inverse map sits after the value tile -- 17.6 instead of 22.8 KB, so
// more chunk CTAs are resident per SM.
__host__ __device__ inline int tc_front_bytes(int kslot, bool un) {
    return un ? (tc_kbuf_bytes(kslot) > kTileBytes ? tc_kbuf_bytes(kslot) : kTileBytes) : tc_kbuf_bytes(kslot) + kTileBytes;
}
__host__ __device__ inline int tc_scratch_bytes(int kslot, bool un = false) {
    return tc_front_bytes(kslot, un) + kTileBytes + (un ? 128 : 0) + 64;
}

__device__ __forceinline__ uint32_t f2h2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// 8 bf16 -> 8 f16 (exact for |x| in the f16 range)
__device__ __forceinline__ uint4 bf16x8_to_f16x8(uint4 w) {
    uint4 o;
    o.x = f2h2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u));
    o.y = f2h2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
    o.z = f2h2(__uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u));
    o.w = f2h2(__uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u));
    return o;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// the key page arrives by 1-D TMA on one mbarrier (one phase per page)
__device__ __forceinline__ void page_fetch(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void page_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "PW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra PW_%=;\n}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ uint32_t fprmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t fand_or(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t fhmul2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Logits of a chunk whose 32 keys all sit in one key page at a 16-token
// aligned offset (the local window at the default shapes): computed from the
// 2-bit codes like the page kernel does (PRMT + LOP3 -> f16 1024 + w c, the
// per-channel scale folded into B = q alpha s, offset and zero points from an
// auxiliary MMA, boosted rows as extra k-steps) instead of dequantising every
// key element.  Warp w covers channels [32 w, 32 w + 32) (k-steps 2w, 2w + 1)
// and boosted k-step w; lane gid's tokens are off0 + 4 gid + j, code j of one
// byte: j = 0 / 1 -> tile 0 rows gid / gid + 8 (w 256 / 4), j = 2 / 3 -> tile 1
// (w 16 / 64).  Writes the warp's partial logits lg[token][8] (columns = query).
template <int GROUP>
__device__ __forceinline__ void qk_from_codes(const uint8_t* kbuf, int d_boost, int off0, const uint16_t* qbase,
                                              const uint8_t* inv, float* lg) {
    constexpr bool kFull = GROUP == 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const bool main_col = kFull || gid < 4;
    const int qcol = kFull ? gid : (gid & 3);
    const bool qok = qcol < GROUP;
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    const uint32_t* kw = reinterpret_cast<const uint32_t*>(kbuf);
    const int wi = (off0 >> 4) + (gid >> 2);
    const uint32_t B = gid & 3;
    const uint32_t sel = B | (B << 4) | ((4 + B) << 8) | ((4 + B) << 12);
    const uint32_t m0 = 0x03000300u, m1 = 0x000C000Cu, m2 = 0x00300030u, m3 = 0x00C000C0u, magic = 0x64006400u;
    const uint32_t ones = 0x3C003C00u;
    const uint16_t* qg = qbase + (qok ? qcol : 0) * D;
    float acc[2][4] = {}, aux[4] = {}, aux2[4] = {};
    auto kstep = [&](const uint32_t* rows, int r0, uint32_t b0, uint32_t b1) {
        // rows r0, r0 + 1, r0 + 8, r0 + 9 of a 32-byte-row code array
        const uint32_t w0 = rows[8 * r0 + wi], w1 = rows[8 * (r0 + 1) + wi];
        const uint32_t w2 = rows[8 * (r0 + 8) + wi], w3 = rows[8 * (r0 + 9) + wi];
        const uint32_t x = fprmt(w0, w1, sel), y = fprmt(w2, w3, sel);
        hmma(acc[0], fand_or(x, m0, magic), fand_or(x, m1, magic), fand_or(y, m0, magic), fand_or(y, m1, magic), b0, b1);
        hmma(acc[1], fand_or(x, m2, magic), fand_or(x, m3, magic), fand_or(y, m2, magic), fand_or(y, m3, magic), b0, b1);
    };
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
        const int c0 = 16 * (2 * warp + k2) + 2 * tig;
        uint32_t qa0 = 0u, qa1 = 0u;
        if (qok) {
            const uint32_t u0 = __ldg(reinterpret_cast<const uint32_t*>(qg + c0));
            const uint32_t u1 = __ldg(reinterpret_cast<const uint32_t*>(qg + c0 + 8));
            qa0 = f2h2(__uint_as_float(u0 << 16) * kAlpha, __uint_as_float(u0 & 0xffff0000u) * kAlpha);
            qa1 = f2h2(__uint_as_float(u1 << 16) * kAlpha, __uint_as_float(u1 & 0xffff0000u) * kAlpha);
        }
        // B columns 0..group-1: q alpha s; group <= 4: columns 4-7 carry q alpha (aux sums)
        const uint32_t s0 = main_col ? *reinterpret_cast<const uint32_t*>(kbuf + scale_off + 2 * c0) : ones;
        const uint32_t s1 = main_col ? *reinterpret_cast<const uint32_t*>(kbuf + scale_off + 2 * (c0 + 8)) : ones;
        const uint32_t b0 = fhmul2(qa0, s0), b1 = fhmul2(qa1, s1);
        const uint32_t z0 = *reinterpret_cast<const uint32_t*>(kbuf + zero_off + 2 * c0);
        const uint32_t z1 = *reinterpret_cast<const uint32_t*>(kbuf + zero_off + 2 * (c0 + 8));
        kstep(kw, c0, b0, b1);
        hmma(aux, ones, z0, ones, z1, b0, b1);  // row 0: sum B; row 8: sum z B
        if (kFull) hmma(aux2, ones, z0, ones, z1, qa0, qa1);
    }
    // boosted rows: warp w takes high-bit rows [16 w, 16 w + 16)
    if (16 * warp < d_boost) {
        const int j0 = 16 * warp + 2 * tig;
        auto qs = [&](int j) -> uint32_t {  // 4 q alpha s of the channel row j boosts (f16 bits), 0 past d_boost
            if (j >= d_boost || !main_col || !qok) return 0u;
            const int ch = inv[j];
            const float qv = __uint_as_float(static_cast<uint32_t>(qg[ch]) << 16) * (4.f * kAlpha);
            const uint16_t sv = *reinterpret_cast<const uint16_t*>(kbuf + scale_off + 2 * ch);
            return __half_as_ushort(__hmul(__float2half_rn(qv), __ushort_as_half(sv)));
        };
        const uint32_t b0 = qs(j0) | (qs(j0 + 1) << 16), b1 = qs(j0 + 8) | (qs(j0 + 9) << 16);
        kstep(kw + (D * G / 4) / 4, j0, b0, b1);
        hmma(aux, ones, 0u, ones, 0u, b0, b1);
    }
    // corrections per column: L = acc / w - (1024 / w) sum B + sum z q alpha
    float sumB[2], cst[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        sumB[j] = __shfl_sync(0xffffffffu, aux[j], kFull ? tig : (tig & 1));
        cst[j] = kFull ? __shfl_sync(0xffffffffu, aux2[2 + j], tig) : __shfl_sync(0xffffffffu, aux[2 + j], 2 + (tig & 1));
    }
    __syncthreads();  // every warp is done reading the page: the logits reuse its bytes
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int g = 2 * tig + j;
        if (g < GROUP && (kFull || tig < 2)) {
            // tile t, row gid + 8 h: code 2 t + h of byte gid -> token 4 gid + 2 t + h
            lg[(4 * gid + 0) * 8 + g] = fmaf(acc[0][j], 1.f / 256.f, cst[j] - 4.f * sumB[j]);
            lg[(4 * gid + 1) * 8 + g] = fmaf(acc[0][2 + j], 1.f / 4.f, cst[j] - 256.f * sumB[j]);
            lg[(4 * gid + 2) * 8 + g] = fmaf(acc[1][j], 1.f / 16.f, cst[j] - 64.f * sumB[j]);
            lg[(4 * gid + 3) * 8 + g] = fmaf(acc[1][2 + j], 1.f / 64.f, cst[j] - 16.f * sumB[j]);
        }
    }
}

template <int GROUP>
__device__ void chunk_tc(const KittyCacheDesc& c, const uint16_t* q, float* part, int nslot, int stride,
                         uint8_t* scratch, int u, int fc, int max_tokens, bool un) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g, d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    uint8_t* kbuf = scratch;
    uint16_t* kt = reinterpret_cast<uint16_t*>(scratch + (un ? 0 : tc_kbuf_bytes(kslot)));  // [32][kRowH] f16 keys
    uint16_t* vt = reinterpret_cast<uint16_t*>(scratch + tc_front_bytes(kslot, un));       // [32][kRowH] f16 values
    uint8_t* inv_buf = un ? reinterpret_cast<uint8_t*>(vt + kChunk * kRowH) : reinterpret_cast<uint8_t*>(kt);
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(vt + kChunk * kRowH) + (un ? 128 : 0));
    // after the dequantisation (a __syncthreads) the key page is dead: logits
    // and P^T live in its bytes (4.5 KB <= the slot)
    float* lgs = reinterpret_cast<float*>(kbuf);                   // [4][32][8] partial logits
    uint16_t* pT = reinterpret_cast<uint16_t*>(lgs + 4 * kChunk * 8);  // [8][32] f16 probabilities
    const Geom gm = geom(c, u, max_tokens);
    const int s_len = min(gm.n, S);
    const int c0 = fc * kChunk;
    const int cnt = min(kChunk, gm.nfp - c0);
    const int vbase = S + gm.vp * G;
    auto token_of = [&](int j) { return j < s_len ? j : vbase + (j - s_len); };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const uint16_t* qbase = q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D;
    // key pages the chunk's tokens sit in (the local window): [pg_lo, pg_hi]
    // chunk index j >= s_len is cache position vbase - S + (j - s_len); the
    // chunk's paged tokens are its post-sink positions below kp * G
    int pg_lo = 1, pg_hi = 0;
    {
        const int j0 = max(c0, s_len), j1 = c0 + cnt - 1;
        const int pc0 = vbase - S + (j0 - s_len), pc1 = vbase - S + (j1 - s_len);
        if (j0 <= j1 && pc0 < gm.kp * G) {
            pg_lo = pc0 / G;
            pg_hi = min(pc1, gm.kp * G - 1) / G;
        }
    }
    auto page_src = [&](int page) { return c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + page] * kslot; };
    // ---- issue every global load first: the page (TMA), the rows, q ----
    if (tid == 0 && pg_lo <= pg_hi) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        page_fetch(kbuf, page_src(pg_lo), kslot, bar);
    }
    const int tk = tid >> 2, qq = tid & 3;
    const int tt = token_of(c0 + min(tk, cnt - 1));
    const int pct = tt - S;
    const bool paged = tt >= S && pct < gm.kp * G;
    uint4 kw[4], vw[4];
    {
        // bf16 rows (the fused path runs for row_dtype KITTY_BF16 only)
        const uint16_t* ksink = static_cast<const uint16_t*>(c.k_sink);
        const uint16_t* vsink = static_cast<const uint16_t*>(c.v_sink);
        const uint16_t* krow = tt < S ? ksink + ((int64_t)u * S + tt) * D : static_cast<const uint16_t*>(c.k_qbuf) + ((int64_t)u * G + (pct % G)) * D;
        const uint16_t* vrow = tt < S ? vsink + ((int64_t)u * S + tt) * D : static_cast<const uint16_t*>(c.v_ring) + ((int64_t)u * W + (pct % W)) * D;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!paged) kw[i] = __ldg(reinterpret_cast<const uint4*>(krow + 32 * qq) + i);
            vw[i] = __ldg(reinterpret_cast<const uint4*>(vrow + 32 * qq) + i);
        }
    }
    // QK split: warp w -> tokens 16 (w & 1) .., k-steps 4 (w >> 1) .. + 3
    const int mrow = warp & 1, khalf = warp >> 1;
    uint32_t qw[8];
    {
        const uint16_t* qg = qbase + (gid < GROUP ? gid : 0) * D;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ch = 16 * (4 * khalf + k) + 2 * tig;
            qw[2 * k] = __ldg(reinterpret_cast<const uint32_t*>(qg + ch));
            qw[2 * k + 1] = __ldg(reinterpret_cast<const uint32_t*>(qg + ch + 8));
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!paged) reinterpret_cast<uint4*>(kt + tk * kRowH + 32 * qq)[i] = bf16x8_to_f16x8(kw[i]);
        reinterpret_cast<uint4*>(vt + tk * kRowH + 32 * qq)[i] = bf16x8_to_f16x8(vw[i]);
    }
    // a chunk whose keys all sit in one key page at a 16-token aligned offset
    // (the local window at the default shapes): logits straight from the codes
    int npart = 2;
    {
        const int pbase = vbase - S + c0 - s_len;
        const int off0 = pbase - pg_lo * G;
        if (pg_lo == pg_hi && c0 >= s_len && pbase + cnt - 1 < gm.kp * G && (off0 & 15) == 0 && off0 + kChunk <= G) {
            uint8_t* inv = inv_buf;  // the key tile is not needed (or shares the page's bytes)
            if (tid == 0) page_wait(bar, 0);
            __syncthreads();
            if (tid < D) {
                const uint8_t bi = kbuf[D * G / 4 + d_boost * G / 4 + tid];
                if (bi < 32) inv[bi] = static_cast<uint8_t>(tid);
            }
            __syncthreads();
            qk_from_codes<GROUP>(kbuf, d_boost, off0, qbase, inv, lgs + warp * kChunk * 8);
            npart = 4;
            pg_hi = pg_lo - 1;  // no dequantisation below
        }
    }
    // keys that sit in key pages: dequantise into the tile.  thread = (channel
    // pair cp, token half th); the half's codes come from one shifted 64-bit
    // window of each channel's code row (16 tokens = 32 bits)
    if (pg_lo <= pg_hi) {
        const int cp = tid & 63, th = tid >> 6, d0 = 2 * cp;
        // chunk token j >= s_len - c0 sits at cache position pct = pbase + j
        const int jpost = max(0, s_len - c0), pbase = vbase - S + c0 - s_len;
        for (int page = pg_lo; page <= pg_hi; ++page) {
            if (page > pg_lo) {
                __syncthreads();  // kbuf reuse
                if (tid == 0) page_fetch(kbuf, page_src(page), kslot, bar);
            }
            if (tid == 0) page_wait(bar, (page - pg_lo) & 1);
            __syncthreads();
            // this half's tokens on this page: j in [jlo, jhi]
            const int lo_pc = page * G, hi_pc = min(page * G + G, gm.kp * G) - 1;
            const int jlo = max(max(16 * th, jpost), lo_pc - pbase);
            const int jhi = min(min(16 * th + 15, cnt - 1), hi_pc - pbase);
            if (jlo > jhi) continue;
            const int w = pbase + jlo - lo_pc;  // page-local token of jlo
            const int word = w >> 4, off = w & 15;
            const uint32_t sc2 = *reinterpret_cast<const uint32_t*>(kbuf + scale_off + 2 * d0);
            const uint32_t zr2 = *reinterpret_cast<const uint32_t*>(kbuf + zero_off + 2 * d0);
            const uint16_t ix2 = *reinterpret_cast<const uint16_t*>(kbuf + D * G / 4 + d_boost * G / 4 + d0);
            float sc[2], zr[2];
            uint32_t lo[2], hi[2];
#pragma unroll
            for (int k2 = 0; k2 < 2; ++k2) {
                sc[k2] = half_bits_to_f32(static_cast<uint16_t>(sc2 >> (16 * k2)));
                zr[k2] = half_bits_to_f32(static_cast<uint16_t>(zr2 >> (16 * k2)));
                const uint32_t* row = reinterpret_cast<const uint32_t*>(kbuf + (d0 + k2) * (G / 4)) + word;
                lo[k2] = static_cast<uint32_t>(((static_cast<uint64_t>(row[1]) << 32) | row[0]) >> (2 * off));
                const uint32_t r = (ix2 >> (8 * k2)) & 0xffu;
                hi[k2] = 0u;
                if (r != kSentinel) {
                    const uint32_t* hrow = reinterpret_cast<const uint32_t*>(kbuf + D * G / 4 + r * (G / 4)) + word;
                    hi[k2] = static_cast<uint32_t>(((static_cast<uint64_t>(hrow[1]) << 32) | hrow[0]) >> (2 * off));
                }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (jlo + i <= jhi) {
                    float kv[2];
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        const uint32_t code = ((lo[k2] >> (2 * i)) & 3u) | (((hi[k2] >> (2 * i)) & 3u) << 2);
                        // Alg. 1: code * scale + zero (the value the reference attends to)
                        kv[k2] = __fadd_rn(__fmul_rn(__uint_as_float(code | 0x4b000000u) - 8388608.f, sc[k2]), zr[k2]);
                    }
                    *reinterpret_cast<uint32_t*>(kt + (jlo + i) * kRowH + d0) = f2h2(kv[0], kv[1]);
                }
            }
        }
    }
    __syncthreads();
    const uint32_t kt_s = static_cast<uint32_t>(__cvta_generic_to_shared(kt));
    const uint32_t vt_s = static_cast<uint32_t>(__cvta_generic_to_shared(vt));
    // ---- QK: N = 8 query columns (q alpha as f16 B fragments) ----
    if (npart == 2) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const int i4 = lane >> 3, r8 = lane & 7;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w0 = qw[2 * k], w1 = qw[2 * k + 1];
            const uint32_t b0 = gid < GROUP ? f2h2(__uint_as_float(w0 << 16) * kAlpha, __uint_as_float(w0 & 0xffff0000u) * kAlpha) : 0u;
            const uint32_t b1 = gid < GROUP ? f2h2(__uint_as_float(w1 << 16) * kAlpha, __uint_as_float(w1 & 0xffff0000u) * kAlpha) : 0u;
            uint32_t a0, a1, a2, a3;
            const int row = 16 * mrow + r8 + 8 * (i4 & 1), cc = 16 * (4 * khalf + k) + 8 * (i4 >> 1);
            ldsm_x4(kt_s + 2 * (row * kRowH + cc), a0, a1, a2, a3);
            hmma(acc, a0, a1, a2, a3, b0, b1);
        }
        // acc: rows (tokens) 16 mrow + gid / + 8, columns 2 tig, 2 tig + 1
        if (un) __syncthreads();  // the logits overwrite the key tile every warp was reading
        float* lg = lgs + khalf * kChunk * 8;
        *reinterpret_cast<float2*>(lg + (16 * mrow + gid) * 8 + 2 * tig) = make_float2(acc[0], acc[1]);
        *reinterpret_cast<float2*>(lg + (16 * mrow + 8 + gid) * 8 + 2 * tig) = make_float2(acc[2], acc[3]);
    }
    __syncthreads();
    // ---- softmax of the chunk, one warp per query (two passes for group 8) ----
    const bool valid = lane < cnt;
#pragma unroll
    for (int pass = 0; pass < (GROUP + 3) / 4; ++pass) {
        const int g = 4 * pass + warp;
        if (g < GROUP) {
            float x = lgs[lane * 8 + g] + lgs[kChunk * 8 + lane * 8 + g];
            if (npart == 4) x += lgs[2 * kChunk * 8 + lane * 8 + g] + lgs[3 * kChunk * 8 + lane * 8 + g];
            x = valid ? x : -INFINITY;
            float mc = x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
            const float p = valid ? ex2f(x - mc) : 0.f;
            float s = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            pT[g * kChunk + lane] = __half_as_ushort(__float2half_rn(p));
            if (lane == 0) {
                float* base = part + ((int64_t)u * nslot + fc) * stride;
                base[GROUP * D + 2 * g] = mc;
                base[GROUP * D + 2 * g + 1] = s;
            }
        } else if (g < 8) {
            pT[g * kChunk + lane] = 0;
        }
    }
    __syncthreads();
    // ---- PV: warp w -> channels 32 w .. 32 w + 31 (two M tiles), K = 32 tokens ----
    {
        float acc[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
        const int i4 = lane >> 3, r8 = lane & 7;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            // B = P [token][query]: b0 = (tokens 16 ks + 2 tig, + 1; query gid)
            const uint32_t b0 = *reinterpret_cast<const uint32_t*>(pT + gid * kChunk + 16 * ks + 2 * tig);
            const uint32_t b1 = *reinterpret_cast<const uint32_t*>(pT + gid * kChunk + 16 * ks + 8 + 2 * tig);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                uint32_t a0, a1, a2, a3;
                // A = V^T [channel][token] via transposed 8x8 loads of V [token][channel]
                const int tok = 16 * ks + r8 + 8 * (i4 >> 1), chn = 32 * warp + 16 * mt + 8 * (i4 & 1);
                ldsm_x4_t(vt_s + 2 * (tok * kRowH + chn), a0, a1, a2, a3);
                hmma(acc[mt], a0, a1, a2, a3, b0, b1);
            }
        }
        float* base = part + ((int64_t)u * nslot + fc) * stride;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int ch = 32 * warp + 16 * mt + gid;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int g = 2 * tig + j;
                if (g < GROUP) {
                    base[g * D + ch] = acc[mt][j];
                    base[g * D + ch + 8] = acc[mt][2 + j];
                }
            }
        }
    }
}

// ---- one warp per 32-token chunk (the aligned geometries: no chunk mixes
// staged and paged keys, i.e. S a multiple of 32) ----------------------------
// Every lane fetches its token's bf16 K row (sink / key q-buffer chunks) and
// V row straight into a padded shared tile with its own 1-D bulk copies (no
// register staging, no conversion); QK runs as a bf16 MMA (q and K exact,
// the 1 / sqrt(d) log2(e) scale applied to the fp32 logits), or from the 2-bit
// codes for a chunk inside one key page (qk_codes_warp); the softmax keeps p
// as a bf16 hi + lo pair so that P V runs as two bf16 MMAs at ~16-bit
// precision.  No CTA-wide barrier: a chunk is one warp's work.
__host__ __device__ inline int cw_front_bytes(int kslot) {
    const int a = tc_kbuf_bytes(kslot) + 128;  // key page + boost inverse map
    return ((a > kTileBytes ? a : kTileBytes) + 127) & ~127;
}
__host__ __device__ inline int cw_warp_bytes(int kslot) {
    // front (key page | key tile; then the logits [32][8] f32 and P^T hi / lo
    // [8][40] bf16 in its first 2.3 KB once QK has read it), value tile, barrier
    return cw_front_bytes(kslot) + kTileBytes + 64;
}

__device__ __forceinline__ void hmma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

// Logits of a chunk inside one key page from its 2-bit codes, all 128
// channels by one warp (qk_from_codes' arithmetic: f16 1024 + w c operands,
// B = q alpha s, offsets and zero points from the auxiliary MMA, boosted rows
// as extra k-steps); lane gid's tokens are off0 + 4 gid + j.  Full logits to
// lg[token][8].
template <int GROUP>
__device__ __forceinline__ void qk_codes_warp(const uint8_t* kbuf, int d_boost, int off0, const uint16_t* qbase,
                                              const uint8_t* inv, float* lg) {
    constexpr bool kFull = GROUP == 8;
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const bool main_col = kFull || gid < 4;
    const int qcol = kFull ? gid : (gid & 3);
    const bool qok = qcol < GROUP;
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    const uint32_t* kw = reinterpret_cast<const uint32_t*>(kbuf);
    const int wi = (off0 >> 4) + (gid >> 2);
    const uint32_t B = gid & 3;
    const uint32_t sel = B | (B << 4) | ((4 + B) << 8) | ((4 + B) << 12);
    const uint32_t m0 = 0x03000300u, m1 = 0x000C000Cu, m2 = 0x00300030u, m3 = 0x00C000C0u, magic = 0x64006400u;
    const uint32_t ones = 0x3C003C00u;
    const uint16_t* qg = qbase + (qok ? qcol : 0) * D;
    float acc[2][4] = {}, aux[4] = {}, aux2[4] = {};
    auto kstep = [&](const uint32_t* rows, int r0, uint32_t b0, uint32_t b1) {
        const uint32_t w0 = rows[8 * r0 + wi], w1 = rows[8 * (r0 + 1) + wi];
        const uint32_t w2 = rows[8 * (r0 + 8) + wi], w3 = rows[8 * (r0 + 9) + wi];
        const uint32_t x = fprmt(w0, w1, sel), y = fprmt(w2, w3, sel);
        hmma(acc[0], fand_or(x, m0, magic), fand_or(x, m1, magic), fand_or(y, m0, magic), fand_or(y, m1, magic), b0, b1);
        hmma(acc[1], fand_or(x, m2, magic), fand_or(x, m3, magic), fand_or(y, m2, magic), fand_or(y, m3, magic), b0, b1);
    };
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        const int c0 = 16 * ks + 2 * tig;
        uint32_t qa0 = 0u, qa1 = 0u;
        if (qok) {
            const uint32_t u0 = __ldg(reinterpret_cast<const uint32_t*>(qg + c0));
            const uint32_t u1 = __ldg(reinterpret_cast<const uint32_t*>(qg + c0 + 8));
            qa0 = f2h2(__uint_as_float(u0 << 16) * kAlpha, __uint_as_float(u0 & 0xffff0000u) * kAlpha);
            qa1 = f2h2(__uint_as_float(u1 << 16) * kAlpha, __uint_as_float(u1 & 0xffff0000u) * kAlpha);
        }
        const uint32_t s0 = main_col ? *reinterpret_cast<const uint32_t*>(kbuf + scale_off + 2 * c0) : ones;
        const uint32_t s1 = main_col ? *reinterpret_cast<const uint32_t*>(kbuf + scale_off + 2 * (c0 + 8)) : ones;
        const uint32_t b0 = fhmul2(qa0, s0), b1 = fhmul2(qa1, s1);
        const uint32_t z0 = *reinterpret_cast<const uint32_t*>(kbuf + zero_off + 2 * c0);
        const uint32_t z1 = *reinterpret_cast<const uint32_t*>(kbuf + zero_off + 2 * (c0 + 8));
        kstep(kw, c0, b0, b1);
        hmma(aux, ones, z0, ones, z1, b0, b1);
        if (kFull) hmma(aux2, ones, z0, ones, z1, qa0, qa1);
    }
    for (int hk = 0; 16 * hk < d_boost; ++hk) {  // boosted rows [16 hk, 16 hk + 16)
        const int j0 = 16 * hk + 2 * tig;
        auto qs = [&](int j) -> uint32_t {
            if (j >= d_boost || !main_col || !qok) return 0u;
            const int ch = inv[j];
            const float qv = __uint_as_float(static_cast<uint32_t>(qg[ch]) << 16) * (4.f * kAlpha);
            const uint16_t sv = *reinterpret_cast<const uint16_t*>(kbuf + scale_off + 2 * ch);
            return __half_as_ushort(__hmul(__float2half_rn(qv), __ushort_as_half(sv)));
        };
        const uint32_t b0 = qs(j0) | (qs(j0 + 1) << 16), b1 = qs(j0 + 8) | (qs(j0 + 9) << 16);
        kstep(kw + (D * G / 4) / 4, j0, b0, b1);
        hmma(aux, ones, 0u, ones, 0u, b0, b1);
    }
    float sumB[2], cst[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        sumB[j] = __shfl_sync(0xffffffffu, aux[j], kFull ? tig : (tig & 1));
        cst[j] = kFull ? __shfl_sync(0xffffffffu, aux2[2 + j], tig) : __shfl_sync(0xffffffffu, aux[2 + j], 2 + (tig & 1));
    }
    __syncwarp();  // every lane is done reading the page (the logits may take its bytes)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int g = 2 * tig + j;
        if (g < GROUP && (kFull || tig < 2)) {
            lg[(4 * gid + 0) * 8 + g] = fmaf(acc[0][j], 1.f / 256.f, cst[j] - 4.f * sumB[j]);
            lg[(4 * gid + 1) * 8 + g] = fmaf(acc[0][2 + j], 1.f / 4.f, cst[j] - 256.f * sumB[j]);
            lg[(4 * gid + 2) * 8 + g] = fmaf(acc[1][j], 1.f / 16.f, cst[j] - 64.f * sumB[j]);
            lg[(4 * gid + 3) * 8 + g] = fmaf(acc[1][2 + j], 1.f / 64.f, cst[j] - 16.f * sumB[j]);
        }
    }
}

template <int GROUP>
__device__ void chunk_warp(const KittyCacheDesc& c, const uint16_t* q, float* part, int nslot, int stride,
                           uint8_t* scratch, int u, int fc, int max_tokens) {
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g, d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    uint8_t* kbuf = scratch;
    uint16_t* kt = reinterpret_cast<uint16_t*>(scratch);  // [32][kRowH] bf16 keys (shares the page's bytes)
    uint8_t* inv = scratch + tc_kbuf_bytes(kslot);
    uint16_t* vt = reinterpret_cast<uint16_t*>(scratch + cw_front_bytes(kslot));  // [32][kRowH] bf16 values
    float* lg = reinterpret_cast<float*>(scratch);                 // [32][8] logits (after QK: over the keys)
    uint16_t* pth = reinterpret_cast<uint16_t*>(lg + kChunk * 8);  // [8][40] bf16 p hi
    uint16_t* ptl = pth + 8 * 40;                                  // [8][40] bf16 p lo
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(vt + kChunk * kRowH));
    const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    const Geom gm = geom(c, u, max_tokens);
    const int s_len = min(gm.n, S);
    const int c0 = fc * kChunk;
    const int cnt = min(kChunk, gm.nfp - c0);
    const int vbase = S + gm.vp * G;
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const uint16_t* qbase = q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D;
    // this chunk: all sink / key q-buffer tokens, or all inside key page pg
    const int pbase = vbase - S + c0 - s_len;  // cache position of chunk token 0 (when c0 >= s_len)
    const bool coded = c0 >= s_len && pbase < gm.kp * G;
    const int pg = coded ? pbase / G : 0, off0 = pbase - pg * G;
    // ---- every load in flight at once: the page (lane 0), each lane's rows ----
    const bool valid = lane < cnt;
    const int tt = valid ? (c0 + lane < s_len ? c0 + lane : vbase + (c0 + lane - s_len)) : 0;
    const int pct = tt - S;
    const uint32_t bytes = (coded ? kslot : 0) + cnt * (coded ? 256 : 512);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(bytes) : "memory");
        if (coded)
            bulk_row(kbuf, c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + pg] * kslot, kslot, bar);
    }
    __syncwarp();
    if (valid) {
        const uint16_t* ksink = static_cast<const uint16_t*>(c.k_sink);
        const uint16_t* vsink = static_cast<const uint16_t*>(c.v_sink);
        const uint16_t* vrow = tt < S ? vsink + ((int64_t)u * S + tt) * D : static_cast<const uint16_t*>(c.v_ring) + ((int64_t)u * W + (pct % W)) * D;
        bulk_row(vt + lane * kRowH, vrow, 256, bar);
        if (!coded) {
            const uint16_t* krow = tt < S ? ksink + ((int64_t)u * S + tt) * D : static_cast<const uint16_t*>(c.k_qbuf) + ((int64_t)u * G + (pct % G)) * D;
            bulk_row(kt + lane * kRowH, krow, 256, bar);
        }
    } else {  // rows past the chunk's tokens: zero values (their p is 0, but 0 x NaN is not)
        uint4* vz = reinterpret_cast<uint4*>(vt + lane * kRowH);
#pragma unroll
        for (int i = 0; i < 16; ++i) vz[i] = make_uint4(0u, 0u, 0u, 0u);
        if (!coded) {
            uint4* kz = reinterpret_cast<uint4*>(kt + lane * kRowH);
#pragma unroll
            for (int i = 0; i < 16; ++i) kz[i] = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    // B fragments of q (bf16 pairs, exact), while the rows are in flight
    uint32_t qb[8][2];
    if (!coded) {
        const uint16_t* qg = qbase + (gid < GROUP ? gid : 0) * D;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int ch = 16 * ks + 2 * tig;
            qb[ks][0] = gid < GROUP ? __ldg(reinterpret_cast<const uint32_t*>(qg + ch)) : 0u;
            qb[ks][1] = gid < GROUP ? __ldg(reinterpret_cast<const uint32_t*>(qg + ch + 8)) : 0u;
        }
    }
    page_wait(bar, 0);
    __syncwarp();
    // ---- logits lg[token][query] (log2 domain) ----
    if (coded) {
        {
            const uint32_t bw = *reinterpret_cast<const uint32_t*>(kbuf + D * G / 4 + d_boost * G / 4 + 4 * lane);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t bi = (bw >> (8 * k)) & 0xffu;
                if (bi < 32u) inv[bi] = static_cast<uint8_t>(4 * lane + k);
            }
        }
        __syncwarp();
        qk_codes_warp<GROUP>(kbuf, d_boost, off0, qbase, inv, lg);  // lg is written after every read of the page
    } else {
        const uint32_t kt_s = static_cast<uint32_t>(__cvta_generic_to_shared(kt));
        const int i4 = lane >> 3, r8 = lane & 7;
        float acc[2][4] = {};
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                uint32_t a0, a1, a2, a3;
                const int row = 16 * mt + r8 + 8 * (i4 & 1), cc = 16 * ks + 8 * (i4 >> 1);
                ldsm_x4(kt_s + 2 * (row * kRowH + cc), a0, a1, a2, a3);
                hmma_bf16(acc[mt], a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
            }
        }
        __syncwarp();  // every lane's key-tile reads are done: the logits take those bytes
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            *reinterpret_cast<float2*>(lg + (16 * mt + gid) * 8 + 2 * tig) = make_float2(acc[mt][0] * kAlpha, acc[mt][1] * kAlpha);
            *reinterpret_cast<float2*>(lg + (16 * mt + 8 + gid) * 8 + 2 * tig) = make_float2(acc[mt][2] * kAlpha, acc[mt][3] * kAlpha);
        }
    }
    __syncwarp();
    // ---- softmax over the chunk's tokens (lane = token), one query at a time ----
    float* base = part + ((int64_t)u * nslot + fc) * stride;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        if (g < GROUP) {
            const float x = valid ? lg[lane * 8 + g] : -INFINITY;
            float mc = x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
            const float p = valid ? ex2f(x - mc) : 0.f;
            float sm = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
            const __nv_bfloat16 ph = __float2bfloat16_rn(p);
            const __nv_bfloat16 pl = __float2bfloat16_rn(p - __bfloat162float(ph));
            pth[g * 40 + lane] = __bfloat16_as_ushort(ph);
            ptl[g * 40 + lane] = __bfloat16_as_ushort(pl);
            if (lane == 0) {
                base[GROUP * D + 2 * g] = mc;
                base[GROUP * D + 2 * g + 1] = sm;
            }
        } else {
            pth[g * 40 + lane] = 0;
            ptl[g * 40 + lane] = 0;
        }
    }
    __syncwarp();
    // ---- P V: out^T [channel][query], A = V^T (ldmatrix.trans), B = p hi / lo ----
    {
        const uint32_t vt_s = static_cast<uint32_t>(__cvta_generic_to_shared(vt));
        const int i4 = lane >> 3, r8 = lane & 7;
        float acc[8][4] = {};
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(pth + gid * 40 + 16 * ks + 2 * tig);
            const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(pth + gid * 40 + 16 * ks + 8 + 2 * tig);
            const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(ptl + gid * 40 + 16 * ks + 2 * tig);
            const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(ptl + gid * 40 + 16 * ks + 8 + 2 * tig);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                const int tok = 16 * ks + r8 + 8 * (i4 >> 1), chn = 16 * mt + 8 * (i4 & 1);
                ldsm_x4_t(vt_s + 2 * (tok * kRowH + chn), a0, a1, a2, a3);
                hmma_bf16(acc[mt], a0, a1, a2, a3, bh0, bh1);
                hmma_bf16(acc[mt], a0, a1, a2, a3, bl0, bl1);
            }
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            const int ch = 16 * mt + gid;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int g = 2 * tig + j;
                if (g < GROUP) {
                    base[g * D + ch] = acc[mt][j];
                    base[g * D + ch + 8] = acc[mt][2 + j];
                }
            }
        }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar_s) : "memory");
}

}  // namespace fptok
}  // namespace kitty
