// The full-precision tokens of a unit -- the sink and the value q-buffer +
// local window (cache.py:196-208) -- in 32-token chunks on CUDA cores, shared
// by both decode-attention kernels.  The keys of those tokens come from the key
// sink, the key q-buffer, or (for the local window, whose keys are already
// packed) a key page dequantised from a shared-memory copy (Alg. 1,
// PAPER.md:425-446).  Lane = token for QK, lane = 4 channels for PV.  Every
// chunk writes one partial record (acc, m, l) like a page item does.
#pragma once

#include "kitty_common.cuh"

namespace kitty {
namespace fptok {

constexpr int D = 128;
constexpr int G = 128;
constexpr int kChunk = 32;
constexpr int kKeySlotMax = 5760;               // d_boost = 32
constexpr float kAlpha = 0.12751743074f;        // log2(e) / sqrt(128)

// scratch per warp: a key page, q * alpha and q * alpha * scale (f32, [D][GROUP])
// and the chunk's probabilities
template <int GROUP>
__host__ __device__ constexpr int scratch_bytes() {
    return (kKeySlotMax + 2 * GROUP * D * 4 + GROUP * kChunk * 4 + 127) / 128 * 128;
}

struct Geom {
    int n, kp, vp, nfp;
};
__device__ __forceinline__ Geom geom(const KittyCacheDesc& c, int u) {
    Geom g;
    g.n = c.unit_len[u];
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

// Chunk fc of unit u.  part: the workspace's partial records, `stride` floats
// each, nslot per unit; the chunk's record is slot fc.  All of the chunk's
// global loads (its value rows and this lane's key row) are issued before any
// of them is used, so a chunk costs one memory round trip, not five.
template <int GROUP>
__device__ void chunk(const KittyCacheDesc& c, const uint16_t* q, float* part, int nslot, int stride,
                      uint8_t* scratch, int u, int fc, int lane) {
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g, d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    uint8_t* kbuf = scratch;
    float* qf = reinterpret_cast<float*>(scratch + kKeySlotMax);                  // [D][GROUP] q * alpha
    float* bs = qf + D * GROUP;                                                    // [D][GROUP] q * alpha * s (paged keys)
    float* ps = bs + D * GROUP;                                                    // [GROUP][32]
    const Geom gm = geom(c, u);
    const int s_len = min(gm.n, S);
    const int c0 = fc * kChunk;
    const int cnt = min(kChunk, gm.nfp - c0);
    const int vbase = S + gm.vp * G;
    auto token_of = [&](int j) { return j < s_len ? j : vbase + (j - s_len); };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const uint16_t* qbase = q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D;
    const bool valid = lane < cnt;
    const int t = token_of(c0 + (valid ? lane : 0));
    const int pc = t - S;
    const bool in_page = t >= S && pc < gm.kp * G;
    // ---- loads, all in flight together ----
    uint2 qw[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) qw[g] = __ldg(reinterpret_cast<const uint2*>(qbase + g * D) + lane);
    const uint16_t* vsink = c.v_sink + (int64_t)u * S * D;
    const uint16_t* vr = c.v_ring + (int64_t)u * W * D;
    uint2 vv[kChunk];
#pragma unroll
    for (int jj = 0; jj < kChunk; ++jj) {
        const int tt = token_of(c0 + min(jj, cnt - 1));
        const uint16_t* vrow = tt < S ? vsink + (int64_t)tt * D : vr + (int64_t)((tt - S) % W) * D;
        vv[jj] = __ldg(reinterpret_cast<const uint2*>(vrow) + lane);
    }
    uint4 kw[16];
    {
        const uint16_t* krow = t < S ? c.k_sink + ((int64_t)u * S + t) * D : c.k_qbuf + ((int64_t)u * G + (pc % G)) * D;
#pragma unroll
        for (int i = 0; i < 16; ++i) kw[i] = in_page ? make_uint4(0u, 0u, 0u, 0u) : __ldg(reinterpret_cast<const uint4*>(krow) + i);
    }
    // q * alpha (f32, channel-major so one vector load serves every query)
#pragma unroll
    for (int g = 0; g < GROUP; ++g) {
        qf[(4 * lane + 0) * GROUP + g] = __uint_as_float(qw[g].x << 16) * kAlpha;
        qf[(4 * lane + 1) * GROUP + g] = __uint_as_float(qw[g].x & 0xffff0000u) * kAlpha;
        qf[(4 * lane + 2) * GROUP + g] = __uint_as_float(qw[g].y << 16) * kAlpha;
        qf[(4 * lane + 3) * GROUP + g] = __uint_as_float(qw[g].y & 0xffff0000u) * kAlpha;
    }
    __syncwarp();
    // q * alpha of channel d for every query, one shared-memory vector load
    auto qrow = [&](const float* arr, int d, float (&out)[GROUP]) {
        if (GROUP == 4) {
            const float4 v = *reinterpret_cast<const float4*>(arr + 4 * d);
            out[0] = v.x;
            out[1 % GROUP] = v.y;
            out[2 % GROUP] = v.z;
            out[3 % GROUP] = v.w;
        } else if (GROUP == 2) {
            const float2 v = *reinterpret_cast<const float2*>(arr + 2 * d);
            out[0] = v.x;
            out[1 % GROUP] = v.y;
        } else {
#pragma unroll
            for (int g = 0; g < GROUP; ++g) out[g] = arr[d * GROUP + g];
        }
    };
    // ---- QK ----
    float lg[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) lg[g] = 0.f;
    if (!in_page) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint4 w = kw[i];
            const float k8[8] = {__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                                 __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u),
                                 __uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u),
                                 __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u)};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                float qv[GROUP];
                qrow(qf, 8 * i + e, qv);
#pragma unroll
                for (int g = 0; g < GROUP; ++g) lg[g] = fmaf(qv[g], k8[e], lg[g]);
            }
        }
    }
    // keys that sit in key pages: stage each such page and dequantise its tokens
    unsigned need = __ballot_sync(0xffffffffu, valid && in_page);
    while (need) {
        const int src = __ffs(need) - 1;
        const int page = __shfl_sync(0xffffffffu, pc / G, src);
        const uint4* gsrc = reinterpret_cast<const uint4*>(c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + page] * kslot);
        uint4 tmp[12];
#pragma unroll
        for (int i = 0; i < 12; ++i)
            if (lane + 32 * i < kslot / 16) tmp[i] = gsrc[lane + 32 * i];
#pragma unroll
        for (int i = 0; i < 12; ++i)
            if (lane + 32 * i < kslot / 16) reinterpret_cast<uint4*>(kbuf)[lane + 32 * i] = tmp[i];
        __syncwarp();
        // scale fold: k = c s + z, so q.k = sum_d (q alpha s)_d c_d + sum_d (q alpha z)_d;
        // bs = q alpha s per channel, the zero-point sum once per page (lane-parallel)
        float zs[GROUP];
#pragma unroll
        for (int g = 0; g < GROUP; ++g) zs[g] = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int d = 4 * lane + k;
            const float s_ = half_bits_to_f32(ld_u16(kbuf + scale_off + 2 * d));
            const float z_ = half_bits_to_f32(ld_u16(kbuf + zero_off + 2 * d));
            float qv[GROUP];
            qrow(qf, d, qv);
#pragma unroll
            for (int g = 0; g < GROUP; ++g) {
                bs[d * GROUP + g] = qv[g] * s_;
                zs[g] = fmaf(qv[g], z_, zs[g]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int g = 0; g < GROUP; ++g) zs[g] += __shfl_xor_sync(0xffffffffu, zs[g], o);
        __syncwarp();
        const bool mine = valid && in_page && pc / G == page;
        if (mine) {
            const int tl = pc % G, sh = 2 * (tl & 3), byte = tl >> 2;
            const uint8_t* hb = kbuf + D * G / 4;
            const uint8_t* ib = kbuf + D * G / 4 + d_boost * G / 4;
            float acc[GROUP];
#pragma unroll
            for (int g = 0; g < GROUP; ++g) acc[g] = zs[g];
#pragma unroll 8
            for (int d = 0; d < D; ++d) {
                uint32_t code = (kbuf[d * (G / 4) + byte] >> sh) & 3u;
                const uint32_t r = ib[d];
                if (r != kSentinel) code |= ((hb[r * (G / 4) + byte] >> sh) & 3u) << 2;
                const float cf = static_cast<float>(code);
                float bv[GROUP];
                qrow(bs, d, bv);
#pragma unroll
                for (int g = 0; g < GROUP; ++g) acc[g] = fmaf(bv[g], cf, acc[g]);
            }
#pragma unroll
            for (int g = 0; g < GROUP; ++g) lg[g] += acc[g];
        }
        __syncwarp();
        need &= ~__ballot_sync(0xffffffffu, mine);
    }
    // ---- softmax of the chunk (log2 domain) ----
    float m[GROUP], l[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) {
        const float x = valid ? lg[g] : -INFINITY;
        float mc = x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        const float p = valid ? ex2f(x - mc) : 0.f;
        float s = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        m[g] = mc;
        l[g] = s;
        ps[g * kChunk + lane] = p;
    }
    __syncwarp();
    // ---- P V: lane owns channels 4 lane .. 4 lane + 3 ----
    float acc[GROUP][4];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
#pragma unroll
    for (int jj = 0; jj < kChunk; ++jj) {
        const float v0 = __uint_as_float(vv[jj].x << 16), v1 = __uint_as_float(vv[jj].x & 0xffff0000u);
        const float v2 = __uint_as_float(vv[jj].y << 16), v3 = __uint_as_float(vv[jj].y & 0xffff0000u);
#pragma unroll
        for (int g = 0; g < GROUP; ++g) {
            const float pg = ps[g * kChunk + jj];  // 0 for tokens past the chunk's count
            acc[g][0] = fmaf(pg, v0, acc[g][0]);
            acc[g][1] = fmaf(pg, v1, acc[g][1]);
            acc[g][2] = fmaf(pg, v2, acc[g][2]);
            acc[g][3] = fmaf(pg, v3, acc[g][3]);
        }
    }
    __syncwarp();
    float* base = part + ((int64_t)u * nslot + fc) * stride;
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

}  // namespace fptok
}  // namespace kitty

namespace kitty {
namespace fptok {

// The same chunk computed by a 128-thread CTA: the 32 tokens' dot products are
// split four ways over the channels (warp w: channels 32w .. 32w + 31, lane =
// token) and the P V sum four ways over the tokens (warp w: tokens 8w .. 8w + 7,
// lane = 4 channels), so one chunk's dependent chain is a quarter as long.
template <int GROUP>
__host__ __device__ constexpr int cta_scratch_bytes() {
    return kKeySlotMax + (4 * GROUP * kChunk + GROUP * kChunk + 4 * GROUP * D + GROUP * D * 2) * 4;
}

template <int GROUP>
__device__ void chunk_cta(const KittyCacheDesc& c, const uint16_t* q, float* part, int nslot, int stride,
                          uint8_t* scratch, int u, int fc) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = c.cfg.s, W = c.cfg.r + c.cfg.g, d_boost = c.cfg.d_boost;
    const int kslot = static_cast<int>(c.key_slot_bytes);
    const int scale_off = D * G / 4 + d_boost * G / 4 + D, zero_off = scale_off + 2 * D;
    uint8_t* kbuf = scratch;                                             // one key page
    float* plg = reinterpret_cast<float*>(scratch + kKeySlotMax);        // [4][GROUP][32] partial logits
    float* ps = plg + 4 * GROUP * kChunk;                                // [GROUP][32] probabilities
    float* pacc = ps + GROUP * kChunk;                                   // [4][GROUP][D] partial P V
    float* qf = pacc + 4 * GROUP * D;                                    // [D][GROUP] q alpha
    float* bs = qf + GROUP * D;                                          // [D][GROUP] q alpha s (paged keys)
    const Geom gm = geom(c, u);
    const int s_len = min(gm.n, S);
    const int c0 = fc * kChunk;
    const int cnt = min(kChunk, gm.nfp - c0);
    const int vbase = S + gm.vp * G;
    auto token_of = [&](int j) { return j < s_len ? j : vbase + (j - s_len); };
    const int b = u / c.cfg.h_kv, h = u - b * c.cfg.h_kv;
    const uint16_t* qbase = q + ((int64_t)b * c.cfg.h_q + (int64_t)h * GROUP) * D;
    // ---- loads: q (thread = channel), this thread's key quarter-row, its value rows ----
    const bool valid = lane < cnt;
    const int t = token_of(c0 + (valid ? lane : 0));
    const int pc = t - S;
    const bool in_page = t >= S && pc < gm.kp * G;
    float qv_own[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) qv_own[g] = bf16_to_f32(__ldg(qbase + g * D + tid)) * kAlpha;
    uint4 kw[4];
    {
        const uint16_t* krow = t < S ? c.k_sink + ((int64_t)u * S + t) * D : c.k_qbuf + ((int64_t)u * G + (pc % G)) * D;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            kw[i] = in_page ? make_uint4(0u, 0u, 0u, 0u) : __ldg(reinterpret_cast<const uint4*>(krow + 32 * warp) + i);
    }
    const uint16_t* vsink = c.v_sink + (int64_t)u * S * D;
    const uint16_t* vr = c.v_ring + (int64_t)u * W * D;
    uint2 vv[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int tt = token_of(c0 + min(8 * warp + jj, cnt - 1));
        const uint16_t* vrow = tt < S ? vsink + (int64_t)tt * D : vr + (int64_t)((tt - S) % W) * D;
        vv[jj] = __ldg(reinterpret_cast<const uint2*>(vrow) + lane);
    }
#pragma unroll
    for (int g = 0; g < GROUP; ++g) qf[tid * GROUP + g] = qv_own[g];
    __syncthreads();
    float lg[GROUP];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) lg[g] = 0.f;
    if (!in_page) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 w = kw[i];
            const float k8[8] = {__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                                 __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u),
                                 __uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u),
                                 __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u)};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int d = 32 * warp + 8 * i + e;
#pragma unroll
                for (int g = 0; g < GROUP; ++g) lg[g] = fmaf(qf[d * GROUP + g], k8[e], lg[g]);
            }
        }
    }
    // paged keys: the pages holding the chunk's tokens, lowest first
    int pg_lo = 0x7fffffff, pg_hi = -1;
    {
        // tokens of a chunk are consecutive: pages of the first / last paged token
        const int first_t = token_of(c0), last_t = token_of(c0 + cnt - 1);
        const int fpc = first_t - S, lpc = last_t - S;
        const bool fp_ = first_t >= S && fpc < gm.kp * G, lp_ = last_t >= S && lpc < gm.kp * G;
        if (fp_ || lp_) {
            pg_lo = fp_ ? fpc / G : (gm.kp - 1);
            pg_hi = lp_ ? lpc / G : (gm.kp - 1);
        }
    }
    for (int page = pg_lo; page <= pg_hi; ++page) {
        const uint4* gsrc = reinterpret_cast<const uint4*>(c.key_pool + (int64_t)c.key_block_table[(int64_t)u * c.max_pages + page] * kslot);
        for (int i = tid; i < kslot / 16; i += 128) reinterpret_cast<uint4*>(kbuf)[i] = gsrc[i];
        __syncthreads();
        {
            const int d = tid;  // scale fold for this page: bs = q alpha s
            const float s_ = half_bits_to_f32(ld_u16(kbuf + scale_off + 2 * d));
#pragma unroll
            for (int g = 0; g < GROUP; ++g) bs[d * GROUP + g] = qf[d * GROUP + g] * s_;
        }
        __syncthreads();
        if (valid && in_page && pc / G == page) {
            const int tl = pc % G, sh = 2 * (tl & 3), byte = tl >> 2;
            const uint8_t* hb = kbuf + D * G / 4;
            const uint8_t* ib = kbuf + D * G / 4 + d_boost * G / 4;
#pragma unroll 8
            for (int e = 0; e < 32; ++e) {
                const int d = 32 * warp + e;
                uint32_t code = (kbuf[d * (G / 4) + byte] >> sh) & 3u;
                const uint32_t r = ib[d];
                if (r != kSentinel) code |= ((hb[r * (G / 4) + byte] >> sh) & 3u) << 2;
                const float cf = static_cast<float>(code);
                const float z_ = half_bits_to_f32(ld_u16(kbuf + zero_off + 2 * d));
#pragma unroll
                for (int g = 0; g < GROUP; ++g) lg[g] = fmaf(bs[d * GROUP + g], cf, fmaf(qf[d * GROUP + g], z_, lg[g]));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int g = 0; g < GROUP; ++g) plg[(warp * GROUP + g) * kChunk + lane] = lg[g];
    __syncthreads();
    // ---- softmax (warp g < GROUP handles query g) ----
    float m_out = 0.f, l_out = 0.f;
    if (warp < GROUP) {
        const int g = warp;
        float x = plg[(0 * GROUP + g) * kChunk + lane] + plg[(1 * GROUP + g) * kChunk + lane] +
                  plg[(2 * GROUP + g) * kChunk + lane] + plg[(3 * GROUP + g) * kChunk + lane];
        x = valid ? x : -INFINITY;
        float mc = x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        const float p = valid ? ex2f(x - mc) : 0.f;
        float s = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        ps[g * kChunk + lane] = p;
        m_out = mc;
        l_out = s;
    }
    // GROUP 8: warps 0-3 handled queries 0-3; queries 4-7 in a second pass
    if (GROUP > 4) {
        __syncthreads();
        if (warp + 4 < GROUP) {
            const int g = warp + 4;
            float x = plg[(0 * GROUP + g) * kChunk + lane] + plg[(1 * GROUP + g) * kChunk + lane] +
                      plg[(2 * GROUP + g) * kChunk + lane] + plg[(3 * GROUP + g) * kChunk + lane];
            x = valid ? x : -INFINITY;
            float mc = x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
            const float p = valid ? ex2f(x - mc) : 0.f;
            float s = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            ps[g * kChunk + lane] = p;
            if (lane == 0) {
                float* base = part + ((int64_t)u * nslot + fc) * stride;
                base[GROUP * D + 2 * g] = mc;
                base[GROUP * D + 2 * g + 1] = s;
            }
        }
    }
    if (warp < GROUP && warp < 4 && lane == 0) {
        float* base = part + ((int64_t)u * nslot + fc) * stride;
        base[GROUP * D + 2 * warp] = m_out;
        base[GROUP * D + 2 * warp + 1] = l_out;
    }
    __syncthreads();
    // ---- P V: warp w sums tokens 8w .. 8w + 7, lane = channels 4 lane .. 4 lane + 3 ----
    float acc[GROUP][4];
#pragma unroll
    for (int g = 0; g < GROUP; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const float v0 = __uint_as_float(vv[jj].x << 16), v1 = __uint_as_float(vv[jj].x & 0xffff0000u);
        const float v2 = __uint_as_float(vv[jj].y << 16), v3 = __uint_as_float(vv[jj].y & 0xffff0000u);
#pragma unroll
        for (int g = 0; g < GROUP; ++g) {
            const float pg = ps[g * kChunk + 8 * warp + jj];
            acc[g][0] = fmaf(pg, v0, acc[g][0]);
            acc[g][1] = fmaf(pg, v1, acc[g][1]);
            acc[g][2] = fmaf(pg, v2, acc[g][2]);
            acc[g][3] = fmaf(pg, v3, acc[g][3]);
        }
    }
#pragma unroll
    for (int g = 0; g < GROUP; ++g)
        reinterpret_cast<float4*>(pacc + (warp * GROUP + g) * D)[lane] = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
    __syncthreads();
    float* base = part + ((int64_t)u * nslot + fc) * stride;
    for (int i = tid; i < GROUP * D; i += 128) {
        base[i] = pacc[i] + pacc[GROUP * D + i] + pacc[2 * GROUP * D + i] + pacc[3 * GROUP * D + i];
    }
}

}  // namespace fptok
}  // namespace kitty
