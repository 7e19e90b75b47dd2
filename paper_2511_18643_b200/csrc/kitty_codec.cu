// Page codec and cache-runtime kernels: quantize + pack (K1/K2), dequantize
// (K6), append with the fused pack trigger (K3) and bulk prefill.
//
// Bit-exactness: channel scores are a sequential fp64
// sum in token order (quant.py:72); the quantizer uses IEEE float32 division
// and round-half-even (quant.py:112-114); dequantisation is multiply-then-add
// with no FMA contraction (quant.py:120, pages.py:143); f16 metadata is RNE.
#include <cstdlib>

#include "kitty_codec.cuh"
#include "kitty_pack_fast.cuh"

namespace kitty {

// ---------------------------------------------------------------------------
// Block-level page packers.  `tile` holds the page rows in token order,
// [g][d] (row = token), staged in shared memory by the caller.
// ---------------------------------------------------------------------------


// pack_key_page (pages.py:81-118) preceded, when `sel` is NULL, by
// channel_scores + select_boost (cache.py:155-158).  Writes the KTYP body to
// `slot_smem` (shared) and the f32 metadata to sc32/ze32 when non-NULL.
template <typename T>
__device__ void pack_key_tile(const T* tile, int g, int d, int d_boost, const int64_t* sel,
                              uint8_t* slot_smem, PackScratch& sc, float* sc32, float* ze32) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const KeyLayout L{d, g, d_boost};
    // boosted flags
    if (sel) {
        for (int c = tid; c < d; c += nt) sc.flag[c] = 0;
        __syncthreads();
        for (int j = tid; j < d_boost; j += nt) sc.flag[sel[j]] = 1;
    } else {
        // channel_scores (quant.py:64-72): sequential fp64 over tokens, / g
        for (int c = tid; c < d; c += nt) {
            double acc = 0.0;
            const T* col = tile + c;
#pragma unroll 8
            for (int t = 0; t < g; ++t) acc += static_cast<double>(fabsf(load_elem(col, t * d)));
            sc.score[c] = acc / static_cast<double>(g);
        }
        __syncthreads();
        // select_boost (quant.py:93): stable top-k on -score
        for (int c = tid; c < d; c += nt) {
            const double s = sc.score[c];
            int rank = 0;
            for (int j = 0; j < d; ++j) {
                const double o = sc.score[j];
                rank += (o > s) || (o == s && j < c);
            }
            sc.flag[c] = rank < d_boost;
        }
    }
    __syncthreads();
    // high_bits row of each boosted channel: ascending channel order (pages.py:103)
    if (d <= nt && d <= 1024) {
        // ballot prefix: rank of c among the boosted channels below it
        __shared__ int warp_cnt[32];
        const int lane = tid & 31, w = tid >> 5;
        const bool f = tid < d && sc.flag[tid] != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) warp_cnt[w] = __popc(bal);
        __syncthreads();
        if (tid < d) {
            int pos = __popc(bal & ((1u << lane) - 1u));
            for (int j = 0; j < w; ++j) pos += warp_cnt[j];
            sc.pos[tid] = pos;
        }
    } else {
        for (int c = tid; c < d; c += nt) {
            int pos = 0;
            for (int j = 0; j < c; ++j) pos += sc.flag[j];
            sc.pos[c] = pos;
        }
    }
    __syncthreads();
    // per-channel quantization (quant.py:102-116) and 2-bit packing (pages.py:42-45)
    const int gb = g / 4;
    uint8_t* dense = slot_smem + L.dense_off();
    uint8_t* high = slot_smem + L.high_off();
    uint8_t* idx = slot_smem + L.idx_off();
    uint8_t* s16 = slot_smem + L.scale_off();
    uint8_t* z16 = slot_smem + L.zero_off();
    for (int c = tid; c < d; c += nt) {
        const T* col = tile + c;
        float mn = load_elem(col, 0), mx = mn;
#pragma unroll 8
        for (int t = 1; t < g; ++t) {
            const float v = load_elem(col, t * d);
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
        if (mn == 0.f || mx == 0.f) {
            // a zero min / max carries the sign of the channel's last zero:
            // np.minimum.reduce / np.maximum.reduce keep the later operand of a tie
            float z = 0.f;
            for (int t = g - 1; t >= 0; --t) {
                const float v = load_elem(col, t * d);
                if (v == 0.f) {
                    z = v;
                    break;
                }
            }
            mn = mn == 0.f ? z : mn;
            mx = mx == 0.f ? z : mx;
        }
        const bool boosted = sc.flag[c] != 0;
        const LaneQuant q(mn, mx, boosted ? 15.f : 3.f);
        const int row = sc.pos[c];
#pragma unroll 2
        for (int b = 0; b < gb; ++b) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t code = q.code(load_elem(col, (4 * b + j) * d));
                lo |= (code & 3u) << (2 * j);
                hi |= (code >> 2) << (2 * j);
            }
            dense[c * gb + b] = static_cast<uint8_t>(lo);
            if (boosted) high[row * gb + b] = static_cast<uint8_t>(hi);
        }
        idx[c] = boosted ? static_cast<uint8_t>(row) : kSentinel;
        // f16 metadata: stored unaligned-safe (2-byte aligned by construction)
        st_u16(s16 + 2 * c, f32_to_half_bits(q.scale));
        st_u16(z16 + 2 * c, f32_to_half_bits(mn));
        if (sc32) sc32[c] = q.scale;
        if (ze32) ze32[c] = mn;
    }
    __syncthreads();
}

// pack_value_page (pages.py:146-162): per-token (row) quantization at 2 bits,
// packed along channels.  One warp per token row.
template <typename T>
__device__ void pack_value_tile(const T* tile, int g, int d, uint8_t* slot_smem, float* sc32,
                                float* ze32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const ValueLayout L{d, g};
    uint8_t* codes = slot_smem + L.codes_off();
    uint8_t* s16 = slot_smem + L.scale_off();
    uint8_t* z16 = slot_smem + L.zero_off();
    const int db = d / 4;
    for (int t = warp; t < g; t += nw) {
        const T* row = tile + (int64_t)t * d;
        float mn = INFINITY, mx = -INFINITY;
        for (int c = lane; c < d; c += 32) {
            const float v = load_elem(row, c);
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (mn == 0.f || mx == 0.f) {  // warp-uniform: the sign of the row's last zero
            int best = -1;
            for (int c = lane; c < d; c += 32) {
                const float v = load_elem(row, c);
                if (v == 0.f) best = (c << 1) | (signbit(v) ? 1 : 0);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
            const float z = (best & 1) ? -0.f : 0.f;
            mn = mn == 0.f ? z : mn;
            mx = mx == 0.f ? z : mx;
        }
        const LaneQuant q(mn, mx, 3.f);
        for (int b = lane; b < db; b += 32) {
            uint32_t byte = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) byte |= q.code(load_elem(row, 4 * b + j)) << (2 * j);
            codes[t * db + b] = static_cast<uint8_t>(byte);
        }
        if (lane == 0) {
            st_u16(s16 + 2 * t, f32_to_half_bits(q.scale));
            st_u16(z16 + 2 * t, f32_to_half_bits(mn));
            if (sc32) sc32[t] = q.scale;
            if (ze32) ze32[t] = mn;
        }
    }
    __syncthreads();
}

__device__ void copy_slot_out(const uint8_t* slot_smem, uint8_t* gslot, int bytes) {
    if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(gslot) & 15) == 0) {
        const uint4* s = reinterpret_cast<const uint4*>(slot_smem);
        uint4* o = reinterpret_cast<uint4*>(gslot);
        for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) o[i] = s[i];
    } else {
        for (int i = threadIdx.x; i < bytes; i += blockDim.x) gslot[i] = slot_smem[i];
    }
}

// Stage g rows [start, start + g) of a row ring of size `wrap` (start < wrap,
// g <= wrap) into smem, checking every element for non-finite values on the
// way (pages.py:88-89, 152-153).  Returns true when all are finite.
__device__ __forceinline__ int bf16x2_nonfinite(uint32_t w) {
    const uint32_t u = (w & 0x7F807F80u) ^ 0x7F807F80u;  // a zero half = exponent all ones
    return ((u & 0xFFFFu) == 0u) | ((u >> 16) == 0u);
}
template <typename T>
__device__ bool stage_rows(T* tile, const T* base, int start, int wrap, int g, int d) {
    int bad = 0;
    if (sizeof(T) == 2 && (d % 8) == 0) {
        const int vpr = d / 8;  // uint4 per row
        const int lg = (vpr & (vpr - 1)) == 0 ? __ffs(vpr) - 1 : -1;
        for (int i = threadIdx.x; i < g * vpr; i += blockDim.x) {
            const int r = lg >= 0 ? (i >> lg) : i / vpr;
            const int v = i - r * vpr;
            int row = start + r;
            if (row >= wrap) row -= wrap;
            const uint4 x = reinterpret_cast<const uint4*>(base + (int64_t)row * d)[v];
            reinterpret_cast<uint4*>(tile + (int64_t)r * d)[v] = x;
            bad |= bf16x2_nonfinite(x.x) | bf16x2_nonfinite(x.y) | bf16x2_nonfinite(x.z) | bf16x2_nonfinite(x.w);
        }
    } else {
        for (int i = threadIdx.x; i < g * d; i += blockDim.x) {
            const int r = i / d, c = i % d;
            int row = start + r;
            if (row >= wrap) row -= wrap;
            tile[i] = base[(int64_t)row * d + c];
            bad |= !isfinite(load_elem(tile, i));
        }
    }
    return __syncthreads_or(bad) == 0;
}

// Shared-memory budget of one pack (tile + slot + scratch), in bytes.
__host__ __device__ size_t pack_smem_bytes(int g, int d, int d_boost, int elem_bytes) {
    size_t tile = (size_t)g * d * elem_bytes;
    tile = (tile + 15) & ~size_t(15);
    size_t slot = (size_t)KeyLayout{d, g, d_boost}.bytes();
    const size_t vslot = (size_t)ValueLayout{d, g}.bytes();
    if (vslot > slot) slot = vslot;
    slot = (slot + 15) & ~size_t(15);
    return tile + slot + PackScratch::bytes(d);
}

__device__ PackScratch carve_scratch(uint8_t* p, int d) {
    PackScratch s;
    s.score = reinterpret_cast<double*>(p);
    s.pos = reinterpret_cast<int*>(p + 8 * (size_t)d);
    s.flag = reinterpret_cast<uint8_t*>(p + 12 * (size_t)d);
    return s;
}

// ---------------------------------------------------------------------------
// Standalone codec kernels (one CTA per page)
// ---------------------------------------------------------------------------

template <typename T>
__global__ void pack_key_pages_kernel(const T* x, int g, int d, int d_boost, const int64_t* sel,
                                      uint8_t* slots, int64_t stride, float* sc32, float* ze32,
                                      uint32_t* status) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int p = blockIdx.x;
    T* tile = reinterpret_cast<T*>(smem);
    size_t off = ((size_t)g * d * sizeof(T) + 15) & ~size_t(15);
    uint8_t* slot = smem + off;
    off += ((size_t)max(KeyLayout{d, g, d_boost}.bytes(), ValueLayout{d, g}.bytes()) + 15) & ~size_t(15);
    PackScratch sc = carve_scratch(smem + off, d);
    if (!stage_rows(tile, x + (int64_t)p * g * d, 0, g, g, d)) {
        if (threadIdx.x == 0) set_status(status, KITTY_STATUS_NONFINITE);
        return;
    }
    pack_key_tile(tile, g, d, d_boost, sel ? sel + (int64_t)p * d_boost : nullptr, slot, sc,
                  sc32 ? sc32 + (int64_t)p * d : nullptr, ze32 ? ze32 + (int64_t)p * d : nullptr);
    copy_slot_out(slot, slots + p * stride, KeyLayout{d, g, d_boost}.bytes());
}

template <typename T>
__global__ void pack_value_pages_kernel(const T* x, int g, int d, uint8_t* slots, int64_t stride,
                                        float* sc32, float* ze32, uint32_t* status) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int p = blockIdx.x;
    T* tile = reinterpret_cast<T*>(smem);
    uint8_t* slot = smem + (((size_t)g * d * sizeof(T) + 15) & ~size_t(15));
    if (!stage_rows(tile, x + (int64_t)p * g * d, 0, g, g, d)) {
        if (threadIdx.x == 0) set_status(status, KITTY_STATUS_NONFINITE);
        return;
    }
    pack_value_tile(tile, g, d, slot, sc32 ? sc32 + (int64_t)p * g : nullptr,
                    ze32 ? ze32 + (int64_t)p * g : nullptr);
    copy_slot_out(slot, slots + p * stride, ValueLayout{d, g}.bytes());
}

template <typename T>
__global__ void channel_scores_kernel(const T* x, int g, int d, double* scores) {
    const int p = blockIdx.x;
    const T* tile = x + (int64_t)p * g * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        double acc = 0.0;
        for (int t = 0; t < g; ++t) acc += static_cast<double>(fabsf(load_elem(tile, (int64_t)t * d + c)));
        scores[(int64_t)p * d + c] = acc / static_cast<double>(g);
    }
}

__global__ void select_boost_kernel(const double* scores, int d, int k, int64_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* flag = smem;
    const double* s = scores + (int64_t)blockIdx.x * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const double v = s[c];
        int rank = 0;
        for (int j = 0; j < d; ++j) rank += (s[j] > v) || (s[j] == v && j < c);
        flag[c] = rank < k;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        if (!flag[c]) continue;
        int pos = 0;
        for (int j = 0; j < c; ++j) pos += flag[j];
        out[(int64_t)blockIdx.x * k + pos] = c;
    }
}

// dequantize_key_page (pages.py:121-143): validate the sentinel pattern, then
// X = low | high[boost_idx] << 2, out = X * scale + zero (mul then add).
// pages.py:128-135 for one key page (block-uniform): d_boost non-sentinel
// entries in boost_idx, forming a bijection onto the high-bit rows 0..d_boost-1.
__device__ bool block_boost_index_ok(const uint8_t* idx, int d, int d_boost) {
    __shared__ int seen[256];
    __shared__ int total;
    for (int j = threadIdx.x; j < 256; j += blockDim.x) seen[j] = 0;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const uint8_t b = idx[c];
        if (b != kSentinel) {
            atomicAdd(&seen[b], 1);
            atomicAdd(&total, 1);
        }
    }
    __syncthreads();
    int bad = total != d_boost;
    for (int j = threadIdx.x; j < 256; j += blockDim.x) bad |= (j < d_boost) ? (seen[j] != 1) : (seen[j] != 0);
    return !__syncthreads_or(bad);
}

__global__ void dequant_key_pages_kernel(const uint8_t* slots, int64_t stride, int g, int d,
                                         int d_boost, const float* sc32, const float* ze32,
                                         float* out, uint32_t* status) {
    const int p = blockIdx.x;
    const KeyLayout L{d, g, d_boost};
    const uint8_t* slot = slots + p * stride;
    const uint8_t* idx = slot + L.idx_off();
    if (!block_boost_index_ok(idx, d, d_boost)) {
        if (threadIdx.x == 0) set_status(status, KITTY_STATUS_PAGE_FORMAT);
        return;
    }
    const int gb = g / 4;
    const uint8_t* dense = slot + L.dense_off();
    const uint8_t* high = slot + L.high_off();
    const uint8_t* s16 = slot + L.scale_off();
    const uint8_t* z16 = slot + L.zero_off();
    float* o = out + (int64_t)p * d * g;
    for (int i = threadIdx.x; i < d * gb; i += blockDim.x) {
        const int c = i / gb, b = i % gb;
        const float s = sc32 ? sc32[(int64_t)p * d + c] : half_bits_to_f32(ld_u16(s16 + 2 * c));
        const float z = ze32 ? ze32[(int64_t)p * d + c] : half_bits_to_f32(ld_u16(z16 + 2 * c));
        const uint32_t lo = dense[c * gb + b];
        const uint8_t r = idx[c];
        const uint32_t hi = (r != kSentinel) ? high[r * gb + b] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t code = ((lo >> (2 * j)) & 3u) | (((hi >> (2 * j)) & 3u) << 2);
            o[(int64_t)c * g + 4 * b + j] = __fadd_rn(__fmul_rn(static_cast<float>(code), s), z);
        }
    }
}

__global__ void dequant_value_pages_kernel(const uint8_t* slots, int64_t stride, int g, int d,
                                           const float* sc32, const float* ze32, float* out) {
    const int p = blockIdx.x;
    const ValueLayout L{d, g};
    const uint8_t* slot = slots + p * stride;
    const uint8_t* s16 = slot + L.scale_off();
    const uint8_t* z16 = slot + L.zero_off();
    const int db = d / 4;
    float* o = out + (int64_t)p * g * d;
    for (int i = threadIdx.x; i < g * db; i += blockDim.x) {
        const int t = i / db, b = i % db;
        const float s = sc32 ? sc32[(int64_t)p * g + t] : half_bits_to_f32(ld_u16(s16 + 2 * t));
        const float z = ze32 ? ze32[(int64_t)p * g + t] : half_bits_to_f32(ld_u16(z16 + 2 * t));
        const uint32_t byte = slot[L.codes_off() + t * db + b];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            o[(int64_t)t * d + 4 * b + j] =
                __fadd_rn(__fmul_rn(static_cast<float>((byte >> (2 * j)) & 3u), s), z);
    }
}

// ---------------------------------------------------------------------------
// Cache runtime: append (insert_token + maybe_pack) and prefill
// ---------------------------------------------------------------------------

// Row element of the cache (bf16 bits or float) as float
__device__ __forceinline__ float row_elem(const uint16_t* p, int64_t i) { return bf16_to_f32(p[i]); }
__device__ __forceinline__ float row_elem(const float* p, int64_t i) { return p[i]; }

template <typename T>
__device__ __forceinline__ void copy_row(T* dst, const T* src, int d) {
    constexpr int kPer = 16 / sizeof(T);  // elements per 16-byte vector
    if ((d % kPer) == 0) {
        for (int i = threadIdx.x; i < d / kPer; i += blockDim.x)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
        for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
    }
}

// The slot of page p of unit u on one side (key / value) for a kernel about
// to write it.  With a page pool (KittyCacheDesc.key_free) thread 0 pops a
// free slot and records it in the unit's block table; without one the
// caller's block table names it.  Block-uniform: every thread calls it and
// gets the slot (-1 = the pool is empty: KITTY_STATUS_OVERFLOW is set).
__device__ int32_t block_claim_slot(const KittyCacheDesc& c, bool key, int u, int p) {
    __shared__ int32_t s_slot;
    __syncthreads();  // a previous call's s_slot has been read by every thread
    if (threadIdx.x == 0) {
        int32_t* e = (key ? c.key_block_table : c.value_block_table) + (int64_t)u * c.max_pages + p;
        int32_t* stack = key ? c.key_free : c.value_free;
        int32_t s = -1;
        if (!stack) {
            s = *e;
        } else {
            int32_t* top = c.free_top + (key ? 0 : 1);
            const int i = atomicSub(top, 1) - 1;
            if (i < 0) {
                atomicAdd(top, 1);
                set_status(c.status, KITTY_STATUS_OVERFLOW);
            } else {
                s = stack[i];
                *e = s;
            }
        }
        s_slot = s;
    }
    __syncthreads();
    return s_slot;
}

// Pack key page `p` of unit `u` from `rows` (g consecutive rows of a ring of
// size `wrap` starting at `start`) into its block-table slot (+ its f32
// metadata into the side table when the cache keeps one).
// A pass-through (16-bit) page (cache.py:150-153,167-170): the block's g rows
// copied as they are (row dtype) into the page's slot.
template <typename T>
__device__ void copy_rows_into_slot(const KittyCacheDesc& c, bool key, int u, int p, const T* base, int start,
                                    int wrap) {
    const int32_t s = block_claim_slot(c, key, u, p);
    if (s < 0) return;
    T* dst = reinterpret_cast<T*>((key ? c.key_pool : c.value_pool) + (int64_t)s * (key ? c.key_slot_bytes : c.value_slot_bytes));
    const int d = c.cfg.d, g = c.cfg.g;
    for (int i = threadIdx.x; i < g * d; i += blockDim.x) {
        const int r = i / d, ch = i - r * d;
        dst[i] = base[(int64_t)((start + r) % wrap) * d + ch];
    }
}

template <typename T>
__device__ void pack_key_into_cache(const KittyCacheDesc& c, int u, int p, const T* base, int start, int wrap,
                                    uint8_t* smem) {
    const KittyConfigC& k = c.cfg;
    if (p >= c.max_pages) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
        return;
    }
    if (k.key_bits == 16) {
        copy_rows_into_slot(c, true, u, p, base, start, wrap);
        return;
    }
    T* tile = reinterpret_cast<T*>(smem);
    size_t off = ((size_t)k.g * k.d * sizeof(T) + 15) & ~size_t(15);
    uint8_t* slot = smem + off;
    off += ((size_t)max(KeyLayout{k.d, k.g, k.d_boost}.bytes(), ValueLayout{k.d, k.g}.bytes()) + 15) & ~size_t(15);
    PackScratch sc = carve_scratch(smem + off, k.d);
    if (!stage_rows(tile, base, start, wrap, k.g, k.d)) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_NONFINITE);
    }
    const int32_t s = block_claim_slot(c, true, u, p);
    if (s < 0) return;
    float* meta = c.key_meta ? c.key_meta + (int64_t)s * 2 * k.d : nullptr;
    pack_key_tile(tile, k.g, k.d, k.d_boost, nullptr, slot, sc, meta, meta ? meta + k.d : nullptr);
    copy_slot_out(slot, c.key_pool + (int64_t)s * c.key_slot_bytes, KeyLayout{k.d, k.g, k.d_boost}.bytes());
}

template <typename T>
__device__ void pack_value_into_cache(const KittyCacheDesc& c, int u, int p, const T* base, int start, int wrap,
                                      uint8_t* smem) {
    const KittyConfigC& k = c.cfg;
    if (p >= c.max_pages) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
        return;
    }
    if (k.value_bits == 16) {
        copy_rows_into_slot(c, false, u, p, base, start, wrap);
        return;
    }
    T* tile = reinterpret_cast<T*>(smem);
    uint8_t* slot = smem + (((size_t)k.g * k.d * sizeof(T) + 15) & ~size_t(15));
    if (!stage_rows(tile, base, start, wrap, k.g, k.d)) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_NONFINITE);
    }
    const int32_t s = block_claim_slot(c, false, u, p);
    if (s < 0) return;
    float* meta = c.value_meta ? c.value_meta + (int64_t)s * 2 * k.g : nullptr;
    pack_value_tile(tile, k.g, k.d, slot, meta, meta ? meta + k.g : nullptr);
    copy_slot_out(slot, c.value_pool + (int64_t)s * c.value_slot_bytes, ValueLayout{k.d, k.g}.bytes());
}

// insert_token (cache.py:107-123) for one unit per CTA, then the pack trigger
// of maybe_pack (cache.py:144-178) on this unit's own counts.  T = the row type.
template <typename T>
__global__ void append_kernel(KittyCacheDesc c, const T* k_new, const T* v_new) {
    extern __shared__ __align__(16) uint8_t smem[];
    // launched as a programmatic dependent of the preceding kernel (e.g. the
    // previous layer's merge): everything below waits for it to complete
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the attention grid that follows may run its prologue now (it waits on us
    // with griddepcontrol.wait before reading the cache)
    asm volatile("griddepcontrol.launch_dependents;");
    const KittyConfigC& k = c.cfg;
    const int u = blockIdx.x;
    const int d = k.d, S = k.s, G = k.g, W = k.r + k.g;
    const T* kr = k_new + (int64_t)u * d;
    const T* vr = v_new + (int64_t)u * d;
    // rows of 16-byte vectors that one pass of the CTA covers: their loads go
    // out together with the length's (one round trip instead of two)
    const int nv = static_cast<int>(d * sizeof(T) / 16);
    const bool vec = (d * sizeof(T)) % 16 == 0 && nv <= static_cast<int>(blockDim.x);
    uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = kv4;
    if (vec && threadIdx.x < nv) {
        kv4 = reinterpret_cast<const uint4*>(kr)[threadIdx.x];
        vv4 = reinterpret_cast<const uint4*>(vr)[threadIdx.x];
    }
    const int t = c.unit_len[u];
    T* ksink = static_cast<T*>(c.k_sink);
    T* vsink = static_cast<T*>(c.v_sink);
    T* kq = static_cast<T*>(c.k_qbuf) + (int64_t)u * G * d;
    T* vring = static_cast<T*>(c.v_ring) + (int64_t)u * W * d;
    T* kd = t < S ? ksink + ((int64_t)u * S + t) * d : kq + (int64_t)((t - S) % G) * d;
    T* vd = t < S ? vsink + ((int64_t)u * S + t) * d : vring + (int64_t)((t - S) % W) * d;
    if (vec) {
        if (threadIdx.x < nv) {
            reinterpret_cast<uint4*>(kd)[threadIdx.x] = kv4;
            reinterpret_cast<uint4*>(vd)[threadIdx.x] = vv4;
        }
    } else {
        copy_row(kd, kr, d);
        copy_row(vd, vr, d);
    }
    const int n = t + 1;
    const int past = n > S ? n - S : 0;
    const int vtot = past > k.r ? past - k.r : 0;  // tokens that left the local window
    const bool kpack = past > 0 && past % G == 0, vpack = vtot > 0 && vtot % G == 0;
    bool fast = false;
    if constexpr (sizeof(T) == 2)
        fast = d == fastpack::kD && G == fastpack::kG && !c.key_meta && !c.value_meta && k.key_bits == 2 && k.value_bits == 2;
    if (fast && (kpack || vpack)) {
        if constexpr (sizeof(T) == 2) {
            // the bulk packer's routines: the page rows arrive by TMA (async proxy),
            // so the row this CTA just stored must be visible to it first
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncthreads();
            fastpack::Smem& s = *reinterpret_cast<fastpack::Smem*>(smem);
            if (kpack) {
                const int p = past / G - 1;
                const int32_t sl = p < c.max_pages ? block_claim_slot(c, true, u, p) : -1;
                if (p >= c.max_pages) {
                    if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
                } else if (sl >= 0) {
                    fastpack::key_page(s, kq, 0, G, k.d_boost, c.key_pool + (int64_t)sl * c.key_slot_bytes, c.status);
                }
                __syncthreads();
            }
            if (vpack) {
                const int p = vtot / G - 1;
                const int32_t sl = p < c.max_pages ? block_claim_slot(c, false, u, p) : -1;
                if (p >= c.max_pages) {
                    if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
                } else if (sl >= 0) {
                    fastpack::value_page(s, vring, (p * G) % W, W, c.value_pool + (int64_t)sl * c.value_slot_bytes,
                                         c.status);
                }
            }
        }
    } else {
        __syncthreads();
        if (kpack) pack_key_into_cache(c, u, past / G - 1, kq, 0, G, smem);
        if (vpack) {
            const int p = vtot / G - 1;
            __syncthreads();
            pack_value_into_cache(c, u, p, vring, (p * G) % W, W, smem);
        }
    }
    if (threadIdx.x == 0) c.unit_len[u] = n;
}

// Prefill, fp rows: every prompt token whose final home (after the fold of
// `P` appends) is a sink / q-buffer / ring row is copied there.
template <typename T>
__global__ void prefill_rows_kernel(KittyCacheDesc c, const T* keys, const T* values, int P) {
    const KittyConfigC& k = c.cfg;
    const int u = blockIdx.y;
    const int d = k.d, S = k.s, G = k.g, W = k.r + k.g;
    const int past = P > S ? P - S : 0;
    const int kp = past / G;
    const int local = min(k.r, past);
    const int vp = (past - local) / G;
    // only the tokens that stay full precision: the sink, the key q-buffer
    // [S + kp G, P) and the value q-buffer + local window [S + vp G, P)
    const int t_fp = S + vp * G;  // <= S + kp * G
    const int n_fp = min(P, S) + (P > t_fp ? P - t_fp : 0);
    for (int i = blockIdx.x; i < n_fp; i += gridDim.x) {
        const int t = i < min(P, S) ? i : t_fp + (i - min(P, S));
        const T* kr = keys + ((int64_t)u * P + t) * d;
        const T* vr = values + ((int64_t)u * P + t) * d;
        if (t < S) {
            copy_row(static_cast<T*>(c.k_sink) + ((int64_t)u * S + t) * d, kr, d);
            copy_row(static_cast<T*>(c.v_sink) + ((int64_t)u * S + t) * d, vr, d);
        } else {
            const int pc = t - S;
            if (pc >= kp * G) copy_row(static_cast<T*>(c.k_qbuf) + ((int64_t)u * G + pc % G) * d, kr, d);
            if (pc >= vp * G) copy_row(static_cast<T*>(c.v_ring) + ((int64_t)u * W + pc % W) * d, vr, d);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) c.unit_len[u] = P;
}

// Prefill, pages: blockIdx.x < kp packs key page blockIdx.x, else value page
// blockIdx.x - kp; a page depends only on its own g tokens.
template <typename T>
__global__ void prefill_pack_kernel(KittyCacheDesc c, const T* keys, const T* values, int P, int kp, int vp) {
    extern __shared__ __align__(16) uint8_t smem[];
    const KittyConfigC& k = c.cfg;
    const int u = blockIdx.y;
    const int y = blockIdx.x;
    if (y < kp) {
        pack_key_into_cache(c, u, y, keys + ((int64_t)u * P + k.s) * k.d, y * k.g, 1 << 30, smem);
    } else if (y < kp + vp) {
        const int p = y - kp;
        pack_value_into_cache(c, u, p, values + ((int64_t)u * P + k.s) * k.d, p * k.g, 1 << 30, smem);
    }
}

// The same pages for d = g = 128 and bf16 rows (kitty_pack_fast.cuh): one
// page per CTA, the page's rows by TMA, bytes straight to the slot.
__global__ void __launch_bounds__(fastpack::kThreads) prefill_pack_fast_kernel(KittyCacheDesc c, const uint16_t* keys,
                                                                              const uint16_t* values, int P, int kp,
                                                                              int vp) {
    extern __shared__ __align__(128) uint8_t smem[];
    fastpack::Smem& s = *reinterpret_cast<fastpack::Smem*>(smem);
    const KittyConfigC& k = c.cfg;
    const int u = blockIdx.y, y = blockIdx.x;
    const bool is_key = y < kp;
    const int p = is_key ? y : y - kp;
    if (!is_key && p >= vp) return;
    if (p >= c.max_pages) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
        return;
    }
    const int64_t row0 = (int64_t)u * P + k.s + (int64_t)p * fastpack::kG;
    const int32_t sl = block_claim_slot(c, is_key, u, p);
    if (sl < 0) return;
    if (is_key) {
        uint8_t* slot = c.key_pool + (int64_t)sl * c.key_slot_bytes;
        fastpack::key_page(s, keys + row0 * fastpack::kD, 0, fastpack::kG, k.d_boost, slot, c.status);
    } else {
        uint8_t* slot = c.value_pool + (int64_t)sl * c.value_slot_bytes;
        fastpack::value_page(s, values + row0 * fastpack::kD, 0, fastpack::kG, slot, c.status);
    }
}

// flatten_keys / flatten_values (cache.py:210-215) of one unit; pages use the
// f32 metadata side table when the cache keeps one, else the slot's f16 copy.
template <typename T>
__global__ void flatten_kernel(KittyCacheDesc c, int u, int n, float* keys_out, float* values_out) {
    const KittyConfigC& k = c.cfg;
    const int d = k.d, S = k.s, G = k.g, W = k.r + k.g;
    const int past = n > S ? n - S : 0;
    const int kp = past / G;
    const int local = min(k.r, past);
    const int vp = (past - local) / G;
    const KeyLayout KL{d, G, k.d_boost};
    const ValueLayout VL{d, G};
    const int gb = G / 4, db = d / 4;
    const T* ksink = static_cast<const T*>(c.k_sink);
    const T* vsink = static_cast<const T*>(c.v_sink);
    const T* kq = static_cast<const T*>(c.k_qbuf);
    const T* vring = static_cast<const T*>(c.v_ring);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)n * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int t = static_cast<int>(i / d), ch = static_cast<int>(i % d);
        float kv, vv;
        if (t < S) {
            kv = row_elem(ksink, ((int64_t)u * S + t) * d + ch);
            vv = row_elem(vsink, ((int64_t)u * S + t) * d + ch);
        } else {
            const int pc = t - S;
            if (pc < kp * G && k.key_bits == 16) {  // pass-through page: the block's rows as stored
                const int32_t sl = c.key_block_table[(int64_t)u * c.max_pages + pc / G];
                kv = row_elem(reinterpret_cast<const T*>(c.key_pool + (int64_t)sl * c.key_slot_bytes), (int64_t)(pc % G) * d + ch);
            } else if (pc < kp * G) {
                const int p = pc / G, tl = pc % G;
                const int32_t sl = c.key_block_table[(int64_t)u * c.max_pages + p];
                const uint8_t* slot = c.key_pool + (int64_t)sl * c.key_slot_bytes;
                uint32_t code = (slot[KL.dense_off() + ch * gb + tl / 4] >> (2 * (tl % 4))) & 3u;
                const uint8_t r = slot[KL.idx_off() + ch];
                if (r != kSentinel) code |= ((slot[KL.high_off() + r * gb + tl / 4] >> (2 * (tl % 4))) & 3u) << 2;
                const float* meta = c.key_meta ? c.key_meta + (int64_t)sl * 2 * d : nullptr;
                const float s = meta ? meta[ch] : half_bits_to_f32(ld_u16(slot + KL.scale_off() + 2 * ch));
                const float z = meta ? meta[d + ch] : half_bits_to_f32(ld_u16(slot + KL.zero_off() + 2 * ch));
                kv = __fadd_rn(__fmul_rn(static_cast<float>(code), s), z);
            } else {
                kv = row_elem(kq, ((int64_t)u * G + pc % G) * d + ch);
            }
            if (pc < vp * G && k.value_bits == 16) {
                const int32_t sl = c.value_block_table[(int64_t)u * c.max_pages + pc / G];
                vv = row_elem(reinterpret_cast<const T*>(c.value_pool + (int64_t)sl * c.value_slot_bytes), (int64_t)(pc % G) * d + ch);
            } else if (pc < vp * G) {
                const int p = pc / G, tl = pc % G;
                const int32_t sl = c.value_block_table[(int64_t)u * c.max_pages + p];
                const uint8_t* slot = c.value_pool + (int64_t)sl * c.value_slot_bytes;
                const uint32_t code = (slot[VL.codes_off() + tl * db + ch / 4] >> (2 * (ch % 4))) & 3u;
                const float* meta = c.value_meta ? c.value_meta + (int64_t)sl * 2 * G : nullptr;
                const float s = meta ? meta[tl] : half_bits_to_f32(ld_u16(slot + VL.scale_off() + 2 * tl));
                const float z = meta ? meta[G + tl] : half_bits_to_f32(ld_u16(slot + VL.zero_off() + 2 * tl));
                vv = __fadd_rn(__fmul_rn(static_cast<float>(code), s), z);
            } else {
                vv = row_elem(vring, ((int64_t)u * W + pc % W) * d + ch);
            }
        }
        keys_out[i] = kv;
        values_out[i] = vv;
    }
}

// fake_quantize_matrix (quant.py:145-177): every lane -- a column of x
// [rows][cols] (per_channel) or a row (per_token) -- quantized and dequantized
// at its own width: 2 / 4 bits with the column quantizer of quant.py:102-120
// (min / max, IEEE scale, rint half-even, clip; multiply then add), 16 = the
// lane passes through.  One thread per lane.
__global__ void fake_quantize_kernel(const float* x, int rows, int cols, int per_token, const int32_t* bits,
                                     float* out) {
    const int lanes = per_token ? rows : cols, len = per_token ? cols : rows;
    const int64_t step = per_token ? 1 : cols;
    for (int lane = blockIdx.x * blockDim.x + threadIdx.x; lane < lanes; lane += gridDim.x * blockDim.x) {
        const float* src = per_token ? x + (int64_t)lane * cols : x + lane;
        float* dst = per_token ? out + (int64_t)lane * cols : out + lane;
        const int b = bits[lane];
        if (b != 2 && b != 4) {
            for (int i = 0; i < len; ++i) dst[i * step] = src[i * step];
            continue;
        }
        float mn = src[0], mx = mn;
        for (int i = 1; i < len; ++i) {
            mn = fminf(mn, src[i * step]);
            mx = fmaxf(mx, src[i * step]);
        }
        if (mn == 0.f || mx == 0.f) {  // a zero min / max carries the sign of the lane's last zero
            float z = 0.f;
            for (int i = len - 1; i >= 0; --i) {
                if (src[i * step] == 0.f) {
                    z = src[i * step];
                    break;
                }
            }
            mn = mn == 0.f ? z : mn;
            mx = mx == 0.f ? z : mx;
        }
        const LaneQuant q(mn, mx, static_cast<float>((1 << b) - 1));
        for (int i = 0; i < len; ++i)
            dst[i * step] = __fadd_rn(__fmul_rn(static_cast<float>(q.code(src[i * step])), q.scale), mn);
    }
}

// _quantize_columns / quantize_values (quant.py:102-132) for every lane of x
// (columns for per_channel, rows for per_token): codes (u8, like x) and the
// lane's f32 scale / zero point.  bits[lane] in {2, 4}.
__global__ void quantize_lanes_kernel(const float* x, int rows, int cols, int per_token, const int32_t* bits,
                                      uint8_t* codes, float* scales, float* zeros) {
    const int lanes = per_token ? rows : cols, len = per_token ? cols : rows;
    const int64_t step = per_token ? 1 : cols;
    for (int lane = blockIdx.x * blockDim.x + threadIdx.x; lane < lanes; lane += gridDim.x * blockDim.x) {
        const float* src = per_token ? x + (int64_t)lane * cols : x + lane;
        uint8_t* dst = per_token ? codes + (int64_t)lane * cols : codes + lane;
        float mn = src[0], mx = mn;
        for (int i = 1; i < len; ++i) {
            mn = fminf(mn, src[i * step]);
            mx = fmaxf(mx, src[i * step]);
        }
        if (mn == 0.f || mx == 0.f) {  // a zero min / max carries the sign of the lane's last zero
            float z = 0.f;
            for (int i = len - 1; i >= 0; --i) {
                if (src[i * step] == 0.f) {
                    z = src[i * step];
                    break;
                }
            }
            mn = mn == 0.f ? z : mn;
            mx = mx == 0.f ? z : mx;
        }
        const LaneQuant q(mn, mx, static_cast<float>((1 << bits[lane]) - 1));
        for (int i = 0; i < len; ++i) dst[i * step] = static_cast<uint8_t>(q.code(src[i * step]));
        scales[lane] = q.scale;
        zeros[lane] = mn;
    }
}

// dequantize_values (quant.py:135-143): code * scale + zero, multiply then add.
__global__ void dequantize_lanes_kernel(const uint8_t* codes, int rows, int cols, int per_token, const float* scales,
                                        const float* zeros, float* out) {
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int lane = per_token ? static_cast<int>(i / cols) : static_cast<int>(i % cols);
        out[i] = __fadd_rn(__fmul_rn(static_cast<float>(codes[i]), scales[lane]), zeros[lane]);
    }
}

cudaError_t launch_quantize_lanes(const float* x, int rows, int cols, int per_token, const int32_t* bits,
                                  uint8_t* codes, float* scales, float* zeros, cudaStream_t st) {
    const int lanes = per_token ? rows : cols;
    if (lanes == 0 || rows == 0 || cols == 0) return cudaSuccess;
    quantize_lanes_kernel<<<(lanes + 127) / 128, 128, 0, st>>>(x, rows, cols, per_token, bits, codes, scales, zeros);
    return cudaGetLastError();
}

cudaError_t launch_dequantize_lanes(const uint8_t* codes, int rows, int cols, int per_token, const float* scales,
                                    const float* zeros, float* out, cudaStream_t st) {
    const int64_t n = (int64_t)rows * cols;
    if (n == 0) return cudaSuccess;
    const int blocks = static_cast<int>(n / 256 + 1 < 4096 ? n / 256 + 1 : 4096);
    dequantize_lanes_kernel<<<blocks, 256, 0, st>>>(codes, rows, cols, per_token, scales, zeros, out);
    return cudaGetLastError();
}

cudaError_t launch_fake_quantize(const float* x, int rows, int cols, int per_token, const int32_t* bits, float* out,
                                 cudaStream_t st) {
    const int lanes = per_token ? rows : cols;
    if (lanes == 0 || rows == 0 || cols == 0) return cudaSuccess;
    fake_quantize_kernel<<<(lanes + 127) / 128, 128, 0, st>>>(x, rows, cols, per_token, bits, out);
    return cudaGetLastError();
}

// Retire sequence seq0 + blockIdx.x / h_kv's unit: its slots go back to the
// pool's free stacks (pushes only: no pop runs in this launch), its block-table
// entries become -1, its length 0.
__global__ void release_kernel(KittyCacheDesc c, int seq0) {
    const int u = seq0 * c.cfg.h_kv + blockIdx.x;
    const int n = c.unit_len[u];
    const int S = c.cfg.s, G = c.cfg.g;
    const int past = n > S ? n - S : 0;
    const int kp = min(past / G, c.max_pages);
    const int vp = min((past - min(c.cfg.r, past)) / G, c.max_pages);
    int32_t* kbt = c.key_block_table + (int64_t)u * c.max_pages;
    int32_t* vbt = c.value_block_table + (int64_t)u * c.max_pages;
    if (c.key_free) {
        for (int p = threadIdx.x; p < kp; p += blockDim.x) {
            const int32_t sl = kbt[p];
            if (sl >= 0) c.key_free[atomicAdd(&c.free_top[0], 1)] = sl;
            kbt[p] = -1;
        }
    }
    if (c.value_free) {
        for (int p = threadIdx.x; p < vp; p += blockDim.x) {
            const int32_t sl = vbt[p];
            if (sl >= 0) c.value_free[atomicAdd(&c.free_top[1], 1)] = sl;
            vbt[p] = -1;
        }
    }
    __syncthreads();  // every thread has read unit_len
    if (threadIdx.x == 0) c.unit_len[u] = 0;
}

// Import page first_page + blockIdx.x of unit u: claim its slot, copy the KTYP
// body in (16-byte vectors: slot sizes are multiples of 16), check a key
// page's boost index (pages.py:128-135) and fill the f32 metadata side table.
__global__ void import_pages_kernel(KittyCacheDesc c, int u, int kind, const uint8_t* bodies, int first_page) {
    const bool key = kind == 0;
    const int p = first_page + blockIdx.x;
    const int64_t bytes = key ? c.key_slot_bytes : c.value_slot_bytes;
    const uint8_t* src = bodies + (int64_t)blockIdx.x * bytes;
    if (p >= c.max_pages) {
        if (threadIdx.x == 0) set_status(c.status, KITTY_STATUS_OVERFLOW);
        return;
    }
    const int32_t sl = block_claim_slot(c, key, u, p);
    if (sl < 0) return;
    uint8_t* dst = (key ? c.key_pool : c.value_pool) + (int64_t)sl * bytes;
    for (int64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    const int d = c.cfg.d, g = c.cfg.g;
    if (key) {
        const KeyLayout L{d, g, c.cfg.d_boost};
        if (!block_boost_index_ok(src + L.idx_off(), d, c.cfg.d_boost) && threadIdx.x == 0)
            set_status(c.status, KITTY_STATUS_PAGE_FORMAT);
        if (c.key_meta) {
            float* m = c.key_meta + (int64_t)sl * 2 * d;
            for (int i = threadIdx.x; i < 2 * d; i += blockDim.x) m[i] = half_bits_to_f32(ld_u16(src + L.scale_off() + 2 * i));
        }
    } else if (c.value_meta) {
        const ValueLayout L{d, g};
        float* m = c.value_meta + (int64_t)sl * 2 * g;
        for (int i = threadIdx.x; i < 2 * g; i += blockDim.x) m[i] = half_bits_to_f32(ld_u16(src + L.scale_off() + 2 * i));
    }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------

cudaError_t launch_pack_key_pages(const void* x, int dtype, int P, int g, int d, int d_boost,
                                  const int64_t* sel, uint8_t* slots, int64_t stride, float* sc32,
                                  float* ze32, uint32_t* status, cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    const size_t sm = pack_smem_bytes(g, d, d_boost, dtype == KITTY_F32 ? 4 : 2);
    if (dtype == KITTY_F32) {
        auto kfn = pack_key_pages_kernel<float>;
        if (cudaError_t e = set_kernel_smem((const void*)kfn, (int)sm)) return e;
        kfn<<<P, 128, sm, st>>>(static_cast<const float*>(x), g, d, d_boost, sel, slots, stride,
                                sc32, ze32, status);
    } else {
        auto kfn = pack_key_pages_kernel<uint16_t>;
        if (cudaError_t e = set_kernel_smem((const void*)kfn, (int)sm)) return e;
        kfn<<<P, 128, sm, st>>>(static_cast<const uint16_t*>(x), g, d, d_boost, sel, slots,
                                stride, sc32, ze32, status);
    }
    return cudaGetLastError();
}

cudaError_t launch_pack_value_pages(const void* x, int dtype, int P, int g, int d, uint8_t* slots,
                                    int64_t stride, float* sc32, float* ze32, uint32_t* status,
                                    cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    const size_t sm = pack_smem_bytes(g, d, 0, dtype == KITTY_F32 ? 4 : 2);
    if (dtype == KITTY_F32) {
        auto kfn = pack_value_pages_kernel<float>;
        if (cudaError_t e = set_kernel_smem((const void*)kfn, (int)sm)) return e;
        kfn<<<P, 128, sm, st>>>(static_cast<const float*>(x), g, d, slots, stride, sc32, ze32, status);
    } else {
        auto kfn = pack_value_pages_kernel<uint16_t>;
        if (cudaError_t e = set_kernel_smem((const void*)kfn, (int)sm)) return e;
        kfn<<<P, 128, sm, st>>>(static_cast<const uint16_t*>(x), g, d, slots, stride, sc32, ze32, status);
    }
    return cudaGetLastError();
}

cudaError_t launch_channel_scores(const void* x, int dtype, int P, int g, int d, double* scores,
                                  cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    if (dtype == KITTY_F32)
        channel_scores_kernel<float><<<P, 128, 0, st>>>(static_cast<const float*>(x), g, d, scores);
    else
        channel_scores_kernel<uint16_t><<<P, 128, 0, st>>>(static_cast<const uint16_t*>(x), g, d, scores);
    return cudaGetLastError();
}

cudaError_t launch_select_boost(const double* scores, int P, int d, int k, int64_t* out,
                                cudaStream_t st) {
    if (P == 0 || k == 0) return cudaSuccess;
    select_boost_kernel<<<P, 128, d, st>>>(scores, d, k, out);
    return cudaGetLastError();
}

cudaError_t launch_dequant_key_pages(const uint8_t* slots, int64_t stride, int P, int g, int d,
                                     int d_boost, const float* sc32, const float* ze32, float* out,
                                     uint32_t* status, cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    dequant_key_pages_kernel<<<P, 256, 0, st>>>(slots, stride, g, d, d_boost, sc32,
                                                                ze32, out, status);
    return cudaGetLastError();
}

cudaError_t launch_dequant_value_pages(const uint8_t* slots, int64_t stride, int P, int g, int d,
                                       const float* sc32, const float* ze32, float* out,
                                       cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    dequant_value_pages_kernel<<<P, 256, 0, st>>>(slots, stride, g, d, sc32, ze32, out);
    return cudaGetLastError();
}

// KITTY_PDL bit 3: the append as a programmatic dependent of the preceding kernel
static const int g_pdl_append = [] {
    const char* e = std::getenv("KITTY_PDL");
    return e ? (std::atoi(e) >> 3) & 1 : 1;
}();

template <typename T>
static cudaError_t append_t(const KittyCacheDesc& c, const void* k_new, const void* v_new, cudaStream_t st) {
    const int units = c.num_seqs * c.cfg.h_kv;
    size_t sm = pack_smem_bytes(c.cfg.g, c.cfg.d, c.cfg.d_boost, sizeof(T));
    if (sizeof(T) == 2 && c.cfg.d == fastpack::kD && c.cfg.g == fastpack::kG && sm < sizeof(fastpack::Smem))
        sm = sizeof(fastpack::Smem);
    auto kfn = append_kernel<T>;
    // the decode kernels all prefer the max-shared carveout: an SM never has to
    // reconfigure between them, and PDL dependents can become resident beside
    // their predecessor
    if (cudaError_t e = set_kernel_smem((const void*)kfn, (int)sm, true)) return e;
    // programmatic dependent launch: the CTAs become resident while the
    // preceding kernel drains and wait for it in griddepcontrol.wait
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = g_pdl_append;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units);
    cfg.blockDim = dim3(fastpack::kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, c, static_cast<const T*>(k_new), static_cast<const T*>(v_new));
}

cudaError_t launch_append(const KittyCacheDesc& c, const void* k_new, const void* v_new, cudaStream_t st) {
    if (c.num_seqs * c.cfg.h_kv == 0) return cudaSuccess;
    return c.row_dtype == KITTY_F32 ? append_t<float>(c, k_new, v_new, st) : append_t<uint16_t>(c, k_new, v_new, st);
}

// KITTY_FAST_PACK=0 keeps prefill on the generic packer (A/B and parity knob)
static const int g_fast_pack = [] {
    const char* e = std::getenv("KITTY_FAST_PACK");
    return e ? std::atoi(e) : 1;
}();

template <typename T>
static cudaError_t prefill_t(const KittyCacheDesc& c, const T* keys, const T* values, int P, cudaStream_t st) {
    const int units = c.num_seqs * c.cfg.h_kv;
    const int S = c.cfg.s, G = c.cfg.g;
    const int past = P > S ? P - S : 0;
    const int kp = past / G;
    const int vp = (past - min(c.cfg.r, past)) / G;
    const int n_fp = min(P, S) + (P > S + vp * G ? P - (S + vp * G) : 0);
    const int gx = n_fp > 0 ? min(n_fp, 1024) : 1;
    prefill_rows_kernel<T><<<dim3(gx, units), 128, 0, st>>>(c, keys, values, P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || kp + vp == 0) return e;
    if constexpr (sizeof(T) == 2) {
        if (c.cfg.d == fastpack::kD && G == fastpack::kG && g_fast_pack && !c.key_meta && !c.value_meta &&
            c.cfg.key_bits == 2 && c.cfg.value_bits == 2) {
            const int sm = static_cast<int>(sizeof(fastpack::Smem));
            if ((e = set_kernel_smem((const void*)prefill_pack_fast_kernel, sm)) != cudaSuccess) return e;
            prefill_pack_fast_kernel<<<dim3(kp + vp, units), fastpack::kThreads, sm, st>>>(c, keys, values, P, kp, vp);
            return cudaGetLastError();
        }
    }
    const size_t sm = pack_smem_bytes(G, c.cfg.d, c.cfg.d_boost, sizeof(T));
    auto kfn = prefill_pack_kernel<T>;
    if ((e = set_kernel_smem((const void*)kfn, (int)sm)) != cudaSuccess) return e;
    kfn<<<dim3(kp + vp, units), 128, sm, st>>>(c, keys, values, P, kp, vp);
    return cudaGetLastError();
}

cudaError_t launch_prefill(const KittyCacheDesc& c, const void* keys, const void* values, int P, cudaStream_t st) {
    if (c.num_seqs * c.cfg.h_kv == 0) return cudaSuccess;
    if (c.row_dtype == KITTY_F32)
        return prefill_t(c, static_cast<const float*>(keys), static_cast<const float*>(values), P, st);
    return prefill_t(c, static_cast<const uint16_t*>(keys), static_cast<const uint16_t*>(values), P, st);
}

cudaError_t launch_release(const KittyCacheDesc& c, int seq0, int nseq, cudaStream_t st) {
    if (nseq <= 0 || c.cfg.h_kv == 0) return cudaSuccess;
    release_kernel<<<nseq * c.cfg.h_kv, 128, 0, st>>>(c, seq0);
    return cudaGetLastError();
}

cudaError_t launch_import_pages(const KittyCacheDesc& c, int u, int kind, const uint8_t* bodies, int first_page,
                                int n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    import_pages_kernel<<<n, 128, 0, st>>>(c, u, kind, bodies, first_page);
    return cudaGetLastError();
}

cudaError_t launch_flatten(const KittyCacheDesc& c, int u, int n, float* ko, float* vo,
                           cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int64_t total = (int64_t)n * c.cfg.d;
    const int64_t want = (total + 255) / 256;
    const int blocks = static_cast<int>(want < 4096 ? want : 4096);
    if (c.row_dtype == KITTY_F32)
        flatten_kernel<float><<<blocks, 256, 0, st>>>(c, u, n, ko, vo);
    else
        flatten_kernel<uint16_t><<<blocks, 256, 0, st>>>(c, u, n, ko, vo);
    return cudaGetLastError();
}

}  // namespace kitty
