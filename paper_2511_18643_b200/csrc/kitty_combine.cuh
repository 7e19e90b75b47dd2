// Split-KV log-sum-exp merge shared by the decode-attention kernels.
//
// A unit's work items each leave a partial record (acc[group][d] = sum p v
// relative to the item's own running max m, then (m, l) per query row, m in
// the log2 domain).  One CTA merges one (unit, query row) (or a channel slice
// of it) into out = acc / l -- the softmax normalisation of cache.py:243-248:
//  * lse_merge_row (long rows, hundreds of parts): the weights 2^(m - max)
//    first (thread = part), then every warp sums a strided subset of the
//    accumulator rows and warp 0 adds the warp sums;
//  * lse_merge_row_1p (<= 128 parts): every lane group keeps a running
//    (max, sum, acc) over its parts, loading (m, l) with the rows in one
//    round trip, and the groups are combined by log-sum-exp at the end.
#pragma once

#include "kitty_common.cuh"

namespace kitty {

constexpr int kMergeWarps = 8;

__device__ __forceinline__ float merge_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// pb: the unit's first record; stride: floats per record; slot_of(i): record
// index of part i; d = 128 (one float4 per lane).
// Thread = part first: (m, l) of every part and the row max, so the weights
// 2^(m - max) are known before the accumulator rows are read; then every warp
// streams a strided subset of the rows (address + weight from shared memory,
// F rows' loads in flight).  Parts are taken in batches of kMaxParts (one
// batch below that: the (m, l) loads of the max pass are reused), so any part
// count is merged -- a 256K-token unit alone on a GPU has ~2 000.
constexpr int kMaxParts = 1024;
// CSPLIT > 1 (long contexts, few rows): the row's channels are split over
// CSPLIT CTAs (`slice` = this CTA's), so a handful of (unit, row) merges still
// fill the GPU; a part's slice is 128 / CSPLIT floats, read by 32 / CSPLIT
// lanes, so a warp covers CSPLIT parts per step.
template <int GROUP, class SlotFn, int WARPS = kMergeWarps, int CSPLIT = 1>
__device__ __forceinline__ void lse_merge_row(const float* pb, int stride, int nparts, SlotFn slot_of, int g,
                                              void* out, int out_dtype, int64_t row, int slice = 0) {
    constexpr int D = 128;
    constexpr int T = WARPS * 32;
    constexpr int F = WARPS == 8 ? 8 : 16;  // accumulator rows in flight per warp
    constexpr int LPP = 32 / CSPLIT;        // lanes per part slice
    __shared__ int s_slot[kMaxParts];
    __shared__ float s_w[kMaxParts];
    __shared__ float s_l[kMaxParts];
    __shared__ float s_red[WARPS];
    __shared__ float s_lsum[WARPS];
    __shared__ float4 s_acc[WARPS][LPP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / LPP, cl = lane - sub * LPP;
    auto load_ml = [&](int i) {
        return __ldcg(reinterpret_cast<const float2*>(pb + (int64_t)slot_of(i) * stride + GROUP * D + 2 * g));
    };
    float mloc = -INFINITY;
    for (int i = threadIdx.x; i < nparts; i += T) {
        const int sl = slot_of(i);
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(pb + (int64_t)sl * stride + GROUP * D + 2 * g));
        if (i < kMaxParts) {
            s_slot[i] = sl;
            s_w[i] = ml.x;
            s_l[i] = ml.y;  // (m, l) in one load: no second round trip for l
        }
        mloc = fmaxf(mloc, ml.x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
    if (lane == 0) s_red[warp] = mloc;
    __syncthreads();
    float M = s_red[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) M = fmaxf(M, s_red[w]);
    float lsum = 0.f;
    const int c0 = slice * (D / CSPLIT);
    const float* rowp = pb + g * D + c0 + 4 * cl;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int b0 = 0; b0 < nparts; b0 += kMaxParts) {
        const int nb = min(kMaxParts, nparts - b0);
        if (b0 > 0) {
            __syncthreads();  // the previous batch's rows are read
            for (int i = threadIdx.x; i < nb; i += T) {
                const float2 ml = load_ml(b0 + i);
                s_slot[i] = slot_of(b0 + i);
                s_w[i] = ml.x;
                s_l[i] = ml.y;
            }
        }
        for (int i = threadIdx.x; i < nb; i += T) {  // this thread's own entries: no barrier needed
            const float m = s_w[i];
            const float w = m == -INFINITY ? 0.f : merge_ex2(m - M);
            s_w[i] = w;
            lsum = fmaf(w, s_l[i], lsum);
        }
        __syncthreads();  // s_w complete
        for (int i0 = warp * CSPLIT + sub; i0 < nb; i0 += F * WARPS * CSPLIT) {
            float4 a[F];
            float w[F];
#pragma unroll
            for (int j = 0; j < F; ++j) {
                const int i = i0 + j * WARPS * CSPLIT;
                const bool ok = i < nb;
                w[j] = ok ? s_w[i] : 0.f;
                a[j] = ok ? __ldcg(reinterpret_cast<const float4*>(rowp + (int64_t)s_slot[i] * stride)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < F; ++j) {
                acc.x = fmaf(w[j], a[j].x, acc.x);
                acc.y = fmaf(w[j], a[j].y, acc.y);
                acc.z = fmaf(w[j], a[j].z, acc.z);
                acc.w = fmaf(w[j], a[j].w, acc.w);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
#pragma unroll
    for (int o = LPP; o < 32; o <<= 1) {  // the warp's CSPLIT parts per step -> one slice sum
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    if (sub == 0) s_acc[warp][cl] = acc;
    if (lane == 0) s_lsum[warp] = lsum;
    __syncthreads();
    if (warp != 0 || lane >= LPP) return;
    float4 o = s_acc[0][lane];
    float lt = s_lsum[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) {
        const float4 x = s_acc[w][lane];
        o.x += x.x;
        o.y += x.y;
        o.z += x.z;
        o.w += x.w;
        lt += s_lsum[w];
    }
    const float inv = 1.f / lt;
    const int64_t ob = row * D + c0 + 4 * lane;
    if (out_dtype == KITTY_F32) {
        *reinterpret_cast<float4*>(static_cast<float*>(out) + ob) = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
    } else {
        uint2 v;
        v.x = f32_to_bf16_bits(o.x * inv) | (f32_to_bf16_bits(o.y * inv) << 16);
        v.y = f32_to_bf16_bits(o.z * inv) | (f32_to_bf16_bits(o.w * inv) << 16);
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + ob) = v;
    }
}

// One-pass variant: every lane group keeps a running (max, sum, acc) over its
// parts, loading each part's (m, l) together with its accumulator slice (one
// round trip per F parts instead of a max pass and a row pass), then the
// groups' partial states are combined by log-sum-exp in shared memory.
template <int GROUP, class SlotFn, int WARPS, int CSPLIT = 1>
__device__ __forceinline__ void lse_merge_row_1p(const float* pb, int stride, int nparts, SlotFn slot_of, int g,
                                                 void* out, int out_dtype, int64_t row, int slice = 0) {
    constexpr int D = 128;
    constexpr int F = GROUP == 8 ? 8 : 16;  // parts in flight per lane group (C2 -0.5 us at 16; C5 +1.8 us)
    constexpr int LPP = 32 / CSPLIT;     // lanes per part slice
    constexpr int NG = WARPS * CSPLIT;   // lane groups in the CTA
    __shared__ float s_m[NG], s_l[NG];
    __shared__ float4 s_acc[NG][LPP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / LPP, cl = lane - sub * LPP;
    const int grp = warp * CSPLIT + sub;
    const int c0 = slice * (D / CSPLIT);
    const float* rowp = pb + g * D + c0 + 4 * cl;
    float m_run = -INFINITY, l_run = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i0 = grp; i0 < nparts; i0 += F * NG) {
        float2 ml[F];
        float4 a[F];
#pragma unroll
        for (int j = 0; j < F; ++j) {
            const int i = i0 + j * NG;
            if (i < nparts) {
                const float* rec = pb + (int64_t)slot_of(i) * stride;
                ml[j] = __ldcg(reinterpret_cast<const float2*>(rec + GROUP * D + 2 * g));
                a[j] = __ldcg(reinterpret_cast<const float4*>(rowp + (rec - pb)));
            } else {
                ml[j] = make_float2(-INFINITY, 0.f);
                a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float mx = m_run;
#pragma unroll
        for (int j = 0; j < F; ++j) mx = fmaxf(mx, ml[j].x);
        if (mx != -INFINITY) {
            const float sc = m_run == -INFINITY ? 0.f : merge_ex2(m_run - mx);
            acc.x *= sc;
            acc.y *= sc;
            acc.z *= sc;
            acc.w *= sc;
            l_run *= sc;
#pragma unroll
            for (int j = 0; j < F; ++j) {
                const float w = ml[j].x == -INFINITY ? 0.f : merge_ex2(ml[j].x - mx);
                l_run = fmaf(w, ml[j].y, l_run);
                acc.x = fmaf(w, a[j].x, acc.x);
                acc.y = fmaf(w, a[j].y, acc.y);
                acc.z = fmaf(w, a[j].z, acc.z);
                acc.w = fmaf(w, a[j].w, acc.w);
            }
            m_run = mx;
        }
    }
    if (cl == 0) {
        s_m[grp] = m_run;
        s_l[grp] = l_run;
    }
    s_acc[grp][cl] = acc;
    __syncthreads();
    if (warp != 0 || lane >= LPP) return;
    float M = -INFINITY;
#pragma unroll
    for (int q = 0; q < NG; ++q) M = fmaxf(M, s_m[q]);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    float lt = 0.f;
#pragma unroll
    for (int q = 0; q < NG; ++q) {
        const float w = s_m[q] == -INFINITY ? 0.f : merge_ex2(s_m[q] - M);
        const float4 x = s_acc[q][lane];
        o.x = fmaf(w, x.x, o.x);
        o.y = fmaf(w, x.y, o.y);
        o.z = fmaf(w, x.z, o.z);
        o.w = fmaf(w, x.w, o.w);
        lt = fmaf(w, s_l[q], lt);
    }
    const float inv = 1.f / lt;
    const int64_t ob = row * D + c0 + 4 * lane;
    if (out_dtype == KITTY_F32) {
        *reinterpret_cast<float4*>(static_cast<float*>(out) + ob) = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
    } else {
        uint2 v;
        v.x = f32_to_bf16_bits(o.x * inv) | (f32_to_bf16_bits(o.y * inv) << 16);
        v.y = f32_to_bf16_bits(o.z * inv) | (f32_to_bf16_bits(o.w * inv) << 16);
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + ob) = v;
    }
}

}  // namespace kitty
