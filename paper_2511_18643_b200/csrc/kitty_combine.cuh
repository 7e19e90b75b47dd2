// Split-KV log-sum-exp merge shared by the decode-attention kernels.
//
// A unit's work items each leave a partial record (acc[group][d] = sum p v
// relative to the item's own running max m, then (m, l) per query row, m in
// the log2 domain).  One CTA of kMergeWarps warps merges one (unit, query row):
// every warp folds a strided subset of the records with online rescaling
// (4 records' loads in flight per step), then warp 0 folds the warp states and
// writes out = acc / l -- the softmax normalisation of cache.py:243-248.
#pragma once

#include "kitty_common.cuh"

namespace kitty {

constexpr int kMergeWarps = 16;

__device__ __forceinline__ float merge_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// pb: the unit's first record; stride: floats per record; slot_of(i): record
// index of part i; d = 128 (one float4 per lane).
template <int GROUP, class SlotFn>
__device__ __forceinline__ void lse_merge_row(const float* pb, int stride, int nparts, SlotFn slot_of, int g,
                                              void* out, int out_dtype, int64_t row) {
    constexpr int D = 128;
    __shared__ float s_m[kMergeWarps], s_l[kMergeWarps];
    __shared__ float4 s_acc[kMergeWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float M = -INFINITY, L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i0 = warp; i0 < nparts; i0 += 4 * kMergeWarps) {
        float4 a[4];
        float m[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + j * kMergeWarps;
            if (i < nparts) {
                const float* p = pb + (int64_t)slot_of(i) * stride;
                a[j] = __ldcg(reinterpret_cast<const float4*>(p + g * D) + lane);
                m[j] = __ldcg(p + GROUP * D + 2 * g);
                l[j] = __ldcg(p + GROUP * D + 2 * g + 1);
            } else {
                a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                m[j] = -INFINITY;
                l[j] = 0.f;
            }
        }
        const float mn = fmaxf(fmaxf(M, fmaxf(m[0], m[1])), fmaxf(m[2], m[3]));
        if (mn == -INFINITY) continue;
        const float sc = merge_ex2(M - mn);
        acc.x *= sc;
        acc.y *= sc;
        acc.z *= sc;
        acc.w *= sc;
        L *= sc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float w = merge_ex2(m[j] - mn);
            acc.x = fmaf(w, a[j].x, acc.x);
            acc.y = fmaf(w, a[j].y, acc.y);
            acc.z = fmaf(w, a[j].z, acc.z);
            acc.w = fmaf(w, a[j].w, acc.w);
            L = fmaf(w, l[j], L);
        }
        M = mn;
    }
    s_acc[warp][lane] = acc;
    if (lane == 0) {
        s_m[warp] = M;
        s_l[warp] = L;
    }
    __syncthreads();
    if (warp != 0) return;
    float mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) mt = fmaxf(mt, s_m[w]);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    float lt = 0.f;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) {
        const float wt = s_m[w] == -INFINITY ? 0.f : merge_ex2(s_m[w] - mt);
        const float4 x = s_acc[w][lane];
        o.x = fmaf(wt, x.x, o.x);
        o.y = fmaf(wt, x.y, o.y);
        o.z = fmaf(wt, x.z, o.z);
        o.w = fmaf(wt, x.w, o.w);
        lt = fmaf(wt, s_l[w], lt);
    }
    const float inv = 1.f / lt;
    if (out_dtype == KITTY_F32) {
        reinterpret_cast<float4*>(static_cast<float*>(out) + row * D)[lane] = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
    } else {
        uint2 v;
        v.x = f32_to_bf16_bits(o.x * inv) | (f32_to_bf16_bits(o.y * inv) << 16);
        v.y = f32_to_bf16_bits(o.z * inv) | (f32_to_bf16_bits(o.w * inv) << 16);
        reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + row * D)[lane] = v;
    }
}

}  // namespace kitty
