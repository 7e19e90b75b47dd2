// Channel-sensitivity and boost-sweep analysis on the device (SURVEY 8(f)
// row 4): the attention-probability MSE of quantizing key channels, in fp64
// like the reference (analysis.py:63-104 channel_sensitivity, :119-142
// attention_mse).
//
// Shapes: queries [h_q][lq][d] f32, keys [h_kv][L][d] f32; query head qh reads
// KV head qh / (h_q / h_kv).  Every probability row is produced by ONE warp
// routine (row_pass): the max, then Z = sum exp(l - max) in a fixed order
// (lane-strided partial sums, then a fixed shuffle tree), then p = exp(l -
// max) / Z -- so a channel whose quantization leaves the keys unchanged (a
// constant channel, bits 16) reproduces the baseline row bit for bit and its
// MSE is exactly 0, as in the reference (test_analysis.py:32-47).
//
// channel_sensitivity: for every (query head, channel) the perturbed logits
// are the rank-1 update base + (q[:, ch] delta[:, ch]) / sqrt(d)
// (analysis.py:98-100); one warp per (row, channel): two passes over the
// row's L logits (max, Z), a third for sum (p' - p)^2.
#include <cmath>

#include "kitty_codec.cuh"

namespace kitty {
namespace analysis {

constexpr int kWarps = 8;

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// logits[qh][i][j] = (q[qh][i] . k[kv][j]) / sqrt(d) in fp64 (analysis.py:95,
// :135-137): one CTA per (row i, query head qh), q row staged as doubles.
__global__ void logits_kernel(const float* q, int lq, const float* k, int L, int d, int group, double inv_sqrt_d,
                              double* logits) {
    extern __shared__ double qs[];
    const int i = blockIdx.x, qh = blockIdx.y, kv = qh / group;
    const float* qr = q + ((int64_t)qh * lq + i) * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = static_cast<double>(qr[c]);
    __syncthreads();
    const float* kb = k + (int64_t)kv * L * d;
    double* out = logits + ((int64_t)qh * lq + i) * L;
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        const float* kr = kb + (int64_t)j * d;
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc = fma(qs[c], static_cast<double>(kr[c]), acc);
        out[j] = acc * inv_sqrt_d;
    }
}

// One softmax row, optionally perturbed: l_j = base_j + (a delta_j) inv
// (delta == nullptr: l_j = base_j).  Returns, per lane, nothing; the warp gets
// (m, Z).  Deterministic order.
struct RowStats {
    double m, z;
};
__device__ __forceinline__ double row_logit(const double* base, const double* delta, double a, double inv, int j) {
    return delta ? base[j] + (a * delta[j]) * inv : base[j];
}
__device__ RowStats row_stats(const double* base, const double* delta, double a, double inv, int L, int lane) {
    double m = -INFINITY;
    for (int j = lane; j < L; j += 32) m = fmax(m, row_logit(base, delta, a, inv, j));
    m = warp_max(m);
    double z = 0.0;
    for (int j = lane; j < L; j += 32) z += exp(row_logit(base, delta, a, inv, j) - m);
    return RowStats{m, warp_sum(z)};
}

// Baseline probabilities of every row: probs[r][j] (one warp per row).
__global__ void probs_kernel(const double* logits, int rows, int L, double* probs) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (r >= rows) return;
    const double* base = logits + (int64_t)r * L;
    const RowStats s = row_stats(base, nullptr, 0.0, 0.0, L, lane);
    double* p = probs + (int64_t)r * L;
    for (int j = lane; j < L; j += 32) p[j] = exp(base[j] - s.m) / s.z;
}

// delta_t[kv][ch][j] = quantized[kv][j][ch] - keys[kv][j][ch] in fp64
// (analysis.py:94), channel-major so a warp reads a channel's column coalesced.
__global__ void delta_kernel(const float* quant, const float* keys, int h_kv, int L, int d, double* delta_t) {
    const int64_t total = (int64_t)h_kv * L * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kv = e / ((int64_t)L * d), rem = e - kv * L * d;
        const int j = static_cast<int>(rem / d), ch = static_cast<int>(rem - (int64_t)j * d);
        delta_t[(kv * d + ch) * L + j] = static_cast<double>(quant[e]) - static_cast<double>(keys[e]);
    }
}

// Sum over j of (p'_j - p_j)^2 for the rank-1 perturbation of channel ch of
// row (qh, i): out[(qh d + ch) lq + i].  One warp per (row, channel).
__global__ void sensitivity_rows_kernel(const float* q, int lq, int L, int d, int group, double inv,
                                        const double* logits, const double* probs, const double* delta_t,
                                        double* out) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x, qh = blockIdx.y, kv = qh / group;
    const int64_t row = (int64_t)qh * lq + i;
    const double* base = logits + row * L;
    const double* p = probs + row * L;
    for (int ch = threadIdx.x >> 5; ch < d; ch += kWarps) {
        const double a = static_cast<double>(q[row * d + ch]);
        const double* dl = delta_t + ((int64_t)kv * d + ch) * L;
        const RowStats s = row_stats(base, dl, a, inv, L, lane);
        double acc = 0.0;
        for (int j = lane; j < L; j += 32) {
            const double e = exp(row_logit(base, dl, a, inv, j) - s.m) / s.z - p[j];
            acc = fma(e, e, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) out[((int64_t)qh * d + ch) * lq + i] = acc;
    }
}

// out[r] = sum_j (pa[r][j] - pb[r][j])^2, one warp per row.
__global__ void sqdiff_rows_kernel(const double* pa, const double* pb, int rows, int L, double* out) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (r >= rows) return;
    double acc = 0.0;
    for (int j = lane; j < L; j += 32) {
        const double e = pa[(int64_t)r * L + j] - pb[(int64_t)r * L + j];
        acc = fma(e, e, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) out[r] = acc;
}

// out[g] = (sum of x[g n .. g n + n)) / denom, one thread per group, in order.
__global__ void group_mean_kernel(const double* x, int groups, int n, double denom, double* out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[(int64_t)g * n + i];
    out[g] = s / denom;
}

// out[0] = mean over heads of the per-head means (analysis.py:138-142).
__global__ void heads_mean_kernel(const double* per_head, int heads, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t = 0.0;
    for (int h = 0; h < heads; ++h) t += per_head[h];
    out[0] = t / heads;
}

__global__ void fill_bits_kernel(int32_t* bits, int n, int v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) bits[i] = v;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace analysis

using namespace analysis;

size_t sensitivity_workspace_bytes(int h_q, int lq, int h_kv, int L, int d) {
    const size_t rows = (size_t)h_q * lq;
    return align256(rows * L * 8) * 2                 // logits, probs
           + align256((size_t)h_kv * d * L * 8)       // delta_t
           + align256((size_t)h_kv * L * d * 4)       // quantized keys
           + align256((size_t)h_q * d * lq * 8)       // per-row sums
           + align256((size_t)d * 4);                 // bits
}

cudaError_t launch_channel_sensitivity(const float* q, int h_q, int lq, const float* keys, int h_kv, int L, int d,
                                       int bits, double* mse, void* ws, cudaStream_t st) {
    const int group = h_q / h_kv;
    const size_t rows = (size_t)h_q * lq;
    uint8_t* w = static_cast<uint8_t*>(ws);
    double* logits = reinterpret_cast<double*>(w);
    w += align256(rows * L * 8);
    double* probs = reinterpret_cast<double*>(w);
    w += align256(rows * L * 8);
    double* delta_t = reinterpret_cast<double*>(w);
    w += align256((size_t)h_kv * d * L * 8);
    float* quant = reinterpret_cast<float*>(w);
    w += align256((size_t)h_kv * L * d * 4);
    double* rowsum = reinterpret_cast<double*>(w);
    w += align256((size_t)h_q * d * lq * 8);
    int32_t* bits_arr = reinterpret_cast<int32_t*>(w);
    const double inv = 1.0 / std::sqrt(static_cast<double>(d));
    fill_bits_kernel<<<1, 128, 0, st>>>(bits_arr, d, bits);
    for (int kv = 0; kv < h_kv; ++kv) {  // fake_quantize_matrix(keys[kv], "per_channel", bits) (analysis.py:93)
        cudaError_t e = launch_fake_quantize(keys + (int64_t)kv * L * d, L, d, 0, bits_arr,
                                             quant + (int64_t)kv * L * d, st);
        if (e != cudaSuccess) return e;
    }
    delta_kernel<<<1184, 256, 0, st>>>(quant, keys, h_kv, L, d, delta_t);
    logits_kernel<<<dim3(lq, h_q), 128, d * sizeof(double), st>>>(q, lq, keys, L, d, group, inv, logits);
    probs_kernel<<<(unsigned)((rows + kWarps - 1) / kWarps), kWarps * 32, 0, st>>>(logits, (int)rows, L, probs);
    sensitivity_rows_kernel<<<dim3(lq, h_q), kWarps * 32, 0, st>>>(q, lq, L, d, group, inv, logits, probs, delta_t,
                                                                   rowsum);
    // mse[qh][ch] = mean over the (lq, L) probability matrix (analysis.py:101)
    group_mean_kernel<<<(h_q * d + 127) / 128, 128, 0, st>>>(rowsum, h_q * d, lq, static_cast<double>(lq) * L, mse);
    return cudaGetLastError();
}

size_t attention_mse_workspace_bytes(int heads, int lq, int L, int d) {
    const size_t rows = (size_t)heads * lq;
    return align256(rows * L * 8) * 3 + align256((size_t)L * d * 4) + align256(rows * 8) + align256((size_t)heads * 8);
}

cudaError_t launch_attention_mse(const float* keys, int L, int d, const float* q, int heads, int lq,
                                 const int32_t* bits, double* out, void* ws, cudaStream_t st) {
    const size_t rows = (size_t)heads * lq;
    uint8_t* w = static_cast<uint8_t*>(ws);
    double* logits = reinterpret_cast<double*>(w);
    w += align256(rows * L * 8);
    double* base = reinterpret_cast<double*>(w);
    w += align256(rows * L * 8);
    double* pert = reinterpret_cast<double*>(w);
    w += align256(rows * L * 8);
    float* quant = reinterpret_cast<float*>(w);
    w += align256((size_t)L * d * 4);
    double* rowsum = reinterpret_cast<double*>(w);
    w += align256(rows * 8);
    double* per_head = reinterpret_cast<double*>(w);
    const double inv = 1.0 / std::sqrt(static_cast<double>(d));
    const unsigned pg = (unsigned)((rows + kWarps - 1) / kWarps);
    // widths: 4 bits for the selection, 2 elsewhere (analysis.py:131-134)
    cudaError_t e = launch_fake_quantize(keys, L, d, 0, bits, quant, st);
    if (e != cudaSuccess) return e;
    logits_kernel<<<dim3(lq, heads), 128, d * sizeof(double), st>>>(q, lq, keys, L, d, heads, inv, logits);
    probs_kernel<<<pg, kWarps * 32, 0, st>>>(logits, (int)rows, L, base);
    logits_kernel<<<dim3(lq, heads), 128, d * sizeof(double), st>>>(q, lq, quant, L, d, heads, inv, logits);
    probs_kernel<<<pg, kWarps * 32, 0, st>>>(logits, (int)rows, L, pert);
    sqdiff_rows_kernel<<<pg, kWarps * 32, 0, st>>>(pert, base, (int)rows, L, rowsum);
    group_mean_kernel<<<(heads + 127) / 128, 128, 0, st>>>(rowsum, heads, lq, static_cast<double>(lq) * L, per_head);
    heads_mean_kernel<<<1, 32, 0, st>>>(per_head, heads, out);
    return cudaGetLastError();
}

}  // namespace kitty
