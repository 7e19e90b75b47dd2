// Decode attention over the heterogeneous Kitty store (K4/K5) and the dense
// fp32 oracle_attend on device.
//
// This file holds the GENERIC split-KV path: any (s, r, g, d, group) the
// reference config accepts.  Pages are dequantised on the fly per element
// (Alg. 1 semantics, mul-then-add), logits are float32 / float32(sqrt(d))
// (cache.py:241), softmax is max-subtracted (cache.py:255-258) per split and
// merged across splits by log-sum-exp.  The specialised tensor-core kernel for
// d = g = 128 lives in kitty_attention_fast.cu and is dispatched from
// launch_decode_attention.
#include "kitty_attention.cuh"
#include "kitty_codec.cuh"

namespace kitty {

constexpr int kGenericChunk = 256;  // tokens per split of the generic path
constexpr int kGenericThreads = 128;

// Row element of the cache rows / queries (row_dtype) as float
__device__ __forceinline__ float rowf(const void* p, int64_t i, int f32) {
    return f32 ? static_cast<const float*>(p)[i] : bf16_to_f32(static_cast<const uint16_t*>(p)[i]);
}

// Reads K/V elements of one unit in global token order (cache.py:12-15);
// pages use the f32 metadata side table when the cache keeps one.
struct CacheSource {
    KittyCacheDesc c;
    int u, n, kp, vp;
    __device__ void init(const KittyCacheDesc& cd, int unit, int max_tokens) {
        c = cd;
        u = unit;
        n = min(cd.unit_len[unit], max_tokens);
        const int past = n > cd.cfg.s ? n - cd.cfg.s : 0;
        kp = past / cd.cfg.g;
        vp = (past - min(cd.cfg.r, past)) / cd.cfg.g;
    }
    __device__ float key(int t, int ch) const {
        const int d = c.cfg.d, S = c.cfg.s, G = c.cfg.g;
        const int f32 = c.row_dtype == KITTY_F32;
        if (t < S) return rowf(c.k_sink, ((int64_t)u * S + t) * d + ch, f32);
        const int pc = t - S;
        if (pc < kp * G && c.cfg.key_bits == 16) {  // pass-through page: the block's rows as stored
            const int32_t sl = c.key_block_table[(int64_t)u * c.max_pages + pc / G];
            return rowf(c.key_pool + (int64_t)sl * c.key_slot_bytes, (int64_t)(pc % G) * d + ch, f32);
        }
        if (pc < kp * G) {
            const int p = pc / G, tl = pc % G, gb = G / 4;
            const KeyLayout L{d, G, c.cfg.d_boost};
            const int32_t sl = c.key_block_table[(int64_t)u * c.max_pages + p];
            const uint8_t* slot = c.key_pool + (int64_t)sl * c.key_slot_bytes;
            uint32_t code = (slot[L.dense_off() + ch * gb + tl / 4] >> (2 * (tl % 4))) & 3u;
            const uint8_t r = slot[L.idx_off() + ch];
            if (r != kSentinel) code |= ((slot[L.high_off() + r * gb + tl / 4] >> (2 * (tl % 4))) & 3u) << 2;
            const float* meta = c.key_meta ? c.key_meta + (int64_t)sl * 2 * d : nullptr;
            const float s = meta ? meta[ch] : half_bits_to_f32(ld_u16(slot + L.scale_off() + 2 * ch));
            const float z = meta ? meta[d + ch] : half_bits_to_f32(ld_u16(slot + L.zero_off() + 2 * ch));
            return __fadd_rn(__fmul_rn(static_cast<float>(code), s), z);
        }
        return rowf(c.k_qbuf, ((int64_t)u * G + pc % G) * d + ch, f32);
    }
    __device__ float val(int t, int ch) const {
        const int d = c.cfg.d, S = c.cfg.s, G = c.cfg.g, W = c.cfg.r + c.cfg.g;
        const int f32 = c.row_dtype == KITTY_F32;
        if (t < S) return rowf(c.v_sink, ((int64_t)u * S + t) * d + ch, f32);
        const int pc = t - S;
        if (pc < vp * G && c.cfg.value_bits == 16) {
            const int32_t sl = c.value_block_table[(int64_t)u * c.max_pages + pc / G];
            return rowf(c.value_pool + (int64_t)sl * c.value_slot_bytes, (int64_t)(pc % G) * d + ch, f32);
        }
        if (pc < vp * G) {
            const int p = pc / G, tl = pc % G;
            const ValueLayout L{d, G};
            const int32_t sl = c.value_block_table[(int64_t)u * c.max_pages + p];
            const uint8_t* slot = c.value_pool + (int64_t)sl * c.value_slot_bytes;
            const uint32_t code = (slot[L.codes_off() + tl * (d / 4) + ch / 4] >> (2 * (ch % 4))) & 3u;
            const float* meta = c.value_meta ? c.value_meta + (int64_t)sl * 2 * G : nullptr;
            const float s = meta ? meta[tl] : half_bits_to_f32(ld_u16(slot + L.scale_off() + 2 * tl));
            const float z = meta ? meta[G + tl] : half_bits_to_f32(ld_u16(slot + L.zero_off() + 2 * tl));
            return __fadd_rn(__fmul_rn(static_cast<float>(code), s), z);
        }
        return rowf(c.v_ring, ((int64_t)u * W + pc % W) * d + ch, f32);
    }
};

struct DenseSource {
    const float* k;
    const float* v;
    int d, n;
    __device__ float key(int t, int ch) const { return k[(int64_t)t * d + ch]; }
    __device__ float val(int t, int ch) const { return v[(int64_t)t * d + ch]; }
};

// One CTA = one (unit, split): tokens [split * chunk, min(n, (split + 1) * chunk)).
// Writes the split's max m, sum l and unnormalised accumulator to the workspace.
template <typename Src>
__device__ void attend_split(const Src& src, int n, int d, int group, const float* qs,
                             float sqrt_d, float* logit, float* ws_acc, float* ws_ml) {
    const int split = blockIdx.x;
    const int t0 = split * kGenericChunk;
    const int t1 = min(n, t0 + kGenericChunk);
    const int cnt = t1 - t0;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    if (cnt <= 0) {
        for (int g = tid; g < group; g += nt) {
            ws_ml[2 * g] = -INFINITY;
            ws_ml[2 * g + 1] = 0.f;
        }
        for (int i = tid; i < group * d; i += nt) ws_acc[i] = 0.f;
        return;
    }
    // logits (cache.py:241): float32 dot products / float32(sqrt(d))
    for (int i = tid; i < cnt; i += nt) {
        const int t = t0 + i;
        for (int g0 = 0; g0 < group; g0 += 8) {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const int gn = min(8, group - g0);
            for (int ch = 0; ch < d; ++ch) {
                const float kv = src.key(t, ch);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < gn) acc[j] = fmaf(qs[(g0 + j) * d + ch], kv, acc[j]);
            }
            for (int j = 0; j < gn; ++j) logit[(g0 + j) * kGenericChunk + i] = __fdiv_rn(acc[j], sqrt_d);
        }
    }
    __syncthreads();
    // max-subtracted exponentials (cache.py:255-258), one warp per query row
    for (int g = warp; g < group; g += nw) {
        float* row = logit + g * kGenericChunk;
        float m = -INFINITY;
        for (int i = lane; i < cnt; i += 32) m = fmaxf(m, row[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float l = 0.f;
        for (int i = lane; i < cnt; i += 32) {
            const float e = expf(row[i] - m);
            row[i] = e;
            l += e;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) {
            ws_ml[2 * g] = m;
            ws_ml[2 * g + 1] = l;
        }
    }
    __syncthreads();
    // p^T @ V over the split (cache.py:245-248)
    for (int i = tid; i < group * d; i += nt) {
        const int g = i / d, ch = i % d;
        const float* p = logit + g * kGenericChunk;
        float acc = 0.f;
        for (int j = 0; j < cnt; ++j) acc = fmaf(p[j], src.val(t0 + j, ch), acc);
        ws_acc[i] = acc;
    }
}

__global__ void attention_generic_kernel(KittyCacheDesc c, const void* q, int splits, int max_tokens,
                                         float* ws_acc, float* ws_ml) {
    extern __shared__ __align__(16) float gsm[];
    const int u = blockIdx.y;
    const int d = c.cfg.d, group = c.cfg.h_q / c.cfg.h_kv;
    const int b = u / c.cfg.h_kv, h = u % c.cfg.h_kv;
    float* qs = gsm;                    // [group][d]
    float* logit = gsm + group * d;     // [group][chunk]
    const int64_t q0 = ((int64_t)b * c.cfg.h_q + (int64_t)h * group) * d;
    for (int i = threadIdx.x; i < group * d; i += blockDim.x) qs[i] = rowf(q, q0 + i, c.row_dtype == KITTY_F32);
    CacheSource src;
    src.init(c, u, max_tokens);
    if (blockIdx.x == 0 && threadIdx.x == 0 && c.unit_len[u] > max_tokens) set_status(c.status, KITTY_STATUS_LENGTH);
    __syncthreads();
    const float sqrt_d = static_cast<float>(sqrt(static_cast<double>(d)));
    const int64_t slot = (int64_t)u * splits + blockIdx.x;
    attend_split(src, src.n, d, group, qs, sqrt_d, logit, ws_acc + slot * group * d,
                 ws_ml + slot * group * 2);
}

__global__ void attention_dense_kernel(const float* keys, const float* values, int length, int d,
                                       const float* queries, const int32_t* kv_map, int splits,
                                       float* ws_acc, float* ws_ml) {
    extern __shared__ __align__(16) float gsm[];
    const int i = blockIdx.y;  // query index: one "unit" per query (group 1)
    float* qs = gsm;
    float* logit = gsm + d;
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) qs[ch] = queries[(int64_t)i * d + ch];
    const int h = kv_map[i];
    DenseSource src{keys + (int64_t)h * length * d, values + (int64_t)h * length * d, d, length};
    __syncthreads();
    const float sqrt_d = static_cast<float>(sqrt(static_cast<double>(d)));
    const int64_t slot = (int64_t)i * splits + blockIdx.x;
    attend_split(src, length, d, 1, qs, sqrt_d, logit, ws_acc + slot * d, ws_ml + slot * 2);
}

// K5: log-sum-exp merge of the splits of every (unit, query row).
// out row r of unit u goes to out_base(u) + r * d.
__global__ void combine_kernel(const float* ws_acc, const float* ws_ml, int splits, int group,
                               int d, int h_kv, int h_q, int dense, void* out, int out_dtype) {
    const int u = blockIdx.x;
    for (int i = threadIdx.x; i < group * d; i += blockDim.x) {
        const int g = i / d, ch = i % d;
        float m = -INFINITY;
        for (int s = 0; s < splits; ++s) m = fmaxf(m, ws_ml[(((int64_t)u * splits + s) * group + g) * 2]);
        float l = 0.f, acc = 0.f;
        for (int s = 0; s < splits; ++s) {
            const int64_t base = ((int64_t)u * splits + s) * group + g;
            const float ms = ws_ml[base * 2];
            if (ms == -INFINITY) continue;
            const float w = expf(ms - m);
            l += ws_ml[base * 2 + 1] * w;
            acc += ws_acc[base * d + ch] * w;
        }
        const float o = l > 0.f ? acc / l : 0.f;  // an empty (retired) unit: zero rows
        int64_t row;
        if (dense) {
            row = u;
        } else {
            const int b = u / h_kv, h = u % h_kv;
            row = (int64_t)b * h_q + (int64_t)h * group + g;
        }
        if (out_dtype == KITTY_F32)
            static_cast<float*>(out)[row * d + ch] = o;
        else
            static_cast<uint16_t*>(out)[row * d + ch] = f32_to_bf16_bits(o);
    }
}

static int generic_splits(int max_tokens) {
    return max_tokens <= 0 ? 1 : (max_tokens + kGenericChunk - 1) / kGenericChunk;
}

size_t attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens) {
    const int units = c.num_seqs * c.cfg.h_kv;
    const int group = c.cfg.h_q / c.cfg.h_kv;
    size_t generic = (size_t)units * generic_splits(max_tokens) * group * (c.cfg.d + 2) * sizeof(float);
    size_t fast = fast_attention_workspace_bytes(c, max_tokens);
    return generic > fast ? generic : fast;
}

cudaError_t launch_decode_attention(const KittyCacheDesc& c, const void* q, void* out,
                                    int out_dtype, int max_tokens, void* ws, size_t ws_bytes,
                                    cudaStream_t st) {
    const int units = c.num_seqs * c.cfg.h_kv;
    if (units == 0) return cudaSuccess;
    // d = g = 128, GQA groups 1/2/4/8: the fused tensor-core kernel
    if (fast_attention_supported(c))
        return launch_fast_attention(c, static_cast<const uint16_t*>(q), out, out_dtype, max_tokens, ws, ws_bytes, st);
    const int group = c.cfg.h_q / c.cfg.h_kv;
    const int d = c.cfg.d;
    const int splits = generic_splits(max_tokens);
    const size_t need = (size_t)units * splits * group * (d + 2) * sizeof(float);
    if (ws_bytes < need) return cudaErrorInvalidValue;
    float* ws_acc = static_cast<float*>(ws);
    float* ws_ml = ws_acc + (size_t)units * splits * group * d;
    const size_t sm = ((size_t)group * d + (size_t)group * kGenericChunk) * sizeof(float);
    if (cudaError_t e0 = set_kernel_smem((const void*)attention_generic_kernel, (int)sm)) return e0;
    attention_generic_kernel<<<dim3(splits, units), kGenericThreads, sm, st>>>(c, q, splits, max_tokens, ws_acc, ws_ml);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    combine_kernel<<<units, 128, 0, st>>>(ws_acc, ws_ml, splits, group, d, c.cfg.h_kv, c.cfg.h_q, 0, out, out_dtype);
    return cudaGetLastError();
}

// The attention probabilities of dense f32 keys (cache.py:241-244,252 and
// oracle_attend's probs, cache.py:291-299): one CTA per query row; logits =
// (k . q) / f32(sqrt d) as the generic kernel computes them, then the
// max-subtracted exponentials (expf) over their sum.  The row of `probs`
// holds the logits, then the exponentials, then the probabilities.
__global__ void dense_probs_kernel(const float* keys, int length, int d, const float* queries,
                                   const int32_t* kv_map, float* probs) {
    extern __shared__ __align__(16) float qsm[];
    __shared__ float red[32];
    const int i = blockIdx.x, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    for (int ch = tid; ch < d; ch += nt) qsm[ch] = queries[(int64_t)i * d + ch];
    __syncthreads();
    const float* kb = keys + (int64_t)kv_map[i] * length * d;
    float* row = probs + (int64_t)i * length;
    const float sqrt_d = static_cast<float>(sqrt(static_cast<double>(d)));
    float m = -INFINITY;
    for (int t = tid; t < length; t += nt) {
        float acc = 0.f;
        for (int ch = 0; ch < d; ++ch) acc = fmaf(qsm[ch], kb[(int64_t)t * d + ch], acc);
        const float l = __fdiv_rn(acc, sqrt_d);
        row[t] = l;
        m = fmaxf(m, l);
    }
    auto block_reduce = [&](float v, bool is_max) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float w = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmaxf(v, w) : v + w;
        }
        __syncthreads();
        if (lane == 0) red[warp] = v;
        __syncthreads();
        v = red[0];
        for (int w = 1; w < (nt + 31) / 32; ++w) v = is_max ? fmaxf(v, red[w]) : v + red[w];
        return v;
    };
    m = block_reduce(m, true);
    float sum = 0.f;
    for (int t = tid; t < length; t += nt) {
        const float e = expf(row[t] - m);
        row[t] = e;
        sum += e;
    }
    sum = block_reduce(sum, false);
    for (int t = tid; t < length; t += nt) row[t] = __fdiv_rn(row[t], sum);
}

cudaError_t launch_dense_probs(const float* keys, int length, int d, const float* queries, int n_q,
                               const int32_t* kv_map, float* probs, cudaStream_t st) {
    if (n_q == 0 || length == 0) return cudaSuccess;
    const int sm = d * static_cast<int>(sizeof(float));
    if (cudaError_t e = set_kernel_smem((const void*)dense_probs_kernel, sm)) return e;
    dense_probs_kernel<<<n_q, 256, sm, st>>>(keys, length, d, queries, kv_map, probs);
    return cudaGetLastError();
}

size_t dense_attention_workspace_bytes(int n_q, int length, int d) {
    return (size_t)n_q * generic_splits(length) * (d + 2) * sizeof(float);
}

cudaError_t launch_dense_attention(const float* keys, const float* values, int h_kv, int length,
                                   int d, const float* queries, int n_q, const int32_t* kv_map,
                                   float* out, void* ws, size_t ws_bytes, cudaStream_t st) {
    (void)h_kv;
    if (n_q == 0) return cudaSuccess;
    const int splits = generic_splits(length);
    if (ws_bytes < dense_attention_workspace_bytes(n_q, length, d)) return cudaErrorInvalidValue;
    float* ws_acc = static_cast<float*>(ws);
    float* ws_ml = ws_acc + (size_t)n_q * splits * d;
    const size_t sm = ((size_t)d + kGenericChunk) * sizeof(float);
    if (cudaError_t e0 = set_kernel_smem((const void*)attention_dense_kernel, (int)sm)) return e0;
    attention_dense_kernel<<<dim3(splits, n_q), kGenericThreads, sm, st>>>(keys, values, length, d, queries, kv_map, splits, ws_acc, ws_ml);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    combine_kernel<<<n_q, 128, 0, st>>>(ws_acc, ws_ml, splits, 1, d, 1, 1, 1, out, KITTY_F32);
    return cudaGetLastError();
}

}  // namespace kitty
