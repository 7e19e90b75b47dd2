// Declarations shared by the codec / runtime kernels and the C ABI.
#pragma once

#include "kitty_common.cuh"

namespace kitty {

// Shared-memory scratch of one key-page pack: fp64 scores, high-bit row of
// each channel and its boosted flag.
struct PackScratch {
    double* score;  // [d]
    int* pos;       // [d]
    uint8_t* flag;  // [d]
    __host__ __device__ static size_t bytes(int d) { return (size_t)d * 13 + 16; }
};

__host__ __device__ size_t pack_smem_bytes(int g, int d, int d_boost, int elem_bytes);

cudaError_t launch_pack_key_pages(const void* x, int dtype, int P, int g, int d, int d_boost,
                                  const int64_t* sel, uint8_t* slots, int64_t stride, float* sc32,
                                  float* ze32, uint32_t* status, cudaStream_t st);
cudaError_t launch_pack_value_pages(const void* x, int dtype, int P, int g, int d, uint8_t* slots,
                                    int64_t stride, float* sc32, float* ze32, uint32_t* status,
                                    cudaStream_t st);
cudaError_t launch_channel_scores(const void* x, int dtype, int P, int g, int d, double* scores,
                                  cudaStream_t st);
cudaError_t launch_select_boost(const double* scores, int P, int d, int k, int64_t* out,
                                cudaStream_t st);
cudaError_t launch_dequant_key_pages(const uint8_t* slots, int64_t stride, int P, int g, int d,
                                     int d_boost, const float* sc32, const float* ze32, float* out,
                                     uint32_t* status, cudaStream_t st);
cudaError_t launch_dequant_value_pages(const uint8_t* slots, int64_t stride, int P, int g, int d,
                                       const float* sc32, const float* ze32, float* out,
                                       cudaStream_t st);
cudaError_t launch_quantize_lanes(const float* x, int rows, int cols, int per_token, const int32_t* bits,
                                  uint8_t* codes, float* scales, float* zeros, cudaStream_t st);
cudaError_t launch_dequantize_lanes(const uint8_t* codes, int rows, int cols, int per_token, const float* scales,
                                    const float* zeros, float* out, cudaStream_t st);
cudaError_t launch_fake_quantize(const float* x, int rows, int cols, int per_token, const int32_t* bits, float* out,
                                 cudaStream_t st);
cudaError_t launch_append(const KittyCacheDesc& c, const void* k_new, const void* v_new, cudaStream_t st);
cudaError_t launch_prefill(const KittyCacheDesc& c, const void* keys, const void* values, int P, cudaStream_t st);
cudaError_t launch_release(const KittyCacheDesc& c, int seq0, int nseq, cudaStream_t st);
cudaError_t launch_import_pages(const KittyCacheDesc& c, int u, int kind, const uint8_t* bodies, int first_page,
                                int n, cudaStream_t st);
cudaError_t launch_flatten(const KittyCacheDesc& c, int u, int n, float* ko, float* vo,
                           cudaStream_t st);

// analysis (kitty_analysis.cu)
size_t sensitivity_workspace_bytes(int h_q, int lq, int h_kv, int L, int d);
cudaError_t launch_channel_sensitivity(const float* q, int h_q, int lq, const float* keys, int h_kv, int L, int d,
                                       int bits, double* mse, void* ws, cudaStream_t st);
size_t attention_mse_workspace_bytes(int heads, int lq, int L, int d);
cudaError_t launch_attention_mse(const float* keys, int L, int d, const float* q, int heads, int lq,
                                 const int32_t* bits, double* out, void* ws, cudaStream_t st);

// attention (kitty_attention.cu)
size_t attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens);
cudaError_t launch_decode_attention(const KittyCacheDesc& c, const void* q, void* out,
                                    int out_dtype, int max_tokens, void* ws, size_t ws_bytes,
                                    cudaStream_t st);
size_t dense_attention_workspace_bytes(int n_q, int length, int d);
cudaError_t launch_dense_probs(const float* keys, int length, int d, const float* queries, int n_q,
                               const int32_t* kv_map, float* probs, cudaStream_t st);
cudaError_t launch_dense_attention(const float* keys, const float* values, int h_kv, int length,
                                   int d, const float* queries, int n_q, const int32_t* kv_map,
                                   float* out, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace kitty
