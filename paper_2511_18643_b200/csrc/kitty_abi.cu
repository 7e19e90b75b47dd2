// extern "C" entry points of libkitty_b200.so (declared in include/kitty_b200.h).
// Each validates its arguments the way the replaced reference function does,
// launches on the caller's stream and returns a KittyStatus.
#include <cstdio>

#include <nvtx3/nvToolsExt.h>

#include "kitty_attention.cuh"
#include "kitty_codec.cuh"

namespace {

thread_local char g_last_error[256] = "";

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return KITTY_OK;
    std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e));
    return KITTY_ERR_CUDA;
}

int invalid(const char* msg, int code = KITTY_ERR_INVALID) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
    return code;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// NVTX range around every compute entry point (host-side enqueue; shows the
// append / pack / attend phases on an Nsight timeline; a no-op without a tool)
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

int check_page_shape(int num_pages, int g, int d) {
    if (num_pages < 0) return invalid("num_pages must be >= 0");
    if (g <= 0 || g % 4 != 0) return invalid("page token count g must be a positive multiple of 4");
    if (d <= 0 || d % 4 != 0) return invalid("channel count d must be a positive multiple of 4");
    if ((size_t)g * d * 4 + 4096 > 200 * 1024) return invalid("page too large for one CTA", KITTY_ERR_UNSUPPORTED);
    return KITTY_OK;
}

int check_cache(const KittyCacheDesc* c) {
    if (!c) return invalid("null cache descriptor");
    const int rc = kitty_validate_config(&c->cfg);
    if (rc != KITTY_OK) return rc;
    if (c->num_seqs < 0 || c->max_pages < 0) return invalid("bad batch geometry");
    // a 2-bit page slot is its KTYP body; a pass-through page slot holds g rows of the row dtype
    const int64_t rows = (int64_t)c->cfg.g * c->cfg.d * (c->row_dtype == KITTY_F32 ? 4 : 2);
    if (c->key_slot_bytes != (c->cfg.key_bits == 16 ? rows : kitty_key_slot_bytes(c->cfg.d, c->cfg.g, c->cfg.d_boost)) ||
        c->value_slot_bytes != (c->cfg.value_bits == 16 ? rows : kitty_value_slot_bytes(c->cfg.d, c->cfg.g)))
        return invalid("slot sizes do not match the page layout");
    if (c->row_dtype != KITTY_BF16 && c->row_dtype != KITTY_F32) return invalid("row_dtype must be KITTY_BF16 or KITTY_F32");
    if ((c->key_free == nullptr) != (c->value_free == nullptr)) return invalid("a page pool needs both free stacks");
    if (c->key_free && (!c->free_top || c->key_slots < 0 || c->value_slots < 0)) return invalid("bad page pool");
    return KITTY_OK;
}

}  // namespace

extern "C" {

int64_t kitty_key_slot_bytes(int32_t d, int32_t g, int32_t d_boost) {
    return kitty::KeyLayout{d, g, d_boost}.bytes();
}

int64_t kitty_value_slot_bytes(int32_t d, int32_t g) { return kitty::ValueLayout{d, g}.bytes(); }

int kitty_validate_config(const KittyConfigC* c) {
    if (!c) return invalid("null config", KITTY_ERR_CONFIG);
    // config.py:35-53
    if (c->s < 0) return invalid("sink size s must be >= 0", KITTY_ERR_CONFIG);
    if (c->r < 1) return invalid("local window r must be >= 1", KITTY_ERR_CONFIG);
    if (c->g < 1 || c->g % 4 != 0) return invalid("group size g must be a positive multiple of 4", KITTY_ERR_CONFIG);
    if (c->d < 1 || c->d % 4 != 0) return invalid("head size d must be a positive multiple of 4", KITTY_ERR_CONFIG);
    if (c->h_kv < 1 || c->h_q < 1 || c->h_q % c->h_kv != 0) return invalid("h_q must be a positive multiple of h_kv", KITTY_ERR_CONFIG);
    if ((c->key_bits != 2 && c->key_bits != 16) || (c->value_bits != 2 && c->value_bits != 16))
        return invalid("key/value bits must be in (2, 16)", KITTY_ERR_CONFIG);
    if (c->d_boost < 0 || c->d_boost > c->d) return invalid("d_boost outside [0, d]", KITTY_ERR_CONFIG);
    if (c->d_boost > 255) return invalid("d_boost exceeds the uint8 boost-index space", KITTY_ERR_CONFIG);
    // device limits (pass-through 16-bit pages run on the generic kernels)
    if ((size_t)c->g * c->d * 2 + 8192 > 200 * 1024) return invalid("page too large for one CTA", KITTY_ERR_UNSUPPORTED);
    return KITTY_OK;
}

const char* kitty_version(void) { return "kitty-b200 0.1.0 (sm_100a)"; }

const char* kitty_last_error(void) { return g_last_error; }

int kitty_channel_scores(const void* x, int32_t dtype, int32_t num_pages, int32_t g, int32_t d,
                         double* scores, void* stream) {
    Range nvtx_range("kitty_channel_scores");
    if (num_pages < 0 || g < 1 || d < 1) return invalid("scores need a (tokens, channels) matrix with tokens >= 1");
    return cuda_status(kitty::launch_channel_scores(x, dtype, num_pages, g, d, scores, as_stream(stream)));
}

int kitty_select_boost(const double* scores, int32_t num_pages, int32_t d, int32_t k,
                       int64_t* boosted, void* stream) {
    Range nvtx_range("kitty_select_boost");
    if (num_pages < 0 || d < 0 || k < 0 || k > d) return invalid("bad selection size");
    return cuda_status(kitty::launch_select_boost(scores, num_pages, d, k, boosted, as_stream(stream)));
}

int kitty_pack_key_pages(const void* x, int32_t dtype, int32_t num_pages, int32_t g, int32_t d,
                         int32_t d_boost, const int64_t* boosted, uint8_t* slots,
                         int64_t slot_stride, float* scales_f32, float* zeros_f32,
                         uint32_t* status, void* stream) {
    Range nvtx_range("kitty_pack_key_pages");
    int rc = check_page_shape(num_pages, g, d);
    if (rc != KITTY_OK) return rc;
    if (d_boost < 0 || d_boost > d) return invalid("boost selection indexes a channel outside the page");
    if (d_boost > 255) return invalid("d_boost exceeds the uint8 index space");
    if (slot_stride < kitty_key_slot_bytes(d, g, d_boost)) return invalid("slot stride smaller than a key page");
    return cuda_status(kitty::launch_pack_key_pages(x, dtype, num_pages, g, d, d_boost, boosted, slots,
                                                    slot_stride, scales_f32, zeros_f32, status,
                                                    as_stream(stream)));
}

int kitty_pack_value_pages(const void* x, int32_t dtype, int32_t num_pages, int32_t g, int32_t d,
                           uint8_t* slots, int64_t slot_stride, float* scales_f32,
                           float* zeros_f32, uint32_t* status, void* stream) {
    Range nvtx_range("kitty_pack_value_pages");
    int rc = check_page_shape(num_pages, g, d);
    if (rc != KITTY_OK) return rc;
    if (slot_stride < kitty_value_slot_bytes(d, g)) return invalid("slot stride smaller than a value page");
    return cuda_status(kitty::launch_pack_value_pages(x, dtype, num_pages, g, d, slots, slot_stride,
                                                      scales_f32, zeros_f32, status, as_stream(stream)));
}

int kitty_dequant_key_pages(const uint8_t* slots, int64_t slot_stride, int32_t num_pages, int32_t g,
                            int32_t d, int32_t d_boost, const float* scales_f32,
                            const float* zeros_f32, float* out, uint32_t* status, void* stream) {
    Range nvtx_range("kitty_dequant_key_pages");
    int rc = check_page_shape(num_pages, g, d);
    if (rc != KITTY_OK) return rc;
    if (d_boost < 0 || d_boost > 255) return invalid("bad d_boost");
    return cuda_status(kitty::launch_dequant_key_pages(slots, slot_stride, num_pages, g, d, d_boost,
                                                       scales_f32, zeros_f32, out, status,
                                                       as_stream(stream)));
}

int kitty_dequant_value_pages(const uint8_t* slots, int64_t slot_stride, int32_t num_pages,
                              int32_t g, int32_t d, const float* scales_f32,
                              const float* zeros_f32, float* out, void* stream) {
    Range nvtx_range("kitty_dequant_value_pages");
    int rc = check_page_shape(num_pages, g, d);
    if (rc != KITTY_OK) return rc;
    return cuda_status(kitty::launch_dequant_value_pages(slots, slot_stride, num_pages, g, d,
                                                         scales_f32, zeros_f32, out, as_stream(stream)));
}

int kitty_quantize_lanes(const float* x, int32_t rows, int32_t cols, int32_t per_token, const int32_t* bits,
                         uint8_t* codes, float* scales, float* zeros, void* stream) {
    Range nvtx_range("kitty_quantize_lanes");
    if (rows < 0 || cols < 0) return invalid("quantize_values needs a 2-D matrix");
    return cuda_status(kitty::launch_quantize_lanes(x, rows, cols, per_token, bits, codes, scales, zeros,
                                                    as_stream(stream)));
}

int kitty_dequantize_lanes(const uint8_t* codes, int32_t rows, int32_t cols, int32_t per_token, const float* scales,
                           const float* zeros, float* out, void* stream) {
    Range nvtx_range("kitty_dequantize_lanes");
    if (rows < 0 || cols < 0) return invalid("dequantize_values needs a 2-D matrix");
    return cuda_status(kitty::launch_dequantize_lanes(codes, rows, cols, per_token, scales, zeros, out,
                                                      as_stream(stream)));
}

int kitty_fake_quantize(const float* x, int32_t rows, int32_t cols, int32_t per_token, const int32_t* bits,
                        float* out, void* stream) {
    Range nvtx_range("kitty_fake_quantize");
    if (rows < 0 || cols < 0) return invalid("fake_quantize_matrix needs a 2-D matrix");
    return cuda_status(kitty::launch_fake_quantize(x, rows, cols, per_token, bits, out, as_stream(stream)));
}

int kitty_append(const KittyCacheDesc* cache, const void* k_new, const void* v_new,
                 void* stream) {
    Range nvtx_range("kitty_append");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    return cuda_status(kitty::launch_append(*cache, k_new, v_new, as_stream(stream)));
}

int kitty_prefill(const KittyCacheDesc* cache, const void* keys, const void* values,
                  int32_t prompt_len, void* stream) {
    Range nvtx_range("kitty_prefill");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    if (prompt_len < 0) return invalid("prompt length must be >= 0");
    return cuda_status(kitty::launch_prefill(*cache, keys, values, prompt_len, as_stream(stream)));
}

int kitty_release_sequences(const KittyCacheDesc* cache, int32_t first_seq, int32_t num_seqs, void* stream) {
    Range nvtx_range("kitty_release_sequences");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    if (first_seq < 0 || num_seqs < 0 || first_seq + num_seqs > cache->num_seqs) return invalid("sequence range out of bounds");
    return cuda_status(kitty::launch_release(*cache, first_seq, num_seqs, as_stream(stream)));
}

int kitty_import_pages(const KittyCacheDesc* cache, int32_t unit, int32_t kind, const uint8_t* bodies,
                       int32_t first_page, int32_t num_pages, void* stream) {
    Range nvtx_range("kitty_import_pages");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    if (unit < 0 || unit >= cache->num_seqs * cache->cfg.h_kv) return invalid("unit out of range");
    if (kind != 0 && kind != 1) return invalid("page kind must be 0 (key) or 1 (value)", KITTY_ERR_PAGE_FORMAT);
    if (first_page < 0 || num_pages < 0) return invalid("bad page range");
    if ((int64_t)first_page + num_pages > cache->max_pages) return invalid("pages beyond the block-table capacity");
    if (num_pages > 0 && !bodies) return invalid("null page bodies");
    return cuda_status(kitty::launch_import_pages(*cache, unit, kind, bodies, first_page, num_pages, as_stream(stream)));
}

int kitty_flatten(const KittyCacheDesc* cache, int32_t unit, int32_t n, float* keys_out,
                  float* values_out, void* stream) {
    Range nvtx_range("kitty_flatten");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    if (unit < 0 || unit >= cache->num_seqs * cache->cfg.h_kv) return invalid("unit out of range");
    return cuda_status(kitty::launch_flatten(*cache, unit, n, keys_out, values_out, as_stream(stream)));
}

size_t kitty_attention_workspace_bytes(const KittyCacheDesc* cache, int32_t max_tokens) {
    if (check_cache(cache) != KITTY_OK) return 0;
    return kitty::attention_workspace_bytes(*cache, max_tokens);
}

int kitty_decode_attention(const KittyCacheDesc* cache, const void* q, void* out,
                           int32_t out_dtype, int32_t max_tokens, void* workspace,
                           size_t workspace_bytes, void* stream) {
    Range nvtx_range("kitty_decode_attention");
    int rc = check_cache(cache);
    if (rc != KITTY_OK) return rc;
    if (max_tokens < 1) return invalid("attend on an empty cache");
    if (out_dtype != KITTY_F32 && out_dtype != KITTY_BF16) return invalid("out_dtype must be F32 or BF16");
    if (workspace_bytes < kitty::attention_workspace_bytes(*cache, max_tokens)) return invalid("workspace too small");
    return cuda_status(kitty::launch_decode_attention(*cache, q, out, out_dtype, max_tokens, workspace,
                                                      workspace_bytes, as_stream(stream)));
}

size_t kitty_dense_attention_workspace_bytes(int32_t n_q, int32_t length, int32_t d) {
    return kitty::dense_attention_workspace_bytes(n_q, length, d);
}

int kitty_dense_attention(const float* keys, const float* values, int32_t h_kv, int32_t length,
                          int32_t d, const float* queries, int32_t n_q,
                          const int32_t* kv_head_map, float* out, void* workspace,
                          size_t workspace_bytes, void* stream) {
    Range nvtx_range("kitty_dense_attention");
    if (length <= 0) return invalid("attention over zero tokens");
    if (h_kv < 1 || d < 1 || n_q < 0) return invalid("bad dense attention shape");
    return cuda_status(kitty::launch_dense_attention(keys, values, h_kv, length, d, queries, n_q,
                                                     kv_head_map, out, workspace, workspace_bytes,
                                                     as_stream(stream)));
}

int kitty_dense_probs(const float* keys, int32_t h_kv, int32_t length, int32_t d, const float* queries,
                      int32_t n_q, const int32_t* kv_head_map, float* probs, void* stream) {
    Range nvtx_range("kitty_dense_probs");
    if (length <= 0) return invalid("attention over zero tokens");
    if (h_kv < 1 || d < 1 || n_q < 0) return invalid("bad dense attention shape");
    return cuda_status(kitty::launch_dense_probs(keys, length, d, queries, n_q, kv_head_map, probs, as_stream(stream)));
}

size_t kitty_sensitivity_workspace_bytes(int32_t h_q, int32_t lq, int32_t h_kv, int32_t length, int32_t d) {
    if (h_q < 0 || lq < 0 || h_kv < 1 || length < 0 || d < 0) return 0;
    return kitty::sensitivity_workspace_bytes(h_q, lq, h_kv, length, d);
}

int kitty_channel_sensitivity(const float* queries, int32_t h_q, int32_t lq, const float* keys, int32_t h_kv,
                              int32_t length, int32_t d, int32_t bits, double* mse, void* workspace,
                              size_t workspace_bytes, void* stream) {
    Range nvtx_range("kitty_channel_sensitivity");
    if (h_q < 1 || h_kv < 1 || lq < 1 || length < 1 || d < 1) return invalid("sensitivity needs non-empty queries and keys");
    if (h_q % h_kv != 0) return invalid("query head count must be a multiple of KV head count");
    if (bits != 2 && bits != 4 && bits != 16) return invalid("bits must be 2, 4 or 16");
    if (workspace_bytes < kitty::sensitivity_workspace_bytes(h_q, lq, h_kv, length, d)) return invalid("workspace too small");
    if (bits == 16) return cuda_status(cudaMemsetAsync(mse, 0, sizeof(double) * h_q * d, as_stream(stream)));
    return cuda_status(kitty::launch_channel_sensitivity(queries, h_q, lq, keys, h_kv, length, d, bits, mse,
                                                         workspace, as_stream(stream)));
}

size_t kitty_attention_mse_workspace_bytes(int32_t heads, int32_t lq, int32_t length, int32_t d) {
    if (heads < 0 || lq < 0 || length < 0 || d < 0) return 0;
    return kitty::attention_mse_workspace_bytes(heads, lq, length, d);
}

int kitty_attention_mse(const float* keys, int32_t length, int32_t d, const float* queries, int32_t heads,
                        int32_t lq, const int32_t* bits, double* out, void* workspace, size_t workspace_bytes,
                        void* stream) {
    Range nvtx_range("kitty_attention_mse");
    if (heads < 1 || lq < 1 || length < 1 || d < 1) return invalid("attention_mse needs non-empty queries and keys");
    if (workspace_bytes < kitty::attention_mse_workspace_bytes(heads, lq, length, d)) return invalid("workspace too small");
    return cuda_status(kitty::launch_attention_mse(keys, length, d, queries, heads, lq, bits, out, workspace,
                                                   as_stream(stream)));
}

}  // extern "C"
