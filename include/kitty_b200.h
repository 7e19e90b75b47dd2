/*
 * kitty_b200.h -- C ABI of the B200-native Kitty decode hot path.
 *
 * The reference (arxiv 2511.18643, package `kittykv`, /root/reference/pkg/src/kittykv)
 * has no FFI: its boundary is the Python API re-exported at __init__.py:61-112.
 * Each entry point below replaces one reference function on the hot path; the
 * replaced symbol is cited next to it (file:line relative to pkg/src/kittykv).
 * A Python shim (paper_2511_18643_b200/) binds these with ctypes and restores
 * the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - plain pointers and sizes only; all buffers are caller-owned device memory
 *     unless stated; no entry point allocates or synchronises;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - every entry point returns a KittyStatus; data-dependent failures that the
 *     reference raises synchronously (non-finite page, broken boost_idx
 *     bijection, cache overflow) are reported through a device status word
 *     (KITTY_STATUS_* bits) that the caller reads after its own sync;
 *   - bf16 tensors are passed as uint16_t*; row-major; D = head size.
 */
#ifndef KITTY_B200_H
#define KITTY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  The shim maps them to the reference exceptions (errors.py:4-33). */
typedef enum KittyStatus {
    KITTY_OK = 0,
    KITTY_ERR_CONFIG = 1,      /* ConfigError      (errors.py:8, config.py:35-53)   */
    KITTY_ERR_INVALID = 2,     /* KittyError       (errors.py:4)                    */
    KITTY_ERR_PAGE_FORMAT = 3, /* PageFormatError  (errors.py:32, pages.py:128-135)  */
    KITTY_ERR_CUDA = 4,        /* launch / runtime failure                          */
    KITTY_ERR_UNSUPPORTED = 5  /* valid for the reference, not built on the device  */
} KittyStatus;

/* Bits of the device status word. */
#define KITTY_STATUS_NONFINITE 0x1u   /* pages.py:88-89,152-153: non-finite page input */
#define KITTY_STATUS_PAGE_FORMAT 0x2u /* pages.py:128-135: sentinel count / bijection   */
#define KITTY_STATUS_OVERFLOW 0x4u    /* append past the block-table capacity          */
#define KITTY_STATUS_LENGTH 0x8u      /* a unit is longer than the attention call's
                                         max_tokens (its tokens beyond it were not read) */

/* Element types for inputs that the reference accepts as float32. */
#define KITTY_F32 0
#define KITTY_BF16 1

/* KittyConfig (config.py:14-65) as a POD.  d_boost = round(boost_fraction * d)
 * is resolved by the caller exactly as quant.py:57-61 does. */
typedef struct KittyConfigC {
    int32_t s;        /* sink tokens                     */
    int32_t r;        /* value local window              */
    int32_t g;        /* page size (tokens)              */
    int32_t d;        /* head size (channels)            */
    int32_t h_kv;     /* KV heads                        */
    int32_t h_q;      /* query heads                     */
    int32_t d_boost;  /* boosted key channels per page   */
    int32_t key_bits; /* 2 on the device (16 = pass-through, not built) */
    int32_t value_bits;
} KittyConfigC;

/*
 * Device state of a batch of sequences (the batched form of KittyCacheState,
 * cache.py:83-192).  One "unit" = (sequence, KV head); unit u = b * h_kv + h.
 * Global token order is the reference's (cache.py:12-15):
 *   keys   = sink | key pages   | key q-buffer
 *   values = sink | value pages | value q-buffer | local
 * Full-precision rows are bf16 (row_dtype KITTY_BF16, the fused decode path)
 * or float32 (KITTY_F32: the reference's own precision, generic kernels).
 * Token t >= s of a unit lives at
 *   k_qbuf[u][(t - s) % g]          while not yet in a key page,
 *   v_ring[u][(t - s) % (r + g)]    while not yet in a value page
 * (the value ring holds q-buffer + local).  Page slots are byte-identical to
 * the KTYP body of pages.py:207-237 (f16 scale/zero), so export is a memcpy.
 */
typedef struct KittyCacheDesc {
    KittyConfigC cfg;
    int32_t num_seqs;          /* B                                           */
    int32_t max_pages;         /* block-table capacity per unit               */
    int64_t key_slot_bytes;    /* = kitty_key_slot_bytes(d, g, d_boost)       */
    int64_t value_slot_bytes;  /* = kitty_value_slot_bytes(d, g)              */
    int32_t* unit_len;         /* [B*h_kv] tokens inserted per unit           */
    void* k_sink;              /* [B*h_kv][s][d]   row_dtype                   */
    void* v_sink;              /* [B*h_kv][s][d]   row_dtype                   */
    void* k_qbuf;              /* [B*h_kv][g][d]   row_dtype                   */
    void* v_ring;              /* [B*h_kv][r+g][d] row_dtype                   */
    uint8_t* key_pool;         /* [slots][key_slot_bytes]                     */
    uint8_t* value_pool;       /* [slots][value_slot_bytes]                   */
    int32_t* key_block_table;  /* [B*h_kv][max_pages] slot index              */
    int32_t* value_block_table;/* [B*h_kv][max_pages] slot index              */
    uint32_t* status;          /* device status word (KITTY_STATUS_*)         */
    int32_t row_dtype;         /* KITTY_BF16 or KITTY_F32: the rows above and the
                                  rows / queries passed to append, prefill and
                                  attention (set it: 0 is KITTY_F32)            */
    int32_t reserved;
    float* key_meta;           /* optional [slots][2 d]: f32 scale | zero of each
                                  key slot, written by the packs; when set,
                                  attention and flatten use it instead of the
                                  slot's f16 copy (the reference keeps f32 in
                                  memory, cache.py:157-161)                     */
    float* value_meta;         /* optional [slots][2 g]: the same for values   */
    /* Page pool (optional; NULL key_free = static block tables written by the
     * caller).  With a pool the block tables start at -1 and a page's slot is
     * popped from the side's free stack by the kernel that packs (or imports)
     * the page, then recorded in the unit's block table; kitty_release_sequences
     * pushes a retired sequence's slots back.  Pops and pushes never share a
     * launch, so a stack is an array plus an atomic top.  An empty stack sets
     * KITTY_STATUS_OVERFLOW and the page is dropped. */
    int32_t* key_free;         /* [key_slots] free key-slot indices (stack)    */
    int32_t* value_free;       /* [value_slots] free value-slot indices        */
    int32_t* free_top;         /* [2] entries on the key / value stacks        */
    int32_t key_slots;         /* key_pool capacity in slots                   */
    int32_t value_slots;       /* value_pool capacity in slots                 */
} KittyCacheDesc;

/* ---- sizes / config --------------------------------------------------- */

/* page_byte_size("key").total (pages.py:189-201): d*g/4 + d_boost*g/4 + d + 4d */
int64_t kitty_key_slot_bytes(int32_t d, int32_t g, int32_t d_boost);
/* page_byte_size("value").total (pages.py:202-203): g*d/4 + 4g */
int64_t kitty_value_slot_bytes(int32_t d, int32_t g);
/* KittyConfig.__post_init__ checks (config.py:35-53) + device limits. */
int kitty_validate_config(const KittyConfigC* cfg);
const char* kitty_version(void);
/* Name of the last CUDA error seen by this library (thread-local). */
const char* kitty_last_error(void);

/* ---- quantize (quant.py) ---------------------------------------------- */

/* channel_scores (quant.py:64-72) of P (g x d) pages: scores[P][d] float64,
 * sequential fp64 sum over tokens then / g. */
int kitty_channel_scores(const void* x, int32_t dtype, int32_t num_pages, int32_t g,
                         int32_t d, double* scores, void* stream);

/* select_boost(..., "magnitude") (quant.py:75-99): boosted[P][k] ascending
 * channel indices, ties to the lower index. */
int kitty_select_boost(const double* scores, int32_t num_pages, int32_t d, int32_t k,
                       int64_t* boosted, void* stream);

/* ---- page codec (pages.py) -------------------------------------------- */

/* channel_scores -> select_boost -> pack_key_page fused (pages.py:81-118,
 * cache.py:155-159), one page per (g x d) block of x.  `boosted` [P][d_boost]
 * overrides the magnitude selection when non-NULL (any ascending selection).
 * Writes KTYP key bodies to slots + p * slot_stride.  Optional f32 metadata
 * outputs scales_f32/zeros_f32 [P][d] carry the in-memory (pre-f16) values. */
int kitty_pack_key_pages(const void* x, int32_t dtype, int32_t num_pages, int32_t g,
                         int32_t d, int32_t d_boost, const int64_t* boosted,
                         uint8_t* slots, int64_t slot_stride, float* scales_f32,
                         float* zeros_f32, uint32_t* status, void* stream);

/* pack_value_page (pages.py:146-162) of P (g x d) blocks. */
int kitty_pack_value_pages(const void* x, int32_t dtype, int32_t num_pages, int32_t g,
                           int32_t d, uint8_t* slots, int64_t slot_stride,
                           float* scales_f32, float* zeros_f32, uint32_t* status,
                           void* stream);

/* dequantize_key_page (pages.py:121-143, Alg. 1): out[P][d][g] float32,
 * code * scale + zero (multiply, then add).  scales_f32/zeros_f32 [P][d] are
 * used when non-NULL, else the slot's f16 metadata.  Sentinel / bijection
 * violations set KITTY_STATUS_PAGE_FORMAT. */
int kitty_dequant_key_pages(const uint8_t* slots, int64_t slot_stride, int32_t num_pages,
                            int32_t g, int32_t d, int32_t d_boost, const float* scales_f32,
                            const float* zeros_f32, float* out, uint32_t* status,
                            void* stream);

/* dequantize_value_page (pages.py:165-168): out[P][g][d] float32. */
int kitty_dequant_value_pages(const uint8_t* slots, int64_t slot_stride, int32_t num_pages,
                              int32_t g, int32_t d, const float* scales_f32,
                              const float* zeros_f32, float* out, void* stream);

/* _quantize_columns / quantize_values (quant.py:102-132) of every lane of x
 * [rows][cols] float32 (lanes = columns, or rows with per_token = 1) at
 * bits[lane] in {2, 4} (device int32): codes [rows][cols] u8, scales / zeros
 * [lanes] f32 (scale = (max - min) / (2^b - 1) in IEEE f32, zero = min, codes
 * = clip(rint((x - min) / scale)), all-zero codes for a constant lane). */
int kitty_quantize_lanes(const float* x, int32_t rows, int32_t cols, int32_t per_token, const int32_t* bits,
                         uint8_t* codes, float* scales, float* zeros, void* stream);

/* dequantize_values (quant.py:135-143): out = code * scale + zero per lane
 * (multiply, then add). */
int kitty_dequantize_lanes(const uint8_t* codes, int32_t rows, int32_t cols, int32_t per_token, const float* scales,
                           const float* zeros, float* out, void* stream);

/* fake_quantize_matrix (quant.py:145-177): x [rows][cols] float32; lanes are
 * columns (per_token = 0, "per_channel") or rows (per_token = 1); bits [lanes]
 * (device int32) in {2, 4, 16}, 16 passing the lane through; out like x. */
int kitty_fake_quantize(const float* x, int32_t rows, int32_t cols, int32_t per_token, const int32_t* bits,
                        float* out, void* stream);

/* ---- cache runtime (cache.py) ----------------------------------------- */

/* insert_token + maybe_pack (cache.py:107-123,144-178) for every unit of the
 * batch: k_new/v_new [B][h_kv][d] bf16.  A unit whose key q-buffer (value
 * q-buffer) reaches g rows is packed into its next key (value) slot inside
 * this call, so a following attention sees the page (pack-before-attend). */
int kitty_append(const KittyCacheDesc* cache, const void* k_new, const void* v_new,
                 void* stream);

/* prefill (cache.py:125-142) of an empty batch: keys/values [B][h_kv][P][d]
 * bf16.  Produces the state of the fold of P appends; all pages of the prompt
 * are packed in parallel. */
int kitty_prefill(const KittyCacheDesc* cache, const void* keys, const void* values,
                  int32_t prompt_len, void* stream);

/* Retire sequences [first_seq, first_seq + num_seqs): every unit's key and
 * value slots go back to the pool's free stacks (no-op without a pool), its
 * block-table entries become -1 and its length 0, so the rows can admit a new
 * sequence (prefill / append).  The reference has one state per sequence and
 * frees it by dropping the object (cache.py:83-105); this is that drop for a
 * batch whose pages live in a shared pool. */
int kitty_release_sequences(const KittyCacheDesc* cache, int32_t first_seq, int32_t num_seqs,
                            void* stream);

/* deserialize_page (pages.py:246-292) into the cache: `bodies` holds
 * num_pages KTYP bodies (header stripped and checked by the caller against
 * the cache's d / g / d_boost) of kind 0 = key, 1 = value, contiguous, in
 * device memory.  Page first_page + i of `unit` gets a slot (popped from the
 * pool, or the block table's entry) and the body is copied in; key pages are
 * checked like dequantize_key_page (pages.py:128-135: d - d_boost sentinels,
 * boost_idx a bijection onto 0..d_boost-1), a violation sets
 * KITTY_STATUS_PAGE_FORMAT.  The f32 metadata side tables, when present, get
 * the bodies' f16 scale / zero promoted to f32 (pages.py:263-264). */
int kitty_import_pages(const KittyCacheDesc* cache, int32_t unit, int32_t kind, const uint8_t* bodies,
                       int32_t first_page, int32_t num_pages, void* stream);

/* flatten_keys / flatten_values (cache.py:210-215) of one unit: [n][d] f32,
 * pages dequantized from their f16 metadata.  n = tokens of the unit. */
int kitty_flatten(const KittyCacheDesc* cache, int32_t unit, int32_t n, float* keys_out,
                  float* values_out, void* stream);

/* ---- attention -------------------------------------------------------- */

/* Workspace needed by kitty_decode_attention for sequences of <= max_tokens. */
size_t kitty_attention_workspace_bytes(const KittyCacheDesc* cache, int32_t max_tokens);

/* attend (cache.py:217-252) for every sequence: q [B][h_q][d] bf16 ->
 * out [B][h_q][d] (out_dtype KITTY_F32 or KITTY_BF16).  Query head i reads KV
 * head i / (h_q / h_kv) (cache.py:240).  Pages are dequantized on the fly
 * inside the QK^T / softmax / PV loop.  max_tokens bounds the unit lengths
 * (the caller's host mirror); it sizes the split-KV grid. */
int kitty_decode_attention(const KittyCacheDesc* cache, const void* q, void* out,
                           int32_t out_dtype, int32_t max_tokens, void* workspace,
                           size_t workspace_bytes, void* stream);

/* oracle_attend (cache.py:261-301) on device: dense f32 keys/values
 * [h_kv][L][d], queries [n_q][d]; query i reads KV head kv_head_map[i]
 * (device int32 [n_q]); out [n_q][d] f32. */
size_t kitty_dense_attention_workspace_bytes(int32_t n_q, int32_t length, int32_t d);
int kitty_dense_attention(const float* keys, const float* values, int32_t h_kv,
                          int32_t length, int32_t d, const float* queries, int32_t n_q,
                          const int32_t* kv_head_map, float* out, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ---- analysis (analysis.py) -------------------------------------------- */

/* channel_sensitivity (analysis.py:63-104): mse[h_q][d] float64 = the mean
 * squared difference of the (lq x length) attention-probability matrix of
 * query head qh when key channel ch alone is fake-quantized per channel at
 * `bits` (rank-1 logit update), fp64 throughout.  queries [h_q][lq][d] and
 * keys [h_kv][length][d] float32; query head qh reads KV head qh / (h_q/h_kv).
 * bits 16 is the identity (all zeros; the caller may skip the launch). */
size_t kitty_sensitivity_workspace_bytes(int32_t h_q, int32_t lq, int32_t h_kv, int32_t length, int32_t d);
int kitty_channel_sensitivity(const float* queries, int32_t h_q, int32_t lq, const float* keys, int32_t h_kv,
                              int32_t length, int32_t d, int32_t bits, double* mse, void* workspace,
                              size_t workspace_bytes, void* stream);

/* attention_mse (analysis.py:119-142): keys [length][d] float32 fake-quantized
 * per channel at bits[d] (device int32: 4 for the boosted selection, 2
 * elsewhere); out[0] float64 = mean over the `heads` query heads
 * (queries [heads][lq][d]) of the probability-matrix MSE against the
 * full-precision keys. */
size_t kitty_attention_mse_workspace_bytes(int32_t heads, int32_t lq, int32_t length, int32_t d);
int kitty_attention_mse(const float* keys, int32_t length, int32_t d, const float* queries, int32_t heads,
                        int32_t lq, const int32_t* bits, double* out, void* workspace, size_t workspace_bytes,
                        void* stream);

/* The attention probabilities oracle_attend returns (cache.py:291-299) and
 * KittyCacheState.attend(return_probs=True) (cache.py:236-251): dense f32
 * keys [h_kv][length][d], queries [n_q][d], query i reads KV head
 * kv_head_map[i]; probs [n_q][length] f32 (max-subtracted softmax of
 * (k . q) / sqrt(d)). */
int kitty_dense_probs(const float* keys, int32_t h_kv, int32_t length, int32_t d, const float* queries,
                      int32_t n_q, const int32_t* kv_head_map, float* probs, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KITTY_B200_H */
