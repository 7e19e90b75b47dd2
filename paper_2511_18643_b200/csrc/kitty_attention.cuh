// Dispatch surface of the specialised decode-attention kernel.
#pragma once

#include "kitty_common.cuh"

namespace kitty {

// True when the tensor-core kernel covers this cache's shape (d = g = 128,
// key/value bits 2, group <= 8).
bool fast_attention_supported(const KittyCacheDesc& c);
size_t fast_attention_workspace_bytes(const KittyCacheDesc& c, int max_tokens);
cudaError_t launch_fast_attention(const KittyCacheDesc& c, const uint16_t* q, void* out,
                                  int out_dtype, int max_tokens, void* ws, size_t ws_bytes,
                                  cudaStream_t st);

}  // namespace kitty
