// Tensor-core fused dequant-attention for d = g = 128 (placeholder: the
// generic path serves every shape until this kernel lands).
#include "kitty_attention.cuh"

namespace kitty {

bool fast_attention_supported(const KittyCacheDesc&) { return false; }
size_t fast_attention_workspace_bytes(const KittyCacheDesc&, int) { return 0; }
cudaError_t launch_fast_attention(const KittyCacheDesc&, const uint16_t*, void*, int, int, void*,
                                  size_t, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace kitty
