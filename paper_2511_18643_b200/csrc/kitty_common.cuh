// Shared device helpers for the Kitty B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kitty_b200.h"

namespace kitty {

constexpr uint8_t kSentinel = 255;  // pages.py:32

__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

__device__ __forceinline__ float load_elem(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float load_elem(const uint16_t* p, int64_t i) {
    return bf16_to_f32(p[i]);
}

__device__ __forceinline__ float half_bits_to_f32(uint16_t h) {
    return __half2float(__ushort_as_half(h));
}
// f32 -> f16 (RNE) bit pattern.  Written with an explicit cvt: going through
// __half_as_ushort and then splitting the result into bytes let nvcc 12.9 fuse
// the byte extraction into a numeric F2I.U8.F16 conversion (wrong bytes).
__device__ __forceinline__ uint32_t f32_to_half_bits(float f) {
    unsigned short h;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
    uint32_t r;
    asm("cvt.u32.u16 %0, %1;" : "=r"(r) : "h"(h));
    return r;
}
__device__ __forceinline__ uint32_t f32_to_bf16_bits(float f) {
    unsigned short h;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f));
    uint32_t r;
    asm("cvt.u32.u16 %0, %1;" : "=r"(r) : "h"(h));
    return r;
}

// Byte offsets of the KTYP key body components (pages.py:215-221).
struct KeyLayout {
    int d, g, d_boost;
    __host__ __device__ int dense_off() const { return 0; }
    __host__ __device__ int high_off() const { return d * g / 4; }
    __host__ __device__ int idx_off() const { return d * g / 4 + d_boost * g / 4; }
    __host__ __device__ int scale_off() const { return idx_off() + d; }
    __host__ __device__ int zero_off() const { return scale_off() + 2 * d; }
    __host__ __device__ int bytes() const { return zero_off() + 2 * d; }
};

// Byte offsets of the KTYP value body (pages.py:228-235).
struct ValueLayout {
    int d, g;
    __host__ __device__ int codes_off() const { return 0; }
    __host__ __device__ int scale_off() const { return g * d / 4; }
    __host__ __device__ int zero_off() const { return scale_off() + 2 * g; }
    __host__ __device__ int bytes() const { return zero_off() + 2 * g; }
};

// Asymmetric quantizer step of quant.py:109-116 for one lane, given its
// min / max: scale = (mx - mn) / qmax in IEEE float32, code =
// clip(rint((x - mn) / safe), 0, qmax), all-zero codes when scale == 0.
struct LaneQuant {
    float mn, scale, safe, inv, qmax;
    bool exact;  // the reciprocal is not usable (scale < 2^-100 or > 2^100): always divide
    __device__ __forceinline__ LaneQuant(float mn_, float mx_, float qmax_) {
        mn = mn_;
        qmax = qmax_;
        scale = __fdiv_rn(__fsub_rn(mx_, mn_), qmax_);
        safe = scale > 0.f ? scale : 1.0f;
        inv = __frcp_rn(safe);
        exact = !(safe >= 0x1p-100f && safe <= 0x1p100f);
    }
    // rint of the IEEE quotient (x - mn) / safe.  x * rcp(safe) is within
    // ~2^-23 relative (< 2e-6 absolute for quotients <= 15) of it, so its
    // rint is the same unless it lies within 1e-5 of a half-integer; only
    // those (rare) elements pay for the IEEE division.
    __device__ __forceinline__ uint32_t code(float x) const {
        if (!(scale != 0.f)) return 0u;  // codes[:, scale == 0] = 0 (also NaN-safe)
        const float dlt = __fsub_rn(x, mn);
        const float qa = __fmul_rn(dlt, inv);
        float r = rintf(qa);
        if (exact || fabsf(__fsub_rn(__fsub_rn(qa, floorf(qa)), 0.5f)) < 1.0e-5f) r = rintf(__fdiv_rn(dlt, safe));
        r = fminf(fmaxf(r, 0.f), qmax);
        return static_cast<uint32_t>(r);
    }
};

// Unaligned-safe 16-bit little-endian access (KTYP metadata offsets are only
// 2-byte aligned when d_boost * g / 4 is even).
__device__ __forceinline__ uint16_t ld_u16(const uint8_t* p) {
    return static_cast<uint16_t>(p[0] | (p[1] << 8));
}
__device__ __forceinline__ void st_u16(uint8_t* p, uint32_t v) {
    p[0] = static_cast<uint8_t>(v & 0xffu);
    p[1] = static_cast<uint8_t>((v >> 8) & 0xffu);
}

__device__ __forceinline__ void set_status(uint32_t* status, uint32_t bits) {
    if (status) atomicOr(status, bits);
}

// ---- host: per-device properties and kernel attributes (kitty_device.cu) ----
// One process may drive several GPUs (one stream each), so nothing here is a
// process-wide static: values are cached per (device ordinal) and kernel
// attributes are set once per (kernel, device, value).
int device_sms();                 // SM count of the current device
int device_smem_per_sm();         // shared memory per SM (bytes)
cudaError_t set_kernel_smem(const void* fn, int bytes, bool max_shared_carveout = false);

}  // namespace kitty
