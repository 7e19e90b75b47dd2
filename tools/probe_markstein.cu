// Verifies on the device that rint(q1), q1 = fma(fma(-q0, s, d), inv, q0),
// q0 = d * inv, inv = RN(1/s), equals rint(RN(d / s)) for the quantiser's
// operand ranges (s in [2^-90, 2^100], d in [0, 16 s]); the bulk packer
// relies on it (kitty_pack_fast.cuh).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hash(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return (uint32_t)x;
}
__device__ unsigned long long g_bad[4], g_q1bad[4];
__global__ void probe(uint64_t seed, int mode, int iters) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bad = 0, qbad = 0;
    for (int it = 0; it < iters; ++it) {
        const uint64_t id = (tid * iters + it) * 4 + seed;
        const uint32_t h0 = hash(id), h1 = hash(id + 1), h2 = hash(id + 2);
        float s, d;
        const float qmax = (h2 & 1) ? 3.f : 15.f;
        if (mode == 0) {  // random f32: s = 2^e * m, d = u * qmax * s
            const int e = (int)(h0 % 190) - 90;
            s = ldexpf(1.f + (h1 >> 9) * (1.f / 8388608.f), e);
            d = __fmul_rn(__fmul_rn((h2 >> 8) * (1.f / 16777216.f), qmax), s);
        } else if (mode == 1) {  // bf16 grid: x, mn, mx bf16 of N-ish magnitudes
            const int e = (int)(h0 % 60) - 30;
            const float a = __uint_as_float(((h1 & 0x7fff) << 16) & 0x3fff0000u | 0x3f800000u) ;
            float mn = -ldexpf(__uint_as_float((0x3f80u | (h1 >> 25)) << 16), e);
            float mx = ldexpf(__uint_as_float((0x3f80u | ((h1 >> 16) & 0x7f)) << 16), e + (int)(h2 >> 29) - 2);
            float x = mn + (mx - mn) * ((h2 >> 8 & 0xffff) * (1.f / 65536.f));
            x = __uint_as_float(__float_as_uint(x) & 0xffff0000u);
            x = fminf(fmaxf(x, mn), mx);
            (void)a;
            s = __fdiv_rn(__fsub_rn(mx, mn), qmax);
            d = __fsub_rn(x, mn);
        } else {  // near ties: d = RN((k + 0.5) s) +- a few ulps
            const int e = (int)(h0 % 180) - 85;
            s = ldexpf(1.f + (h1 >> 9) * (1.f / 8388608.f), e);
            const float k = (float)(h2 % (uint32_t)qmax) + 0.5f;
            d = __fmul_rn(k, s);
            const int off = (int)((h2 >> 8) % 9) - 4;
            d = __uint_as_float(__float_as_uint(d) + off);
        }
        if (!(s > 0.f)) continue;
        const float inv = __frcp_rn(s);
        const float q0 = __fmul_rn(d, inv);
        const float r = __fmaf_rn(-q0, s, d);
        const float q1 = __fmaf_rn(r, inv, q0);
        const float ref = __fdiv_rn(d, s);
        bad += rintf(q1) != rintf(ref);
        qbad += q1 != ref;
    }
    atomicAdd(&g_bad[mode], bad);
    atomicAdd(&g_q1bad[mode], qbad);
}
int main() {
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 4; ++rep) probe<<<148 * 16, 256>>>(rep * 0x9e3779b97f4a7c15ull + mode * 77, mode, 1024);
        cudaDeviceSynchronize();
        unsigned long long b[4], q[4];
        cudaMemcpyFromSymbol(b, g_bad, sizeof(b));
        cudaMemcpyFromSymbol(q, g_q1bad, sizeof(q));
        printf("mode %d: %.3g samples, rint mismatches %llu, quotient mismatches %llu\n", mode,
               4.0 * 148 * 16 * 256 * 1024, b[mode], q[mode]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
