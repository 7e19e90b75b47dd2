// Tensor-pipe throughput of the legacy mma.sync shapes on sm_100a: cycles per
// instruction per SM sub-partition with 8 independent accumulators per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe_mma_kinds.cu
#include <cstdio>
#include <cstdint>
#define ITERS 4096

#define KERNEL(NAME, ACC_T, CONSTR, ASM, AREGS)                                                          \
    __global__ void NAME(float* out, uint32_t seed) {                                                    \
        ACC_T acc[8][4] = {};                                                                            \
        uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13; \
        for (int i = 0; i < ITERS; ++i) {                                                                \
            _Pragma("unroll") for (int j = 0; j < 8; ++j) asm volatile(ASM                              \
                                                                       : CONSTR(acc[j][0]), CONSTR(acc[j][1]), CONSTR(acc[j][2]), CONSTR(acc[j][3]) \
                                                                       : AREGS);                         \
        }                                                                                                \
        float s = 0;                                                                                     \
        for (int j = 0; j < 8; ++j) s += (float)acc[j][0] + (float)acc[j][1] + (float)acc[j][2] + (float)acc[j][3]; \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                                  \
    }
#define CF(x) "+f"(x)
#define CR(x) "+r"(x)
#define A4B2 "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1)
#define A2B1 "r"(a0), "r"(a1), "r"(b0)

KERNEL(hmma_f32, float, CF, "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};", A4B2)
KERNEL(hmma_k8, float, CF, "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};", A2B1)
KERNEL(imma_k32, int, CR, "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};", A4B2)
KERNEL(fp8_k32, float, CF, "mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};", A4B2)
KERNEL(bf16_f32, float, CF, "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};", A4B2)

__global__ void hmma_f16acc(float* out, uint32_t seed) {
    uint32_t acc[8][2] = {};
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                         : "+r"(acc[j][0]), "+r"(acc[j][1])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    uint32_t s = 0;
    for (int j = 0; j < 8; ++j) s ^= acc[j][0] ^ acc[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

typedef void (*K)(float*, uint32_t);
int main() {
    float* o;
    cudaMalloc(&o, 148 * 1024 * 4 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    K ks[] = {hmma_f32, hmma_f16acc, hmma_k8, bf16_f32, imma_k32, fp8_k32};
    const char* nm[] = {"f16 m16n8k16 f32acc", "f16 m16n8k16 f16acc", "f16 m16n8k8 f32acc", "bf16 m16n8k16 f32acc",
                        "u8s8 m16n8k32 s32", "e4m3 m16n8k32 f32acc"};
    for (int k = 0; k < 6; ++k) {
        for (int warps : {8, 16}) {
            float best = 1e9;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                ks[k]<<<148 * 2, warps * 32>>>(o, r);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            const double mmas_per_smsp = 2.0 * warps * ITERS * 8 / 4;
            printf("%-24s warps/CTA %2d (2 CTA/SM): %.3f ms  %.2f cycles/mma/SMSP @1.965GHz\n", nm[k], warps, best,
                   best * 1e-3 * 1.965e9 / mmas_per_smsp);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
