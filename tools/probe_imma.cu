// Throughput probe: legacy mma.sync f16 m16n8k16 vs s8/u8 m16n8k32 on sm_100a.
// 8 warps/SM x 148 SMs x ITERS x 8 independent accumulators.
#include <cstdio>
#include <cstdint>
#define ITERS 4096
__global__ void hmma_k(float* out, uint32_t seed) {
    float acc[8][4] = {};
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imma_k(int* out, uint32_t seed) {
    int acc[8][4] = {};
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(acc[j][0]), "+r"(acc[j][1]), "+r"(acc[j][2]), "+r"(acc[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imma16_k(int* out, uint32_t seed) {
    int acc[8][4] = {};
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, b0 = a0 * 11;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+r"(acc[j][0]), "+r"(acc[j][1]), "+r"(acc[j][2]), "+r"(acc[j][3])
                         : "r"(a0), "r"(a1), "r"(b0));
    }
    int s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 1024 * 4 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps = 4; warps <= 16; warps *= 2) {
        for (int k = 0; k < 3; ++k) {
            float best = 1e9;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                if (k == 0) hmma_k<<<148, warps * 32>>>(o, r);
                if (k == 1) imma_k<<<148, warps * 32>>>((int*)o, r);
                if (k == 2) imma16_k<<<148, warps * 32>>>((int*)o, r);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            const double mmas = 148.0 * warps * ITERS * 8;
            const double kdim = k == 1 ? 32 : 16;
            const char* nm[3] = {"HMMA f16 m16n8k16", "IMMA u8s8 m16n8k32", "IMMA u8s8 m16n8k16"};
            printf("%-20s warps/SM %2d: %.3f ms, %.1f cycles/mma/SM-subpartition @1.9GHz, %.1f TOPS\n", nm[k], warps, best,
                   best * 1e-3 * 1.9e9 / (mmas / 148 / 4), mmas * 16 * 8 * kdim * 2 / (best * 1e-3) / 1e12);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
