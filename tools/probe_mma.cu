// Throughput probe: legacy mma.sync.m16n8k16 (f16 in, f32 accumulate) and the
// ALU ops of the 2-bit -> fp16 conversion (PRMT / LOP3) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_mma tools/probe_mma.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void mma_loop(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void alu_loop(uint32_t* out, int iters) {
    uint32_t x = threadIdx.x * 0x9E3779B9u, y = x ^ 0x5bd1e995u, acc[8] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t p;
            asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(p) : "r"(x + j), "r"(y));
            uint32_t l;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(l) : "r"(p), "r"(0x00300030u), "r"(0x64006400u));
            acc[j] += l;
        }
        x += 1;
    }
    uint32_t s = 0;
    for (int j = 0; j < 8; ++j) s ^= acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps : {4, 8, 16}) {
        const int iters = 4096;
        mma_loop<<<sms * 2, 32 * warps>>>(out, 16);
        cudaEventRecord(a);
        mma_loop<<<sms * 2, 32 * warps>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * (sms * 2) * warps;
        printf("mma.sync m16n8k16 f16->f32: warps/CTA=%d  %.1f TFLOP/s  (%.0f FLOP/clk/SM @1.9GHz)\n", warps,
               flops / ms / 1e9, flops / (ms * 1e-3) / sms / 1.9e9);
    }
    for (int warps : {8, 16, 32}) {
        const int iters = 4096;
        alu_loop<<<sms * 2, 32 * warps>>>((uint32_t*)out, 16);
        cudaEventRecord(a);
        alu_loop<<<sms * 2, 32 * warps>>>((uint32_t*)out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = 8.0 * 2 * iters * (sms * 2) * warps;  // warp-instructions of PRMT+LOP3
        printf("PRMT+LOP3: warps/CTA=%d  %.3f warp-instr/clk/SM @1.9GHz\n", warps, ops / (ms * 1e-3) / sms / 1.9e9);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock attr %d kHz, SMs %d\n", clk, sms);
    return 0;
}
