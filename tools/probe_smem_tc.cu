// Probe: do tcgen05.mma shared-memory operand reads share bandwidth with the
// LSU (ld/st.shared) path?  Per SM: warps 1..7 stream st.shared.v4 (mode 1) or
// ld.shared.v4 (mode 3) over 32 KB while thread 0 of warp 0 issues kind::i8
// M=128 N=16 K=32 MMAs from a 16 KB A tile (mode 2), or both (mode 1|2, 3|2).
// Prints bytes/cycle/SM of each stream.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int kIters = 4096;
constexpr int kMma = 8192;

__global__ void __launch_bounds__(256, 1) probe(int mode, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* a = sm;             // 16 KB A tile
    uint8_t* b = sm + 16384;     // 512 B B tile
    uint8_t* buf = sm + 32768;   // 32 KB LSU stream area
    __shared__ uint32_t tbase;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 16384 / 16; i += 256) reinterpret_cast<uint4*>(a)[i] = make_uint4(1, 2, 3, 4);
    for (int i = tid; i < 512 / 16; i += 256) reinterpret_cast<uint4*>(b)[i] = make_uint4(1, 1, 1, 1);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    long long t0 = clock64();
    unsigned long long lsu_bytes = 0, mma_bytes = 0;
    long long t_lsu = 0, t_mma = 0;
    if (warp == 0) {
        if ((mode & 2) && tid == 0) {
            const uint32_t id = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (2u << 17) | (8u << 24);
            for (int i = 0; i < kMma; ++i) {
                const int s = i & 3;
                const uint64_t da = desc(smem_u32(a) + 4096 * s, 1024, 128);
                const uint64_t db = desc(smem_u32(b), 128, 128);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                             "l"(da), "l"(db), "r"(id), "r"(1u));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                smem_u32(&bar)) : "memory");
            t_mma = clock64() - t0;
            mma_bytes = (unsigned long long)kMma * (4096 + 512);
        }
    } else if (mode & 1) {
        const uint32_t base = smem_u32(buf) + 16 * (tid - 32);
        for (int it = 0; it < kIters; ++it) {
            const uint32_t ad = base + (uint32_t)((it * 3584) % (32768 - 3584));
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(ad), "r"(it) : "memory");
        }
        asm volatile("bar.sync 1, 224;");
        t_lsu = clock64() - t0;
        lsu_bytes = (unsigned long long)kIters * 224 * 16;
    } else if (mode & 4) {
        const uint32_t base = smem_u32(buf) + 16 * (tid - 32);
        uint32_t acc = 0;
        for (int it = 0; it < kIters; ++it) {
            const uint32_t ad = base + (uint32_t)((it * 3584) % (32768 - 3584));
            uint32_t x, y, z, w;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(ad));
            acc ^= x ^ y ^ z ^ w;
        }
        asm volatile("bar.sync 1, 224;");
        t_lsu = clock64() - t0;
        lsu_bytes = (unsigned long long)kIters * 224 * 16;
        if (acc == 0x12345678) out[3] = acc;
    }
    if (tid == 0 && blockIdx.x == 0) {
        out[0] = mma_bytes;
        out[1] = t_mma;
    }
    if (tid == 32 && blockIdx.x == 0) {
        out[2] = lsu_bytes;
        out[4] = t_lsu;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const char* names[] = {"", "STS only", "MMA only", "STS + MMA", "LDS only", "", "LDS + MMA"};
    for (int mode : {1, 2, 3, 4, 6}) {
        unsigned long long h[5] = {0, 0, 0, 0, 0};
        cudaMemset(d, 0, 64);
        probe<<<148, 256, 65536>>>(mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
        printf("%-10s %s: MMA A+B reads %.1f B/cyc (%llu cyc)   LSU %.1f B/cyc (%llu cyc)\n", names[mode],
               cudaGetErrorString(e), h[1] ? (double)h[0] / h[1] : 0.0, h[1], h[4] ? (double)h[2] / h[4] : 0.0, h[4]);
    }
    return 0;
}
