// Probe: tcgen05.mma kind::i8 with MN-major (no swizzle) shared-memory operands.
// Checks the descriptor encoding the fused attention kernel relies on:
//   A u8  [M=128][K] MN-major: addr(m,k) = m%16 + 16 (k%8) + SBO_A (m/16) + LBO_A (k/8)
//   B s8  [K][N=16]  MN-major: addr(k,n) = n + 16 (k%8) + LBO_B (k/8)
//   D s32 in TMEM, lane = m, column = n.
// Build+run on a B200:  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/p tools/probe_umma_i8.cu && /tmp/p
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N>
__device__ __forceinline__ uint32_t idesc_i8(bool a_mn, bool b_mn, bool b_signed) {
    return (2u << 4) | (0u << 7) | ((b_signed ? 1u : 0u) << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

constexpr int KT = 64;  // two MMA k-steps
constexpr int LBO_A = 1024, SBO_A = 128, LBO_B = 128;

__global__ void probe(const uint8_t* A, const int8_t* B, int* D, int mode) {
    __shared__ __align__(1024) uint8_t sa[128 * KT];
    __shared__ __align__(1024) int8_t sb[KT * 16];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // A logical [m][k] -> MN-major interleaved
    for (int i = tid; i < 128 * KT; i += blockDim.x) {
        const int m = i / KT, k = i % KT;
        sa[(m % 16) + 16 * (k % 8) + SBO_A * (m / 16) + LBO_A * (k / 8)] = A[i];
    }
    for (int i = tid; i < KT * 16; i += blockDim.x) {
        const int k = i / 16, n = i % 16;
        sb[n + 16 * (k % 8) + LBO_B * (k / 8)] = B[i];
    }
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
    if (tid == 0) {
        const uint32_t id = idesc_i8<16>(true, true, true);
        for (int s = 0; s < KT / 32; ++s) {
            const uint64_t da = desc(smem_u32(sa) + s * 4 * LBO_A, LBO_A, SBO_A);
            const uint64_t db = desc(smem_u32(sb) + s * 4 * LBO_B, LBO_B, 256);
            const uint32_t acc = s > 0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                "l"(da), "l"(db), "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    // wait for the MMA
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tm + ((uint32_t)(32 * warp) << 16)));
    for (int n = 0; n < 16; ++n) D[tid * 16 + n] = (int)v[n];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    std::vector<uint8_t> A(128 * KT);
    std::vector<int8_t> B(KT * 16);
    srand(1);
    for (auto& a : A) a = rand() % 256;
    for (auto& b : B) b = (int8_t)(rand() % 256 - 128);
    uint8_t* dA;
    int8_t* dB;
    int* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 128 * 16 * 4);
    probe<<<1, 128>>>(dA, dB, dD, 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> D(128 * 16);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            int ref = 0;
            for (int k = 0; k < KT; ++k) ref += (int)A[m * KT + k] * (int)B[k * 16 + n];
            if (ref != D[m * 16 + n]) {
                if (bad < 8) printf("m %d n %d ref %d got %d\n", m, n, ref, D[m * 16 + n]);
                ++bad;
            }
        }
    printf("probe_umma_i8: %s, mismatches %d / %d\n", cudaGetErrorString(e), bad, 128 * 16);
    return bad != 0;
}
