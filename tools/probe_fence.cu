// Probe: which synchronisation instructions wait for a thread's outstanding
// global loads?  A warp issues an LDG (cold, ~1 us) it does not consume, then
// st.shared and one of: fence.proxy.async.shared::cta, mbarrier.arrive
// (release), mbarrier.arrive.relaxed, bar.sync, __syncwarp.  Prints cycles.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint4* g, int mode, long long* out) {
    __shared__ __align__(16) uint4 buf[64];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1024;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint4 v;
    const uint4* p = g + ((size_t)blockIdx.x * 1000003ull + threadIdx.x * 7919ull) % (1ull << 26);
    long long t0 = clock64();
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    long long t1 = clock64();
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(smem_u32(&buf[threadIdx.x])), "r"(threadIdx.x) : "memory");
    if (mode == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode == 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (mode == 2) asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (mode == 3) asm volatile("bar.sync 1, 32;" ::: "memory");
    if (mode == 4) __syncwarp();
    if (mode == 5) asm volatile("membar.cta;" ::: "memory");
    if (mode == 6) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // same as 0, after flush
    long long t2 = clock64();
    // consume the load afterwards
    long long t3 = clock64();
    const uint32_t s = v.x ^ v.y ^ v.z ^ v.w;
    long long t4 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[mode * 4 + 0] = t1 - t0;
        out[mode * 4 + 1] = t2 - t1;
        out[mode * 4 + 2] = t4 - t3;
        out[mode * 4 + 3] = s;
    }
}

int main() {
    uint4* g;
    long long* d;
    cudaMalloc(&g, (size_t)1 << 30);
    cudaMemset(g, 1, (size_t)1 << 30);
    char* flush;
    cudaMalloc(&flush, (size_t)512 << 20);
    cudaMalloc(&d, 8 * 4 * 8);
    const char* names[] = {"fence.proxy.async", "mbarrier.arrive (release)", "mbarrier.arrive.relaxed", "bar.sync(32)", "__syncwarp", "membar.cta", "fence.proxy.async", "none"};
    for (int mode = 0; mode < 8; ++mode) {
        cudaMemset(d, 0, 8 * 4 * 8);
        cudaMemset(flush, mode, (size_t)512 << 20);
        // evict: touch another buffer so the loads are cold
        probe<<<148, 32>>>(g, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[32];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-28s %s: issue %lld cyc, sync op %lld cyc, use-after %lld cyc\n", names[mode], cudaGetErrorString(e),
               h[mode * 4], h[mode * 4 + 1], h[mode * 4 + 2]);
    }
    return 0;
}
