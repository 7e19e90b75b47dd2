// Host helpers: per-device property cache and once-per-device kernel attributes.
#include <mutex>
#include <vector>

#include "kitty_common.cuh"

namespace kitty {

namespace {

std::mutex g_mu;
struct DevProps {
    int sms = 0, smem_per_sm = 0;
};
std::vector<DevProps> g_props;
struct AttrKey {
    const void* fn;
    int dev, bytes, carve;
};
std::vector<AttrKey> g_attrs;

DevProps props() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    if ((int)g_props.size() <= dev) g_props.resize(dev + 1);
    DevProps& p = g_props[dev];
    if (p.sms == 0) {
        cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        if (p.sms <= 0) p.sms = 148;
        if (p.smem_per_sm <= 0) p.smem_per_sm = 233472;
    }
    return p;
}

}  // namespace

int device_sms() { return props().sms; }
int device_smem_per_sm() { return props().smem_per_sm; }

cudaError_t set_kernel_smem(const void* fn, int bytes, bool max_shared_carveout) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (const AttrKey& k : g_attrs)
            if (k.fn == fn && k.dev == dev && k.bytes >= bytes && k.carve == (int)max_shared_carveout) return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && max_shared_carveout)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    g_attrs.push_back(AttrKey{fn, dev, bytes, (int)max_shared_carveout});
    return cudaSuccess;
}

}  // namespace kitty
