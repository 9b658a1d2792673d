// Device selection, tracked device allocations and releasable scratch caches.
//
// The reference counts live and peak full-state amplitude buffers
// (AllocStats, state.hpp:56-83,154-161) so its tests can check the memory
// contract of the gradient sweep (tests/test_autodiff.cpp:132-145). The
// device path does the same for its amplitude buffers and also counts bytes,
// scratch included; cached buffers stay counted as live until
// vqb_release_caches() frees them.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "common.hpp"

namespace vqb {

namespace {
std::atomic<int64_t> g_live_states{0}, g_peak_states{0};
std::atomic<uint64_t> g_live_bytes{0}, g_peak_bytes{0};

template <typename T> void raise_peak(std::atomic<T> &peak, T v) {
    T seen = peak.load();
    while (seen < v && !peak.compare_exchange_weak(seen, v)) {
    }
}

std::mutex &reg_mu() {
    static std::mutex m;
    return m;
}
std::unordered_set<DevMem *> &registry() {
    static std::unordered_set<DevMem *> r;
    return r;
}
std::vector<void (*)()> &release_fns() {
    static std::vector<void (*)()> v;
    return v;
}
} // namespace

int current_device() {
    int d = 0;
    VQB_CUDA(cudaGetDevice(&d));
    if (d < 0 || d >= kMaxDevices) raise(VQB_ERR_UNSUPPORTED, "device ordinal beyond 16");
    return d;
}

DevScope::DevScope(int dev) {
    int cur = 0;
    VQB_CUDA(cudaGetDevice(&cur));
    if (cur != dev) {
        VQB_CUDA(cudaSetDevice(dev));
        prev = cur;
    }
}

DevScope::~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
}

void *dev_alloc(size_t bytes, bool state, bool raise_on_fail) {
    void *p = nullptr;
    if (dry_run()) return reinterpret_cast<void *>(uintptr_t(256)); // planning only: never dereferenced
    const cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (!raise_on_fail) return nullptr;
        raise(VQB_ERR_SIZE, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                cudaGetErrorString(e));
    }
    raise_peak(g_peak_bytes, g_live_bytes.fetch_add(bytes) + bytes);
    if (state) raise_peak(g_peak_states, g_live_states.fetch_add(1) + 1);
    return p;
}

void dev_free(void *p, size_t bytes, bool state) {
    if (!p || dry_run()) return;
    cudaFree(p);
    g_live_bytes.fetch_sub(bytes);
    if (state) g_live_states.fetch_sub(1);
}

AllocStats alloc_stats() {
    return {g_live_states.load(), g_peak_states.load(), g_live_bytes.load(), g_peak_bytes.load()};
}

void reset_alloc_peak() {
    g_peak_states.store(g_live_states.load());
    g_peak_bytes.store(g_live_bytes.load());
}

DevMem::DevMem() {
    std::lock_guard<std::mutex> lk(reg_mu());
    registry().insert(this);
}

DevMem::~DevMem() {
    {
        std::lock_guard<std::mutex> lk(reg_mu());
        registry().erase(this);
    }
    release();
}

void DevMem::ensure(size_t bytes) {
    const int d = current_device();
    if (bytes > cap[d]) {
        dev_free(ptr[d], cap[d], false);
        ptr[d] = nullptr;
        cap[d] = 0;
        ptr[d] = dev_alloc(bytes, false);
        cap[d] = bytes;
    }
    p = ptr[d];
}

void DevMem::release() {
    for (int d = 0; d < kMaxDevices; ++d) {
        if (!ptr[d]) continue;
        dev_free(ptr[d], cap[d], false); // cudaFree resolves the owning device (UVA)
        ptr[d] = nullptr;
        cap[d] = 0;
    }
    p = nullptr;
}

void register_cache_release(void (*fn)()) {
    std::lock_guard<std::mutex> lk(reg_mu());
    if (std::find(release_fns().begin(), release_fns().end(), fn) == release_fns().end())
        release_fns().push_back(fn);
}

void release_caches() {
    cudaDeviceSynchronize();
    std::vector<void (*)()> fns;
    {
        std::lock_guard<std::mutex> lk(reg_mu());
        for (DevMem *m : registry()) m->release();
        fns = release_fns();
    }
    for (auto fn : fns) fn();
}

} // namespace vqb
