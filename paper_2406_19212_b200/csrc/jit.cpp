// Run-time specialisation of stage kernels (see jit_rt.cuh): NVRTC compiles a
// generated kernel for sm_100a once per stage-program *shape*; the cubin is
// loaded with the runtime's library API (cudaLibraryLoadData) and launched
// with cudaLaunchKernel. NVRTC is opened lazily with dlopen, so the library
// loads (and the interpreter runs) where NVRTC is absent; VQB_JIT=0 disables
// specialisation. Compiled kernels are cached in-process by source text, and
// on disk under $VQB_JIT_CACHE (if set) by a hash of it.
#include "jit.hpp"

#include <dlfcn.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

namespace vqb::jit {

namespace {

const char *kRuntimeSource =
#include "jit_rt.inc"
    ;

// ---- NVRTC, opened lazily ----
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
    void *h = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                            const char *const *) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *) = nullptr;
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*log)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t *) = nullptr;
    bool ok = false;
    Nvrtc() {
        for (const char *name : {"libnvrtc.so.12", "libnvrtc.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (h) break;
        }
        if (!h) return;
        create = reinterpret_cast<decltype(create)>(dlsym(h, "nvrtcCreateProgram"));
        compile = reinterpret_cast<decltype(compile)>(dlsym(h, "nvrtcCompileProgram"));
        log_size = reinterpret_cast<decltype(log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        log = reinterpret_cast<decltype(log)>(dlsym(h, "nvrtcGetProgramLog"));
        cubin_size = reinterpret_cast<decltype(cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        cubin = reinterpret_cast<decltype(cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        ok = create && compile && log_size && log && cubin_size && cubin && destroy;
    }
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    return n;
}

std::string cache_dir() {
    const char *d = std::getenv("VQB_JIT_CACHE");
    return d && *d ? std::string(d) : std::string();
}

std::string hex_hash(const std::string &s) {
    const size_t h1 = std::hash<std::string>{}(s);
    const size_t h2 = std::hash<std::string>{}(s + "#vqb");
    char buf[40];
    std::snprintf(buf, sizeof buf, "%016zx%016zx", h1, h2);
    return buf;
}

// source -> cubin (NVRTC), or from the disk cache
std::string compile_cubin(const std::string &src, const std::string &name) {
    const std::string dir = cache_dir();
    const std::string path = dir.empty() ? "" : dir + "/" + hex_hash(src) + ".cubin";
    if (!path.empty()) {
        std::ifstream f(path, std::ios::binary);
        if (f) {
            std::stringstream ss;
            ss << f.rdbuf();
            if (!ss.str().empty()) return ss.str();
        }
    }
    Nvrtc &nv = nvrtc();
    if (!nv.ok) raise(VQB_ERR_UNSUPPORTED, "jit: libnvrtc.so.12 not available");
    nvrtcProgram_t prog = nullptr;
    const char *hdr_src[1] = {kRuntimeSource};
    const char *hdr_name[1] = {"jit_rt.cuh"};
    if (nv.create(&prog, src.c_str(), (name + ".cu").c_str(), 1, hdr_src, hdr_name) != 0)
        raise(VQB_ERR_INTERNAL, "jit: nvrtcCreateProgram failed");
    const char *opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device",
                          "--fmad=true", "-lineinfo"};
    const int rc = nv.compile(prog, 5, opts);
    if (rc != 0) {
        size_t n = 0;
        nv.log_size(prog, &n);
        std::string log(n, '\0');
        nv.log(prog, log.data());
        nv.destroy(&prog);
        raise(VQB_ERR_INTERNAL, "jit: NVRTC compile failed: " + log.substr(0, 2000));
    }
    size_t n = 0;
    nv.cubin_size(prog, &n);
    std::string bin(n, '\0');
    nv.cubin(prog, bin.data());
    nv.destroy(&prog);
    if (!path.empty()) {
        std::ofstream(dir + "/" + hex_hash(src) + ".cu") << src; // for inspection
        const std::string tmp = path + ".tmp" + std::to_string(::getpid());
        std::ofstream f(tmp, std::ios::binary);
        f.write(bin.data(), (std::streamsize)bin.size());
        f.close();
        std::rename(tmp.c_str(), path.c_str());
    }
    return bin;
}

struct Entry {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    size_t max_smem = 0;
    std::unordered_map<size_t, int> per_sm; // by dynamic smem bytes
};

std::mutex g_mu;
std::unordered_map<std::string, Entry *> g_cache; // by source text (entries never freed)
std::atomic<int64_t> g_compiles{0};

Entry *load(const std::string &cubin, const std::string &name) {
    auto *e = new Entry();
    VQB_CUDA(cudaLibraryLoadData(&e->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    VQB_CUDA(cudaLibraryGetKernel(&e->kern, e->lib, name.c_str()));
    return e;
}

} // namespace

bool available() { return nvrtc().ok; }

bool enabled(int pn) {
    const char *v = std::getenv("VQB_JIT");
    if (v && *v) return std::atoi(v) != 0 && available();
    return pn >= 20 && available(); // small states: compile time would dominate
}

int64_t compiles() { return g_compiles.load(); }

std::vector<Kernel> get(const std::vector<std::string> &sources, const std::string &name) {
    std::vector<Kernel> out(sources.size());
    if (dry_run()) { // planning only: no compilation, a placeholder handle
        static Entry placeholder;
        for (auto &k : out) k.e = &placeholder;
        return out;
    }
    std::vector<size_t> miss;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (size_t i = 0; i < sources.size(); ++i) {
            auto it = g_cache.find(sources[i]);
            if (it != g_cache.end()) out[i].e = it->second;
            else miss.push_back(i);
        }
    }
    if (!miss.empty()) {
        // distinct misses, compiled in parallel on the host cores
        std::vector<size_t> uniq;
        {
            std::unordered_map<std::string, size_t> seen;
            for (size_t i : miss)
                if (seen.emplace(sources[i], i).second) uniq.push_back(i);
        }
        std::vector<std::string> bins(uniq.size());
        std::vector<std::string> errs(uniq.size());
        std::atomic<size_t> next{0};
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const size_t nt = std::min<size_t>(uniq.size(), hw);
        std::vector<std::thread> pool;
        for (size_t w = 0; w < nt; ++w)
            pool.emplace_back([&] {
                for (size_t k; (k = next.fetch_add(1)) < uniq.size();) {
                    try {
                        bins[k] = compile_cubin(sources[uniq[k]], name);
                    } catch (const std::exception &ex) {
                        errs[k] = ex.what();
                    }
                }
            });
        for (auto &th : pool) th.join();
        for (size_t k = 0; k < uniq.size(); ++k)
            if (!errs[k].empty()) raise(VQB_ERR_INTERNAL, errs[k]);
        std::lock_guard<std::mutex> lk(g_mu);
        for (size_t k = 0; k < uniq.size(); ++k) {
            const std::string &src = sources[uniq[k]];
            if (g_cache.find(src) == g_cache.end()) {
                g_cache[src] = load(bins[k], name);
                g_compiles.fetch_add(1);
            }
        }
        for (size_t i : miss) out[i].e = g_cache[sources[i]];
    }
    return out;
}

void launch(const Kernel &k, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
            void **args) {
    Entry *e = static_cast<Entry *>(k.e);
    if (dry_run()) return;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (smem > e->max_smem) {
            VQB_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void *>(e->kern),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            e->max_smem = smem;
        }
    }
    VQB_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(e->kern), dim3(grid), dim3(block),
                              args, smem, st));
}

int blocks_per_sm(const Kernel &k, unsigned block, size_t smem) {
    Entry *e = static_cast<Entry *>(k.e);
    if (dry_run()) return 4;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = e->per_sm.find(smem);
    if (it != e->per_sm.end()) return it->second;
    if (smem > e->max_smem) {
        VQB_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void *>(e->kern),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        e->max_smem = smem;
    }
    int b = 0;
    VQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &b, reinterpret_cast<const void *>(e->kern), (int)block, smem));
    b = std::max(b, 1);
    e->per_sm[smem] = b;
    return b;
}

std::string compile_only(const std::string &src, const std::string &name) {
    return compile_cubin(src, name);
}

} // namespace vqb::jit
