// Common host/device definitions for libvqcs_b200.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vqcs_b200.h"

namespace vqb {

// Accumulating host timer (VQB_HOST_TIMING): add the scope's time to *acc.
struct HostAcc {
    double *acc;
    std::chrono::steady_clock::time_point t0;
    explicit HostAcc(double *a) : acc(a), t0(std::chrono::steady_clock::now()) {}
    ~HostAcc() {
        *acc += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    }
};

// Host-side phase timing for diagnostics (VQB_HOST_TIMING=1 prints to stderr).
struct HostTimer {
    const char *what;
    std::chrono::steady_clock::time_point t0;
    bool on;
    explicit HostTimer(const char *w) : what(w), t0(std::chrono::steady_clock::now()) {
        static const bool enabled = std::getenv("VQB_HOST_TIMING") != nullptr;
        on = enabled;
    }
    ~HostTimer() {
        if (!on) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[host] %-28s %9.1f us\n", what, us);
    }
};

using cplx = std::complex<double>;
using cvec = std::vector<cplx>;

// Status-carrying exception; the C-ABI layer turns it into a vqb_status and a
// thread-local message (errors.hpp:23-96 taxonomy).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string &msg) { throw Error(code, msg); }

// Planning-only mode for development on a host without a GPU (VQB_DRYRUN=1):
// CUDA runtime calls and kernel launches are skipped, so the host side --
// reverse programs, stage planning, lowering, kernel generation and
// VQB_JIT_DUMP -- runs to completion and can be inspected; every result read
// back from the "device" is garbage. Never set in production.
inline bool dry_run() {
    static const bool on = [] {
        const char *v = std::getenv("VQB_DRYRUN");
        return v && *v == '1';
    }();
    return on;
}

#define VQB_CUDA(call)                                                                     \
    do {                                                                                   \
        if (::vqb::dry_run()) break;                                                       \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            ::vqb::raise(VQB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Launch accounting (vqb_kernel_launch_count).
void note_launch(int64_t n = 1);

inline int popcount64(uint64_t x) { return __builtin_popcountll(x); }

} // namespace vqb

namespace vqb {
// Optional per-launch CUDA-event profiling (vqb_profile_begin/end): a mark is
// taken before a launch and closed by check_launch after it.
struct ProfMark {
    int slot = -1;
    cudaStream_t st = nullptr;
};
ProfMark prof_begin(cudaStream_t st);
void check_launch(const char *what, const ProfMark &m);
void prof_annotate(const ProfMark &m, double flops, double bytes);
} // namespace vqb

namespace vqb {
// ---- devices and device memory (memory.cpp) ----
constexpr int kMaxDevices = 16;
int current_device();
// Makes `dev` the calling thread's current device for the scope (no-op when
// it already is); every entry point that touches a state opens one on the
// state's device, so states on several devices can be driven from one thread.
struct DevScope {
    int prev = -1;
    explicit DevScope(int dev);
    ~DevScope();
    DevScope(const DevScope &) = delete;
    DevScope &operator=(const DevScope &) = delete;
};

// Tracked device allocations: `state` buffers are full amplitude vectors
// (the reference's AmpBuffer bookkeeping, state.hpp:56-83), the rest scratch.
void *dev_alloc(size_t bytes, bool state, bool raise_on_fail = true);
void dev_free(void *p, size_t bytes, bool state);
struct AllocStats {
    int64_t live_states, peak_states;
    uint64_t live_bytes, peak_bytes;
};
AllocStats alloc_stats();
void reset_alloc_peak();

// Grow-only device scratch, one buffer per device (a thread may drive states
// on several devices). ensure() makes `p` the current device's buffer.
// Instances register themselves so release_caches() can free every one.
struct DevMem {
    void *p = nullptr;
    void *ptr[kMaxDevices] = {};
    size_t cap[kMaxDevices] = {};
    DevMem();
    ~DevMem();
    DevMem(const DevMem &) = delete;
    DevMem &operator=(const DevMem &) = delete;
    void ensure(size_t bytes);
    void release();
};
// Callbacks run by release_caches() (cached working states, batch slots).
void register_cache_release(void (*fn)());
// Frees every cached device buffer of this process (scratch, cached working
// states); must not run concurrently with other calls.
void release_caches();
} // namespace vqb
