// Common host/device definitions for libvqcs_b200.
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vqcs_b200.h"

namespace vqb {

using cplx = std::complex<double>;
using cvec = std::vector<cplx>;

// Status-carrying exception; the C-ABI layer turns it into a vqb_status and a
// thread-local message (errors.hpp:23-96 taxonomy).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string &msg) { throw Error(code, msg); }

#define VQB_CUDA(call)                                                                     \
    do {                                                                                   \
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
} // namespace vqb
