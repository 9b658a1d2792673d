// Run-time specialised stage kernels (jit.cpp, jit_rt.cuh).
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace vqb::jit {

struct Kernel {
    void *e = nullptr; // cache entry
};

// NVRTC present (dlopen'ed on first use)
bool available();
// specialise stage programs on a (pseudo) state of pn qubits? (VQB_JIT=0/1
// overrides; default: pn >= 20, where a compile amortises over a few calls)
bool enabled(int pn);
// Kernels for the given sources (entry point `name`), compiling cache misses
// in parallel; raises if compilation fails.
std::vector<Kernel> get(const std::vector<std::string> &sources, const std::string &name);
void launch(const Kernel &k, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
            void **args);
int blocks_per_sm(const Kernel &k, unsigned block, size_t smem);
// number of kernels compiled (or loaded from the disk cache) so far
int64_t compiles();
// cubin of a source (tests / tools; no device needed)
std::string compile_only(const std::string &src, const std::string &name);

} // namespace vqb::jit
