// Launch accounting and optional per-launch CUDA-event timing.
//
// Profiling is off by default (zero cost beyond an atomic increment). When a
// benchmark enables it (vqb_profile_begin), every kernel launch is bracketed
// by two CUDA events on its own stream; vqb_profile_end synchronises and
// reports, per kernel name, the launch count and summed device time. Used by
// bench.py to measure the dominant kernel's average launch duration live.
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace vqb {

namespace {

std::atomic<int64_t> g_launches{0};
std::atomic<bool> g_prof{false};
std::mutex g_mu;

struct Rec {
    const char *name = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    double flops = 0, bytes = 0; // algorithmic FP64 flops / HBM bytes, if annotated
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    VQB_CUDA(cudaEventCreate(&e));
    return e;
}

} // namespace

void note_launch(int64_t n) { g_launches += n; }
int64_t launch_count() { return g_launches.load(); }

// Algorithmic FP64 flops issued by the fused executors (complex MAC = 8 flops).
static std::atomic<double> g_flops{0.0};
void note_flops(double f) {
    double cur = g_flops.load();
    while (!g_flops.compare_exchange_weak(cur, cur + f)) {
    }
}
double flop_count() { return g_flops.load(); }

ProfMark prof_begin(cudaStream_t st) {
    ProfMark m;
    if (!g_prof.load(std::memory_order_relaxed)) return m;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r;
    r.a = take_event();
    r.b = take_event();
    VQB_CUDA(cudaEventRecord(r.a, st));
    m.slot = (int)g_recs.size();
    m.st = st;
    g_recs.push_back(r);
    return m;
}

void check_launch(const char *what, const ProfMark &m) {
    note_launch(1);
    const cudaError_t e = cudaGetLastError();
    if (dry_run()) return;
    if (e != cudaSuccess) raise(VQB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    if (m.slot >= 0) {
        std::lock_guard<std::mutex> lk(g_mu);
        Rec &r = g_recs[m.slot];
        r.name = what;
        VQB_CUDA(cudaEventRecord(r.b, m.st));
    }
}

// Attach the launch's FP64 flops and HBM bytes (per-launch roofline).
void prof_annotate(const ProfMark &m, double flops, double bytes) {
    if (m.slot < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    g_recs[m.slot].flops = flops;
    g_recs[m.slot].bytes = bytes;
}

// Starts a profiling window (clears earlier records).
void prof_start() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    g_prof = true;
}

// Ends the window: "name count total_ms" lines, one per kernel name.
std::string prof_stop() {
    g_prof = false;
    VQB_CUDA(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<long, double>> agg;
    for (auto &r : g_recs) {
        if (!r.name) continue;
        float ms = 0;
        VQB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        auto &x = agg[r.name];
        x.first += 1;
        x.second += ms;
    }
    std::string out;
    char buf[256];
    for (auto &[k, v] : agg) {
        std::snprintf(buf, sizeof buf, "%s %ld %.6f\n", k.c_str(), v.first, v.second);
        out += buf;
    }
    // annotated launches, one line each: "#L name ms flops bytes"
    for (auto &r : g_recs) {
        if (!r.name || (r.flops == 0 && r.bytes == 0)) continue;
        float ms = 0;
        VQB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        std::snprintf(buf, sizeof buf, "#L %s %.6f %.6g %.6g\n", r.name, ms, r.flops, r.bytes);
        out += buf;
    }
    return out;
}

} // namespace vqb
