// Losses and adjoint gradients on the device (autodiff.hpp:80-329).
//
// Algorithm 2 of the paper: forward to |Phi_M>, |Psi> = H|Phi_M>,
// then per element in reverse pull both states back through the inverse and
// accumulate <Psi| dU |Phi> for every active parameter. Only two full-size
// working states are held. Gradient partials are reduced on the device and
// written straight into a device gradient vector; the host reads it once at
// the end (no per-gate synchronisation).
#include "autodiff.hpp"

#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <mutex>
#include <thread>

#include "engine.hpp"

namespace vqb {

namespace {

// ---- host-parallel adjoint ----
// One persistent worker thread (its thread-local executor buffers and kernel
// lookups stay warm across calls) runs the reverse sweep's host work --
// reverse program, folding, analysis, stage planning, block fusion, lowering,
// kernel lookup -- while the calling thread plans and launches the forward
// pass; the worker launches only after the caller opens the gate (stream
// order: forward, costate, loss, then the sweep).
struct LaunchGate {
    std::mutex mu;
    std::condition_variable cv;
    bool open = false, abort = false;
};
thread_local LaunchGate *g_gate = nullptr;

class Worker {
  public:
    Worker() : th_([this] { loop(); }) {}
    ~Worker() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    std::future<void> submit(std::function<void()> fn) {
        std::packaged_task<void()> task(std::move(fn));
        auto fut = task.get_future();
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(task));
        }
        cv_.notify_one();
        return fut;
    }

  private:
    void loop() {
        for (;;) {
            std::packaged_task<void()> task;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                task = std::move(q_.front());
                q_.pop_front();
            }
            task();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::packaged_task<void()>> q_;
    bool stop_ = false;
    std::thread th_;
};

Worker &worker() {
    static Worker w;
    return w;
}

bool parallel_adjoint() {
    static const bool on = [] {
        const char *v = std::getenv("VQB_PARALLEL_ADJOINT");
        return !(v && *v == '0');
    }();
    return on;
}

// Runs `sweep` on the worker behind a gate; open() lets it launch, finish()
// waits for it (rethrowing its error). If the caller unwinds without opening,
// the sweep is aborted before any launch.
class GatedSweep {
  public:
    explicit GatedSweep(std::function<void()> sweep) {
        // the worker drives the caller's device (its buffers and the states'
        // streams live there)
        const int dev = current_device();
        fut_ = worker().submit([this, dev, sweep = std::move(sweep)] {
            VQB_CUDA(cudaSetDevice(dev));
            g_gate = &gate_;
            struct Reset {
                ~Reset() { g_gate = nullptr; }
            } reset;
            sweep();
        });
    }
    void open() {
        {
            std::lock_guard<std::mutex> lk(gate_.mu);
            gate_.open = true;
        }
        gate_.cv.notify_all();
    }
    void finish() {
        done_ = true;
        fut_.get();
    }
    ~GatedSweep() {
        if (done_) return;
        {
            std::lock_guard<std::mutex> lk(gate_.mu);
            gate_.abort = true;
        }
        gate_.cv.notify_all();
        fut_.wait();
    }

  private:
    LaunchGate gate_;
    std::future<void> fut_;
    bool done_ = false;
};

// Device buffer for the gradient vector and the loss, reused across calls
// on a thread (grow-only, per device): a cudaMalloc/cudaFree pair per call
// would cost more than a small gradient (and cudaFree synchronises the device).
struct DevBuf {
    void *p = nullptr;
    explicit DevBuf(size_t bytes) {
        static thread_local DevMem cached;
        cached.ensure(bytes);
        p = cached.p;
    }
    template <typename T> T *as() { return static_cast<T *>(p); }
};

// Working states of the losses / gradients, kept for the next call instead
// of being freed (allocation, stream and workspace setup otherwise dominate
// small problems such as config 0, and allocating and freeing 2 x 16 GiB per
// 30-qubit gradient cost 100-500 ms of cudaMalloc/cudaFree against a ~0.8 s
// gradient). One process-wide pool keyed by (device, shape): any number of
// states up to 2^26 amplitudes (1 GiB) up to 8 in total, and at most two of
// one larger shape (<= 2^31 amplitudes: a 30-qubit gradient's Phi and Psi;
// caching a new large shape drops the old one). Cached states stay counted in
// vqb_alloc_stats; vqb_release_caches() frees them.
constexpr uint64_t kCacheLimit = 1ull << 26;
constexpr uint64_t kLargeCacheLimit = 1ull << 31;
constexpr int kLargeCacheCount = 2;
constexpr size_t kSmallCacheCount = 8;

struct ScratchPool {
    std::mutex mu;
    std::vector<DeviceState *> free_list;
};
ScratchPool &pool() {
    static ScratchPool *p = [] {
        register_cache_release([] {
            ScratchPool &sp = pool();
            std::vector<DeviceState *> v;
            {
                std::lock_guard<std::mutex> lk(sp.mu);
                v.swap(sp.free_list);
            }
            for (DeviceState *s : v) state_destroy(s);
        });
        return new ScratchPool; // never destroyed: states may outlive static teardown
    }();
    return *p;
}

DeviceState *scratch(int n, int mixed) {
    const uint64_t size = 1ull << (mixed ? 2 * n : n);
    const int dev = current_device();
    if (size <= kLargeCacheLimit) {
        ScratchPool &sp = pool();
        std::lock_guard<std::mutex> lk(sp.mu);
        for (size_t i = 0; i < sp.free_list.size(); ++i) {
            DeviceState *s = sp.free_list[i];
            if (s->n == n && s->mixed == mixed && s->device == dev) {
                sp.free_list.erase(sp.free_list.begin() + i);
                return s;
            }
        }
    }
    return state_create(n, mixed);
}

struct StateGuard {
    DeviceState *s;
    ~StateGuard() {
        cudaStreamSynchronize(s->stream);
        std::vector<DeviceState *> drop;
        {
            ScratchPool &sp = pool();
            std::lock_guard<std::mutex> lk(sp.mu);
            int small_n = 0, large_n = 0;
            for (DeviceState *c : sp.free_list) ++(c->size > kCacheLimit ? large_n : small_n);
            const bool small = s->size <= kCacheLimit && small_n < (int)kSmallCacheCount;
            const bool large = s->size > kCacheLimit && s->size <= kLargeCacheLimit;
            if (large) {
                // keep the newest shape: drop cached large states of other shapes
                for (size_t i = 0; i < sp.free_list.size();) {
                    DeviceState *c = sp.free_list[i];
                    if (c->size > kCacheLimit &&
                        (c->n != s->n || c->mixed != s->mixed || c->device != s->device)) {
                        drop.push_back(c);
                        sp.free_list.erase(sp.free_list.begin() + i);
                        --large_n;
                    } else {
                        ++i;
                    }
                }
            }
            if (small || (large && large_n < kLargeCacheCount)) sp.free_list.push_back(s);
            else drop.push_back(s);
        }
        for (DeviceState *d : drop) state_destroy(d);
    }
};

DeviceState *clone(const DeviceState *src) {
    DeviceState *d = scratch(src->n, src->mixed);
    VQB_CUDA(cudaStreamSynchronize(src->stream));
    VQB_CUDA(cudaMemcpyAsync(d->amps, src->amps, sizeof(double2) * src->size,
                             cudaMemcpyDeviceToDevice, d->stream));
    return d;
}

// The reverse steps after the last parametric one only bring Phi back to the
// initial state (autodiff.hpp:151-154 reports max |Phi_end - s0|): without a
// residual request nothing reads their result, so they are not run.
void drop_dead_tail(std::vector<RevOp> &rprog, bool want_residual) {
    if (want_residual) return;
    while (!rprog.empty() && rprog.back().dmats.empty()) rprog.pop_back();
}

void check_operator(const PauliPack &op, int n, const char *what) {
    if (op.max_qubit > n)
        raise(VQB_ERR_INDEX, std::string(what) + ": operator acts on qubit " +
                                 std::to_string(op.max_qubit) + " but the state has " +
                                 std::to_string(n) + " qubits");
}

void reject_channels(const vqb_op *ops, int64_t count, const char *what) {
    for (int64_t i = 0; i < count; ++i)
        if (ops[i].elem == VQB_ELEM_CHANNEL)
            raise(VQB_ERR_TYPE, std::string(what) +
                                    ": circuit contains quantum channels; use the mixed-state variant");
}

} // namespace

double loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms, int64_t nterms,
                 DeviceState *s0, bool fused) {
    if (s0->mixed) raise(VQB_ERR_TYPE, "loss_pure: pure initial state required");
    reject_channels(ops, count, "loss_pure");
    const PauliPack op = pack_operator(terms, nterms, false);
    const auto es = build_elements(ops, count);
    std::vector<Gate> prog;
    for (const auto &e : es) {
        check_fit(e.gate.pos, e.gate.m, s0->n);
        prog.push_back(e.gate);
    }
    check_operator(op, s0->n, "loss_pure");
    DeviceState *s = clone(s0);
    StateGuard g{s};
    run_program(s, prog, fused);
    return expectation(s, op).real();
}

double loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms, int64_t nterms,
                  DeviceState *dm0, bool fused) {
    if (!dm0->mixed) raise(VQB_ERR_TYPE, "loss_mixed: mixed initial state required");
    const PauliPack op = pack_operator(terms, nterms, false);
    check_operator(op, dm0->n, "loss_mixed");
    const auto es = build_elements(ops, count);
    for (const auto &e : es) {
        if (e.channel) check_fit(e.chan.pos, e.chan.m, dm0->n);
        else check_fit(e.gate.pos, e.gate.m, dm0->n);
    }
    DeviceState *s = clone(dm0);
    StateGuard g{s};
    run_program(s, mixed_forward_program(es, dm0->n), fused);
    return expectation(s, op).real();
}

void wait_issue_gate() {
    LaunchGate *g = g_gate;
    if (!g) return;
    std::unique_lock<std::mutex> lk(g->mu);
    g->cv.wait(lk, [&] { return g->open || g->abort; });
    if (g->abort) raise(VQB_ERR_INTERNAL, "adjoint sweep aborted: the forward pass failed");
    g_gate = nullptr; // open: later launches need not wait
}

GradientOut gradient_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                          int64_t nterms, DeviceState *s0, bool want_residual, bool fused) {
    if (s0->mixed) raise(VQB_ERR_TYPE, "gradient_pure: pure initial state required");
    reject_channels(ops, count, "gradient_pure");
    const int n = s0->n;
    const PauliPack op = pack_operator(terms, nterms, false);
    check_operator(op, n, "gradient_pure");
    const auto es = build_elements(ops, count);
    std::vector<int64_t> base(count);
    int64_t total = 0;
    std::vector<Gate> fwd;
    for (int64_t i = 0; i < count; ++i) {
        base[i] = total;
        total += es[i].gate.num_active();
        check_fit(es[i].gate.pos, es[i].gate.m, n);
        fwd.push_back(es[i].gate);
    }

    DeviceState *phi = clone(s0);
    StateGuard gphi{phi};
    GradientOut out;
    out.grads.assign(total, 0.0);
    if (total == 0) {
        run_program(phi, fwd, fused);
        out.loss = expectation(phi, op).real();
        return out;
    }
    DeviceState *psi = scratch(n, 0); // fully overwritten by apply_operator
    StateGuard gpsi{psi};
    const size_t gbytes = sizeof(double2) * ((total + 1) / 2); // keep dloss 16-B aligned
    DevBuf dbuf(gbytes + sizeof(double2));
    double *dgrads = dbuf.as<double>();
    double2 *dloss = reinterpret_cast<double2 *>(dbuf.as<char>() + gbytes);
    // every writer accumulates (steps may share a gradient entry)
    VQB_CUDA(cudaMemsetAsync(dgrads, 0, gbytes, phi->stream));
    auto sweep = [&] {
        HostTimer ht("gradient_pure reverse");
        std::vector<RevOp> rprog;
        {
            HostTimer ht2("reverse program");
            rprog = pure_reverse_program(es, base);
            drop_dead_tail(rprog, want_residual);
        }
        run_reverse(phi, psi, rprog, dgrads, fused);
    };
    std::unique_ptr<GatedSweep> gs;
    if (parallel_adjoint()) gs = std::make_unique<GatedSweep>(sweep);
    {
        HostTimer ht("gradient_pure forward");
        run_program(phi, fwd, fused);
    }
    VQB_CUDA(cudaStreamSynchronize(psi->stream));
    apply_operator(phi, psi->amps, op, false);
    dot_async(phi, phi->amps, psi->amps, dloss); // loss = Re <phi|H phi>
    if (gs) {
        gs->open();
        gs->finish();
    } else {
        sweep();
    }

    double2 hl;
    VQB_CUDA(cudaMemcpyAsync(out.grads.data(), dgrads, sizeof(double) * total,
                             cudaMemcpyDeviceToHost, phi->stream));
    VQB_CUDA(cudaMemcpyAsync(&hl, dloss, sizeof(double2), cudaMemcpyDeviceToHost, phi->stream));
    VQB_CUDA(cudaStreamSynchronize(phi->stream));
    out.loss = hl.x;
    if (want_residual) out.residual = max_abs_diff(phi, phi->amps, s0->amps);
    return out;
}

GradientOut gradient_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                           int64_t nterms, DeviceState *dm0, bool want_residual, bool fused) {
    if (!dm0->mixed) raise(VQB_ERR_TYPE, "gradient_mixed: mixed initial state required");
    const int n = dm0->n;
    const PauliPack op = pack_operator(terms, nterms, true); // op.conjugated() (autodiff.hpp:247)
    check_operator(op, n, "gradient_mixed");
    const auto es = build_elements(ops, count);
    std::vector<int64_t> base(count);
    int64_t total = 0;
    for (int64_t i = 0; i < count; ++i) {
        base[i] = total;
        if (es[i].channel) {
            check_fit(es[i].chan.pos, es[i].chan.m, n);
        } else {
            total += es[i].gate.num_active();
            check_fit(es[i].gate.pos, es[i].gate.m, n);
        }
    }
    // Channel inverses on the host first (LU, condition limit;
    // autodiff.hpp:263-276), so a non-invertible channel fails before any
    // device work.
    std::vector<cvec> chan_inv(count), chan_adj(count);
    if (total > 0) {
        for (int64_t i = count; i-- > 0;) {
            if (!es[i].channel) continue;
            const Channel &ch = es[i].chan;
            const cvec s = channel_superop(ch);
            const int d = 1 << (2 * ch.m);
            const Inverse lu = channel_inverse(ch, s);
            if (lu.singular || lu.condition > kChannelConditionLimit) {
                static const char *names[] = {"Generic", "AmplitudeDamping", "PhaseDamping",
                                              "Depolarizing"};
                raise(VQB_ERR_NONINVERTIBLE,
                      std::string("gradient_mixed: the superoperator of channel '") +
                          names[ch.kind & 3] + "' on qubit " + std::to_string(ch.pos[0]) +
                          " (element " + std::to_string(i + 1) +
                          ") is singular or too ill-conditioned to invert");
            }
            chan_inv[i] = lu.inv;
            chan_adj[i] = adjoint(s, d);
        }
    }

    DeviceState *phi = clone(dm0);
    StateGuard gphi{phi};
    DeviceState *psi = scratch(n, 1); // fully overwritten by identity_costate
    StateGuard gpsi{psi};
    GradientOut out;
    out.grads.assign(total, 0.0);
    const size_t gbytes = sizeof(double2) * ((std::max<int64_t>(total, 1) + 1) / 2);
    DevBuf dbuf(gbytes + sizeof(double2));
    double *dgrads = dbuf.as<double>();
    double2 *dloss = reinterpret_cast<double2 *>(dbuf.as<char>() + gbytes);
    // every writer accumulates: the ket and bra halves of a gate share its entries
    VQB_CUDA(cudaMemsetAsync(dgrads, 0, gbytes, phi->stream));
    auto sweep = [&] {
        std::vector<RevOp> rprog = mixed_reverse_program(es, n, base, chan_inv, chan_adj);
        drop_dead_tail(rprog, want_residual);
        run_reverse(phi, psi, rprog, dgrads, fused);
    };
    std::unique_ptr<GatedSweep> gs;
    if (total > 0 && parallel_adjoint()) gs = std::make_unique<GatedSweep>(sweep);
    run_program(phi, mixed_forward_program(es, n), fused);
    identity_costate(psi, op); // <<Psi| = <<I| H (autodiff.hpp:241-248)
    VQB_CUDA(cudaStreamSynchronize(psi->stream));
    dot_async(phi, psi->amps, phi->amps, dloss); // loss = Re <<psi|phi>>
    if (total > 0) {
        if (gs) {
            gs->open();
            gs->finish();
        } else {
            sweep();
        }
        VQB_CUDA(cudaMemcpyAsync(out.grads.data(), dgrads, sizeof(double) * total,
                                 cudaMemcpyDeviceToHost, phi->stream));
    }
    double2 hl;
    VQB_CUDA(cudaMemcpyAsync(&hl, dloss, sizeof(double2), cudaMemcpyDeviceToHost, phi->stream));
    VQB_CUDA(cudaStreamSynchronize(phi->stream));
    out.loss = hl.x;
    if (want_residual && total > 0) out.residual = max_abs_diff(phi, phi->amps, dm0->amps);
    return out;
}

} // namespace vqb
