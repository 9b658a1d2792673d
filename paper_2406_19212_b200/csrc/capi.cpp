// extern "C" boundary (include/vqcs_b200.h). Every entry point catches all
// exceptions and returns a vqb_status; messages go to a thread-local buffer.
#include <cstring>
#include <mutex>
#include <string>

#include "autodiff.hpp"
#include "engine.hpp"
#include "plan.hpp"
#include "sharded.hpp"

using namespace vqb;

struct vqb_state : DeviceState {};
struct vqb_sharded {
    Sharded *p;
};

namespace vqb {
std::string bench_report(const vqb_bench_record *recs, int64_t count, int format);
std::string debug_jit_source(int regs, const void *params, size_t nbytes, bool rev, double *flops);
int64_t launch_count();
double flop_count();
void prof_start();
std::string prof_stop();
}

namespace {

thread_local std::string g_err;

template <typename F> int guard(F &&f) {
    try {
        f();
        return VQB_OK;
    } catch (const vqb::Error &e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "host allocation failed";
        return VQB_ERR_SIZE;
    } catch (const std::exception &e) {
        g_err = e.what();
        return VQB_ERR_INTERNAL;
    }
}

DeviceState *ds(vqb_state *s) {
    if (!s) raise(VQB_ERR_USAGE, "null state handle");
    return static_cast<DeviceState *>(s);
}
DeviceState *ds(const vqb_state *s) { return ds(const_cast<vqb_state *>(s)); }

void same_device(const DeviceState *a, const DeviceState *b) {
    if (a->device != b->device)
        raise(VQB_ERR_USAGE, "states on different devices (" + std::to_string(a->device) + " and " +
                                 std::to_string(b->device) + ")");
}

void need(const void *p, const char *what) {
    if (!p) raise(VQB_ERR_USAGE, std::string("null argument: ") + what);
}

void check_count(const DeviceState *s, uint64_t count, const char *what) {
    if (count != s->size)
        raise(VQB_ERR_SHAPE, std::string(what) + ": count " + std::to_string(count) +
                                 " does not match the state's " + std::to_string(s->size) +
                                 " amplitudes");
}

void write_grads(const GradientOut &r, double *loss, double *grads, int64_t cap, int64_t *ng,
                 double *res) {
    if ((int64_t)r.grads.size() > cap)
        raise(VQB_ERR_SHAPE, "gradient buffer too small: need " + std::to_string(r.grads.size()));
    *loss = r.loss;
    if (!r.grads.empty()) std::memcpy(grads, r.grads.data(), sizeof(double) * r.grads.size());
    *ng = (int64_t)r.grads.size();
    if (res) *res = r.residual;
}

// Device states of vqb_apply_circuit_copy_batch, kept for the next call of
// the same shape; freed by vqb_release_caches().
struct BatchSlots {
    std::mutex mu;
    std::vector<DeviceState *> states;
};
BatchSlots &batch_slots() {
    static BatchSlots *b = [] {
        register_cache_release([] {
            BatchSlots &bs = batch_slots();
            std::lock_guard<std::mutex> lk(bs.mu);
            for (DeviceState *d : bs.states) state_destroy(d);
            bs.states.clear();
        });
        return new BatchSlots;
    }();
    return *b;
}

} // namespace

extern "C" {

VQB_API const char *vqb_last_error(void) { return g_err.c_str(); }

VQB_API const char *vqb_build_info(void) {
    return "libvqcs_b200: sm_100a complex128 state-vector/density-matrix core (CUDA "
#ifdef __CUDACC_VER_MAJOR__
        "nvcc"
#endif
        ")";
}

VQB_API int64_t vqb_kernel_launch_count(void) { return vqb::launch_count(); }

VQB_API double vqb_flop_count(void) { return vqb::flop_count(); }

VQB_API int vqb_debug_jit_source(int regs, const void *params, size_t nbytes, int rev, char *out,
                                 size_t cap, double *flops_per_amp) {
    return guard([&] {
        const std::string src = vqb::debug_jit_source(regs, params, nbytes, rev != 0, flops_per_amp);
        if (src.size() + 1 > cap) raise(VQB_ERR_SIZE, "output buffer too small");
        std::memcpy(out, src.c_str(), src.size() + 1);
    });
}

VQB_API int vqb_profile_begin(void) {
    return guard([&] { prof_start(); });
}

VQB_API int vqb_profile_end(char *buf, int64_t cap) {
    return guard([&] {
        const std::string r = prof_stop();
        if (buf && cap > 0) {
            const size_t n = std::min<size_t>(r.size(), size_t(cap - 1));
            std::memcpy(buf, r.data(), n);
            buf[n] = 0;
        }
    });
}

VQB_API int vqb_alloc_stats(int64_t *live_states, int64_t *peak_states, uint64_t *live_bytes,
                            uint64_t *peak_bytes) {
    return guard([&] {
        const AllocStats a = alloc_stats();
        if (live_states) *live_states = a.live_states;
        if (peak_states) *peak_states = a.peak_states;
        if (live_bytes) *live_bytes = a.live_bytes;
        if (peak_bytes) *peak_bytes = a.peak_bytes;
    });
}

VQB_API int vqb_reset_alloc_peak(void) {
    return guard([&] { reset_alloc_peak(); });
}

VQB_API int vqb_release_caches(void) {
    return guard([&] { release_caches(); });
}

VQB_API int vqb_state_stream(const vqb_state *s, void **stream) {
    return guard([&] {
        need(stream, "stream");
        *stream = ds(s)->stream;
    });
}

VQB_API int vqb_state_create(int32_t n, int32_t mixed, vqb_state **out) {
    return guard([&] {
        need(out, "out");
        *out = static_cast<vqb_state *>(state_create(n, mixed));
    });
}

VQB_API int vqb_state_wrap(void *ptr, int32_t n, int32_t mixed, uint64_t goff, int32_t gq,
                           vqb_state **out) {
    return guard([&] {
        need(ptr, "device_ptr");
        need(out, "out");
        *out = static_cast<vqb_state *>(state_wrap(ptr, n, mixed, goff, gq));
    });
}

VQB_API int vqb_state_destroy(vqb_state *s) {
    return guard([&] { state_destroy(static_cast<DeviceState *>(s)); });
}

VQB_API int vqb_state_info(const vqb_state *s, int32_t *n, int32_t *mixed, uint64_t *count) {
    return guard([&] {
        const DeviceState *d = ds(s);
        DevScope on_(d->device);
        if (n) *n = d->n;
        if (mixed) *mixed = d->mixed;
        if (count) *count = d->size;
    });
}

VQB_API int vqb_state_device_ptr(const vqb_state *s, void **ptr) {
    return guard([&] { *ptr = ds(s)->amps; });
}

VQB_API int vqb_state_set_zero(vqb_state *s) {
    return guard([&] {
        DevScope on_(ds(s)->device);
        state_set_zero(ds(s));
    });
}

VQB_API int vqb_state_upload(vqb_state *s, const vqb_c128 *host, uint64_t count) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(host, "host");
        check_count(d, count, "state_upload");
        VQB_CUDA(cudaMemcpyAsync(d->amps, host, sizeof(double2) * count, cudaMemcpyHostToDevice,
                                 d->stream));
        sync(d);
    });
}

VQB_API int vqb_state_upload_async(vqb_state *s, const vqb_c128 *host, uint64_t count) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(host, "host");
        check_count(d, count, "state_upload_async");
        cudaPointerAttributes attr{};
        if (!dry_run() && (cudaPointerGetAttributes(&attr, host) != cudaSuccess ||
                           attr.type != cudaMemoryTypeHost)) {
            cudaGetLastError();
            raise(VQB_ERR_USAGE, "state_upload_async: the host buffer must be page-locked "
                                 "(cudaMallocHost / cudaHostRegister); use vqb_state_upload");
        }
        VQB_CUDA(cudaMemcpyAsync(d->amps, host, sizeof(double2) * count, cudaMemcpyHostToDevice,
                                 d->stream));
    });
}

VQB_API int vqb_state_download(const vqb_state *s, vqb_c128 *host, uint64_t count) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(host, "host");
        check_count(d, count, "state_download");
        VQB_CUDA(cudaMemcpyAsync(host, d->amps, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                                 d->stream));
        sync(d);
    });
}

VQB_API int vqb_state_download_range(const vqb_state *s, uint64_t offset, uint64_t count,
                                     vqb_c128 *host) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        if (count > 0) need(host, "host");
        if (offset > d->size || count > d->size - offset)
            raise(VQB_ERR_INDEX, "state_download_range: range [" + std::to_string(offset) + ", " +
                                     std::to_string(offset + count) + ") exceeds the state's " +
                                     std::to_string(d->size) + " amplitudes");
        if (count == 0) return;
        VQB_CUDA(cudaMemcpyAsync(host, d->amps + offset, sizeof(double2) * count,
                                 cudaMemcpyDeviceToHost, d->stream));
        sync(d);
    });
}

VQB_API int vqb_state_copy(vqb_state *dst, const vqb_state *src) {
    return guard([&] {
        DeviceState *a = ds(dst), *b = ds(src);
        same_device(a, b);
        DevScope on_(a->device);
        if (a->size != b->size) raise(VQB_ERR_SHAPE, "state_copy: shape mismatch");
        sync(b);
        VQB_CUDA(cudaMemcpyAsync(a->amps, b->amps, sizeof(double2) * b->size,
                                 cudaMemcpyDeviceToDevice, a->stream));
        sync(a);
    });
}

VQB_API int vqb_apply_gate(vqb_state *s, const vqb_op *op) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(op, "gate");
        const Gate g = gate_from_op(*op);
        check_fit(g.pos, g.m, d->n);
        if (d->mixed) apply_gate_both_sides(d, g);
        else apply_gate_fast(d->amps, d->pn, g, d->stream);
        sync(d);
    });
}

VQB_API int vqb_apply_channel(vqb_state *s, const vqb_op *op) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(op, "channel");
        if (!d->mixed)
            raise(VQB_ERR_TYPE, "apply_channel: a quantum channel cannot act on a pure state");
        const Channel c = channel_from_op(*op);
        check_fit(c.pos, c.m, d->n);
        apply_superop(d, c);
        sync(d);
    });
}

VQB_API int vqb_apply_matrix(vqb_state *s, const int32_t *pos, int32_t m, const vqb_c128 *mat) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(pos, "positions");
        need(mat, "matrix");
        if (m < 1 || m > VQB_MAX_POSITIONS) raise(VQB_ERR_UNSUPPORTED, "apply_matrix: 1..6 positions");
        check_fit(pos, m, d->pn);
        const size_t dd = size_t(1) << (2 * m);
        cvec M(dd);
        for (size_t i = 0; i < dd; ++i) M[i] = cplx(mat[i].re, mat[i].im);
        int bits[VQB_MAX_POSITIONS];
        for (int k = 0; k < m; ++k) bits[k] = pos[k] - 1;
        launch_dense(d->amps, d->pn, bits, m, M, d->stream);
        sync(d);
    });
}

static void apply_circuit_impl(vqb_state *s, const vqb_op *ops, int64_t count, bool fused) {
    DeviceState *d = ds(s);
        DevScope on_(d->device);
    HostTimer ht_call("apply_circuit (to launch end)");
    if (count > 0) need(ops, "ops");
    std::vector<Element> es;
    {
        HostTimer ht("build_elements");
        es = build_elements(ops, count);
    }
    for (const auto &e : es) {
        if (e.channel) {
            if (!d->mixed)
                raise(VQB_ERR_TYPE,
                      "apply_circuit: a quantum channel cannot act on a pure state; use a MixedState");
            check_fit(e.chan.pos, e.chan.m, d->n);
        } else {
            check_fit(e.gate.pos, e.gate.m, d->n);
        }
    }
    if (d->mixed) {
        run_program(d, mixed_forward_program(es, d->n), fused);
    } else {
        std::vector<Gate> prog;
        prog.reserve(es.size());
        for (const auto &e : es) prog.push_back(e.gate);
        run_program(d, prog, fused);
    }
    HostTimer ht_sync("apply_circuit sync");
    sync(d);
}

VQB_API int vqb_apply_circuit(vqb_state *s, const vqb_op *ops, int64_t count) {
    return guard([&] { apply_circuit_impl(s, ops, count, true); });
}

// apply_circuit_copy (circuit.hpp:132-146) over a batch of host-resident
// input states: job j uploads inputs[j], runs the circuit and downloads the
// result into outputs[j]. Three device states rotate through the jobs, each
// with its own stream, so job j+1's upload and job j-1's download (the two
// copy engines, both PCIe directions) overlap job j's circuit. Pinned host
// buffers are needed for the overlap (pageable ones still give correct
// results). Returns when every output has been written.
VQB_API int vqb_apply_circuit_copy_batch(int32_t num_qubits, int32_t mixed, const vqb_op *ops, int64_t count,
                                         const vqb_c128 *const *inputs, vqb_c128 *const *outputs,
                                         int64_t batch) {
    return guard([&] {
        if (batch < 0) raise(VQB_ERR_SIZE, "apply_circuit_copy_batch: negative batch");
        if (batch == 0) return;
        need(inputs, "inputs");
        need(outputs, "outputs");
        if (count > 0) need(ops, "ops");
        const std::vector<Element> es = build_elements(ops, count);
        // the rotating device states are kept for the next call of the same
        // shape (allocating and freeing 3 x 2^n amplitudes per call costs
        // more than a job); a call of another shape releases them first
        constexpr int kSlots = 3;
        BatchSlots &bs = batch_slots();
        std::lock_guard<std::mutex> lk(bs.mu);
        std::vector<DeviceState *> &cache = bs.states;
        if (!cache.empty() && (cache[0]->n != num_qubits || cache[0]->mixed != (mixed ? 1 : 0) ||
                               cache[0]->device != current_device())) {
            for (DeviceState *d : cache) state_destroy(d);
            cache.clear();
        }
        while ((int64_t)cache.size() < std::min<int64_t>(kSlots, batch))
            cache.push_back(state_create(num_qubits, mixed));
        std::vector<DeviceState *> slots(cache.begin(), cache.begin() + std::min<int64_t>(kSlots, batch));
        DeviceState *d0 = slots[0];
        for (const auto &e : es) {
            if (e.channel) {
                if (!d0->mixed)
                    raise(VQB_ERR_TYPE,
                          "apply_circuit: a quantum channel cannot act on a pure state; use a MixedState");
                check_fit(e.chan.pos, e.chan.m, d0->n);
            } else {
                check_fit(e.gate.pos, e.gate.m, d0->n);
            }
        }
        std::vector<Gate> prog;
        if (d0->mixed) prog = mixed_forward_program(es, d0->n);
        else
            for (const auto &e : es) prog.push_back(e.gate);
        const size_t bytes = sizeof(double2) * d0->size;
        for (int64_t j = 0; j < batch; ++j) {
            need(inputs[j], "inputs[j]");
            need(outputs[j], "outputs[j]");
            DeviceState *d = slots[(size_t)(j % (int64_t)slots.size())];
            VQB_CUDA(cudaMemcpyAsync(d->amps, inputs[j], bytes, cudaMemcpyHostToDevice, d->stream));
            run_program(d, prog, true); // enqueues on d->stream, no host synchronisation
            VQB_CUDA(cudaMemcpyAsync(outputs[j], d->amps, bytes, cudaMemcpyDeviceToHost, d->stream));
        }
        for (DeviceState *d : slots) sync(d);
    });
}

VQB_API int vqb_apply_circuit_unfused(vqb_state *s, const vqb_op *ops, int64_t count) {
    return guard([&] { apply_circuit_impl(s, ops, count, false); });
}

VQB_API int vqb_norm(const vqb_state *s, double *out) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(out, "out");
        if (d->mixed) raise(VQB_ERR_TYPE, "norm: pure states only (use trace)");
        *out = std::sqrt(norm_sq(d));
    });
}

VQB_API int vqb_trace(const vqb_state *s, vqb_c128 *out) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(out, "out");
        if (!d->mixed) raise(VQB_ERR_TYPE, "trace: mixed states only");
        const cplx t = trace(d);
        out->re = t.real();
        out->im = t.imag();
    });
}

VQB_API int vqb_expectation(const vqb_state *s, const vqb_pauli_term *terms, int64_t nt,
                            vqb_c128 *out) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(out, "out");
        const PauliPack p = pack_operator(terms, nt, false);
        if (p.max_qubit > d->n)
            raise(VQB_ERR_INDEX, "expectation: operator acts on qubit " + std::to_string(p.max_qubit) +
                                     " but the state has " + std::to_string(d->n) + " qubits");
        const cplx e = expectation(d, p);
        out->re = e.real();
        out->im = e.imag();
    });
}

VQB_API int vqb_apply_operator(const vqb_state *src, vqb_state *dst, const vqb_pauli_term *terms,
                               int64_t nt) {
    return guard([&] {
        DeviceState *a = ds(src), *b = ds(dst);
        same_device(a, b);
        DevScope on_(a->device);
        if (a->mixed || b->mixed) raise(VQB_ERR_TYPE, "apply_operator: pure states only");
        if (a->size != b->size) raise(VQB_ERR_SHAPE, "apply_operator: shape mismatch");
        if (a == b) raise(VQB_ERR_USAGE, "apply_operator: src and dst must differ");
        const PauliPack p = pack_operator(terms, nt, false);
        if (p.max_qubit > a->n)
            raise(VQB_ERR_INDEX, "apply_operator: operator acts on qubit " +
                                     std::to_string(p.max_qubit) + " but the state has " +
                                     std::to_string(a->n) + " qubits");
        sync(b);
        if (p.groups.empty()) {
            VQB_CUDA(cudaMemsetAsync(b->amps, 0, sizeof(double2) * b->size, a->stream));
        } else {
            apply_operator(a, b->amps, p, false);
        }
        sync(a);
    });
}

VQB_API int vqb_bilinear_form(const vqb_state *bra, const vqb_state *ket, const int32_t *pos,
                              int32_t m, const vqb_c128 *local, vqb_c128 *out) {
    return guard([&] {
        DeviceState *a = ds(bra), *b = ds(ket);
        same_device(a, b);
        DevScope on_(a->device);
        need(pos, "positions");
        need(local, "local");
        need(out, "out");
        if (a->size != b->size) raise(VQB_ERR_SHAPE, "bilinear_form: shape mismatch");
        check_fit(pos, m, b->pn);
        const size_t dd = size_t(1) << (2 * m);
        cvec L(dd);
        for (size_t i = 0; i < dd; ++i) L[i] = cplx(local[i].re, local[i].im);
        const cplx r = bilinear_form(a, b, pos, m, L);
        out->re = r.real();
        out->im = r.imag();
    });
}

VQB_API int vqb_reverse_step(vqb_state *phi, vqb_state *psi, const int32_t *pos, int32_t m,
                             const vqb_c128 *inv, const vqb_c128 *dmats, int32_t np, vqb_c128 *out) {
    return guard([&] {
        DeviceState *a = ds(phi), *b = ds(psi);
        same_device(a, b);
        DevScope on_(a->device);
        need(pos, "positions");
        need(inv, "inv");
        if (np > 0) {
            need(dmats, "dmats");
            need(out, "out");
        }
        if (a->size != b->size) raise(VQB_ERR_SHAPE, "reverse_step: shape mismatch");
        check_fit(pos, m, a->pn);
        const size_t dd = size_t(1) << (2 * m);
        cvec I(dd);
        for (size_t i = 0; i < dd; ++i) I[i] = cplx(inv[i].re, inv[i].im);
        sync(b);
        if (np == 0) {
            Gate g;
            g.m = m;
            for (int k = 0; k < m; ++k) g.pos[k] = pos[k];
            g.mat = I;
            apply_gate_fast(a->amps, a->pn, g, a->stream);
            apply_gate_fast(b->amps, b->pn, g, a->stream);
            sync(a);
            return;
        }
        std::vector<cvec> D(np, cvec(dd));
        for (int p = 0; p < np; ++p)
            for (size_t i = 0; i < dd; ++i) D[p][i] = cplx(dmats[p * dd + i].re, dmats[p * dd + i].im);
        reverse_step_async(a->amps, b->amps, a->pn, pos, m, I, D, a, a->ws.result, nullptr, 0.0);
        VQB_CUDA(cudaMemcpyAsync(a->ws.host_result, a->ws.result, sizeof(double2) * np,
                                 cudaMemcpyDeviceToHost, a->stream));
        sync(a);
        for (int p = 0; p < np; ++p) {
            out[p].re = a->ws.host_result[p].x;
            out[p].im = a->ws.host_result[p].y;
        }
    });
}

VQB_API int vqb_loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms, int64_t nt,
                          const vqb_state *s0, double *loss) {
    return guard([&] {
        need(loss, "loss");
        DevScope on_(ds(s0)->device);
        *loss = loss_pure(ops, count, terms, nt, ds(s0), true);
    });
}

VQB_API int vqb_loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                           int64_t nt, const vqb_state *dm0, double *loss) {
    return guard([&] {
        need(loss, "loss");
        DevScope on_(ds(dm0)->device);
        *loss = loss_mixed(ops, count, terms, nt, ds(dm0), true);
    });
}

VQB_API int vqb_gradient_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                              int64_t nt, const vqb_state *s0, double *loss, double *grads,
                              int64_t cap, int64_t *ng, double *res) {
    return guard([&] {
        need(loss, "loss");
        need(ng, "num_grads");
        DevScope on_(ds(s0)->device);
        const auto r = gradient_pure(ops, count, terms, nt, ds(s0), res != nullptr, true);
        if (!r.grads.empty()) need(grads, "grads");
        write_grads(r, loss, grads, cap, ng, res);
    });
}

VQB_API int vqb_gradient_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                               int64_t nt, const vqb_state *dm0, double *loss, double *grads,
                               int64_t cap, int64_t *ng, double *res) {
    return guard([&] {
        need(loss, "loss");
        need(ng, "num_grads");
        DevScope on_(ds(dm0)->device);
        const auto r = gradient_mixed(ops, count, terms, nt, ds(dm0), res != nullptr, true);
        if (!r.grads.empty()) need(grads, "grads");
        write_grads(r, loss, grads, cap, ng, res);
    });
}

// ---- batched reverse steps (autodiff.hpp:130-150 with explicit matrices) ----
VQB_API int vqb_reverse_sweep(vqb_state *phi, vqb_state *psi, const vqb_rev_step *steps,
                              int64_t count, double scale, double *grads, int64_t grads_len) {
    return guard([&] {
        DeviceState *a = ds(phi), *b = ds(psi);
        same_device(a, b);
        DevScope on_(a->device);
        if (a == b) raise(VQB_ERR_USAGE, "reverse_sweep: phi and psi must be distinct states");
        if (a->size != b->size) raise(VQB_ERR_SHAPE, "reverse_sweep: shape mismatch");
        if (count > 0) need(steps, "steps");
        std::vector<RevOp> prog;
        prog.reserve((size_t)count);
        bool any_param = false;
        // every step gets private device slots (the executor writes, not
        // adds, a step's contributions); the host adds them into grads at
        // grad_index, so steps sharing an index (tied parameters) accumulate
        int64_t nslots = 0;
        std::vector<int64_t> dst;
        for (int64_t i = 0; i < count; ++i) {
            const vqb_rev_step &st = steps[i];
            const int m = st.num_positions;
            if (m < 1 || m > 4) raise(VQB_ERR_SHAPE, "reverse_sweep: steps act on 1..4 positions");
            check_positions(st.positions, m, "reverse_sweep");
            check_fit(st.positions, m, a->pn);
            need(st.inv, "inv");
            if (st.num_dmats < 0 || st.num_dmats > VQB_MAX_PARAMS)
                raise(VQB_ERR_SHAPE, "reverse_sweep: at most 5 derivative matrices per step");
            const size_t dd = size_t(1) << (2 * m);
            RevOp r;
            r.phi_op.m = m;
            for (int k = 0; k < m; ++k) r.phi_op.pos[k] = st.positions[k];
            r.phi_op.mat.resize(dd);
            for (size_t e = 0; e < dd; ++e) r.phi_op.mat[e] = cplx(st.inv[e].re, st.inv[e].im);
            r.psi_op = r.phi_op;
            if (st.num_dmats > 0) {
                need(st.dmats, "dmats");
                need(grads, "grads");
                if (st.grad_index < 0 || st.grad_index + st.num_dmats > grads_len)
                    raise(VQB_ERR_INDEX, "reverse_sweep: gradient slot out of range");
                for (int p = 0; p < st.num_dmats; ++p) {
                    cvec d(dd);
                    for (size_t e = 0; e < dd; ++e)
                        d[e] = cplx(st.dmats[p * dd + e].re, st.dmats[p * dd + e].im);
                    r.dmats.push_back(std::move(d));
                }
                r.grad_base = nslots;
                for (int p = 0; p < st.num_dmats; ++p) dst.push_back(st.grad_index + p);
                nslots += st.num_dmats;
                r.scale = scale;
                any_param = true;
            }
            prog.push_back(std::move(r));
        }
        double *dg = nullptr;
        static thread_local DevMem slots;
        if (any_param) {
            slots.ensure(sizeof(double) * (size_t)nslots + 16);
            dg = static_cast<double *>(slots.p);
            VQB_CUDA(cudaMemsetAsync(dg, 0, sizeof(double) * (size_t)nslots, a->stream));
        }
        sync(b);
        run_reverse(a, b, prog, dg, true);
        sync(a);
        if (any_param) {
            std::vector<double> h((size_t)nslots);
            VQB_CUDA(cudaMemcpy(h.data(), dg, sizeof(double) * (size_t)nslots, cudaMemcpyDeviceToHost));
            for (int64_t k = 0; k < nslots; ++k) grads[dst[(size_t)k]] += h[(size_t)k];
        }
    });
}

// ---- measurement (circuit.hpp:303-375) ----
namespace {
void check_qubit(const DeviceState *d, int32_t qubit) {
    if (qubit < 1 || qubit > d->n)
        raise(VQB_ERR_INDEX, "measure: qubit " + std::to_string(qubit) + " does not fit a " +
                                 std::to_string(d->n) + "-qubit state");
}
double clamp_probability(double p) { return p < 0 ? 0.0 : (p > 1 ? 1.0 : p); } // :283-285
} // namespace

VQB_API int vqb_measure(vqb_state *s, int32_t qubit, double uniform, int32_t *outcome,
                        double *probability) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(outcome, "outcome");
        need(probability, "probability");
        check_qubit(d, qubit);
        const double p1 = clamp_probability(prob_one(d, qubit));
        const double p0 = clamp_probability(1.0 - p1);
        if (p0 == 0 && p1 == 0)
            raise(VQB_ERR_DEGENERATE, "measure: both outcome probabilities vanish");
        const int o = uniform < p1 ? 1 : 0;
        const double p = o == 1 ? p1 : p0;
        if (p == 0) raise(VQB_ERR_DEGENERATE, "measure: drawn outcome has zero probability");
        collapse(d, qubit, o, d->mixed ? 1.0 / p : 1.0 / std::sqrt(p));
        *outcome = o;
        *probability = p;
    });
}

VQB_API int vqb_measure_probability(const vqb_state *s, int32_t qubit, double *p1) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        need(p1, "p1");
        check_qubit(d, qubit);
        *p1 = prob_one(d, qubit);
    });
}

VQB_API int vqb_collapse(vqb_state *s, int32_t qubit, int32_t outcome, double probability) {
    return guard([&] {
        DeviceState *d = ds(s);
        DevScope on_(d->device);
        check_qubit(d, qubit);
        if (outcome != 0 && outcome != 1) raise(VQB_ERR_DOMAIN, "collapse: outcome must be 0 or 1");
        if (!(probability > 0)) raise(VQB_ERR_DEGENERATE, "collapse: outcome probability must be > 0");
        collapse(d, qubit, outcome, d->mixed ? 1.0 / probability : 1.0 / std::sqrt(probability));
    });
}

// ---- multi-device sharded state ----
namespace {
Sharded *sh(const vqb_sharded *s) {
    if (!s || !s->p) raise(VQB_ERR_USAGE, "null sharded state handle");
    return s->p;
}
} // namespace

VQB_API int vqb_sharded_create(int32_t n, int32_t ndev, const int32_t *devices, vqb_sharded **out) {
    return guard([&] {
        need(devices, "devices");
        need(out, "out");
        if (n < 1 || n > 40) raise(VQB_ERR_SIZE, "sharded state: qubit count must be in 1..40");
        std::vector<int> d(devices, devices + std::max(ndev, 0));
        Sharded *s = sharded_create(n, ndev, d.data());
        *out = new vqb_sharded{s};
    });
}

VQB_API int vqb_sharded_destroy(vqb_sharded *s) {
    return guard([&] {
        if (!s) return;
        sharded_destroy(s->p);
        delete s;
    });
}

VQB_API int vqb_sharded_set_zero(vqb_sharded *s) {
    return guard([&] { sharded_set_zero(sh(s)); });
}

VQB_API int vqb_sharded_apply_circuit(vqb_sharded *s, const vqb_op *ops, int64_t count) {
    return guard([&] {
        if (count > 0) need(ops, "ops");
        sharded_apply_circuit(sh(s), ops, count);
    });
}

VQB_API int vqb_sharded_norm(vqb_sharded *s, double *out) {
    return guard([&] {
        need(out, "out");
        *out = sharded_norm(sh(s));
    });
}

VQB_API int vqb_sharded_expectation(vqb_sharded *s, const vqb_pauli_term *terms, int64_t nt, vqb_c128 *out) {
    return guard([&] {
        need(out, "out");
        if (nt > 0) need(terms, "terms");
        const cplx e = sharded_expectation(sh(s), terms, nt);
        out->re = e.real();
        out->im = e.imag();
    });
}

VQB_API int vqb_sharded_download(vqb_sharded *s, vqb_c128 *host, uint64_t count) {
    return guard([&] {
        need(host, "host");
        sharded_download(sh(s), host, count);
    });
}

VQB_API int vqb_sharded_upload(vqb_sharded *s, const vqb_c128 *host, uint64_t count) {
    return guard([&] {
        need(host, "host");
        sharded_upload(sh(s), host, count);
    });
}

VQB_API int vqb_sharded_stats(const vqb_sharded *s, int64_t *rounds, int64_t *swapped_bits,
                              uint64_t *bytes_moved, int32_t *log2phys) {
    return guard([&] {
        const Sharded *p = sh(s);
        if (rounds) *rounds = p->rounds;
        if (swapped_bits) *swapped_bits = p->bits_swapped;
        if (bytes_moved) *bytes_moved = p->bytes_moved;
        if (log2phys)
            for (int q = 0; q < p->n; ++q) log2phys[q] = p->log2phys[q];
    });
}

VQB_API int vqb_sharded_gradient_pure(vqb_sharded *s, const vqb_op *ops, int64_t count,
                                      const vqb_pauli_term *terms, int64_t nt, double *loss, double *grads,
                                      int64_t cap, int64_t *ng) {
    return guard([&] {
        need(loss, "loss");
        need(ng, "num_grads");
        if (count > 0) need(ops, "ops");
        if (nt > 0) need(terms, "terms");
        const ShardedGradient r = sharded_gradient_pure(sh(s), ops, count, terms, nt);
        if ((int64_t)r.grads.size() > cap)
            raise(VQB_ERR_SHAPE, "gradient buffer too small: need " + std::to_string(r.grads.size()));
        if (!r.grads.empty()) need(grads, "grads");
        *loss = r.loss;
        if (!r.grads.empty()) std::memcpy(grads, r.grads.data(), sizeof(double) * r.grads.size());
        *ng = (int64_t)r.grads.size();
    });
}

VQB_API int vqb_sharded_save(vqb_sharded *s, const char *path) {
    return guard([&] {
        need(path, "path");
        sharded_save(sh(s), path);
    });
}

VQB_API int vqb_sharded_load(vqb_sharded *s, const char *path, int32_t *precision) {
    return guard([&] {
        need(path, "path");
        int prec = 0;
        sharded_load(sh(s), path, &prec);
        if (precision) *precision = prec;
    });
}

// ---- state dumps (io.hpp:40-128) ----
VQB_API int vqb_state_save(const vqb_state *s, const char *path) {
    return guard([&] {
        need(path, "path");
        DevScope on_(ds(s)->device);
        state_save(ds(s), path);
    });
}

VQB_API int vqb_state_load(const char *path, vqb_state **out, int32_t *precision) {
    return guard([&] {
        need(path, "path");
        need(out, "out");
        int prec = 0;
        *out = static_cast<vqb_state *>(state_load(path, &prec));
        if (precision) *precision = prec;
    });
}

// ---- BenchRecord reports (src/bench.cpp:329-369) ----
VQB_API int vqb_bench_report(const vqb_bench_record *recs, int64_t count, int32_t format, char *out,
                             int64_t cap, int64_t *length) {
    return guard([&] {
        if (count > 0) need(recs, "records");
        if (format != 0 && format != 1) raise(VQB_ERR_DOMAIN, "bench_report: format must be 0 (JSON) or 1 (CSV)");
        const std::string r = bench_report(recs, count, format);
        if (length) *length = (int64_t)r.size();
        if (out && cap > 0) {
            const size_t n = std::min<size_t>(r.size(), size_t(cap - 1));
            std::memcpy(out, r.data(), n);
            out[n] = 0;
        }
    });
}

// ---- fuse_gates (circuit.hpp:199-276) ----
VQB_API int vqb_fuse_gates(const vqb_op *ops, int64_t count, int64_t cap, vqb_op *out_ops,
                           int64_t matrix_cap, vqb_c128 *out_matrices, int64_t *num_out,
                           int64_t *num_entries) {
    return guard([&] {
        need(num_out, "num_out");
        need(num_entries, "num_entries");
        if (count > 0) need(ops, "ops");
        std::vector<Gate> flat;
        for (int64_t i = 0; i < count; ++i) {
            if (ops[i].elem == VQB_ELEM_CHANNEL)
                raise(VQB_ERR_UNSUPPORTED, "fuse_gates: circuit contains quantum channels");
        }
        for (int64_t i = 0; i < count; ++i) flat.push_back(gate_from_op(ops[i]));
        const std::vector<Gate> fused = fuse_gates(flat);
        int64_t entries = 0;
        for (const auto &g : fused) entries += (int64_t)g.mat.size();
        *num_out = (int64_t)fused.size();
        *num_entries = entries;
        if (cap == 0) return;
        if (cap < (int64_t)fused.size() || matrix_cap < entries)
            raise(VQB_ERR_SHAPE, "fuse_gates: output buffers too small");
        need(out_ops, "out_ops");
        need(out_matrices, "out_matrices");
        int64_t off = 0;
        for (size_t i = 0; i < fused.size(); ++i) {
            const Gate &g = fused[i];
            vqb_op o;
            std::memset(&o, 0, sizeof o);
            o.elem = VQB_ELEM_GATE;
            o.kind = VQB_GATE_GENERIC;
            o.num_positions = g.m;
            for (int k = 0; k < g.m; ++k) o.positions[k] = g.pos[k];
            o.matrix = out_matrices + off;
            for (const cplx &x : g.mat) {
                out_matrices[off].re = x.real();
                out_matrices[off].im = x.imag();
                ++off;
            }
            out_ops[i] = o;
        }
    });
}

VQB_API int vqb_plan_blocks(const vqb_op *ops, int64_t count, int32_t n, int32_t mixed,
                            int32_t tile_bits, int32_t max_support, int64_t cap,
                            int64_t *num_blocks, int64_t *num_stages, int32_t *num_positions,
                            int32_t *positions, vqb_c128 *matrices) {
    return guard([&] {
        need(num_blocks, "num_blocks");
        need(num_stages, "num_stages");
        if (count > 0) need(ops, "ops");
        const auto es = build_elements(ops, count);
        std::vector<Gate> prog;
        if (mixed) {
            prog = mixed_forward_program(es, n);
        } else {
            for (const auto &e : es) {
                if (e.channel) raise(VQB_ERR_TYPE, "plan_blocks: channel in a pure-state program");
                prog.push_back(e.gate);
            }
        }
        const int pn = mixed ? 2 * n : n;
        for (const auto &g : prog) check_fit(g.pos, g.m, pn);
        std::vector<FusedOp> fops;
        for (const auto &g : prog) fops.push_back(analyse_gate(g));
        const auto stages = plan_stages(fops, pn, tile_bits);
        int64_t nb = 0;
        std::deque<FusedOp> store;
        for (const auto &sg : stages) {
            std::vector<const FusedOp *> blocks;
            if (sg.fused && max_support > 0) {
                blocks = fuse_blocks_ref(fops, sg.ops, max_support, store);
            } else {
                for (int i : sg.ops) blocks.push_back(&fops[i]);
            }
            for (const FusedOp *bp : blocks) {
                const FusedOp &b = *bp;
                if (nb < cap) {
                    const Gate &g = b.gate;
                    if (g.m > 4) raise(VQB_ERR_UNSUPPORTED, "plan_blocks: block wider than 4 positions");
                    num_positions[nb] = g.m;
                    for (int k = 0; k < g.m; ++k) positions[6 * nb + k] = g.pos[k];
                    for (size_t i = 0; i < g.mat.size(); ++i) {
                        matrices[256 * nb + i].re = g.mat[i].real();
                        matrices[256 * nb + i].im = g.mat[i].imag();
                    }
                }
                ++nb;
            }
        }
        *num_blocks = nb;
        *num_stages = (int64_t)stages.size();
    });
}

static void to_c128(const cvec &v, vqb_c128 *out) {
    for (size_t i = 0; i < v.size(); ++i) {
        out[i].re = v[i].real();
        out[i].im = v[i].imag();
    }
}

VQB_API int vqb_gate_matrix(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { to_c128(gate_from_op(*op).mat, out); });
}

VQB_API int vqb_gate_derivative(const vqb_op *op, int32_t p, vqb_c128 *out) {
    return guard([&] { to_c128(gate_derivative(gate_from_op(*op), p), out); });
}

VQB_API int vqb_gate_inverse(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { to_c128(gate_inverse(gate_from_op(*op)).mat, out); });
}

VQB_API int vqb_channel_inverse(const vqb_op *op, vqb_c128 *out, double *condition, int32_t *singular) {
    return guard([&] {
        need(op, "channel");
        const Channel c = channel_from_op(*op);
        const Inverse r = channel_inverse(c, channel_superop(c));
        if (condition) *condition = r.condition;
        if (singular) *singular = r.singular ? 1 : 0;
        if (!r.singular && out) to_c128(r.inv, out);
    });
}

VQB_API int vqb_channel_superop(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { to_c128(channel_superop(channel_from_op(*op)), out); });
}

} // extern "C"
