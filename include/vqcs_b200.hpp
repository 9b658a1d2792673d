// vqcs_b200.hpp — the reference-side binding of libvqcs_b200 (C++20, header-only).
//
// A maintainer of the reference library `vqcs` adds this header next to
// include/vqcs/*.hpp and links libvqcs_b200.so. It lowers the reference's own
// types (vqcs::Circuit<double>, vqcs::GateOp<double>, vqcs::ChannelOp<double>,
// vqcs::PauliOperator, vqcs::PureState<double>, vqcs::MixedState<double>) to the
// plain-C descriptors of vqcs_b200.h and exposes functions with the same names,
// arguments and exceptions as the reference calls they replace:
//
//   vqcs::apply_circuit   (circuit.hpp:110-129)    -> vqb::apply_circuit
//   vqcs::expectation     (observables.hpp:176-213)-> vqb::expectation
//   vqcs::apply_operator  (observables.hpp:216-237)-> vqb::apply_operator
//   vqcs::loss_pure / gradient_pure   (autodiff.hpp:80-156)  -> vqb::...
//   vqcs::loss_mixed / gradient_mixed (autodiff.hpp:160-329) -> vqb::...
//   vqcs::measure         (circuit.hpp:303-385)    -> vqb::measure
//   vqcs::fuse_gates      (circuit.hpp:199-276)    -> vqb::fuse_gates
//   vqcs::save_state / load_state (io.hpp:56-128)  -> vqb::save_state / load_state
//
// States stay host objects (as in the reference); each call uploads the state,
// runs on the B200 and downloads the result. vqb::DeviceState keeps a state
// resident on the device across calls for pipelines that want to avoid the
// PCIe round trip. Errors come back as the reference's vqcs::*Error classes.
//
// The reference headers are NOT part of this repository; this header compiles
// against them where they live.
#pragma once

#include <complex>
#include <memory>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "vqcs/autodiff.hpp"
#include "vqcs/circuit.hpp"
#include "vqcs/errors.hpp"
#include "vqcs/io.hpp"
#include "vqcs/observables.hpp"
#include "vqcs/state.hpp"
#include "vqcs_b200.h"

namespace vqb {

// ---- errors: vqb_status -> the reference exception of the same meaning ----
[[noreturn]] inline void throw_status(int rc) {
    const std::string m = std::string("libvqcs_b200: ") + vqb_last_error();
    switch (rc) {
    case VQB_ERR_SIZE: throw vqcs::SizeError(m);
    case VQB_ERR_SHAPE: throw vqcs::ShapeError(m);
    case VQB_ERR_VALIDITY: throw vqcs::ValidityError(m);
    case VQB_ERR_DOMAIN: throw vqcs::DomainError(m);
    case VQB_ERR_INDEX: throw vqcs::IndexError(m);
    case VQB_ERR_TYPE: throw vqcs::TypeError(m);
    case VQB_ERR_UNSUPPORTED: throw vqcs::UnsupportedError(m);
    case VQB_ERR_DEGENERATE: throw vqcs::DegenerateStateError(m);
    case VQB_ERR_NONINVERTIBLE: throw vqcs::NonInvertibleChannelError(m);
    case VQB_ERR_IO: throw vqcs::IoError(m);
    case VQB_ERR_USAGE: throw vqcs::UsageError(m);
    default: throw vqcs::Error(m);
    }
}

inline void check(int rc) {
    if (rc != VQB_OK) throw_status(rc);
}

// ---- descriptor lowering ----
struct LoweredCircuit {
    std::vector<vqb_op> ops;
    std::vector<std::vector<vqb_c128>> store; // keeps matrices / Kraus alive

    static vqb_c128 c(std::complex<double> z) { return {z.real(), z.imag()}; }

    void add(const vqcs::GateOp<double> &g) {
        vqb_op o{};
        o.elem = VQB_ELEM_GATE;
        o.kind = static_cast<int32_t>(g.kind);
        o.num_positions = static_cast<int32_t>(g.positions.size());
        for (size_t i = 0; i < g.positions.size() && i < VQB_MAX_POSITIONS; ++i)
            o.positions[i] = g.positions[i];
        o.num_params = static_cast<int32_t>(g.params.size());
        for (size_t i = 0; i < g.params.size() && i < VQB_MAX_PARAMS; ++i) {
            o.params[i] = g.params[i];
            o.is_param[i] = g.is_param[i] ? 1 : 0;
        }
        auto &m = store.emplace_back();
        for (const auto &z : g.matrix) m.push_back(c(z));
        o.matrix = nullptr; // pointers fixed up in finish()
        ops.push_back(o);
    }

    void add(const vqcs::ChannelOp<double> &ch) {
        vqb_op o{};
        o.elem = VQB_ELEM_CHANNEL;
        o.kind = static_cast<int32_t>(ch.kind);
        o.num_positions = static_cast<int32_t>(ch.positions.size());
        for (size_t i = 0; i < ch.positions.size() && i < VQB_MAX_POSITIONS; ++i)
            o.positions[i] = ch.positions[i];
        auto &k = store.emplace_back();
        for (const auto &mat : ch.kraus)
            for (const auto &z : mat) k.push_back(c(z));
        o.num_kraus = static_cast<int32_t>(ch.kraus.size());
        ops.push_back(o);
    }

    void finish() {
        for (size_t i = 0; i < ops.size(); ++i) {
            if (ops[i].elem == VQB_ELEM_GATE) ops[i].matrix = store[i].data();
            else ops[i].kraus = store[i].data();
        }
    }
};

inline LoweredCircuit lower(const vqcs::Circuit<double> &c) {
    LoweredCircuit L;
    c.for_each_element([&](const vqcs::GateOp<double> &g) { L.add(g); },
                       [&](const vqcs::ChannelOp<double> &ch) { L.add(ch); });
    L.finish();
    return L;
}

struct LoweredOperator {
    std::vector<vqb_pauli_term> terms;
    std::vector<std::vector<int32_t>> qubits;
    std::vector<std::string> labels;
};

inline LoweredOperator lower(const vqcs::PauliOperator &op) {
    LoweredOperator L;
    L.qubits.reserve(op.size());
    L.labels.reserve(op.size());
    for (const auto &t : op.terms()) {
        auto &q = L.qubits.emplace_back();
        auto &l = L.labels.emplace_back();
        for (const auto &[qb, lab] : t.factors) {
            q.push_back(qb);
            l.push_back(static_cast<char>(lab));
        }
        vqb_pauli_term pt{};
        pt.coeff = {t.coeff.real(), t.coeff.imag()};
        pt.num_factors = static_cast<int32_t>(q.size());
        L.terms.push_back(pt);
    }
    for (size_t i = 0; i < L.terms.size(); ++i) {
        L.terms[i].qubits = L.qubits[i].data();
        L.terms[i].labels = L.labels[i].c_str();
    }
    return L;
}

// ---- a device-resident state (RAII over vqb_state) ----
class DeviceState {
  public:
    DeviceState(int n, bool mixed) { check(vqb_state_create(n, mixed ? 1 : 0, &s_)); }
    explicit DeviceState(const vqcs::PureState<double> &h) : DeviceState(h.num_qubits(), false) {
        upload(h.amplitudes());
    }
    explicit DeviceState(const vqcs::MixedState<double> &h) : DeviceState(h.num_qubits(), true) {
        upload(h.entries());
    }
    DeviceState(const DeviceState &) = delete;
    DeviceState &operator=(const DeviceState &) = delete;
    ~DeviceState() { vqb_state_destroy(s_); }

    void upload(std::span<const std::complex<double>> a) {
        check(vqb_state_upload(s_, reinterpret_cast<const vqb_c128 *>(a.data()), a.size()));
    }
    // `a` must be page-locked and unchanged until the next call on this state
    // that returns a result (vqb_state_upload_async)
    void upload_async(std::span<const std::complex<double>> a) {
        check(vqb_state_upload_async(s_, reinterpret_cast<const vqb_c128 *>(a.data()), a.size()));
    }
    void download(std::span<std::complex<double>> a) const {
        check(vqb_state_download(s_, reinterpret_cast<vqb_c128 *>(a.data()), a.size()));
    }
    vqb_state *get() const { return s_; }
    // adopt a handle created by the library (vqb_state_load)
    static std::unique_ptr<DeviceState> adopt(vqb_state *s) {
        return std::unique_ptr<DeviceState>(new DeviceState(s));
    }

  private:
    explicit DeviceState(vqb_state *s) : s_(s) {}
    vqb_state *s_ = nullptr;
};

// ---- a pure state sharded over the devices of this process (vqb_sharded_*) ----
// The top log2(devices.size()) qubits are global; every call below has the
// reference's semantics for a PureState<double> of n qubits (the unsharded
// result is the oracle), see vqcs_b200.h.
class ShardedState {
  public:
    ShardedState(int n, const std::vector<int> &devices) : n_(n) {
        std::vector<int32_t> d(devices.begin(), devices.end());
        check(vqb_sharded_create(n, static_cast<int32_t>(d.size()), d.data(), &s_));
    }
    ShardedState(const ShardedState &) = delete;
    ShardedState &operator=(const ShardedState &) = delete;
    ~ShardedState() { vqb_sharded_destroy(s_); }

    int num_qubits() const { return n_; }
    void set_zero() { check(vqb_sharded_set_zero(s_)); }
    void upload(std::span<const std::complex<double>> a) {
        check(vqb_sharded_upload(s_, reinterpret_cast<const vqb_c128 *>(a.data()), a.size()));
    }
    void download(std::span<std::complex<double>> a) const {
        check(vqb_sharded_download(s_, reinterpret_cast<vqb_c128 *>(a.data()), a.size()));
    }
    double norm() const {
        double v = 0;
        check(vqb_sharded_norm(s_, &v));
        return v;
    }
    void save(const std::string &path) { check(vqb_sharded_save(s_, path.c_str())); }
    vqb_sharded *get() const { return s_; }

  private:
    int n_;
    vqb_sharded *s_ = nullptr;
};

inline void apply_circuit(const vqcs::Circuit<double> &c, ShardedState &s);
inline std::complex<double> expectation(const vqcs::PauliOperator &op, ShardedState &s);

// ---- the replaced reference calls (same names and semantics) ----
inline void apply_circuit(const vqcs::Circuit<double> &c, DeviceState &s) {
    const auto L = lower(c);
    check(vqb_apply_circuit(s.get(), L.ops.data(), static_cast<int64_t>(L.ops.size())));
}

inline void apply_circuit(const vqcs::Circuit<double> &c, vqcs::PureState<double> &state) {
    DeviceState d(state);
    apply_circuit(c, d);
    d.download(state.amplitudes());
}

inline void apply_circuit(const vqcs::Circuit<double> &c, vqcs::MixedState<double> &dm) {
    DeviceState d(dm);
    apply_circuit(c, d);
    d.download(dm.entries());
}

// apply_circuit_copy (circuit.hpp:132-146) over a batch of host states: one
// call, uploads / circuits / downloads of consecutive states overlapped
// (vqb_apply_circuit_copy_batch). Host buffers of the reference's states are
// pageable; register them (cudaHostRegister) for full copy overlap.
inline std::vector<vqcs::PureState<double>> apply_circuit_copy(const vqcs::Circuit<double> &c,
                                                              const std::vector<vqcs::PureState<double>> &in) {
    std::vector<vqcs::PureState<double>> out(in.begin(), in.end());
    if (in.empty()) return out;
    const auto L = lower(c);
    std::vector<const vqb_c128 *> src;
    std::vector<vqb_c128 *> dst;
    for (size_t j = 0; j < in.size(); ++j) {
        if (in[j].num_qubits() != in[0].num_qubits())
            throw vqcs::ShapeError("apply_circuit_copy: states of different sizes in one batch");
        src.push_back(reinterpret_cast<const vqb_c128 *>(in[j].amplitudes().data()));
        dst.push_back(reinterpret_cast<vqb_c128 *>(out[j].amplitudes().data()));
    }
    check(vqb_apply_circuit_copy_batch(in[0].num_qubits(), 0, L.ops.data(), static_cast<int64_t>(L.ops.size()),
                                       src.data(), dst.data(), static_cast<int64_t>(in.size())));
    return out;
}

inline std::complex<double> expectation(const vqcs::PauliOperator &op, const DeviceState &s) {
    const auto L = lower(op);
    vqb_c128 out{};
    check(vqb_expectation(s.get(), L.terms.data(), static_cast<int64_t>(L.terms.size()), &out));
    return {out.re, out.im};
}

inline std::complex<double> expectation(const vqcs::PauliOperator &op,
                                        const vqcs::PureState<double> &state) {
    return expectation(op, DeviceState(state));
}

inline std::complex<double> expectation(const vqcs::PauliOperator &op,
                                        const vqcs::MixedState<double> &dm) {
    return expectation(op, DeviceState(dm));
}

inline vqcs::PureState<double> apply_operator(const vqcs::PauliOperator &op,
                                              const vqcs::PureState<double> &state) {
    const auto L = lower(op);
    DeviceState src(state), dst(state.num_qubits(), false);
    check(vqb_apply_operator(src.get(), dst.get(), L.terms.data(),
                             static_cast<int64_t>(L.terms.size())));
    vqcs::PureState<double> out(vqcs::unchecked, vqcs::cvector<double>(state.size()));
    dst.download(out.amplitudes());
    return out;
}

inline double loss_pure(const vqcs::PauliOperator &op, const vqcs::Circuit<double> &c,
                        const vqcs::PureState<double> &s0) {
    const auto L = lower(c);
    const auto O = lower(op);
    DeviceState d(s0);
    double loss = 0;
    check(vqb_loss_pure(L.ops.data(), static_cast<int64_t>(L.ops.size()), O.terms.data(),
                        static_cast<int64_t>(O.terms.size()), d.get(), &loss));
    return loss;
}

inline double loss_mixed(const vqcs::PauliOperator &op, const vqcs::Circuit<double> &c,
                         const vqcs::MixedState<double> &dm0) {
    const auto L = lower(c);
    const auto O = lower(op);
    DeviceState d(dm0);
    double loss = 0;
    check(vqb_loss_mixed(L.ops.data(), static_cast<int64_t>(L.ops.size()), O.terms.data(),
                         static_cast<int64_t>(O.terms.size()), d.get(), &loss));
    return loss;
}

namespace detail {
template <typename Fn, typename State>
vqcs::GradientResult gradient(Fn fn, const vqcs::PauliOperator &op, const vqcs::Circuit<double> &c,
                              const State &s0, vqcs::GradientDiagnostics *diag) {
    const auto L = lower(c);
    const auto O = lower(op);
    DeviceState d(s0);
    const auto params = vqcs::active_parameters(c);
    vqcs::GradientResult r;
    r.grads.assign(params.size(), 0.0);
    int64_t ng = 0;
    double residual = 0;
    check(fn(L.ops.data(), static_cast<int64_t>(L.ops.size()), O.terms.data(),
             static_cast<int64_t>(O.terms.size()), d.get(), &r.loss, r.grads.data(),
             static_cast<int64_t>(r.grads.size()), &ng, diag ? &residual : nullptr));
    r.grads.resize(static_cast<size_t>(ng));
    if (diag) diag->reverse_residual = residual;
    return r;
}
} // namespace detail

inline vqcs::GradientResult gradient_pure(const vqcs::PauliOperator &op,
                                          const vqcs::Circuit<double> &c,
                                          const vqcs::PureState<double> &s0,
                                          vqcs::GradientDiagnostics *diag = nullptr) {
    return detail::gradient(vqb_gradient_pure, op, c, s0, diag);
}

// gradient_pure on a sharded s0 (left as the reverse-swept Phi = s0 up to
// rounding; see vqb_sharded_gradient_pure)
inline vqcs::GradientResult gradient_pure(const vqcs::PauliOperator &op, const vqcs::Circuit<double> &c,
                                          ShardedState &s0) {
    const auto L = lower(c);
    const auto O = lower(op);
    vqcs::GradientResult r;
    r.grads.assign(vqcs::active_parameters(c).size(), 0.0);
    int64_t ng = 0;
    check(vqb_sharded_gradient_pure(s0.get(), L.ops.data(), static_cast<int64_t>(L.ops.size()),
                                    O.terms.data(), static_cast<int64_t>(O.terms.size()), &r.loss,
                                    r.grads.data(), static_cast<int64_t>(r.grads.size()), &ng));
    r.grads.resize(static_cast<size_t>(ng));
    return r;
}

inline vqcs::GradientResult gradient_mixed(const vqcs::PauliOperator &op,
                                           const vqcs::Circuit<double> &c,
                                           const vqcs::MixedState<double> &dm0,
                                           vqcs::GradientDiagnostics *diag = nullptr) {
    return detail::gradient(vqb_gradient_mixed, op, c, dm0, diag);
}

// ---- measure (circuit.hpp:303-385): the uniform is drawn from the caller's
// stream exactly as the reference draws it (detail::uniform_unit), so the
// same std::mt19937_64 yields the same outcomes ----
inline vqcs::MeasurementOutcome measure(DeviceState &s, int qubit, std::mt19937_64 &rng) {
    const double u = vqcs::detail::uniform_unit(rng);
    int32_t outcome = 0;
    double p = 0;
    check(vqb_measure(s.get(), qubit, u, &outcome, &p));
    return {outcome, p};
}

inline vqcs::MeasurementOutcome measure(vqcs::PureState<double> &state, int qubit,
                                        std::mt19937_64 &rng) {
    DeviceState d(state);
    const auto r = measure(d, qubit, rng);
    d.download(state.amplitudes());
    return r;
}

inline vqcs::MeasurementOutcome measure(vqcs::MixedState<double> &dm, int qubit,
                                        std::mt19937_64 &rng) {
    DeviceState d(dm);
    const auto r = measure(d, qubit, rng);
    d.download(dm.entries());
    return r;
}

// ---- fuse_gates (circuit.hpp:199-276) ----
inline vqcs::Circuit<double> fuse_gates(const vqcs::Circuit<double> &c) {
    const auto L = lower(c);
    int64_t nout = 0, nent = 0;
    check(vqb_fuse_gates(L.ops.data(), static_cast<int64_t>(L.ops.size()), 0, nullptr, 0, nullptr,
                         &nout, &nent));
    std::vector<vqb_op> ops(static_cast<size_t>(std::max<int64_t>(nout, 1)));
    std::vector<std::complex<double>> mats(static_cast<size_t>(std::max<int64_t>(nent, 1)));
    check(vqb_fuse_gates(L.ops.data(), static_cast<int64_t>(L.ops.size()),
                         static_cast<int64_t>(ops.size()), ops.data(),
                         static_cast<int64_t>(mats.size()),
                         reinterpret_cast<vqb_c128 *>(mats.data()), &nout, &nent));
    vqcs::Circuit<double> out;
    for (int64_t i = 0; i < nout; ++i) {
        const vqb_op &o = ops[static_cast<size_t>(i)];
        const size_t d = size_t(1) << o.num_positions;
        const auto *m = reinterpret_cast<const std::complex<double> *>(o.matrix);
        out.push_back(vqcs::make_gate<double>(
            std::vector<int>(o.positions, o.positions + o.num_positions),
            vqcs::cvector<double>(m, m + d * d)));
    }
    return out;
}

// ---- state dumps (io.hpp:56-128), device-resident states ----
inline void save_state(const DeviceState &s, const std::string &path) {
    check(vqb_state_save(s.get(), path.c_str()));
}

inline std::unique_ptr<DeviceState> load_state(const std::string &path,
                                               vqcs::Precision *precision = nullptr) {
    vqb_state *h = nullptr;
    int32_t prec = 0;
    check(vqb_state_load(path.c_str(), &h, &prec));
    if (precision) *precision = static_cast<vqcs::Precision>(prec);
    return DeviceState::adopt(h);
}

inline void apply_circuit(const vqcs::Circuit<double> &c, ShardedState &s) {
    const auto L = lower(c);
    check(vqb_sharded_apply_circuit(s.get(), L.ops.data(), static_cast<int64_t>(L.ops.size())));
}

inline std::complex<double> expectation(const vqcs::PauliOperator &op, ShardedState &s) {
    const auto O = lower(op);
    vqb_c128 v{};
    check(vqb_sharded_expectation(s.get(), O.terms.data(), static_cast<int64_t>(O.terms.size()), &v));
    return {v.re, v.im};
}

} // namespace vqb
