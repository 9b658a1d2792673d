// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product). Exposes the UNMODIFIED reference library `vqcs`
// (header-only, /root/reference/proj/include/vqcs) behind the same C-ABI as
// include/vqcs_b200.h, with the prefix `vqcsref_` instead of `vqb_`.
//
// Built by oracle/Makefile directly from the reference headers where they lie
// (no sources are copied); output goes to oracle/_ref/libvqcs_ref.so. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs load it, as the checker and as the CPU baseline.
//
// Every function forwards to the reference call it names; state handles own
// vqcs::PureState<double> / vqcs::MixedState<double> host buffers.

#include <cstring>
#include <memory>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "vqcs/autodiff.hpp"
#include "vqcs/circuit.hpp"
#include "vqcs/gates.hpp"
#include "vqcs/io.hpp"
#include "vqcs/kernels.hpp"
#include "vqcs/observables.hpp"
#include "vqcs/state.hpp"

#include "../include/vqcs_b200.h"

using namespace vqcs;
using C = std::complex<double>;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_last_error;
int g_threads = 0; // 0 = reference default (VQCS_NUM_THREADS / hw concurrency)

ThreadConfig cfg() {
    ThreadConfig c;
    if (g_threads > 0) {
        c.num_threads = g_threads;
    }
    return c;
}

struct RefState {
    std::optional<PureState<double>> pure;
    std::optional<MixedState<double>> mixed;
    std::span<C> amps() {
        return pure ? pure->amplitudes() : mixed->entries();
    }
    std::span<const C> amps() const {
        return pure ? std::span<const C>(pure->amplitudes())
                    : std::span<const C>(mixed->entries());
    }
    int pseudo_qubits() const {
        return pure ? pure->num_qubits() : 2 * mixed->num_qubits();
    }
};

template <typename F> int guard(F &&f) {
    try {
        f();
        return VQB_OK;
    } catch (const SizeError &e) {
        g_last_error = e.what();
        return VQB_ERR_SIZE;
    } catch (const ShapeError &e) {
        g_last_error = e.what();
        return VQB_ERR_SHAPE;
    } catch (const ValidityError &e) {
        g_last_error = e.what();
        return VQB_ERR_VALIDITY;
    } catch (const DomainError &e) {
        g_last_error = e.what();
        return VQB_ERR_DOMAIN;
    } catch (const IndexError &e) {
        g_last_error = e.what();
        return VQB_ERR_INDEX;
    } catch (const TypeError &e) {
        g_last_error = e.what();
        return VQB_ERR_TYPE;
    } catch (const UnsupportedError &e) {
        g_last_error = e.what();
        return VQB_ERR_UNSUPPORTED;
    } catch (const DegenerateStateError &e) {
        g_last_error = e.what();
        return VQB_ERR_DEGENERATE;
    } catch (const NonInvertibleChannelError &e) {
        g_last_error = e.what();
        return VQB_ERR_NONINVERTIBLE;
    } catch (const IoError &e) {
        g_last_error = e.what();
        return VQB_ERR_IO;
    } catch (const UsageError &e) {
        g_last_error = e.what();
        return VQB_ERR_USAGE;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return VQB_ERR_INTERNAL;
    }
}

cvector<double> to_cvec(const vqb_c128 *p, std::size_t count) {
    cvector<double> v(count);
    for (std::size_t i = 0; i < count; ++i) {
        v[i] = C(p[i].re, p[i].im);
    }
    return v;
}

void from_cvec(const cvector<double> &v, vqb_c128 *out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[i].re = v[i].real();
        out[i].im = v[i].imag();
    }
}

std::vector<int> positions_of(const vqb_op &op) {
    return std::vector<int>(op.positions, op.positions + op.num_positions);
}

// A GateOp exactly as a reference caller would hold it.
GateOp<double> to_gate(const vqb_op &op) {
    const auto kind = static_cast<GateKind>(op.kind);
    auto pos = positions_of(op);
    const std::size_t d = std::size_t(1) << pos.size();
    if (op.matrix == nullptr) {
        if (op.num_params == 0) {
            return standard_gate<double>(kind, std::move(pos));
        }
        std::vector<double> params(op.params, op.params + op.num_params);
        std::vector<bool> flags;
        for (int i = 0; i < op.num_params; ++i) {
            flags.push_back(op.is_param[i] != 0);
        }
        return parametric_gate<double>(kind, std::move(pos), std::move(params),
                                       std::move(flags));
    }
    if (kind == GateKind::Generic) {
        return make_gate<double>(std::move(pos), to_cvec(op.matrix, d * d));
    }
    GateOp<double> g;
    g.positions = std::move(pos);
    g.matrix = to_cvec(op.matrix, d * d);
    g.kind = kind;
    g.params.assign(op.params, op.params + op.num_params);
    for (int i = 0; i < op.num_params; ++i) {
        g.is_param.push_back(op.is_param[i] != 0);
    }
    return g;
}

ChannelOp<double> to_channel(const vqb_op &op) {
    const auto kind = static_cast<ChannelKind>(op.kind);
    if (op.kraus == nullptr) {
        return standard_channel<double>(kind, op.positions[0], op.params[0]);
    }
    const std::size_t d = std::size_t(1) << op.num_positions;
    std::vector<cvector<double>> kraus;
    for (int s = 0; s < op.num_kraus; ++s) {
        kraus.push_back(to_cvec(op.kraus + s * d * d, d * d));
    }
    ChannelOp<double> c = make_channel<double>(positions_of(op), std::move(kraus));
    c.kind = kind;
    return c;
}

Circuit<double> to_circuit(const vqb_op *ops, int64_t count) {
    Circuit<double> c;
    for (int64_t i = 0; i < count; ++i) {
        if (ops[i].elem == VQB_ELEM_CHANNEL) {
            c.push_back(to_channel(ops[i]));
        } else {
            c.push_back(to_gate(ops[i]));
        }
    }
    return c;
}

PauliOperator to_operator(const vqb_pauli_term *terms, int64_t n) {
    PauliOperator op;
    for (int64_t t = 0; t < n; ++t) {
        std::vector<std::pair<int, PauliLabel>> f;
        for (int k = 0; k < terms[t].num_factors; ++k) {
            f.push_back({terms[t].qubits[k], parse_pauli_label(terms[t].labels[k])});
        }
        op.add_term(PauliTerm(std::move(f), C(terms[t].coeff.re, terms[t].coeff.im)));
    }
    return op;
}

} // namespace

REF_API const char *vqcsref_last_error(void) { return g_last_error.c_str(); }
REF_API void vqcsref_set_num_threads(int t) { g_threads = t; }
REF_API int vqcsref_get_num_threads(void) { return cfg().num_threads; }

// ---- allocation bookkeeping: state_alloc_stats (state.hpp:154-161) ----
REF_API int vqcsref_alloc_stats(int64_t *live, int64_t *peak, uint64_t *live_bytes,
                                uint64_t *peak_bytes) {
    const auto a = vqcs::state_alloc_stats();
    if (live) *live = a.live;
    if (peak) *peak = a.peak;
    if (live_bytes) *live_bytes = 0; // the reference counts buffers, not bytes
    if (peak_bytes) *peak_bytes = 0;
    return VQB_OK;
}
REF_API int vqcsref_reset_alloc_peak(void) {
    vqcs::reset_state_alloc_peak();
    return VQB_OK;
}
REF_API int vqcsref_release_caches(void) { return VQB_OK; } // the reference caches nothing

// ---- state ----
REF_API int vqcsref_state_create(int32_t n, int32_t mixed, RefState **out) {
    return guard([&] {
        auto s = std::make_unique<RefState>();
        if (mixed) {
            s->mixed.emplace(n); // MixedState(n) state.hpp:264-268
        } else {
            s->pure.emplace(n); // PureState(n) state.hpp:182-185
        }
        *out = s.release();
    });
}

// The reference harness's per-repetition reset (src/bench.cpp:138-141):
// std::fill with zero, then amplitude 0 = 1 (pure) / entry (0,0) = 1 (mixed).
REF_API int vqcsref_state_set_zero(RefState *s) {
    return guard([&] {
        auto a = s->amps();
        std::fill(a.begin(), a.end(), C(0));
        a[0] = 1;
    });
}

REF_API int vqcsref_state_destroy(RefState *s) {
    delete s;
    return VQB_OK;
}

REF_API int vqcsref_state_info(const RefState *s, int32_t *n, int32_t *mixed,
                               uint64_t *count) {
    if (n) *n = s->pure ? s->pure->num_qubits() : s->mixed->num_qubits();
    if (mixed) *mixed = s->mixed ? 1 : 0;
    if (count) *count = s->amps().size();
    return VQB_OK;
}

REF_API int vqcsref_state_upload(RefState *s, const vqb_c128 *host, uint64_t count) {
    return guard([&] {
        auto a = s->amps();
        if (count != a.size()) {
            throw ShapeError("state_upload: count mismatch");
        }
        std::memcpy(a.data(), host, count * sizeof(C));
    });
}

REF_API int vqcsref_state_download(const RefState *s, vqb_c128 *host, uint64_t count) {
    return guard([&] {
        auto a = s->amps();
        if (count != a.size()) {
            throw ShapeError("state_download: count mismatch");
        }
        std::memcpy(host, a.data(), count * sizeof(C));
    });
}

REF_API int vqcsref_state_download_range(const RefState *s, uint64_t offset, uint64_t count,
                                         vqb_c128 *host) {
    return guard([&] {
        auto a = s->amps();
        if (offset > a.size() || count > a.size() - offset) {
            throw IndexError("state_download_range: range exceeds the state");
        }
        std::memcpy(host, a.data() + offset, count * sizeof(C));
    });
}

REF_API int vqcsref_state_copy(RefState *dst, const RefState *src) {
    return guard([&] {
        if (dst->amps().size() != src->amps().size()) {
            throw ShapeError("state_copy: shape mismatch");
        }
        std::copy(src->amps().begin(), src->amps().end(), dst->amps().begin());
    });
}

// ---- application ----
REF_API int vqcsref_apply_gate(RefState *s, const vqb_op *op) {
    return guard([&] {
        const auto g = to_gate(*op);
        if (s->pure) {
            apply_gate_fast(s->pure->amplitudes(), s->pure->num_qubits(), g, cfg());
        } else {
            apply_gate_mixed(*s->mixed, g, cfg());
        }
    });
}

REF_API int vqcsref_apply_gate_naive(RefState *s, const vqb_op *op) {
    return guard([&] {
        const auto g = to_gate(*op);
        apply_gate_naive(s->amps(), s->pseudo_qubits(), g);
    });
}

REF_API int vqcsref_apply_channel(RefState *s, const vqb_op *op) {
    return guard([&] {
        if (!s->mixed) {
            throw TypeError("apply_channel: a quantum channel cannot act on a pure state");
        }
        apply_channel(*s->mixed, to_channel(*op), cfg());
    });
}

REF_API int vqcsref_apply_matrix(RefState *s, const int32_t *positions, int32_t m,
                                 const vqb_c128 *matrix) {
    return guard([&] {
        const std::vector<int> pos(positions, positions + m);
        const std::size_t d = std::size_t(1) << m;
        apply_matrix(s->amps(), s->pseudo_qubits(), std::span<const int>(pos),
                     to_cvec(matrix, d * d), cfg());
    });
}

REF_API int vqcsref_apply_circuit(RefState *s, const vqb_op *ops, int64_t count) {
    return guard([&] {
        const auto c = to_circuit(ops, count);
        if (s->pure) {
            apply_circuit(c, *s->pure, cfg());
        } else {
            apply_circuit(c, *s->mixed, cfg());
        }
    });
}

// ---- reductions ----
REF_API int vqcsref_norm(const RefState *s, double *out) {
    return guard([&] {
        if (!s->pure) {
            throw TypeError("norm: pure states only");
        }
        *out = s->pure->norm();
    });
}

REF_API int vqcsref_trace(const RefState *s, vqb_c128 *out) {
    return guard([&] {
        if (!s->mixed) {
            throw TypeError("trace: mixed states only");
        }
        const C t = s->mixed->trace();
        out->re = t.real();
        out->im = t.imag();
    });
}

REF_API int vqcsref_expectation(const RefState *s, const vqb_pauli_term *terms,
                                int64_t nterms, vqb_c128 *out) {
    return guard([&] {
        const auto op = to_operator(terms, nterms);
        const C e = s->pure ? expectation(op, *s->pure, cfg())
                            : expectation(op, *s->mixed, cfg());
        out->re = e.real();
        out->im = e.imag();
    });
}

REF_API int vqcsref_apply_operator(const RefState *src, RefState *dst,
                                   const vqb_pauli_term *terms, int64_t nterms) {
    return guard([&] {
        if (!src->pure || !dst->pure) {
            throw TypeError("apply_operator: pure states only");
        }
        const auto op = to_operator(terms, nterms);
        *dst->pure = apply_operator(op, *src->pure, cfg());
    });
}

REF_API int vqcsref_bilinear_form(const RefState *bra, const RefState *ket,
                                  const int32_t *positions, int32_t m,
                                  const vqb_c128 *local, vqb_c128 *out) {
    return guard([&] {
        const std::vector<int> pos(positions, positions + m);
        const std::size_t d = std::size_t(1) << m;
        const C r = bilinear_gate_form<double>(bra->amps(), ket->amps(),
                                               ket->pseudo_qubits(), pos,
                                               to_cvec(local, d * d), cfg());
        out->re = r.real();
        out->im = r.imag();
    });
}

REF_API int vqcsref_reverse_step(RefState *phi, RefState *psi, const int32_t *positions,
                                 int32_t m, const vqb_c128 *inv, const vqb_c128 *dmats,
                                 int32_t np, vqb_c128 *out) {
    return guard([&] {
        const std::vector<int> pos(positions, positions + m);
        const std::size_t d = std::size_t(1) << m;
        std::vector<cvector<double>> dm;
        for (int p = 0; p < np; ++p) {
            dm.push_back(to_cvec(dmats + p * d * d, d * d));
        }
        const auto acc = reverse_sweep_step<double>(
            phi->amps(), psi->amps(), phi->pseudo_qubits(), pos, to_cvec(inv, d * d),
            std::span<const cvector<double>>(dm), cfg());
        for (int p = 0; p < np; ++p) {
            out[p].re = acc[p].real();
            out[p].im = acc[p].imag();
        }
    });
}

// ---- losses / gradients ----
REF_API int vqcsref_loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                              int64_t nterms, const RefState *s0, double *loss) {
    return guard([&] {
        if (!s0->pure) {
            throw TypeError("loss_pure: pure initial state required");
        }
        *loss = loss_pure(to_operator(terms, nterms), to_circuit(ops, count), *s0->pure,
                          cfg());
    });
}

REF_API int vqcsref_gradient_pure(const vqb_op *ops, int64_t count,
                                  const vqb_pauli_term *terms, int64_t nterms,
                                  const RefState *s0, double *loss, double *grads,
                                  int64_t capacity, int64_t *num_grads, double *residual) {
    return guard([&] {
        if (!s0->pure) {
            throw TypeError("gradient_pure: pure initial state required");
        }
        GradientDiagnostics diag;
        const auto r = gradient_pure(to_operator(terms, nterms), to_circuit(ops, count),
                                     *s0->pure, cfg(), &diag);
        if (static_cast<int64_t>(r.grads.size()) > capacity) {
            throw ShapeError("gradient_pure: gradient buffer too small");
        }
        *loss = r.loss;
        std::copy(r.grads.begin(), r.grads.end(), grads);
        *num_grads = static_cast<int64_t>(r.grads.size());
        if (residual) *residual = diag.reverse_residual;
    });
}

REF_API int vqcsref_loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                               int64_t nterms, const RefState *dm0, double *loss) {
    return guard([&] {
        if (!dm0->mixed) {
            throw TypeError("loss_mixed: mixed initial state required");
        }
        *loss = loss_mixed(to_operator(terms, nterms), to_circuit(ops, count), *dm0->mixed,
                           cfg());
    });
}

REF_API int vqcsref_gradient_mixed(const vqb_op *ops, int64_t count,
                                   const vqb_pauli_term *terms, int64_t nterms,
                                   const RefState *dm0, double *loss, double *grads,
                                   int64_t capacity, int64_t *num_grads, double *residual) {
    return guard([&] {
        if (!dm0->mixed) {
            throw TypeError("gradient_mixed: mixed initial state required");
        }
        GradientDiagnostics diag;
        const auto r = gradient_mixed(to_operator(terms, nterms), to_circuit(ops, count),
                                      *dm0->mixed, cfg(), &diag);
        if (static_cast<int64_t>(r.grads.size()) > capacity) {
            throw ShapeError("gradient_mixed: gradient buffer too small");
        }
        *loss = r.loss;
        std::copy(r.grads.begin(), r.grads.end(), grads);
        *num_grads = static_cast<int64_t>(r.grads.size());
        if (residual) *residual = diag.reverse_residual;
    });
}

// ---- gate algebra ----
REF_API int vqcsref_gate_matrix(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { from_cvec(to_gate(*op).matrix, out); });
}

REF_API int vqcsref_gate_derivative(const vqb_op *op, int32_t p, vqb_c128 *out) {
    return guard([&] { from_cvec(gate_derivative(to_gate(*op), p), out); });
}

REF_API int vqcsref_gate_inverse(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { from_cvec(gate_inverse(to_gate(*op)).matrix, out); });
}

// the reference's rule: LU inverse of the superoperator (autodiff.hpp:263-276)
REF_API int vqcsref_channel_inverse(const vqb_op *op, vqb_c128 *out, double *condition,
                                    int32_t *singular) {
    return guard([&] {
        const auto c = to_channel(*op);
        const auto s = channel_superoperator(c);
        const auto lu = linalg::lu_inverse(s.matrix, s.dim());
        if (condition) *condition = lu.condition;
        if (singular) *singular = lu.singular ? 1 : 0;
        if (!lu.singular && out) std::memcpy(out, lu.inverse.data(), lu.inverse.size() * sizeof(C));
    });
}

REF_API int vqcsref_channel_superop(const vqb_op *op, vqb_c128 *out) {
    return guard([&] { from_cvec(channel_superoperator(to_channel(*op)).matrix, out); });
}

// ---- measurement (circuit.hpp:303-375) ----
// The reference draws the outcome from a caller-supplied std::mt19937_64; the
// C-ABI takes the drawn uniform instead. These two entry points let tests
// reproduce a reference draw: the uniform a stream (seed, after `skip`
// draws) yields, and measure() run on that very stream.
REF_API int vqcsref_uniform_unit(uint64_t seed, uint64_t skip, double *u) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        rng.discard(skip);
        *u = detail::uniform_unit(rng);
    });
}

REF_API int vqcsref_measure_seeded(RefState *s, int32_t qubit, uint64_t seed, uint64_t skip,
                                   int32_t *outcome, double *probability) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        rng.discard(skip);
        const MeasurementOutcome r =
            s->pure ? measure(*s->pure, qubit, rng) : measure(*s->mixed, qubit, rng);
        *outcome = r.outcome;
        *probability = r.probability;
    });
}

// ---- state dumps (io.hpp) ----
REF_API int vqcsref_state_save(const RefState *s, const char *path) {
    return guard([&] {
        if (!s->pure) {
            throw TypeError("save_state: only pure states can be dumped");
        }
        save_state(*s->pure, std::string(path));
    });
}

REF_API int vqcsref_state_load(const char *path, RefState **out, int32_t *precision) {
    return guard([&] {
        const LoadedState ls = load_state(std::string(path));
        auto s = std::make_unique<RefState>();
        s->pure.emplace(ls.to_pure<double>());
        if (precision) *precision = static_cast<int32_t>(ls.precision);
        *out = s.release();
    });
}

// ---- fuse_gates (circuit.hpp:199-276) ----
REF_API int vqcsref_fuse_gates(const vqb_op *ops, int64_t count, int64_t cap, vqb_op *out_ops,
                               int64_t matrix_cap, vqb_c128 *out_matrices, int64_t *num_out,
                               int64_t *num_entries) {
    return guard([&] {
        const Circuit<double> fused = fuse_gates(to_circuit(ops, count));
        std::vector<GateOp<double>> gates;
        fused.for_each_gate([&](const GateOp<double> &g) { gates.push_back(g); });
        int64_t entries = 0;
        for (const auto &g : gates) entries += (int64_t)g.matrix.size();
        *num_out = (int64_t)gates.size();
        *num_entries = entries;
        if (cap == 0) {
            return;
        }
        if (cap < (int64_t)gates.size() || matrix_cap < entries) {
            throw ShapeError("fuse_gates: output buffers too small");
        }
        int64_t off = 0;
        for (std::size_t i = 0; i < gates.size(); ++i) {
            vqb_op o;
            std::memset(&o, 0, sizeof o);
            o.elem = VQB_ELEM_GATE;
            o.kind = static_cast<int32_t>(gates[i].kind);
            o.num_positions = (int32_t)gates[i].positions.size();
            for (std::size_t k = 0; k < gates[i].positions.size(); ++k) {
                o.positions[k] = gates[i].positions[k];
            }
            o.matrix = out_matrices + off;
            from_cvec(gates[i].matrix, out_matrices + off);
            off += (int64_t)gates[i].matrix.size();
            out_ops[i] = o;
        }
    });
}

// ---- batched reverse steps: reverse_sweep_step (kernels.hpp:659-697) per step ----
REF_API int vqcsref_reverse_sweep(RefState *phi, RefState *psi, const vqb_rev_step *steps,
                                  int64_t count, double scale, double *grads, int64_t grads_len) {
    return guard([&] {
        if (phi == psi) {
            throw UsageError("reverse_sweep: phi and psi must be distinct states");
        }
        for (int64_t i = 0; i < count; ++i) {
            const vqb_rev_step &st = steps[i];
            const std::vector<int> pos(st.positions, st.positions + st.num_positions);
            const std::size_t d = std::size_t(1) << st.num_positions;
            std::vector<cvector<double>> dm;
            for (int p = 0; p < st.num_dmats; ++p) {
                dm.push_back(to_cvec(st.dmats + p * d * d, d * d));
            }
            if (st.num_dmats > 0 && (st.grad_index < 0 || st.grad_index + st.num_dmats > grads_len)) {
                throw IndexError("reverse_sweep: gradient slot out of range");
            }
            const auto acc = reverse_sweep_step<double>(
                phi->amps(), psi->amps(), phi->pseudo_qubits(), pos, to_cvec(st.inv, d * d),
                std::span<const cvector<double>>(dm), cfg());
            for (int p = 0; p < st.num_dmats; ++p) {
                grads[st.grad_index + p] += scale * acc[p].real();
            }
        }
    });
}
