// Program layer: circuits lowered to flat gate programs on the (pseudo) state,
// executed either element by element or as fused shared-memory tile passes.
#pragma once

#include "device.hpp"

namespace vqb {

constexpr double kChannelConditionLimit = 1e12; // autodiff.hpp:51

struct Element {
    bool channel = false;
    Gate gate;
    Channel chan;
};

std::vector<Element> build_elements(const vqb_op *ops, int64_t count);

// Forward program of a density-matrix circuit on the 2n-qubit pseudo state:
// gates act on the ket positions and (conjugated) on the bra mirrors
// (apply_gate_mixed kernels.hpp:434-449); channels become superoperators on
// (pos..., pos+n...) (apply_channel kernels.hpp:453-461).
std::vector<Gate> mixed_forward_program(const std::vector<Element> &es, int n);

// One reverse-sweep step on (phi, psi): phi <- phi_op phi, psi <- psi_op psi,
// and, when dmats is non-empty, grads[grad_base + p] = scale * Re <psi|D_p|phi>
// taken between the two updates (reverse_sweep_step kernels.hpp:659-697).
struct RevOp {
    Gate phi_op;
    Gate psi_op;
    std::vector<cvec> dmats;
    int64_t grad_base = -1;
    double scale = 1.0;
};

std::vector<RevOp> pure_reverse_program(const std::vector<Element> &es,
                                        const std::vector<int64_t> &base);
std::vector<RevOp> mixed_reverse_program(const std::vector<Element> &es, int n,
                                         const std::vector<int64_t> &base,
                                         const std::vector<cvec> &chan_inv,
                                         const std::vector<cvec> &chan_adj);

// Launch gate of the host-parallel adjoint: the reverse sweep is planned on
// a worker thread while the calling thread launches the forward pass; the
// worker's executors call wait_issue_gate() before their first device work,
// which returns once the caller has enqueued everything that must precede
// the sweep on the stream (no-op on threads without a gate).
void wait_issue_gate();

// Execute a forward program on s (asynchronous on s->stream).
void run_program(DeviceState *s, const std::vector<Gate> &prog, bool fused);
// Execute a reverse program on (phi, psi); gradients go to the device vector.
void run_reverse(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                 double *dgrads, bool fused);

// Fused executor (fused.cu).
void run_program_fused(DeviceState *s, const std::vector<Gate> &prog);
void run_reverse_fused(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                       double *dgrads);

} // namespace vqb
