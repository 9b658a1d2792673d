// Device losses and adjoint gradients (autodiff.hpp:80-329 of the reference).
#pragma once

#include "device.hpp"

namespace vqb {

struct GradientOut {
    double loss = 0;
    std::vector<double> grads;
    double residual = 0;
};

GradientOut gradient_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                          int64_t nterms, DeviceState *s0, bool want_residual, bool fused);
GradientOut gradient_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                           int64_t nterms, DeviceState *dm0, bool want_residual, bool fused);
double loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms, int64_t nterms,
                 DeviceState *s0, bool fused);
double loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms, int64_t nterms,
                  DeviceState *dm0, bool fused);

} // namespace vqb
