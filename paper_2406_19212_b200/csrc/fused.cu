// Fused tile executor (placeholder: element-by-element until the tile kernels land).
#include "engine.hpp"

namespace vqb {

void run_program_fused(DeviceState *s, const std::vector<Gate> &prog) { run_program(s, prog, false); }

void run_reverse_fused(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                       double *dgrads) {
    run_reverse(phi, psi, prog, dgrads, false);
}

} // namespace vqb
