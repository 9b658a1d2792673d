// fuse_gates (circuit.hpp:199-276): the reference's own circuit-level fusion,
// a host-side caller of the path. Single-qubit gates are absorbed into the
// next two-qubit gate touching their qubit, else into the previous one; gates
// absorbed earlier multiply from the right, later ones from the left. The
// fused executor (plan.cpp) does strictly more (k-qubit blocks with qubit
// remapping), so this exists for API parity: vqb_apply_circuit on its output
// runs through the same executor.
#include "gates.hpp"

#include <cstddef>

namespace vqb {

namespace {

// detail::embed_1q_in_2q (circuit.hpp:190-196)
cvec embed_1q_in_2q(const cvec &m, int local_bit) {
    const cvec eye = {cplx(1), cplx(0), cplx(0), cplx(1)};
    return local_bit == 0 ? kron(eye, 2, m, 2) : kron(m, 2, eye, 2);
}

bool touches(const Gate &g, int q) {
    for (int i = 0; i < g.m; ++i)
        if (g.pos[i] == q) return true;
    return false;
}

} // namespace

std::vector<Gate> fuse_gates(const std::vector<Gate> &flat) {
    const std::ptrdiff_t count = (std::ptrdiff_t)flat.size();
    std::vector<std::ptrdiff_t> merge_into(flat.size(), -1);
    for (std::ptrdiff_t i = 0; i < count; ++i) {
        if (flat[i].m != 1) continue;
        const int q = flat[i].pos[0];
        std::ptrdiff_t prev = -1, next = -1;
        for (std::ptrdiff_t j = i - 1; j >= 0; --j)
            if (touches(flat[j], q)) {
                prev = j;
                break;
            }
        for (std::ptrdiff_t j = i + 1; j < count; ++j)
            if (touches(flat[j], q)) {
                next = j;
                break;
            }
        if (next >= 0 && flat[next].m == 2) merge_into[i] = next;
        else if (prev >= 0 && flat[prev].m == 2) merge_into[i] = prev;
    }
    std::vector<Gate> fused;
    for (std::ptrdiff_t i = 0; i < count; ++i) {
        if (merge_into[i] >= 0) continue;
        Gate out; // generic, non-parametric
        out.m = flat[i].m;
        for (int k = 0; k < out.m; ++k) out.pos[k] = flat[i].pos[k];
        out.mat = flat[i].mat;
        if (flat[i].m == 2) {
            for (std::ptrdiff_t k = 0; k < count; ++k) {
                if (merge_into[k] != i) continue;
                const int bit = flat[k].pos[0] == out.pos[0] ? 0 : 1;
                const cvec e = embed_1q_in_2q(flat[k].mat, bit);
                out.mat = k < i ? matmul(out.mat, e, 4) : matmul(e, out.mat, 4);
            }
        }
        fused.push_back(std::move(out));
    }
    return fused;
}

} // namespace vqb
