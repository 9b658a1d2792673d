// Host-side gate / channel algebra: descriptors -> small dense matrices.
//
// Semantics follow the reference builders (gates.hpp:161-733): matrices are
// column-major, first listed position = local LSB. These are tiny host
// computations that feed the device kernels.
#pragma once

#include "common.hpp"

namespace vqb {

struct Gate {
    int kind = VQB_GATE_GENERIC;
    int m = 0;
    int pos[VQB_MAX_POSITIONS] = {}; // 1-based
    int np = 0;
    double params[VQB_MAX_PARAMS] = {};
    bool is_param[VQB_MAX_PARAMS] = {};
    cvec mat; // 4^m entries

    int dim() const { return 1 << m; }
    int num_active() const {
        int c = 0;
        for (int i = 0; i < np; ++i) c += is_param[i] ? 1 : 0;
        return c;
    }
    bool has_active() const { return num_active() > 0; }
};

struct Channel {
    int kind = VQB_CHANNEL_GENERIC;
    int m = 0;
    int pos[3] = {};
    std::vector<cvec> kraus;
};

int gate_arity(int kind);
int param_arity(int kind);

// Validates positions and builds the matrix (caller's matrix, or the closed
// form of the named kind).
Gate gate_from_op(const vqb_op &op);
Channel channel_from_op(const vqb_op &op);

cvec gate_derivative(const Gate &g, int p);   // gates.hpp:543-577
Gate gate_inverse(const Gate &g);             // gates.hpp:581-619
cvec channel_superop(const Channel &c);       // gates.hpp:708-732
std::vector<Gate> fuse_gates(const std::vector<Gate> &flat); // circuit.hpp:199-276

// Small dense linear algebra on column-major d x d matrices.
cvec kron(const cvec &high, int dh, const cvec &low, int dl); // linalg.hpp:75-93
cvec adjoint(const cvec &a, int d);
cvec conjugated(const cvec &a);
cvec matmul(const cvec &a, const cvec &b, int d);
struct Inverse {
    cvec inv;
    double condition;
    bool singular;
};
Inverse lu_inverse(const cvec &a, int d); // linalg.hpp:140-200 (singularity / condition rule)
// Inverse of a channel's superoperator S: closed form for the named 1-qubit
// channels (gates.hpp:657-704), lu_inverse for Generic ones.
Inverse channel_inverse(const Channel &c, const cvec &S);

void check_positions(const int *pos, int m, const char *what);
void check_fit(const int *pos, int m, int n); // kernels.hpp:71-87

} // namespace vqb
