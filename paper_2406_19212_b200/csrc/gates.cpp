// Host-side gate / channel algebra (see gates.hpp). Closed forms restate the
// reference definitions cited per function.
#include "gates.hpp"

#include <cmath>
#include <cstring>

namespace vqb {

namespace {

const double kIsq = 0.70710678118654752440; // sqrt(2)/2

cvec eye(int d) {
    cvec m(size_t(d) * d);
    for (int i = 0; i < d; ++i) m[i + i * d] = 1.0;
    return m;
}

// gates.hpp:188-259
cvec fixed_matrix(int kind) {
    using C = cplx;
    switch (kind) {
    case VQB_GATE_X: return {0.0, 1.0, 1.0, 0.0};
    case VQB_GATE_Y: return {0.0, C(0, 1), C(0, -1), 0.0};
    case VQB_GATE_Z: return {1.0, 0.0, 0.0, -1.0};
    case VQB_GATE_H: return {kIsq, kIsq, kIsq, -kIsq};
    case VQB_GATE_S: return {1.0, 0.0, 0.0, C(0, 1)};
    case VQB_GATE_T: return {1.0, 0.0, 0.0, C(kIsq, kIsq)};
    case VQB_GATE_SQRTX: return {C(.5, .5), C(.5, -.5), C(.5, -.5), C(.5, .5)};
    case VQB_GATE_SQRTY: return {C(.5, .5), C(.5, .5), C(-.5, -.5), C(.5, .5)};
    case VQB_GATE_SWAP: {
        cvec m(16);
        m[0] = m[2 + 4] = m[1 + 8] = m[15] = 1.0;
        return m;
    }
    case VQB_GATE_ISWAP: {
        cvec m(16);
        m[0] = m[15] = 1.0;
        m[2 + 4] = m[1 + 8] = C(0, 1);
        return m;
    }
    case VQB_GATE_CZ: {
        cvec m = eye(4);
        m[15] = -1.0;
        return m;
    }
    case VQB_GATE_CNOT: { // first position = control
        cvec m(16);
        m[0] = m[2 + 8] = m[3 + 4] = m[1 + 12] = 1.0;
        return m;
    }
    case VQB_GATE_TOFFOLI: {
        cvec m = eye(8);
        m[3 + 24] = m[7 + 56] = 0.0;
        m[7 + 24] = m[3 + 56] = 1.0;
        return m;
    }
    case VQB_GATE_FREDKIN: {
        cvec m = eye(8);
        m[3 + 24] = m[5 + 40] = 0.0;
        m[5 + 24] = m[3 + 40] = 1.0;
        return m;
    }
    default:
        raise(VQB_ERR_UNSUPPORTED, "standard_gate: kind is not a fixed named gate");
    }
}

// gates.hpp:309-345
cvec rotation(int kind, double theta, bool derivative) {
    const double f = derivative ? 0.5 : 1.0;
    const double c = f * std::cos(theta / 2), s = f * std::sin(theta / 2);
    using C = cplx;
    const bool x = kind == VQB_GATE_RX || kind == VQB_GATE_CRX;
    const bool y = kind == VQB_GATE_RY || kind == VQB_GATE_CRY;
    if (!derivative) {
        if (x) return {c, C(0, -s), C(0, -s), c};
        if (y) return {c, s, -s, c};
        return {C(c, -s), 0.0, 0.0, C(c, s)};
    }
    if (x) return {-s, C(0, -c), C(0, -c), -s};
    if (y) return {-s, c, -c, -s};
    return {C(-s, -c), 0.0, 0.0, C(-s, c)};
}

// gates.hpp:349-358: identity on control = 0, block on control = 1.
cvec controlled_block(const cvec &u) {
    cvec m(16);
    m[0] = m[2 + 8] = 1.0;
    m[1 + 4] = u[0];
    m[3 + 4] = u[1];
    m[1 + 12] = u[2];
    m[3 + 12] = u[3];
    return m;
}

// gates.hpp:360-416. index < 0: the matrix itself; else d/dparam[index].
cvec fsim(const double *p, int index) {
    const double th = p[0], ph = p[1], dp = p[2], dm = p[3], doff = p[4];
    const double ct = std::cos(th), st = std::sin(th);
    const cplx i1(0, 1), mi(0, -1);
    const cplx e11 = std::polar(ct, dp + dm);
    const cplx e21 = mi * std::polar(st, dp + doff);
    const cplx e12 = mi * std::polar(st, dp - doff);
    const cplx e22 = std::polar(ct, dp - dm);
    const cplx e33 = std::polar(1.0, 2 * dp - ph);
    cvec m(16);
    switch (index) {
    case -1:
        m[0] = 1.0;
        m[1 + 4] = e11;
        m[2 + 4] = e21;
        m[1 + 8] = e12;
        m[2 + 8] = e22;
        m[15] = e33;
        break;
    case 0:
        m[1 + 4] = -std::polar(st, dp + dm);
        m[2 + 4] = -i1 * std::polar(ct, dp + doff);
        m[1 + 8] = -i1 * std::polar(ct, dp - doff);
        m[2 + 8] = -std::polar(st, dp - dm);
        break;
    case 1:
        m[15] = -i1 * e33;
        break;
    case 2:
        m[1 + 4] = i1 * e11;
        m[2 + 4] = i1 * e21;
        m[1 + 8] = i1 * e12;
        m[2 + 8] = i1 * e22;
        m[15] = 2.0 * i1 * e33;
        break;
    case 3:
        m[1 + 4] = i1 * e11;
        m[2 + 8] = -i1 * e22;
        break;
    case 4:
        m[2 + 4] = i1 * e21;
        m[1 + 8] = -i1 * e12;
        break;
    default:
        raise(VQB_ERR_DOMAIN, "fsim_derivative: parameter index out of range");
    }
    return m;
}

cvec parametric_matrix(int kind, const double *params) {
    switch (kind) {
    case VQB_GATE_RX:
    case VQB_GATE_RY:
    case VQB_GATE_RZ:
        return rotation(kind, params[0], false);
    case VQB_GATE_CRX:
    case VQB_GATE_CRY:
    case VQB_GATE_CRZ:
        return controlled_block(rotation(kind, params[0], false));
    case VQB_GATE_FSIM:
        return fsim(params, -1);
    default:
        raise(VQB_ERR_UNSUPPORTED, "parametric_matrix: kind has no parametric form");
    }
}

double max_abs(const cvec &a) {
    double m = 0;
    for (const auto &x : a) m = std::max(m, std::abs(x));
    return m;
}

double unitarity_defect(const cvec &a, int d) {
    double m = 0;
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) {
            cplx s = 0;
            for (int k = 0; k < d; ++k) s += std::conj(a[k + i * d]) * a[k + j * d];
            if (i == j) s -= 1.0;
            m = std::max(m, std::abs(s));
        }
    return m;
}

double norm1(const cvec &a, int d) {
    double best = 0;
    for (int j = 0; j < d; ++j) {
        double col = 0;
        for (int i = 0; i < d; ++i) col += std::abs(a[i + j * d]);
        best = std::max(best, col);
    }
    return best;
}

cvec from_c128(const vqb_c128 *p, size_t count) {
    cvec v(count);
    for (size_t i = 0; i < count; ++i) v[i] = cplx(p[i].re, p[i].im);
    return v;
}

} // namespace

int gate_arity(int kind) {
    switch (kind) {
    case VQB_GATE_X: case VQB_GATE_Y: case VQB_GATE_Z: case VQB_GATE_H: case VQB_GATE_S:
    case VQB_GATE_T: case VQB_GATE_SQRTX: case VQB_GATE_SQRTY: case VQB_GATE_RX:
    case VQB_GATE_RY: case VQB_GATE_RZ:
        return 1;
    case VQB_GATE_SWAP: case VQB_GATE_ISWAP: case VQB_GATE_CZ: case VQB_GATE_CNOT:
    case VQB_GATE_CRX: case VQB_GATE_CRY: case VQB_GATE_CRZ: case VQB_GATE_FSIM:
        return 2;
    case VQB_GATE_TOFFOLI: case VQB_GATE_FREDKIN:
        return 3;
    default:
        return 0;
    }
}

int param_arity(int kind) {
    switch (kind) {
    case VQB_GATE_RX: case VQB_GATE_RY: case VQB_GATE_RZ: case VQB_GATE_CRX: case VQB_GATE_CRY:
    case VQB_GATE_CRZ:
        return 1;
    case VQB_GATE_FSIM:
        return 5;
    default:
        return 0;
    }
}

void check_positions(const int *pos, int m, const char *what) {
    if (m < 1 || m > VQB_MAX_POSITIONS)
        raise(VQB_ERR_SHAPE, std::string(what) + ": needs 1..6 positions");
    for (int i = 0; i < m; ++i) {
        if (pos[i] < 1) raise(VQB_ERR_VALIDITY, std::string(what) + ": positions must be >= 1");
        for (int j = i + 1; j < m; ++j)
            if (pos[i] == pos[j])
                raise(VQB_ERR_VALIDITY,
                      std::string(what) + ": duplicate position " + std::to_string(pos[i]));
    }
}

void check_fit(const int *pos, int m, int n) {
    for (int i = 0; i < m; ++i)
        if (pos[i] < 1 || pos[i] > n)
            raise(VQB_ERR_INDEX, "gate position " + std::to_string(pos[i]) +
                                     " does not fit a " + std::to_string(n) + "-qubit state");
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            if (pos[i] == pos[j])
                raise(VQB_ERR_VALIDITY, "duplicate gate position " + std::to_string(pos[i]));
}

Gate gate_from_op(const vqb_op &op) {
    if (op.elem != VQB_ELEM_GATE) raise(VQB_ERR_TYPE, "expected a gate element");
    check_positions(op.positions, op.num_positions, "gate");
    if (op.num_params < 0 || op.num_params > VQB_MAX_PARAMS)
        raise(VQB_ERR_SHAPE, "gate: bad parameter count");
    Gate g;
    g.kind = op.kind;
    g.m = op.num_positions;
    std::memcpy(g.pos, op.positions, sizeof(int) * g.m);
    g.np = op.num_params;
    for (int i = 0; i < g.np; ++i) {
        g.params[i] = op.params[i];
        g.is_param[i] = op.is_param[i] != 0;
    }
    const int d = g.dim();
    if (op.matrix != nullptr) {
        g.mat = from_c128(op.matrix, size_t(d) * d);
        // make_gate validates unitarity (gates.hpp:161-173)
        if (g.kind == VQB_GATE_GENERIC && unitarity_defect(g.mat, d) > 1e-8)
            raise(VQB_ERR_VALIDITY, "make_gate: matrix is not unitary within 1e-8");
        return g;
    }
    const int arity = gate_arity(g.kind);
    if (arity == 0) raise(VQB_ERR_UNSUPPORTED, "gate: kind needs an explicit matrix");
    if (arity != g.m)
        raise(VQB_ERR_SHAPE, "gate: kind needs " + std::to_string(arity) + " position(s)");
    if (param_arity(g.kind) == 0) {
        if (g.np != 0) raise(VQB_ERR_UNSUPPORTED, "standard_gate: kind is not a fixed named gate");
        g.mat = fixed_matrix(g.kind);
    } else {
        if (g.np != param_arity(g.kind))
            raise(VQB_ERR_SHAPE, "parametric_gate: wrong parameter count");
        g.mat = parametric_matrix(g.kind, g.params);
    }
    return g;
}

Channel channel_from_op(const vqb_op &op) {
    if (op.elem != VQB_ELEM_CHANNEL) raise(VQB_ERR_TYPE, "expected a channel element");
    check_positions(op.positions, op.num_positions, "channel");
    if (op.num_positions > 3) raise(VQB_ERR_UNSUPPORTED, "channels act on at most 3 qubits");
    Channel c;
    c.kind = op.kind;
    c.m = op.num_positions;
    std::memcpy(c.pos, op.positions, sizeof(int) * c.m);
    const int d = 1 << c.m;
    if (op.kraus != nullptr) {
        if (op.num_kraus < 1) raise(VQB_ERR_SHAPE, "make_channel: needs at least one Kraus operator");
        cvec sum(size_t(d) * d);
        for (int s = 0; s < op.num_kraus; ++s) {
            c.kraus.push_back(from_c128(op.kraus + size_t(s) * d * d, size_t(d) * d));
            const cvec p = matmul(adjoint(c.kraus.back(), d), c.kraus.back(), d);
            for (size_t i = 0; i < sum.size(); ++i) sum[i] += p[i];
        }
        for (int i = 0; i < d; ++i) sum[i + i * d] -= 1.0;
        if (max_abs(sum) > 1e-8)
            raise(VQB_ERR_VALIDITY,
                  "make_channel: Kraus operators violate the completeness relation within 1e-8");
        return c;
    }
    // standard_channel gates.hpp:657-704
    const double p = op.params[0];
    if (c.m != 1) raise(VQB_ERR_SHAPE, "named channels act on one qubit");
    if (p < 0 || p > 1) raise(VQB_ERR_DOMAIN, "standard_channel: parameter must lie in [0,1]");
    switch (c.kind) {
    case VQB_CHANNEL_AMPLITUDE_DAMPING:
        c.kraus = {{1.0, 0.0, 0.0, std::sqrt(1 - p)}, {0.0, 0.0, std::sqrt(p), 0.0}};
        break;
    case VQB_CHANNEL_PHASE_DAMPING:
        c.kraus = {{1.0, 0.0, 0.0, std::sqrt(1 - p)}, {0.0, 0.0, 0.0, std::sqrt(p)}};
        break;
    case VQB_CHANNEL_DEPOLARIZING: {
        const double w0 = std::sqrt(1 - 0.75 * p), w = 0.5 * std::sqrt(p);
        c.kraus = {{w0, 0.0, 0.0, w0}};
        for (int k : {VQB_GATE_X, VQB_GATE_Y, VQB_GATE_Z}) {
            cvec m = fixed_matrix(k);
            for (auto &x : m) x *= w;
            c.kraus.push_back(m);
        }
        break;
    }
    default:
        raise(VQB_ERR_UNSUPPORTED, "standard_channel: not a named channel kind");
    }
    return c;
}

cvec gate_derivative(const Gate &g, int p) {
    if (g.kind == VQB_GATE_GENERIC || param_arity(g.kind) == 0)
        raise(VQB_ERR_UNSUPPORTED, "gate_derivative: gate has no closed form");
    if (p < 0 || p >= g.np) raise(VQB_ERR_DOMAIN, "gate_derivative: parameter index out of range");
    if (!g.is_param[p])
        raise(VQB_ERR_DOMAIN,
              "gate_derivative: parameter " + std::to_string(p) + " is not variational");
    switch (g.kind) {
    case VQB_GATE_RX:
    case VQB_GATE_RY:
    case VQB_GATE_RZ:
        return rotation(g.kind, g.params[0], true);
    case VQB_GATE_CRX:
    case VQB_GATE_CRY:
    case VQB_GATE_CRZ: {
        const cvec dr = rotation(g.kind, g.params[0], true);
        cvec m(16);
        m[1 + 4] = dr[0];
        m[3 + 4] = dr[1];
        m[1 + 12] = dr[2];
        m[3 + 12] = dr[3];
        return m;
    }
    default:
        return fsim(g.params, p);
    }
}

Gate gate_inverse(const Gate &g) {
    Gate inv;
    inv.m = g.m;
    std::memcpy(inv.pos, g.pos, sizeof(g.pos));
    switch (g.kind) {
    case VQB_GATE_X: case VQB_GATE_Y: case VQB_GATE_Z: case VQB_GATE_H: case VQB_GATE_SWAP:
    case VQB_GATE_CZ: case VQB_GATE_CNOT: case VQB_GATE_TOFFOLI: case VQB_GATE_FREDKIN:
        inv.kind = g.kind;
        inv.mat = g.mat;
        return inv;
    case VQB_GATE_RX: case VQB_GATE_RY: case VQB_GATE_RZ: case VQB_GATE_CRX: case VQB_GATE_CRY:
    case VQB_GATE_CRZ:
        inv.kind = g.kind;
        inv.np = 1;
        inv.params[0] = -g.params[0];
        inv.mat = parametric_matrix(g.kind, inv.params);
        return inv;
    case VQB_GATE_FSIM:
        inv.kind = g.kind;
        inv.np = 5;
        for (int i = 0; i < 4; ++i) inv.params[i] = -g.params[i];
        inv.params[4] = g.params[4];
        inv.mat = parametric_matrix(g.kind, inv.params);
        return inv;
    default:
        inv.kind = VQB_GATE_GENERIC;
        inv.mat = adjoint(g.mat, g.dim());
        return inv;
    }
}

cvec channel_superop(const Channel &c) {
    const int d = 1 << c.m, dd = d * d;
    cvec s(size_t(dd) * dd);
    for (const auto &k : c.kraus)
        for (int tp = 0; tp < d; ++tp)
            for (int sp = 0; sp < d; ++sp) {
                const cplx kc = std::conj(k[tp + sp * d]);
                if (kc == cplx(0)) continue;
                for (int sig = 0; sig < d; ++sig)
                    for (int tau = 0; tau < d; ++tau)
                        s[(tau + tp * d) + size_t(sig + sp * d) * dd] += k[tau + sig * d] * kc;
            }
    return s;
}

cvec kron(const cvec &high, int dh, const cvec &low, int dl) {
    const int d = dh * dl;
    cvec r(size_t(d) * d);
    for (int ch = 0; ch < dh; ++ch)
        for (int cl = 0; cl < dl; ++cl)
            for (int rh = 0; rh < dh; ++rh)
                for (int rl = 0; rl < dl; ++rl)
                    r[(rl + rh * dl) + size_t(cl + ch * dl) * d] =
                        high[rh + ch * dh] * low[rl + cl * dl];
    return r;
}

cvec adjoint(const cvec &a, int d) {
    cvec r(size_t(d) * d);
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) r[j + i * d] = std::conj(a[i + j * d]);
    return r;
}

cvec conjugated(const cvec &a) {
    cvec r(a.size());
    for (size_t i = 0; i < a.size(); ++i) r[i] = std::conj(a[i]);
    return r;
}

cvec matmul(const cvec &a, const cvec &b, int d) {
    cvec r(size_t(d) * d);
    for (int j = 0; j < d; ++j)
        for (int k = 0; k < d; ++k) {
            const cplx bkj = b[k + j * d];
            if (bkj == cplx(0)) continue; // linalg.hpp:46-48
            for (int i = 0; i < d; ++i) r[i + j * d] += a[i + k * d] * bkj;
        }
    return r;
}

// Dense inverse for the channel-inversion rule of gradient_mixed
// (autodiff.hpp:263-276, linalg.hpp:140-200): Gauss-Jordan elimination with
// partial pivoting on [A | I]. The pivot sequence equals the reference LU's
// (same column maxima), so "singular" (a pivot at or below 1e-300 of max|A|)
// is decided identically, and condition = ||A||_1 ||A^-1||_1 as there.
Inverse lu_inverse(const cvec &a, int d) {
    const int w = 2 * d; // row-major augmented rows [A row | I row]
    std::vector<cplx> m(size_t(d) * w, cplx(0));
    for (int r = 0; r < d; ++r) {
        for (int c = 0; c < d; ++c) m[size_t(r) * w + c] = a[r + size_t(c) * d];
        m[size_t(r) * w + d + r] = 1.0;
    }
    const double tiny = std::max(max_abs(a), 1e-300) * 1e-300;
    for (int col = 0; col < d; ++col) {
        int piv = col;
        for (int r = col + 1; r < d; ++r)
            if (std::abs(m[size_t(r) * w + col]) > std::abs(m[size_t(piv) * w + col])) piv = r;
        if (std::abs(m[size_t(piv) * w + col]) <= tiny) return {{}, INFINITY, true};
        if (piv != col)
            std::swap_ranges(m.begin() + size_t(piv) * w, m.begin() + size_t(piv + 1) * w,
                             m.begin() + size_t(col) * w);
        const cplx inv_p = 1.0 / m[size_t(col) * w + col];
        for (int c = col; c < w; ++c) m[size_t(col) * w + c] *= inv_p;
        for (int r = 0; r < d; ++r) {
            if (r == col) continue;
            const cplx f = m[size_t(r) * w + col];
            if (f == cplx(0)) continue;
            for (int c = col; c < w; ++c) m[size_t(r) * w + c] -= f * m[size_t(col) * w + c];
        }
    }
    cvec inv(size_t(d) * d);
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) inv[r + size_t(c) * d] = m[size_t(r) * w + d + c];
    const double cond = norm1(a, d) * norm1(inv, d);
    return {std::move(inv), cond, false};
}

// Closed-form inverse of a named single-qubit channel's superoperator
// (standard_channel, gates.hpp:657-704). Amplitude damping, phase damping and
// depolarizing all map populations to populations and scale each coherence:
// in the (tau + 2 tau') order the superoperator is block diagonal with the
// 2x2 population block on {0, 3} and the coherences 1, 2 on the diagonal, so
// its inverse is that block's 2x2 inverse and two reciprocals (e.g.
// depolarizing: [[1-p/2, p/2], [p/2, 1-p/2]]^-1 = [[1-p/2, -p/2], [-p/2,
// 1-p/2]] / (1-p), coherences 1/(1-p)). Generic channels keep the
// elimination (the reference's rule for every channel, autodiff.hpp:263-276).
Inverse channel_inverse(const Channel &c, const cvec &S) {
    const int d = 1 << (2 * c.m);
    if (c.kind == VQB_CHANNEL_GENERIC || c.m != 1) return lu_inverse(S, d);
    auto at = [&](int r, int col) { return S[r + size_t(col) * 4]; };
    for (int r = 0; r < 4; ++r)
        for (int col = 0; col < 4; ++col) {
            const bool pop = (r == 0 || r == 3) && (col == 0 || col == 3);
            if (!pop && r != col && at(r, col) != cplx(0)) return lu_inverse(S, d); // not the named form
        }
    const double tiny = std::max(max_abs(S), 1e-300) * 1e-300;
    const cplx det = at(0, 0) * at(3, 3) - at(0, 3) * at(3, 0);
    if (std::abs(det) <= tiny || std::abs(at(1, 1)) <= tiny || std::abs(at(2, 2)) <= tiny)
        return {{}, INFINITY, true};
    cvec inv(16, cplx(0));
    inv[0 + 0 * 4] = at(3, 3) / det;
    inv[0 + 3 * 4] = -at(0, 3) / det;
    inv[3 + 0 * 4] = -at(3, 0) / det;
    inv[3 + 3 * 4] = at(0, 0) / det;
    inv[1 + 1 * 4] = 1.0 / at(1, 1);
    inv[2 + 2 * 4] = 1.0 / at(2, 2);
    const double cond = norm1(S, 4) * norm1(inv, 4);
    return {std::move(inv), cond, false};
}

} // namespace vqb
