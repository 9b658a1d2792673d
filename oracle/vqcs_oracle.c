/*
 * oracle/vqcs_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A serial, plain-C restatement of the reference `vqcs` hot path
 * (/root/reference/proj/include/vqcs/ headers), exposing the C-ABI of
 * include/vqcs_b200.h with the prefix `vqcsorc_`. It is the parity checker
 * for the CUDA path; it is never linked into, called by, or measured as the
 * product. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.
 *
 * Pinning: tests/test_oracle.py checks it against (a) the reference itself
 * compiled from /root/reference (oracle/_ref/libvqcs_ref.so, ref_shim.cpp),
 * and (b) the golden vectors under tests/golden/ generated from that build by
 * tests/golden/make_golden.py, and (c) the reference tests' known answers.
 *
 * Arithmetic follows the reference's operation order (complex products as
 * (ac - bd, ad + bc), sums left to right) and is compiled with
 * -ffp-contract=off so results are expected to agree with the reference
 * bit for bit on single-threaded runs.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/vqcs_b200.h"

#define ORC_API __attribute__((visibility("default")))

typedef vqb_c128 cd;

static _Thread_local char g_err[512];

static int fail(int code, const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

ORC_API const char *vqcsorc_last_error(void) { return g_err; }

/* ---- complex arithmetic in the reference's (std::complex) order ---- */
static inline cd C(double re, double im) {
    cd z = {re, im};
    return z;
}
static inline cd cmul(cd a, cd b) { return C(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cd cadd(cd a, cd b) { return C(a.re + b.re, a.im + b.im); }
static inline cd csub(cd a, cd b) { return C(a.re - b.re, a.im - b.im); }
static inline cd cconj(cd a) { return C(a.re, -a.im); }
static inline double cabs_(cd a) { return hypot(a.re, a.im); }
/* std::polar(r, t) = (r cos t, r sin t) */
static inline cd cpolar(double r, double t) { return C(r * cos(t), r * sin(t)); }
/* std::complex<double> division compiles to libgcc's __divdc3 under GCC
 * without -ffast-math; C99 complex division calls the same routine. */
static inline cd cdiv(cd a, cd b) {
    const _Complex double r = __builtin_complex(a.re, a.im) / __builtin_complex(b.re, b.im);
    return C(__real__ r, __imag__ r);
}

/* ================= gate algebra: gates.hpp ================= */

/* gate_arity gates.hpp:261-291 */
static int gate_arity(int kind) {
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

/* param_arity gates.hpp:293-307 */
static int param_arity(int kind) {
    switch (kind) {
    case VQB_GATE_RX: case VQB_GATE_RY: case VQB_GATE_RZ: case VQB_GATE_CRX:
    case VQB_GATE_CRY: case VQB_GATE_CRZ:
        return 1;
    case VQB_GATE_FSIM:
        return 5;
    default:
        return 0;
    }
}

static void identity(cd *m, int d) {
    memset(m, 0, sizeof(cd) * d * d);
    for (int i = 0; i < d; ++i) m[i + i * d] = C(1, 0);
}

/* fixed_gate_matrix gates.hpp:188-259 */
static int fixed_matrix(int kind, cd *m) {
    const double isq = 0.70710678118654752440; /* std::numbers::sqrt2 / 2 */
    switch (kind) {
    case VQB_GATE_X: m[0] = C(0, 0); m[1] = C(1, 0); m[2] = C(1, 0); m[3] = C(0, 0); return 0;
    case VQB_GATE_Y: m[0] = C(0, 0); m[1] = C(0, 1); m[2] = C(0, -1); m[3] = C(0, 0); return 0;
    case VQB_GATE_Z: m[0] = C(1, 0); m[1] = C(0, 0); m[2] = C(0, 0); m[3] = C(-1, 0); return 0;
    case VQB_GATE_H: m[0] = C(isq, 0); m[1] = C(isq, 0); m[2] = C(isq, 0); m[3] = C(-isq, 0); return 0;
    case VQB_GATE_S: m[0] = C(1, 0); m[1] = C(0, 0); m[2] = C(0, 0); m[3] = C(0, 1); return 0;
    case VQB_GATE_T: m[0] = C(1, 0); m[1] = C(0, 0); m[2] = C(0, 0); m[3] = C(isq, isq); return 0;
    case VQB_GATE_SQRTX:
        m[0] = C(0.5, 0.5); m[1] = C(0.5, -0.5); m[2] = C(0.5, -0.5); m[3] = C(0.5, 0.5); return 0;
    case VQB_GATE_SQRTY:
        m[0] = C(0.5, 0.5); m[1] = C(0.5, 0.5); m[2] = C(-0.5, -0.5); m[3] = C(0.5, 0.5); return 0;
    case VQB_GATE_SWAP:
        memset(m, 0, sizeof(cd) * 16);
        m[0] = C(1, 0); m[2 + 4] = C(1, 0); m[1 + 8] = C(1, 0); m[15] = C(1, 0); return 0;
    case VQB_GATE_ISWAP:
        memset(m, 0, sizeof(cd) * 16);
        m[0] = C(1, 0); m[2 + 4] = C(0, 1); m[1 + 8] = C(0, 1); m[15] = C(1, 0); return 0;
    case VQB_GATE_CZ:
        identity(m, 4); m[15] = C(-1, 0); return 0;
    case VQB_GATE_CNOT: /* first position controls */
        memset(m, 0, sizeof(cd) * 16);
        m[0] = C(1, 0); m[2 + 8] = C(1, 0); m[3 + 4] = C(1, 0); m[1 + 12] = C(1, 0); return 0;
    case VQB_GATE_TOFFOLI:
        identity(m, 8); m[3 + 24] = C(0, 0); m[7 + 56] = C(0, 0);
        m[7 + 24] = C(1, 0); m[3 + 56] = C(1, 0); return 0;
    case VQB_GATE_FREDKIN:
        identity(m, 8); m[3 + 24] = C(0, 0); m[5 + 40] = C(0, 0);
        m[5 + 24] = C(1, 0); m[3 + 40] = C(1, 0); return 0;
    default:
        return -1;
    }
}

/* rotation_matrix gates.hpp:309-326 */
static void rotation(int kind, double theta, cd *m) {
    const double c = cos(theta / 2), s = sin(theta / 2);
    switch (kind) {
    case VQB_GATE_RX: case VQB_GATE_CRX:
        m[0] = C(c, 0); m[1] = C(0, -s); m[2] = C(0, -s); m[3] = C(c, 0); break;
    case VQB_GATE_RY: case VQB_GATE_CRY:
        m[0] = C(c, 0); m[1] = C(s, 0); m[2] = C(-s, 0); m[3] = C(c, 0); break;
    default: /* Rz, CRz */
        m[0] = C(c, -s); m[1] = C(0, 0); m[2] = C(0, 0); m[3] = C(c, s); break;
    }
}

/* rotation_derivative gates.hpp:328-345 */
static void rotation_deriv(int kind, double theta, cd *m) {
    const double c = 0.5 * cos(theta / 2), s = 0.5 * sin(theta / 2);
    switch (kind) {
    case VQB_GATE_RX: case VQB_GATE_CRX:
        m[0] = C(-s, 0); m[1] = C(0, -c); m[2] = C(0, -c); m[3] = C(-s, 0); break;
    case VQB_GATE_RY: case VQB_GATE_CRY:
        m[0] = C(-s, 0); m[1] = C(c, 0); m[2] = C(-c, 0); m[3] = C(-s, 0); break;
    default:
        m[0] = C(-s, -c); m[1] = C(0, 0); m[2] = C(0, 0); m[3] = C(-s, c); break;
    }
}

/* controlled_block gates.hpp:349-358 */
static void controlled_block(const cd *u, cd *m) {
    memset(m, 0, sizeof(cd) * 16);
    m[0] = C(1, 0); m[2 + 8] = C(1, 0);
    m[1 + 4] = u[0]; m[3 + 4] = u[1]; m[1 + 12] = u[2]; m[3 + 12] = u[3];
}


/* fsim_matrix gates.hpp:360-373 */
static void fsim(const double *p, cd *m) {
    const double th = p[0], ph = p[1], dp = p[2], dm = p[3], doff = p[4];
    const double ct = cos(th), st = sin(th);
    memset(m, 0, sizeof(cd) * 16);
    m[0] = C(1, 0);
    m[1 + 4] = cpolar(ct, dp + dm);
    m[2 + 4] = cmul(C(0, -1), cpolar(st, dp + doff));
    m[1 + 8] = cmul(C(0, -1), cpolar(st, dp - doff));
    m[2 + 8] = cpolar(ct, dp - dm);
    m[3 + 12] = cpolar(1.0, 2 * dp - ph);
}

/* fsim_derivative gates.hpp:375-416 */
static int fsim_deriv(const double *p, int index, cd *m) {
    const double th = p[0], ph = p[1], dp = p[2], dm = p[3], doff = p[4];
    const double ct = cos(th), st = sin(th);
    const cd i1 = C(0, 1);
    const cd e11 = cpolar(ct, dp + dm);
    const cd e21 = cmul(C(-0.0, -1), cpolar(st, dp + doff)); /* -i1 * ... */
    const cd e12 = cmul(C(-0.0, -1), cpolar(st, dp - doff));
    const cd e22 = cpolar(ct, dp - dm);
    const cd e33 = cpolar(1.0, 2 * dp - ph);
    memset(m, 0, sizeof(cd) * 16);
    switch (index) {
    case 0: {
        cd a = cpolar(st, dp + dm);
        m[1 + 4] = C(-a.re, -a.im);
        m[2 + 4] = cmul(C(-0.0, -1), cpolar(ct, dp + doff));
        m[1 + 8] = cmul(C(-0.0, -1), cpolar(ct, dp - doff));
        a = cpolar(st, dp - dm);
        m[2 + 8] = C(-a.re, -a.im);
        break;
    }
    case 1:
        m[3 + 12] = cmul(C(-0.0, -1), e33);
        break;
    case 2:
        m[1 + 4] = cmul(i1, e11);
        m[2 + 4] = cmul(i1, e21);
        m[1 + 8] = cmul(i1, e12);
        m[2 + 8] = cmul(i1, e22);
        m[3 + 12] = cmul(cmul(C(2.0, 0), i1), e33);
        break;
    case 3:
        m[1 + 4] = cmul(i1, e11);
        m[2 + 8] = cmul(C(-0.0, -1), e22);
        break;
    case 4:
        m[2 + 4] = cmul(i1, e21);
        m[1 + 8] = cmul(C(-0.0, -1), e12);
        break;
    default:
        return -1;
    }
    return 0;
}

/* parametric_matrix gates.hpp:418-434 */
static void parametric_matrix(int kind, const double *params, cd *m) {
    if (kind == VQB_GATE_FSIM) {
        fsim(params, m);
    } else if (kind == VQB_GATE_CRX || kind == VQB_GATE_CRY || kind == VQB_GATE_CRZ) {
        cd u[4];
        rotation(kind, params[0], u);
        controlled_block(u, m);
    } else {
        rotation(kind, params[0], m);
    }
}

static int check_positions(const int32_t *pos, int m) {
    if (m < 1 || m > VQB_MAX_POSITIONS) return fail(VQB_ERR_SHAPE, "needs 1..6 positions");
    for (int i = 0; i < m; ++i) {
        if (pos[i] < 1) return fail(VQB_ERR_VALIDITY, "positions must be >= 1");
        for (int j = i + 1; j < m; ++j)
            if (pos[i] == pos[j]) return fail(VQB_ERR_VALIDITY, "duplicate position");
    }
    return VQB_OK;
}

/* The GateOp a reference caller would build from the descriptor:
 * standard_gate / parametric_gate / make_gate (gates.hpp:161-173,439-533). */
typedef struct {
    int kind, m, np;
    int32_t pos[VQB_MAX_POSITIONS];
    double params[VQB_MAX_PARAMS];
    int is_param[VQB_MAX_PARAMS];
    cd mat[64 * 64];
} gate_t;

static double unitarity_defect(const cd *a, int d) { /* linalg.hpp unitarity_defect */
    double mx = 0;
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) {
            cd s = C(0, 0);
            for (int k = 0; k < d; ++k) s = cadd(s, cmul(cconj(a[k + i * d]), a[k + j * d]));
            if (i == j) s.re -= 1.0;
            const double v = cabs_(s);
            if (v > mx) mx = v;
        }
    return mx;
}

static int build_gate(const vqb_op *op, gate_t *g) {
    int rc = check_positions(op->positions, op->num_positions);
    if (rc) return rc;
    g->kind = op->kind;
    g->m = op->num_positions;
    g->np = op->num_params;
    memcpy(g->pos, op->positions, sizeof(int32_t) * g->m);
    for (int i = 0; i < g->np; ++i) {
        g->params[i] = op->params[i];
        g->is_param[i] = op->is_param[i] != 0;
    }
    const int d = 1 << g->m;
    if (op->matrix != NULL) {
        memcpy(g->mat, op->matrix, sizeof(cd) * d * d);
        if (g->kind == VQB_GATE_GENERIC && unitarity_defect(g->mat, d) > 1e-8)
            return fail(VQB_ERR_VALIDITY, "make_gate: matrix is not unitary within 1e-8");
        return VQB_OK;
    }
    const int arity = gate_arity(g->kind);
    if (arity == 0) return fail(VQB_ERR_UNSUPPORTED, "gate kind needs an explicit matrix");
    if (arity != g->m) return fail(VQB_ERR_SHAPE, "wrong number of positions for gate kind");
    if (param_arity(g->kind) == 0) {
        if (g->np != 0) return fail(VQB_ERR_UNSUPPORTED, "standard_gate: not a fixed named gate");
        fixed_matrix(g->kind, g->mat);
    } else {
        if (g->np != param_arity(g->kind)) return fail(VQB_ERR_SHAPE, "wrong parameter count");
        parametric_matrix(g->kind, g->params, g->mat);
    }
    return VQB_OK;
}

static int has_active(const gate_t *g) {
    for (int i = 0; i < g->np; ++i)
        if (g->is_param[i]) return 1;
    return 0;
}

/* gate_derivative gates.hpp:543-577 */
static int gate_derivative(const gate_t *g, int p, cd *out) {
    if (g->kind == VQB_GATE_GENERIC || param_arity(g->kind) == 0)
        return fail(VQB_ERR_UNSUPPORTED, "gate_derivative: gate has no closed form");
    if (p < 0 || p >= g->np) return fail(VQB_ERR_DOMAIN, "gate_derivative: index out of range");
    if (!g->is_param[p]) return fail(VQB_ERR_DOMAIN, "gate_derivative: parameter is not variational");
    switch (g->kind) {
    case VQB_GATE_RX: case VQB_GATE_RY: case VQB_GATE_RZ:
        rotation_deriv(g->kind, g->params[0], out);
        return VQB_OK;
    case VQB_GATE_CRX: case VQB_GATE_CRY: case VQB_GATE_CRZ: {
        cd dr[4];
        rotation_deriv(g->kind, g->params[0], dr);
        memset(out, 0, sizeof(cd) * 16);
        out[1 + 4] = dr[0]; out[3 + 4] = dr[1]; out[1 + 12] = dr[2]; out[3 + 12] = dr[3];
        return VQB_OK;
    }
    default:
        fsim_deriv(g->params, p, out);
        return VQB_OK;
    }
}

/* gate_inverse gates.hpp:581-619: kind kept for self-inverse kinds and
 * parametric kinds (angles negated); everything else becomes the Generic
 * adjoint. */
static void gate_inverse(const gate_t *g, gate_t *inv) {
    const int d = 1 << g->m;
    inv->m = g->m;
    memcpy(inv->pos, g->pos, sizeof(int32_t) * g->m);
    inv->np = 0;
    switch (g->kind) {
    case VQB_GATE_X: case VQB_GATE_Y: case VQB_GATE_Z: case VQB_GATE_H: case VQB_GATE_SWAP:
    case VQB_GATE_CZ: case VQB_GATE_CNOT: case VQB_GATE_TOFFOLI: case VQB_GATE_FREDKIN:
        inv->kind = g->kind;
        memcpy(inv->mat, g->mat, sizeof(cd) * d * d);
        return;
    case VQB_GATE_RX: case VQB_GATE_RY: case VQB_GATE_RZ: case VQB_GATE_CRX: case VQB_GATE_CRY:
    case VQB_GATE_CRZ:
        inv->kind = g->kind;
        inv->np = 1;
        inv->params[0] = -g->params[0];
        inv->is_param[0] = 0;
        parametric_matrix(g->kind, inv->params, inv->mat);
        return;
    case VQB_GATE_FSIM:
        inv->kind = g->kind;
        inv->np = 5;
        for (int i = 0; i < 4; ++i) inv->params[i] = -g->params[i];
        inv->params[4] = g->params[4];
        for (int i = 0; i < 5; ++i) inv->is_param[i] = 0;
        parametric_matrix(g->kind, inv->params, inv->mat);
        return;
    default:
        inv->kind = VQB_GATE_GENERIC;
        for (int j = 0; j < d; ++j)
            for (int i = 0; i < d; ++i) inv->mat[j + i * d] = cconj(g->mat[i + j * d]);
        return;
    }
}

/* ---- channels: standard_channel gates.hpp:657-704, superop :708-732 ---- */
typedef struct {
    int kind, m, nk;
    int32_t pos[3];
    cd kraus[16 * 64];
} channel_t;

static int build_channel(const vqb_op *op, channel_t *c) {
    int rc = check_positions(op->positions, op->num_positions);
    if (rc) return rc;
    if (op->num_positions > 3) return fail(VQB_ERR_UNSUPPORTED, "channels act on at most 3 qubits");
    c->kind = op->kind;
    c->m = op->num_positions;
    memcpy(c->pos, op->positions, sizeof(int32_t) * c->m);
    const int d = 1 << c->m;
    if (op->kraus != NULL) {
        if (op->num_kraus < 1 || op->num_kraus * d * d > 16 * 64)
            return fail(VQB_ERR_SHAPE, "make_channel: bad Kraus operator count");
        c->nk = op->num_kraus;
        memcpy(c->kraus, op->kraus, sizeof(cd) * d * d * c->nk);
        /* completeness relation within 1e-8 (gates.hpp:631-648) */
        double mx = 0;
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) {
                cd s = C(0, 0);
                for (int k = 0; k < c->nk; ++k)
                    for (int r = 0; r < d; ++r)
                        s = cadd(s, cmul(cconj(c->kraus[k * d * d + r + i * d]),
                                         c->kraus[k * d * d + r + j * d]));
                if (i == j) s.re -= 1;
                if (cabs_(s) > mx) mx = cabs_(s);
            }
        if (mx > 1e-8)
            return fail(VQB_ERR_VALIDITY, "make_channel: Kraus operators violate the completeness relation within 1e-8");
        return VQB_OK;
    }
    const double p = op->params[0];
    if (c->m != 1) return fail(VQB_ERR_SHAPE, "named channels act on one qubit");
    if (p < 0 || p > 1) return fail(VQB_ERR_DOMAIN, "standard_channel: parameter must lie in [0,1]");
    cd *k = c->kraus;
    memset(k, 0, sizeof(cd) * 16);
    switch (c->kind) {
    case VQB_CHANNEL_AMPLITUDE_DAMPING:
        c->nk = 2;
        k[0] = C(1, 0); k[3] = C(sqrt(1 - p), 0);
        k[4 + 2] = C(sqrt(p), 0);
        return VQB_OK;
    case VQB_CHANNEL_PHASE_DAMPING:
        c->nk = 2;
        k[0] = C(1, 0); k[3] = C(sqrt(1 - p), 0);
        k[4 + 3] = C(sqrt(p), 0);
        return VQB_OK;
    case VQB_CHANNEL_DEPOLARIZING: {
        c->nk = 4;
        const double w0 = sqrt(1 - 0.75 * p), w = 0.5 * sqrt(p);
        k[0] = C(w0, 0); k[3] = C(w0, 0);
        cd px[4] = {C(0, 0), C(1, 0), C(1, 0), C(0, 0)};
        cd py[4] = {C(0, 0), C(0, 1), C(0, -1), C(0, 0)};
        cd pz[4] = {C(1, 0), C(0, 0), C(0, 0), C(-1, 0)};
        for (int i = 0; i < 4; ++i) {
            /* x *= w for a real w scales both components (gates.hpp:686-691) */
            k[4 + i] = C(px[i].re * w, px[i].im * w);
            k[8 + i] = C(py[i].re * w, py[i].im * w);
            k[12 + i] = C(pz[i].re * w, pz[i].im * w);
        }
        return VQB_OK;
    }
    default:
        return fail(VQB_ERR_UNSUPPORTED, "standard_channel: not a named channel kind");
    }
}

/* channel_superoperator gates.hpp:708-732 */
static void superop(const channel_t *c, cd *s) {
    const int d = 1 << c->m, dd = d * d;
    memset(s, 0, sizeof(cd) * dd * dd);
    for (int q = 0; q < c->nk; ++q) {
        const cd *k = c->kraus + q * dd;
        for (int tp = 0; tp < d; ++tp)
            for (int sp = 0; sp < d; ++sp) {
                const cd kc = cconj(k[tp + sp * d]);
                if (kc.re == 0 && kc.im == 0) continue;
                for (int sig = 0; sig < d; ++sig)
                    for (int tau = 0; tau < d; ++tau) {
                        cd *e = &s[(tau + tp * d) + (sig + sp * d) * dd];
                        *e = cadd(*e, cmul(k[tau + sig * d], kc));
                    }
            }
    }
}

/* linalg::kron(high, low) linalg.hpp:75-93 */
static void kron(const cd *hi, int dh, const cd *lo, int dl, cd *r) {
    const int d = dh * dl;
    for (int ch = 0; ch < dh; ++ch)
        for (int cl = 0; cl < dl; ++cl)
            for (int rh = 0; rh < dh; ++rh)
                for (int rl = 0; rl < dl; ++rl)
                    r[(rl + rh * dl) + (cl + ch * dl) * d] = cmul(hi[rh + ch * dh], lo[rl + cl * dl]);
}

static double norm1(const cd *a, int d) { /* linalg.hpp norm1 */
    double best = 0;
    for (int j = 0; j < d; ++j) {
        double col = 0;
        for (int i = 0; i < d; ++i) col += cabs_(a[i + j * d]);
        if (col > best) best = col;
    }
    return best;
}

/* lu_inverse linalg.hpp:140-200 (partial pivoting, one-norm condition). */
static int lu_inverse(const cd *a, int d, cd *inv, double *cond) {
    cd lu[64 * 64];
    int piv[64];
    memcpy(lu, a, sizeof(cd) * d * d);
    for (int i = 0; i < d; ++i) piv[i] = i;
    double scale = 0;
    for (int i = 0; i < d * d; ++i)
        if (cabs_(a[i]) > scale) scale = cabs_(a[i]);
    if (scale < 1e-300) scale = 1e-300;
    for (int k = 0; k < d; ++k) {
        int p = k;
        double best = cabs_(lu[k + k * d]);
        for (int i = k + 1; i < d; ++i) {
            const double v = cabs_(lu[i + k * d]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        if (best <= scale * 1e-300) return 1; /* singular */
        if (p != k) {
            const int t = piv[p];
            piv[p] = piv[k];
            piv[k] = t;
            for (int j = 0; j < d; ++j) {
                const cd x = lu[p + j * d];
                lu[p + j * d] = lu[k + j * d];
                lu[k + j * d] = x;
            }
        }
        const cd pivot = lu[k + k * d];
        for (int i = k + 1; i < d; ++i) {
            const cd f = cdiv(lu[i + k * d], pivot);
            lu[i + k * d] = f;
            for (int j = k + 1; j < d; ++j) lu[i + j * d] = csub(lu[i + j * d], cmul(f, lu[k + j * d]));
        }
    }
    cd x[64];
    for (int col = 0; col < d; ++col) {
        for (int i = 0; i < d; ++i) x[i] = (piv[i] == col) ? C(1, 0) : C(0, 0);
        for (int i = 1; i < d; ++i)
            for (int j = 0; j < i; ++j) x[i] = csub(x[i], cmul(lu[i + j * d], x[j]));
        for (int ii = d; ii-- > 0;) {
            for (int j = ii + 1; j < d; ++j) x[ii] = csub(x[ii], cmul(lu[ii + j * d], x[j]));
            x[ii] = cdiv(x[ii], lu[ii + ii * d]);
        }
        for (int i = 0; i < d; ++i) inv[i + col * d] = x[i];
    }
    *cond = norm1(a, d) * norm1(inv, d);
    return 0;
}

/* ================= state: state.hpp ================= */
typedef struct {
    int n;      /* qubits (pure) or physical qubits (mixed) */
    int mixed;
    int pn;     /* pseudo qubits: n or 2n */
    uint64_t size;
    cd *a;
} ostate;

/* AllocStats state.hpp:56-83,154-161: live/peak full-state buffers */
static int64_t g_live, g_peak;
ORC_API int vqcsorc_alloc_stats(int64_t *live, int64_t *peak, uint64_t *live_bytes, uint64_t *peak_bytes) {
    if (live) *live = g_live;
    if (peak) *peak = g_peak;
    if (live_bytes) *live_bytes = 0;
    if (peak_bytes) *peak_bytes = 0;
    return VQB_OK;
}
ORC_API int vqcsorc_reset_alloc_peak(void) {
    g_peak = g_live;
    return VQB_OK;
}
ORC_API int vqcsorc_release_caches(void) { return VQB_OK; }

ORC_API int vqcsorc_state_create(int32_t n, int32_t mixed, ostate **out) {
    const int maxq = mixed ? 20 : 40; /* state.hpp:179,261 */
    if (n < 1) return fail(VQB_ERR_SIZE, "qubit count must be >= 1");
    if (n > maxq) return fail(VQB_ERR_SIZE, "qubit count exceeds the supported maximum");
    ostate *s = (ostate *)calloc(1, sizeof(ostate));
    s->n = n;
    s->mixed = mixed != 0;
    s->pn = mixed ? 2 * n : n;
    s->size = (uint64_t)1 << s->pn;
    s->a = (cd *)calloc(s->size, sizeof(cd));
    if (!s->a) {
        free(s);
        return fail(VQB_ERR_SIZE, "cannot allocate state");
    }
    s->a[0] = C(1, 0);
    if (++g_live > g_peak) g_peak = g_live;
    *out = s;
    return VQB_OK;
}

ORC_API int vqcsorc_state_destroy(ostate *s) {
    if (s) {
        --g_live;
        free(s->a);
        free(s);
    }
    return VQB_OK;
}

ORC_API int vqcsorc_state_info(const ostate *s, int32_t *n, int32_t *mixed, uint64_t *count) {
    if (n) *n = s->n;
    if (mixed) *mixed = s->mixed;
    if (count) *count = s->size;
    return VQB_OK;
}

ORC_API int vqcsorc_state_upload(ostate *s, const cd *h, uint64_t count) {
    if (count != s->size) return fail(VQB_ERR_SHAPE, "state_upload: count mismatch");
    memcpy(s->a, h, sizeof(cd) * count);
    return VQB_OK;
}

ORC_API int vqcsorc_state_download(const ostate *s, cd *h, uint64_t count) {
    if (count != s->size) return fail(VQB_ERR_SHAPE, "state_download: count mismatch");
    memcpy(h, s->a, sizeof(cd) * count);
    return VQB_OK;
}

ORC_API int vqcsorc_state_download_range(const ostate *s, uint64_t offset, uint64_t count, cd *h) {
    if (offset > s->size || count > s->size - offset)
        return fail(VQB_ERR_INDEX, "state_download_range: range exceeds the state");
    memcpy(h, s->a + offset, sizeof(cd) * count);
    return VQB_OK;
}

ORC_API int vqcsorc_state_set_zero(ostate *s) {
    memset(s->a, 0, sizeof(cd) * s->size);
    s->a[0].re = 1.0;
    return VQB_OK;
}

ORC_API int vqcsorc_state_copy(ostate *dst, const ostate *src) {
    if (dst->size != src->size) return fail(VQB_ERR_SHAPE, "state_copy: shape mismatch");
    memcpy(dst->a, src->a, sizeof(cd) * src->size);
    return VQB_OK;
}

/* ================= kernels: kernels.hpp ================= */

/* check_targets_fit kernels.hpp:71-87 */
static int check_fit(const int32_t *pos, int m, int n) {
    for (int i = 0; i < m; ++i)
        if (pos[i] < 1 || pos[i] > n) return fail(VQB_ERR_INDEX, "gate position does not fit the state");
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            if (pos[i] == pos[j]) return fail(VQB_ERR_VALIDITY, "duplicate gate position");
    return VQB_OK;
}

/* expand_index kernels.hpp:116-122 over ascending strides */
static inline uint64_t expand(uint64_t c, const uint64_t *strides, int m) {
    for (int i = 0; i < m; ++i) {
        const uint64_t s = strides[i];
        c = ((c & ~(s - 1)) << 1) | (c & (s - 1));
    }
    return c;
}

static void sorted_strides(const int32_t *pos, int m, uint64_t *s) {
    for (int i = 0; i < m; ++i) s[i] = (uint64_t)1 << (pos[i] - 1);
    for (int i = 1; i < m; ++i)
        for (int j = i; j > 0 && s[j - 1] > s[j]; --j) {
            const uint64_t t = s[j];
            s[j] = s[j - 1];
            s[j - 1] = t;
        }
}

/* group_offsets kernels.hpp:101-113 */
static void group_offsets(const int32_t *pos, int m, uint64_t *off) {
    for (int r = 0; r < (1 << m); ++r) {
        off[r] = 0;
        for (int k = 0; k < m; ++k)
            if ((r >> k) & 1) off[r] += (uint64_t)1 << (pos[k] - 1);
    }
}

/* apply_dense_range kernels.hpp:180-202 (also the 1q/2q aggregated kernels:
 * they evaluate the same products in the same order). */
static void apply_dense(cd *a, int n, const int32_t *pos, int m, const cd *mat) {
    const int d = 1 << m;
    uint64_t off[64], st[VQB_MAX_POSITIONS];
    cd in[64], out[64];
    group_offsets(pos, m, off);
    sorted_strides(pos, m, st);
    const uint64_t bases = (uint64_t)1 << (n - m);
    for (uint64_t c = 0; c < bases; ++c) {
        const uint64_t b = expand(c, st, m);
        for (int r = 0; r < d; ++r) in[r] = a[b + off[r]];
        for (int r = 0; r < d; ++r) {
            cd acc = cmul(mat[r], in[0]);
            for (int s = 1; s < d; ++s) acc = cadd(acc, cmul(mat[r + s * d], in[s]));
            out[r] = acc;
        }
        for (int r = 0; r < d; ++r) a[b + off[r]] = out[r];
    }
}

/* swap_pairs_range kernels.hpp:291-299 */
static void swap_pairs(cd *a, int n, const int32_t *pos, int m, uint64_t base_add, uint64_t delta) {
    uint64_t st[VQB_MAX_POSITIONS];
    sorted_strides(pos, m, st);
    const uint64_t bases = (uint64_t)1 << (n - m);
    for (uint64_t c = 0; c < bases; ++c) {
        const uint64_t i = expand(c, st, m) + base_add;
        const cd t = a[i];
        a[i] = a[i + delta];
        a[i + delta] = t;
    }
}

/* phase_range kernels.hpp:301-308 */
static void phase(cd *a, int n, const int32_t *pos, int m, cd ph, uint64_t base_add) {
    uint64_t st[VQB_MAX_POSITIONS];
    sorted_strides(pos, m, st);
    const uint64_t bases = (uint64_t)1 << (n - m);
    for (uint64_t c = 0; c < bases; ++c) {
        const uint64_t i = expand(c, st, m) + base_add;
        a[i] = cmul(a[i], ph);
    }
}

/* apply_gate_fast kernels.hpp:365-430 */
static int apply_gate_fast(cd *a, int n, const gate_t *g) {
    int rc = check_fit(g->pos, g->m, n);
    if (rc) return rc;
    if (((uint64_t)1 << (n - g->m)) < 8) { /* bases < kAggregationBatch -> naive */
        apply_dense(a, n, g->pos, g->m, g->mat);
        return VQB_OK;
    }
    uint64_t off[64];
    group_offsets(g->pos, g->m, off);
    const double isq = 0.70710678118654752440;
    switch (g->kind) {
    case VQB_GATE_X: swap_pairs(a, n, g->pos, 1, 0, off[1]); return VQB_OK;
    case VQB_GATE_Z: phase(a, n, g->pos, 1, C(-1, 0), off[1]); return VQB_OK;
    case VQB_GATE_S: phase(a, n, g->pos, 1, C(0, 1), off[1]); return VQB_OK;
    case VQB_GATE_T: phase(a, n, g->pos, 1, C(isq, isq), off[1]); return VQB_OK;
    case VQB_GATE_CZ: phase(a, n, g->pos, 2, C(-1, 0), off[3]); return VQB_OK;
    case VQB_GATE_CNOT: swap_pairs(a, n, g->pos, 2, off[1], off[2]); return VQB_OK;
    case VQB_GATE_SWAP: {
        const uint64_t lo = off[1] < off[2] ? off[1] : off[2];
        const uint64_t hi = off[1] < off[2] ? off[2] : off[1];
        swap_pairs(a, n, g->pos, 2, lo, hi - lo);
        return VQB_OK;
    }
    default:
        apply_dense(a, n, g->pos, g->m, g->mat);
        return VQB_OK;
    }
}

static int mat_equal(const cd *a, const cd *b, int count) {
    for (int i = 0; i < count; ++i)
        if (a[i].re != b[i].re || a[i].im != b[i].im) return 0;
    return 1;
}

/* Both sides of a unitary on vec(rho): ket pass, then conj on +n with the
 * same kind when conj(U) == U (apply_gate_mixed kernels.hpp:434-449 and
 * autodiff.hpp:214-226). */
static int apply_both_sides(ostate *s, const gate_t *g) {
    int rc = apply_gate_fast(s->a, s->pn, g);
    if (rc) return rc;
    static _Thread_local gate_t bra;
    const int d = 1 << g->m;
    bra.m = g->m;
    bra.np = 0;
    for (int i = 0; i < g->m; ++i) bra.pos[i] = g->pos[i] + s->n;
    for (int i = 0; i < d * d; ++i) bra.mat[i] = cconj(g->mat[i]);
    bra.kind = mat_equal(bra.mat, g->mat, d * d) ? g->kind : VQB_GATE_GENERIC;
    return apply_gate_fast(s->a, s->pn, &bra);
}

ORC_API int vqcsorc_apply_gate(ostate *s, const vqb_op *op) {
    static _Thread_local gate_t g;
    int rc = build_gate(op, &g);
    if (rc) return rc;
    if (s->mixed) {
        rc = check_fit(g.pos, g.m, s->n);
        if (rc) return rc;
        return apply_both_sides(s, &g);
    }
    return apply_gate_fast(s->a, s->n, &g);
}

ORC_API int vqcsorc_apply_matrix(ostate *s, const int32_t *pos, int32_t m, const cd *mat) {
    int rc = check_fit(pos, m, s->pn);
    if (rc) return rc;
    apply_dense(s->a, s->pn, pos, m, mat);
    return VQB_OK;
}

static void bound_positions(const channel_t *c, int n, int32_t *pos) {
    for (int i = 0; i < c->m; ++i) {
        pos[i] = c->pos[i];
        pos[i + c->m] = c->pos[i] + n;
    }
}

/* apply_channel kernels.hpp:453-461 */
static int apply_channel(ostate *s, const channel_t *c) {
    int rc = check_fit(c->pos, c->m, s->n);
    if (rc) return rc;
    static _Thread_local cd sop[64 * 64];
    int32_t pos[6];
    superop(c, sop);
    bound_positions(c, s->n, pos);
    apply_dense(s->a, s->pn, pos, 2 * c->m, sop);
    return VQB_OK;
}

ORC_API int vqcsorc_apply_channel(ostate *s, const vqb_op *op) {
    if (!s->mixed) return fail(VQB_ERR_TYPE, "apply_channel: a quantum channel cannot act on a pure state");
    static _Thread_local channel_t c;
    int rc = build_channel(op, &c);
    if (rc) return rc;
    return apply_channel(s, &c);
}

/* apply_circuit circuit.hpp:110-129 */
ORC_API int vqcsorc_apply_circuit(ostate *s, const vqb_op *ops, int64_t count) {
    for (int64_t i = 0; i < count; ++i) {
        int rc;
        if (ops[i].elem == VQB_ELEM_CHANNEL) {
            if (!s->mixed)
                return fail(VQB_ERR_TYPE, "apply_circuit: a quantum channel cannot act on a pure state; use a MixedState");
            rc = vqcsorc_apply_channel(s, &ops[i]);
        } else {
            rc = vqcsorc_apply_gate(s, &ops[i]);
        }
        if (rc) return rc;
    }
    return VQB_OK;
}

/* ================= reductions: state.hpp, observables.hpp ================= */
ORC_API int vqcsorc_norm(const ostate *s, double *out) { /* state.hpp:236-242 */
    if (s->mixed) return fail(VQB_ERR_TYPE, "norm: pure states only");
    double sq = 0;
    for (uint64_t k = 0; k < s->size; ++k) sq += s->a[k].re * s->a[k].re + s->a[k].im * s->a[k].im;
    *out = sqrt(sq);
    return VQB_OK;
}

ORC_API int vqcsorc_trace(const ostate *s, cd *out) { /* state.hpp:329-336 */
    if (!s->mixed) return fail(VQB_ERR_TYPE, "trace: mixed states only");
    const uint64_t dim = (uint64_t)1 << s->n;
    cd t = C(0, 0);
    for (uint64_t k = 0; k < dim; ++k) t = cadd(t, s->a[k + k * dim]);
    *out = t;
    return VQB_OK;
}

static int check_terms(const vqb_pauli_term *t, int64_t nt, int n) {
    for (int64_t i = 0; i < nt; ++i)
        for (int k = 0; k < t[i].num_factors; ++k) {
            const char l = t[i].labels[k] | 0x20;
            if (l != 'x' && l != 'y' && l != 'z') return fail(VQB_ERR_VALIDITY, "unknown Pauli label");
            if (t[i].qubits[k] < 1) return fail(VQB_ERR_VALIDITY, "PauliTerm: qubit indices must be >= 1");
            for (int j = k + 1; j < t[i].num_factors; ++j)
                if (t[i].qubits[k] == t[i].qubits[j]) return fail(VQB_ERR_VALIDITY, "PauliTerm: duplicate qubit index");
            if (t[i].qubits[k] > n) return fail(VQB_ERR_INDEX, "operator acts on a qubit beyond the state");
        }
    return VQB_OK;
}

/* apply_term_factors observables.hpp:155-162: X/Y/Z gates, one per factor. */
static void apply_term(cd *a, int pn, const vqb_pauli_term *t, int shift) {
    static _Thread_local gate_t g;
    for (int k = 0; k < t->num_factors; ++k) {
        const char l = t->labels[k] | 0x20;
        g.kind = l == 'x' ? VQB_GATE_X : (l == 'y' ? VQB_GATE_Y : VQB_GATE_Z);
        g.m = 1;
        g.np = 0;
        g.pos[0] = t->qubits[k] + shift;
        fixed_matrix(g.kind, g.mat);
        apply_gate_fast(a, pn, &g);
    }
}

static cd dot(const cd *a, const cd *b, uint64_t size) { /* observables.hpp:164-171 */
    cd acc = C(0, 0);
    for (uint64_t k = 0; k < size; ++k) acc = cadd(acc, cmul(cconj(a[k]), b[k]));
    return acc;
}

/* expectation observables.hpp:176-213 */
ORC_API int vqcsorc_expectation(const ostate *s, const vqb_pauli_term *t, int64_t nt, cd *out) {
    int rc = check_terms(t, nt, s->n);
    if (rc) return rc;
    cd *scratch = (cd *)malloc(sizeof(cd) * s->size);
    cd acc = C(0, 0);
    const uint64_t dim = (uint64_t)1 << s->n;
    for (int64_t i = 0; i < nt; ++i) {
        memcpy(scratch, s->a, sizeof(cd) * s->size);
        apply_term(scratch, s->pn, &t[i], 0);
        cd v;
        if (s->mixed) {
            v = C(0, 0);
            for (uint64_t k = 0; k < dim; ++k) v = cadd(v, scratch[k + k * dim]);
        } else {
            v = dot(s->a, scratch, s->size);
        }
        acc = cadd(acc, cmul(t[i].coeff, v));
    }
    free(scratch);
    *out = acc;
    return VQB_OK;
}

/* apply_operator observables.hpp:216-237 (pure) */
static void apply_operator_raw(const cd *src, cd *dst, int pn, uint64_t size, const vqb_pauli_term *t,
                               int64_t nt) {
    cd *scratch = (cd *)malloc(sizeof(cd) * size);
    memset(dst, 0, sizeof(cd) * size);
    for (int64_t i = 0; i < nt; ++i) {
        memcpy(scratch, src, sizeof(cd) * size);
        apply_term(scratch, pn, &t[i], 0);
        for (uint64_t k = 0; k < size; ++k) dst[k] = cadd(dst[k], cmul(t[i].coeff, scratch[k]));
    }
    free(scratch);
}

ORC_API int vqcsorc_apply_operator(const ostate *src, ostate *dst, const vqb_pauli_term *t, int64_t nt) {
    if (src->mixed || dst->mixed) return fail(VQB_ERR_TYPE, "apply_operator: pure states only");
    if (src->size != dst->size) return fail(VQB_ERR_SHAPE, "apply_operator: shape mismatch");
    int rc = check_terms(t, nt, src->n);
    if (rc) return rc;
    apply_operator_raw(src->a, dst->a, src->pn, src->size, t, nt);
    return VQB_OK;
}

/* bilinear_gate_form kernels.hpp:466-503 */
ORC_API int vqcsorc_bilinear_form(const ostate *bra, const ostate *ket, const int32_t *pos, int32_t m,
                                  const cd *local, cd *out) {
    int rc = check_fit(pos, m, ket->pn);
    if (rc) return rc;
    const int d = 1 << m;
    uint64_t off[64], st[VQB_MAX_POSITIONS];
    cd in[64];
    group_offsets(pos, m, off);
    sorted_strides(pos, m, st);
    cd acc = C(0, 0);
    const uint64_t bases = (uint64_t)1 << (ket->pn - m);
    for (uint64_t c = 0; c < bases; ++c) {
        const uint64_t b = expand(c, st, m);
        for (int r = 0; r < d; ++r) in[r] = ket->a[b + off[r]];
        for (int r = 0; r < d; ++r) {
            cd w = cmul(local[r], in[0]);
            for (int s = 1; s < d; ++s) w = cadd(w, cmul(local[r + s * d], in[s]));
            acc = cadd(acc, cmul(cconj(bra->a[b + off[r]]), w));
        }
    }
    *out = acc;
    return VQB_OK;
}

/* reverse_sweep_step kernels.hpp:659-697 (generic/dense form :609-652; the
 * 1q and 2q specialisations evaluate the same expressions). */
static void reverse_step_raw(cd *fp, cd *sp, int n, const int32_t *pos, int m, const cd *iv,
                             const cd *dmats, int np, cd *acc) {
    const int d = 1 << m;
    uint64_t off[64], st[VQB_MAX_POSITIONS];
    cd f[64], g[64], w[64];
    group_offsets(pos, m, off);
    sorted_strides(pos, m, st);
    for (int p = 0; p < np; ++p) acc[p] = C(0, 0);
    const uint64_t bases = (uint64_t)1 << (n - m);
    for (uint64_t c = 0; c < bases; ++c) {
        const uint64_t b = expand(c, st, m);
        for (int r = 0; r < d; ++r) {
            f[r] = fp[b + off[r]];
            g[r] = sp[b + off[r]];
        }
        for (int r = 0; r < d; ++r) {
            cd v = cmul(iv[r], f[0]);
            for (int s = 1; s < d; ++s) v = cadd(v, cmul(iv[r + s * d], f[s]));
            w[r] = v;
            fp[b + off[r]] = v;
        }
        for (int p = 0; p < np; ++p) {
            const cd *dm = dmats + p * d * d;
            cd a = C(0, 0);
            for (int r = 0; r < d; ++r) {
                cd v = cmul(dm[r], w[0]);
                for (int s = 1; s < d; ++s) v = cadd(v, cmul(dm[r + s * d], w[s]));
                a = cadd(a, cmul(cconj(g[r]), v));
            }
            acc[p] = cadd(acc[p], a);
        }
        for (int r = 0; r < d; ++r) {
            cd v = cmul(iv[r], g[0]);
            for (int s = 1; s < d; ++s) v = cadd(v, cmul(iv[r + s * d], g[s]));
            sp[b + off[r]] = v;
        }
    }
}

ORC_API int vqcsorc_reverse_step(ostate *phi, ostate *psi, const int32_t *pos, int32_t m, const cd *inv,
                                 const cd *dmats, int32_t np, cd *out) {
    int rc = check_fit(pos, m, phi->pn);
    if (rc) return rc;
    reverse_step_raw(phi->a, psi->a, phi->pn, pos, m, inv, dmats, np, out);
    return VQB_OK;
}

/* ================= autodiff.hpp ================= */

typedef struct {
    int64_t count;
    gate_t *gates;      /* gate elements (NULL slot for channels) */
    channel_t *chans;   /* channel elements */
    int *is_channel;
} elems_t;

static int build_elems(const vqb_op *ops, int64_t count, elems_t *e) {
    e->count = count;
    e->gates = (gate_t *)calloc(count > 0 ? count : 1, sizeof(gate_t));
    e->chans = (channel_t *)calloc(count > 0 ? count : 1, sizeof(channel_t));
    e->is_channel = (int *)calloc(count > 0 ? count : 1, sizeof(int));
    for (int64_t i = 0; i < count; ++i) {
        int rc;
        if (ops[i].elem == VQB_ELEM_CHANNEL) {
            e->is_channel[i] = 1;
            rc = build_channel(&ops[i], &e->chans[i]);
        } else {
            rc = build_gate(&ops[i], &e->gates[i]);
        }
        if (rc) return rc;
    }
    return VQB_OK;
}

static void free_elems(elems_t *e) {
    free(e->gates);
    free(e->chans);
    free(e->is_channel);
}

static double max_abs_diff(const cd *a, const cd *b, uint64_t size) {
    double m = 0;
    for (uint64_t k = 0; k < size; ++k) {
        const double v = cabs_(csub(a[k], b[k]));
        if (v > m) m = v;
    }
    return m;
}

/* loss_pure autodiff.hpp:80-89 */
ORC_API int vqcsorc_loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *t, int64_t nt,
                              const ostate *s0, double *loss) {
    if (s0->mixed) return fail(VQB_ERR_TYPE, "loss_pure: pure initial state required");
    for (int64_t i = 0; i < count; ++i)
        if (ops[i].elem == VQB_ELEM_CHANNEL) return fail(VQB_ERR_TYPE, "loss_pure: circuit contains quantum channels");
    ostate *s;
    int rc = vqcsorc_state_create(s0->n, 0, &s);
    if (rc) return rc;
    vqcsorc_state_copy(s, s0);
    rc = vqcsorc_apply_circuit(s, ops, count);
    cd e = C(0, 0);
    if (!rc) rc = vqcsorc_expectation(s, t, nt, &e);
    vqcsorc_state_destroy(s);
    *loss = e.re;
    return rc;
}

/* gradient_pure autodiff.hpp:95-156 */
ORC_API int vqcsorc_gradient_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *t, int64_t nt,
                                  const ostate *s0, double *loss, double *grads, int64_t capacity,
                                  int64_t *num_grads, double *residual) {
    if (s0->mixed) return fail(VQB_ERR_TYPE, "gradient_pure: pure initial state required");
    for (int64_t i = 0; i < count; ++i)
        if (ops[i].elem == VQB_ELEM_CHANNEL)
            return fail(VQB_ERR_TYPE, "gradient_pure: circuit contains quantum channels; use the mixed-state variant");
    const int n = s0->n;
    int rc = check_terms(t, nt, n);
    if (rc) return rc;
    elems_t e;
    rc = build_elems(ops, count, &e);
    if (rc) {
        free_elems(&e);
        return rc;
    }
    int64_t *base = (int64_t *)calloc(count > 0 ? count : 1, sizeof(int64_t));
    int64_t total = 0;
    for (int64_t i = 0; i < count; ++i) {
        base[i] = total;
        for (int p = 0; p < e.gates[i].np; ++p) total += e.gates[i].is_param[p] ? 1 : 0;
    }
    if (total > capacity) {
        free(base);
        free_elems(&e);
        return fail(VQB_ERR_SHAPE, "gradient_pure: gradient buffer too small");
    }
    cd *phi = (cd *)malloc(sizeof(cd) * s0->size);
    memcpy(phi, s0->a, sizeof(cd) * s0->size);
    for (int64_t i = 0; i < count && !rc; ++i) rc = apply_gate_fast(phi, n, &e.gates[i]);
    *num_grads = total;
    if (!rc && total == 0) {
        ostate tmp = *s0;
        tmp.a = phi;
        cd ex;
        rc = vqcsorc_expectation(&tmp, t, nt, &ex);
        *loss = ex.re;
        if (residual) *residual = 0;
    } else if (!rc) {
        cd *psi = (cd *)malloc(sizeof(cd) * s0->size);
        apply_operator_raw(phi, psi, n, s0->size, t, nt);
        *loss = dot(phi, psi, s0->size).re;
        for (int64_t k = 0; k < total; ++k) grads[k] = 0;
        static _Thread_local gate_t inv;
        cd dmats[5 * 64], acc[5];
        for (int64_t i = count; i-- > 0 && !rc;) {
            const gate_t *g = &e.gates[i];
            gate_inverse(g, &inv);
            if (!has_active(g)) {
                rc = apply_gate_fast(phi, n, &inv);
                if (!rc) rc = apply_gate_fast(psi, n, &inv);
                continue;
            }
            const int dd = (1 << g->m) * (1 << g->m);
            int np = 0;
            for (int p = 0; p < g->np; ++p)
                if (g->is_param[p]) gate_derivative(g, p, dmats + (np++) * dd);
            rc = check_fit(g->pos, g->m, n);
            if (rc) break;
            reverse_step_raw(phi, psi, n, g->pos, g->m, inv.mat, dmats, np, acc);
            for (int k = 0; k < np; ++k) grads[base[i] + k] = 2.0 * acc[k].re;
        }
        if (residual) *residual = max_abs_diff(phi, s0->a, s0->size);
        free(psi);
    }
    free(phi);
    free(base);
    free_elems(&e);
    return rc;
}

/* loss_mixed autodiff.hpp:160-167 */
ORC_API int vqcsorc_loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *t, int64_t nt,
                               const ostate *dm0, double *loss) {
    if (!dm0->mixed) return fail(VQB_ERR_TYPE, "loss_mixed: mixed initial state required");
    int rc = check_terms(t, nt, dm0->n);
    if (rc) return rc;
    ostate *s;
    rc = vqcsorc_state_create(dm0->n, 1, &s);
    if (rc) return rc;
    vqcsorc_state_copy(s, dm0);
    rc = vqcsorc_apply_circuit(s, ops, count);
    cd e = C(0, 0);
    if (!rc) rc = vqcsorc_expectation(s, t, nt, &e);
    vqcsorc_state_destroy(s);
    *loss = e.re;
    return rc;
}

/* gradient_mixed autodiff.hpp:184-329 */
ORC_API int vqcsorc_gradient_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *t, int64_t nt,
                                   const ostate *dm0, double *loss, double *grads, int64_t capacity,
                                   int64_t *num_grads, double *residual) {
    if (!dm0->mixed) return fail(VQB_ERR_TYPE, "gradient_mixed: mixed initial state required");
    const int n = dm0->n, big = 2 * n;
    int rc = check_terms(t, nt, n);
    if (rc) return rc;
    elems_t e;
    rc = build_elems(ops, count, &e);
    if (rc) {
        free_elems(&e);
        return rc;
    }
    int64_t *base = (int64_t *)calloc(count > 0 ? count : 1, sizeof(int64_t));
    int64_t total = 0;
    for (int64_t i = 0; i < count; ++i) {
        base[i] = total;
        if (!e.is_channel[i])
            for (int p = 0; p < e.gates[i].np; ++p) total += e.gates[i].is_param[p] ? 1 : 0;
    }
    if (total > capacity) {
        free(base);
        free_elems(&e);
        return fail(VQB_ERR_SHAPE, "gradient_mixed: gradient buffer too small");
    }
    *num_grads = total;
    ostate phi = *dm0, psi = *dm0;
    phi.a = (cd *)malloc(sizeof(cd) * dm0->size);
    psi.a = (cd *)calloc(dm0->size, sizeof(cd));
    memcpy(phi.a, dm0->a, sizeof(cd) * dm0->size);
    /* forward */
    for (int64_t i = 0; i < count && !rc; ++i) {
        if (e.is_channel[i]) {
            rc = apply_channel(&phi, &e.chans[i]);
        } else {
            rc = check_fit(e.gates[i].pos, e.gates[i].m, n);
            if (!rc) rc = apply_both_sides(&phi, &e.gates[i]);
        }
    }
    /* <<Psi| = <<I| H: apply the conjugated operator to |I>> (autodiff.hpp:241-248) */
    if (!rc) {
        const uint64_t dim = (uint64_t)1 << n;
        cd *ident = (cd *)calloc(dm0->size, sizeof(cd));
        for (uint64_t k = 0; k < dim; ++k) ident[k + k * dim] = C(1, 0);
        vqb_pauli_term *tc = (vqb_pauli_term *)malloc(sizeof(vqb_pauli_term) * (nt > 0 ? nt : 1));
        for (int64_t i = 0; i < nt; ++i) {
            tc[i] = t[i];
            tc[i].coeff = cconj(t[i].coeff);
        }
        apply_operator_raw(ident, psi.a, big, dm0->size, tc, nt);
        free(tc);
        free(ident);
        *loss = dot(psi.a, phi.a, dm0->size).re;
        for (int64_t k = 0; k < total; ++k) grads[k] = 0;
    }
    static _Thread_local gate_t inv, tmpg;
    static _Thread_local cd sop[64 * 64], sinv[64 * 64], sadj[64 * 64];
    cd dmats[5 * 256], acc[5];
    for (int64_t i = count; total > 0 && i-- > 0 && !rc;) {
        if (e.is_channel[i]) {
            const channel_t *ch = &e.chans[i];
            const int d = 1 << (2 * ch->m);
            double cond = 0;
            superop(ch, sop);
            if (lu_inverse(sop, d, sinv, &cond) || cond > 1e12) {
                static const char *names[] = {"Generic", "AmplitudeDamping", "PhaseDamping", "Depolarizing"};
                char msg[256];
                snprintf(msg, sizeof msg,
                         "gradient_mixed: the superoperator of channel '%s' on qubit %d (element %lld) is singular or too ill-conditioned to invert",
                         names[ch->kind & 3], ch->pos[0], (long long)(i + 1));
                rc = fail(VQB_ERR_NONINVERTIBLE, msg);
                break;
            }
            for (int a = 0; a < d; ++a)
                for (int b = 0; b < d; ++b) sadj[b + a * d] = cconj(sop[a + b * d]);
            int32_t pos[6];
            bound_positions(ch, n, pos);
            apply_dense(phi.a, big, pos, 2 * ch->m, sinv);
            apply_dense(psi.a, big, pos, 2 * ch->m, sadj);
            continue;
        }
        const gate_t *g = &e.gates[i];
        gate_inverse(g, &inv);
        const int d = 1 << g->m;
        if (!has_active(g)) {
            rc = apply_both_sides(&phi, &inv);
            if (!rc) rc = apply_both_sides(&psi, &inv);
            continue;
        }
        /* inv_local = kron(conj(inv), inv); dS = dU (x) conj U + U (x) conj dU */
        static _Thread_local cd inv_bra[64], inv_local[256], du[64], conj_u[64], conj_du[64], second[256];
        for (int k = 0; k < d * d; ++k) inv_bra[k] = cconj(inv.mat[k]);
        kron(inv_bra, d, inv.mat, d, inv_local);
        for (int k = 0; k < d * d; ++k) conj_u[k] = cconj(g->mat[k]);
        int np = 0;
        for (int p = 0; p < g->np; ++p) {
            if (!g->is_param[p]) continue;
            gate_derivative(g, p, du);
            for (int k = 0; k < d * d; ++k) conj_du[k] = cconj(du[k]);
            cd *ds = dmats + np * d * d * d * d;
            kron(conj_u, d, du, d, ds);
            kron(conj_du, d, g->mat, d, second);
            for (int k = 0; k < d * d * d * d; ++k) ds[k] = cadd(ds[k], second[k]);
            ++np;
        }
        int32_t pos[6];
        for (int k = 0; k < g->m; ++k) {
            pos[k] = g->pos[k];
            pos[k + g->m] = g->pos[k] + n;
        }
        rc = check_fit(pos, 2 * g->m, big);
        if (rc) break;
        reverse_step_raw(phi.a, psi.a, big, pos, 2 * g->m, inv_local, dmats, np, acc);
        for (int k = 0; k < np; ++k) grads[base[i] + k] = acc[k].re;
    }
    (void)tmpg;
    if (!rc && residual) *residual = total > 0 ? max_abs_diff(phi.a, dm0->a, dm0->size) : 0;
    free(phi.a);
    free(psi.a);
    free(base);
    free_elems(&e);
    return rc;
}

/* ================= gate algebra exports ================= */
ORC_API int vqcsorc_gate_matrix(const vqb_op *op, cd *out) {
    static _Thread_local gate_t g;
    int rc = build_gate(op, &g);
    if (rc) return rc;
    memcpy(out, g.mat, sizeof(cd) << (2 * g.m));
    return VQB_OK;
}

ORC_API int vqcsorc_gate_derivative(const vqb_op *op, int32_t p, cd *out) {
    static _Thread_local gate_t g;
    int rc = build_gate(op, &g);
    if (rc) return rc;
    return gate_derivative(&g, p, out);
}

ORC_API int vqcsorc_gate_inverse(const vqb_op *op, cd *out) {
    static _Thread_local gate_t g, inv;
    int rc = build_gate(op, &g);
    if (rc) return rc;
    gate_inverse(&g, &inv);
    memcpy(out, inv.mat, sizeof(cd) << (2 * g.m));
    return VQB_OK;
}

ORC_API int vqcsorc_channel_superop(const vqb_op *op, cd *out) {
    static _Thread_local channel_t c;
    int rc = build_channel(op, &c);
    if (rc) return rc;
    superop(&c, out);
    return VQB_OK;
}

/* ================= measurement: circuit.hpp:278-375 ================= */
static double clamp_probability(double p) { return p < 0 ? 0.0 : (p > 1 ? 1.0 : p); } /* :283-285 */

static int check_measure_qubit(const ostate *s, int32_t q) {
    if (q < 1 || q > s->n) return fail(VQB_ERR_INDEX, "measure: qubit does not fit the state");
    return VQB_OK;
}

/* p1 loop of measure (circuit.hpp:311-317 pure, :346-352 mixed) */
ORC_API int vqcsorc_measure_probability(const ostate *s, int32_t q, double *p1) {
    int rc = check_measure_qubit(s, q);
    if (rc) return rc;
    const uint64_t mask = (uint64_t)1 << (q - 1);
    double p = 0;
    if (!s->mixed) {
        for (uint64_t k = 0; k < s->size; ++k)
            if (k & mask) p += s->a[k].re * s->a[k].re + s->a[k].im * s->a[k].im; /* std::norm */
    } else {
        const uint64_t dim = (uint64_t)1 << s->n;
        for (uint64_t k = 0; k < dim; ++k)
            if (k & mask) p += s->a[k + k * dim].re;
    }
    *p1 = p;
    return VQB_OK;
}

/* collapse loops (circuit.hpp:328-335 pure, :363-373 mixed) */
ORC_API int vqcsorc_collapse(ostate *s, int32_t q, int32_t outcome, double p) {
    int rc = check_measure_qubit(s, q);
    if (rc) return rc;
    if (outcome != 0 && outcome != 1) return fail(VQB_ERR_DOMAIN, "collapse: outcome must be 0 or 1");
    if (!(p > 0)) return fail(VQB_ERR_DEGENERATE, "collapse: outcome probability must be > 0");
    const uint64_t mask = (uint64_t)1 << (q - 1);
    if (!s->mixed) {
        const double scale = 1.0 / sqrt(p);
        for (uint64_t k = 0; k < s->size; ++k) {
            if (((k & mask) != 0) == (outcome == 1)) s->a[k] = C(s->a[k].re * scale, s->a[k].im * scale);
            else s->a[k] = C(0, 0);
        }
    } else {
        const double scale = 1.0 / p;
        const uint64_t dim = (uint64_t)1 << s->n;
        for (uint64_t col = 0; col < dim; ++col) {
            const int col_keep = ((col & mask) != 0) == (outcome == 1);
            for (uint64_t row = 0; row < dim; ++row) {
                const int keep = col_keep && (((row & mask) != 0) == (outcome == 1));
                cd *e = &s->a[row + col * dim];
                *e = keep ? C(e->re * scale, e->im * scale) : C(0, 0);
            }
        }
    }
    return VQB_OK;
}

/* measure (circuit.hpp:303-337, :339-375) with the drawn uniform given */
ORC_API int vqcsorc_measure(ostate *s, int32_t q, double uniform, int32_t *outcome, double *prob) {
    double p1;
    int rc = vqcsorc_measure_probability(s, q, &p1);
    if (rc) return rc;
    p1 = clamp_probability(p1);
    const double p0 = clamp_probability(1.0 - p1);
    if (p0 == 0 && p1 == 0) return fail(VQB_ERR_DEGENERATE, "measure: both outcome probabilities vanish");
    const int o = uniform < p1 ? 1 : 0;
    const double p = o == 1 ? p1 : p0;
    if (p == 0) return fail(VQB_ERR_DEGENERATE, "measure: drawn outcome has zero probability");
    rc = vqcsorc_collapse(s, q, o, p);
    if (rc) return rc;
    *outcome = o;
    *prob = p;
    return VQB_OK;
}

/* ================= state dumps: io.hpp:15-128 ================= */
ORC_API int vqcsorc_state_save(const ostate *s, const char *path) { /* io.hpp:56-82 */
    if (s->mixed) return fail(VQB_ERR_TYPE, "save_state: only pure states can be dumped");
    FILE *f = fopen(path, "wb");
    if (!f) return fail(VQB_ERR_IO, "save_state: cannot open file for writing");
    const uint32_t version = 1, n = (uint32_t)s->n;
    const uint8_t prec = 2;
    int ok = fwrite("VQCS", 1, 4, f) == 4 && fwrite(&version, 4, 1, f) == 1 && fwrite(&n, 4, 1, f) == 1 &&
             fwrite(&prec, 1, 1, f) == 1;
    for (uint64_t k = 0; ok && k < s->size; ++k) {
        const double pair[2] = {s->a[k].re, s->a[k].im};
        ok = fwrite(pair, sizeof pair, 1, f) == 1;
    }
    if (fclose(f) != 0) ok = 0;
    return ok ? VQB_OK : fail(VQB_ERR_IO, "save_state: write failed");
}

ORC_API int vqcsorc_state_load(const char *path, ostate **out, int32_t *precision) { /* io.hpp:84-128 */
    FILE *f = fopen(path, "rb");
    if (!f) return fail(VQB_ERR_IO, "load_state: cannot open file");
    char magic[4] = {0, 0, 0, 0};
    uint32_t version = 0, n = 0;
    uint8_t prec = 0;
    const int hdr = fread(magic, 1, 4, f) == 4 && fread(&version, 4, 1, f) == 1 && fread(&n, 4, 1, f) == 1 &&
                    fread(&prec, 1, 1, f) == 1;
    int rc = VQB_OK;
    if (!hdr || memcmp(magic, "VQCS", 4) != 0) rc = fail(VQB_ERR_IO, "load_state: not a state dump (bad magic)");
    else if (version != 1) rc = fail(VQB_ERR_IO, "load_state: unsupported format version");
    else if (n < 1 || n > 40) rc = fail(VQB_ERR_IO, "load_state: qubit count out of range");
    else if (prec != 1 && prec != 2) rc = fail(VQB_ERR_IO, "load_state: unknown precision tag");
    ostate *s = NULL;
    if (!rc) rc = vqcsorc_state_create((int32_t)n, 0, &s);
    for (uint64_t k = 0; !rc && k < s->size; ++k) {
        double pair[2];
        if (fread(pair, sizeof pair, 1, f) != 1) rc = fail(VQB_ERR_IO, "load_state: truncated amplitude payload");
        else s->a[k] = C(pair[0], pair[1]);
    }
    fclose(f);
    if (rc) {
        vqcsorc_state_destroy(s);
        return rc;
    }
    if (precision) *precision = prec;
    *out = s;
    return VQB_OK;
}

/* ================= fuse_gates: circuit.hpp:190-276 ================= */
static void matmul(const cd *a, const cd *b, int d, cd *c) { /* linalg.hpp:40-55 */
    for (int i = 0; i < d * d; ++i) c[i] = C(0, 0);
    for (int j = 0; j < d; ++j)
        for (int k = 0; k < d; ++k) {
            const cd bkj = b[k + j * d];
            if (bkj.re == 0 && bkj.im == 0) continue;
            for (int i = 0; i < d; ++i) c[i + j * d] = cadd(c[i + j * d], cmul(a[i + k * d], bkj));
        }
}

typedef struct {
    int m;
    int32_t pos[VQB_MAX_POSITIONS];
    cd *mat; /* 4^m */
} small_gate;

ORC_API int vqcsorc_fuse_gates(const vqb_op *ops, int64_t count, int64_t cap, vqb_op *out_ops,
                               int64_t matrix_cap, cd *out_matrices, int64_t *num_out, int64_t *num_entries) {
    for (int64_t i = 0; i < count; ++i)
        if (ops[i].elem == VQB_ELEM_CHANNEL)
            return fail(VQB_ERR_UNSUPPORTED, "fuse_gates: circuit contains quantum channels");
    small_gate *flat = (small_gate *)calloc(count > 0 ? count : 1, sizeof(small_gate));
    int64_t *merge = (int64_t *)malloc(sizeof(int64_t) * (count > 0 ? count : 1));
    gate_t *g = (gate_t *)malloc(sizeof(gate_t));
    int rc = VQB_OK;
    for (int64_t i = 0; i < count && !rc; ++i) {
        rc = build_gate(&ops[i], g);
        if (rc) break;
        const int dd = 1 << (2 * g->m);
        flat[i].m = g->m;
        memcpy(flat[i].pos, g->pos, sizeof(int32_t) * g->m);
        flat[i].mat = (cd *)malloc(sizeof(cd) * dd);
        memcpy(flat[i].mat, g->mat, sizeof(cd) * dd);
    }
    free(g);
    int64_t nout = 0, entries = 0;
    if (!rc) {
        for (int64_t i = 0; i < count; ++i) { /* circuit.hpp:219-246 */
            merge[i] = -1;
            if (flat[i].m != 1) continue;
            const int q = flat[i].pos[0];
            int64_t prev = -1, next = -1;
            for (int64_t j = i - 1; j >= 0 && prev < 0; --j)
                for (int k = 0; k < flat[j].m; ++k)
                    if (flat[j].pos[k] == q) prev = j;
            for (int64_t j = i + 1; j < count && next < 0; ++j)
                for (int k = 0; k < flat[j].m; ++k)
                    if (flat[j].pos[k] == q) next = j;
            if (next >= 0 && flat[next].m == 2) merge[i] = next;
            else if (prev >= 0 && flat[prev].m == 2) merge[i] = prev;
        }
        for (int64_t i = 0; i < count; ++i)
            if (merge[i] < 0) {
                ++nout;
                entries += (int64_t)1 << (2 * flat[i].m);
            }
        *num_out = nout;
        *num_entries = entries;
        if (cap > 0 && (cap < nout || matrix_cap < entries)) rc = fail(VQB_ERR_SHAPE, "fuse_gates: output buffers too small");
    }
    if (!rc && cap > 0) {
        int64_t o = 0, off = 0;
        for (int64_t i = 0; i < count; ++i) { /* circuit.hpp:248-275 */
            if (merge[i] >= 0) continue;
            const int d = 1 << flat[i].m;
            cd cur[16], emb[16], tmp[16];
            cd *dst = out_matrices + off;
            memcpy(dst, flat[i].mat, sizeof(cd) * d * d);
            if (flat[i].m == 2) {
                memcpy(cur, flat[i].mat, sizeof cur);
                for (int64_t k = 0; k < count; ++k) {
                    if (merge[k] != i) continue;
                    const cd eye[4] = {C(1, 0), C(0, 0), C(0, 0), C(1, 0)};
                    if (flat[k].pos[0] == flat[i].pos[0]) kron(eye, 2, flat[k].mat, 2, emb); /* low bit */
                    else kron(flat[k].mat, 2, eye, 2, emb);
                    if (k < i) matmul(cur, emb, 4, tmp);
                    else matmul(emb, cur, 4, tmp);
                    memcpy(cur, tmp, sizeof cur);
                }
                memcpy(dst, cur, sizeof cur);
            }
            vqb_op op;
            memset(&op, 0, sizeof op);
            op.elem = VQB_ELEM_GATE;
            op.kind = VQB_GATE_GENERIC;
            op.num_positions = flat[i].m;
            memcpy(op.positions, flat[i].pos, sizeof(int32_t) * flat[i].m);
            op.matrix = dst;
            out_ops[o++] = op;
            off += (int64_t)d * d;
        }
    }
    for (int64_t i = 0; i < count; ++i) free(flat[i].mat);
    free(flat);
    free(merge);
    return rc;
}

/* ================= batched reverse steps (autodiff.hpp:130-150) ================= */
ORC_API int vqcsorc_reverse_sweep(ostate *phi, ostate *psi, const vqb_rev_step *steps, int64_t count,
                                  double scale, double *grads, int64_t grads_len) {
    if (phi == psi) return fail(VQB_ERR_USAGE, "reverse_sweep: phi and psi must be distinct states");
    if (phi->size != psi->size) return fail(VQB_ERR_SHAPE, "reverse_sweep: shape mismatch");
    for (int64_t i = 0; i < count; ++i) {
        const vqb_rev_step *st = &steps[i];
        if (st->num_positions < 1 || st->num_positions > 4)
            return fail(VQB_ERR_SHAPE, "reverse_sweep: steps act on 1..4 positions");
        int rc = check_positions(st->positions, st->num_positions);
        if (!rc) rc = check_fit(st->positions, st->num_positions, phi->pn);
        if (rc) return rc;
        if (st->num_dmats < 0 || st->num_dmats > VQB_MAX_PARAMS)
            return fail(VQB_ERR_SHAPE, "reverse_sweep: at most 5 derivative matrices per step");
        if (st->num_dmats > 0 && (st->grad_index < 0 || st->grad_index + st->num_dmats > grads_len))
            return fail(VQB_ERR_INDEX, "reverse_sweep: gradient slot out of range");
        cd acc[VQB_MAX_PARAMS];
        reverse_step_raw(phi->a, psi->a, phi->pn, st->positions, st->num_positions, st->inv, st->dmats,
                         st->num_dmats, acc);
        for (int p = 0; p < st->num_dmats; ++p) grads[st->grad_index + p] += scale * acc[p].re;
    }
    return VQB_OK;
}
