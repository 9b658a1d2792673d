// Lowering of circuits to gate programs and the element-by-element executor.
#include "engine.hpp"
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>

namespace vqb {

std::vector<Element> build_elements(const vqb_op *ops, int64_t count) {
    std::vector<Element> es(count);
    for (int64_t i = 0; i < count; ++i) {
        if (ops[i].elem == VQB_ELEM_CHANNEL) {
            es[i].channel = true;
            es[i].chan = channel_from_op(ops[i]);
        } else {
            es[i].gate = gate_from_op(ops[i]);
        }
    }
    return es;
}

namespace {

// The bra-side copy of a gate: conj(U) on positions + n, keeping the kind
// only when conj(U) == U (kernels.hpp:441-448).
Gate bra_side(const Gate &g, int n) {
    Gate b = g;
    for (int k = 0; k < g.m; ++k) b.pos[k] = g.pos[k] + n;
    b.mat = conjugated(g.mat);
    b.np = 0;
    if (b.mat != g.mat) b.kind = VQB_GATE_GENERIC;
    return b;
}

Gate dense_gate(const int *pos, int m, cvec mat) {
    Gate g;
    g.kind = VQB_GATE_GENERIC;
    g.m = m;
    for (int k = 0; k < m; ++k) g.pos[k] = pos[k];
    g.mat = std::move(mat);
    return g;
}

Gate superop_gate(const Channel &c, int n, cvec mat) {
    int pos[6];
    for (int k = 0; k < c.m; ++k) {
        pos[k] = c.pos[k];
        pos[k + c.m] = c.pos[k] + n;
    }
    return dense_gate(pos, 2 * c.m, std::move(mat));
}

} // namespace

std::vector<Gate> mixed_forward_program(const std::vector<Element> &es, int n) {
    std::vector<Gate> prog;
    for (const auto &e : es) {
        if (e.channel) {
            prog.push_back(superop_gate(e.chan, n, channel_superop(e.chan)));
        } else {
            prog.push_back(e.gate);
            prog.push_back(bra_side(e.gate, n));
        }
    }
    return prog;
}

// gradient_pure reverse loop (autodiff.hpp:130-150)
std::vector<RevOp> pure_reverse_program(const std::vector<Element> &es,
                                        const std::vector<int64_t> &base) {
    const size_t n = es.size();
    std::vector<RevOp> prog(n);
    parallel_chunks(n, 96, [&](size_t b, size_t e) {
        for (size_t k = b; k < e; ++k) {
            const size_t i = n - 1 - k; // reverse order
            const Gate &g = es[i].gate;
            RevOp &r = prog[k];
            r.phi_op = gate_inverse(g);
            r.psi_op = r.phi_op;
            if (g.has_active()) {
                for (int p = 0; p < g.np; ++p)
                    if (g.is_param[p]) r.dmats.push_back(gate_derivative(g, p));
                r.grad_base = base[i];
                r.scale = 2.0; // grads = 2 Re(acc) (autodiff.hpp:147-149)
            }
        }
    });
    return prog;
}

// gradient_mixed reverse loop (autodiff.hpp:263-323)
std::vector<RevOp> mixed_reverse_program(const std::vector<Element> &es, int n,
                                         const std::vector<int64_t> &base,
                                         const std::vector<cvec> &chan_inv,
                                         const std::vector<cvec> &chan_adj) {
    std::vector<RevOp> prog;
    for (size_t i = es.size(); i-- > 0;) {
        if (es[i].channel) {
            RevOp r;
            r.phi_op = superop_gate(es[i].chan, n, chan_inv[i]); // S^-1 on phi
            r.psi_op = superop_gate(es[i].chan, n, chan_adj[i]); // S^dag on psi
            prog.push_back(std::move(r));
            continue;
        }
        const Gate &g = es[i].gate;
        const Gate inv = gate_inverse(g);
        if (!g.has_active()) {
            RevOp ket, bra;
            ket.phi_op = ket.psi_op = inv;
            bra.phi_op = bra.psi_op = bra_side(inv, n);
            prog.push_back(std::move(ket));
            prog.push_back(std::move(bra));
            continue;
        }
        // The superoperator conj(U) (x) U is the product of its ket half and its
        // bra half, which act on different bits: the step splits into two, each
        // with the derivative of its own factor, both adding into the gate's
        // gradient entries. dS S^-1 = (dU U^-1) (x) 1 + 1 (x) conj(dU U^-1) and the
        // halves commute, so the two contributions sum to the reference's
        // Re<<psi| dS |S^-1 phi>> (autodiff.hpp:297-322) while each half costs a
        // 2^m x 2^m product instead of one 4^m x 4^m. VQB_MIXED_SPLIT=0 keeps
        // the single step.
        const char *split_env = std::getenv("VQB_MIXED_SPLIT");
        const bool split = !(split_env && *split_env == '0');
        // (a diagonal gate stays one step: the ket and bra phases cancel on
        // half of the entries, which the single diagonal superoperator skips)
        bool diagonal = true;
        for (int r = 0; r < g.dim() && diagonal; ++r)
            for (int c = 0; c < g.dim(); ++c)
                if (r != c && inv.mat[r + (size_t)c * g.dim()] != cplx(0)) {
                    diagonal = false;
                    break;
                }
        if (split && !diagonal) {
            RevOp ket, bra;
            ket.phi_op = ket.psi_op = inv;
            bra.phi_op = bra.psi_op = bra_side(inv, n);
            for (int p = 0; p < g.np; ++p) {
                if (!g.is_param[p]) continue;
                const cvec du = gate_derivative(g, p);
                bra.dmats.push_back(conjugated(du));
                ket.dmats.push_back(du);
            }
            ket.grad_base = bra.grad_base = base[i];
            ket.scale = bra.scale = 1.0; // grads = Re(acc) (autodiff.hpp:320-322)
            prog.push_back(std::move(ket));
            prog.push_back(std::move(bra));
            continue;
        }
        const int d = g.dim();
        int pos[6];
        for (int k = 0; k < g.m; ++k) {
            pos[k] = g.pos[k];
            pos[k + g.m] = g.pos[k] + n;
        }
        RevOp r;
        // inv_local = kron(high = conj(U^-1) on bra, low = U^-1 on ket) (autodiff.hpp:297)
        r.phi_op = dense_gate(pos, 2 * g.m, kron(conjugated(inv.mat), d, inv.mat, d));
        r.psi_op = r.phi_op;
        const cvec conj_u = conjugated(g.mat);
        for (int p = 0; p < g.np; ++p) {
            if (!g.is_param[p]) continue;
            // dS = dU (x) conj(U) + U (x) conj(dU) (autodiff.hpp:303-311)
            const cvec du = gate_derivative(g, p);
            cvec ds = kron(conj_u, d, du, d);
            const cvec second = kron(conjugated(du), d, g.mat, d);
            for (size_t k = 0; k < ds.size(); ++k) ds[k] += second[k];
            r.dmats.push_back(std::move(ds));
        }
        r.grad_base = base[i];
        r.scale = 1.0; // grads = Re(acc) (autodiff.hpp:320-322)
        prog.push_back(std::move(r));
    }
    return prog;
}

namespace {

// Matrix over positions P (1-based) embedded into the sorted union U.
cvec embed_into(const cvec &M, const int *P, int m, const std::vector<int> &U) {
    const int u = (int)U.size(), du = 1 << u, dp = 1 << m;
    int where[VQB_MAX_POSITIONS];
    int pmask = 0;
    for (int i = 0; i < m; ++i) {
        where[i] = (int)(std::find(U.begin(), U.end(), P[i]) - U.begin());
        pmask |= 1 << where[i];
    }
    cvec out(size_t(du) * du);
    for (int c = 0; c < du; ++c)
        for (int r = 0; r < du; ++r) {
            if ((r & ~pmask) != (c & ~pmask)) continue;
            int rp = 0, cp = 0;
            for (int i = 0; i < m; ++i) {
                rp |= ((r >> where[i]) & 1) << i;
                cp |= ((c >> where[i]) & 1) << i;
            }
            out[r + size_t(c) * du] = M[rp + size_t(cp) * dp];
        }
    return out;
}

std::vector<int> union_of(const Gate &a, const Gate &b) {
    std::vector<int> u(a.pos, a.pos + a.m);
    for (int i = 0; i < b.m; ++i)
        if (std::find(u.begin(), u.end(), b.pos[i]) == u.end()) u.push_back(b.pos[i]);
    std::sort(u.begin(), u.end());
    return u;
}

bool overlaps(const Gate &a, const Gate &b) {
    for (int i = 0; i < a.m; ++i)
        for (int j = 0; j < b.m; ++j)
            if (a.pos[i] == b.pos[j]) return true;
    return false;
}

Gate on_union(const std::vector<int> &U, cvec mat) {
    Gate g;
    g.kind = VQB_GATE_GENERIC;
    g.m = (int)U.size();
    for (int i = 0; i < g.m; ++i) g.pos[i] = U[i];
    g.mat = std::move(mat);
    return g;
}

// A unitary non-parametric step (same matrix on both states) may be folded
// into an adjacent parametric step when their supports overlap and the union
// has at most two qubits.
bool is_unitary(const cvec &a, int d) {
    const cvec p = matmul(adjoint(a, d), a, d);
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i)
            if (std::abs(p[i + j * d] - (i == j ? cplx(1) : cplx(0))) > 1e-12) return false;
    return true;
}

bool foldable(const RevOp &x, const RevOp &p) {
    return x.dmats.empty() && x.phi_op.mat == x.psi_op.mat && overlaps(x.phi_op, p.phi_op) &&
           union_of(x.phi_op, p.phi_op).size() <= 2 && is_unitary(x.phi_op.mat, x.phi_op.dim());
}

} // namespace

// Reverse-program rewrite: [A][P][B] -> [P'] with inv' = B inv A and
// D'_p = A^dag D_p B^dag (A, B unitary). Same gradient contributions
// (acc = <A psi| D |inv A phi> = <psi| A^dag D B^dag |B inv A phi>), fewer
// passes over the two states. Applied to both the pure and the mixed sweep
// (where A, B are the ket/bra halves of unitary gates; channel steps, whose
// phi and psi matrices differ, are never folded).
std::vector<RevOp> fold_reverse_program(const std::vector<RevOp> &prog) {
    std::vector<RevOp> out;
    out.reserve(prog.size());
    for (const RevOp &r : prog) {
        if (!r.dmats.empty() && !out.empty() && foldable(out.back(), r)) {
            // A = out.back() runs before P: inv' = inv A, D' = A^dag D
            const RevOp A = out.back();
            out.pop_back();
            const std::vector<int> U = union_of(A.phi_op, r.phi_op);
            const int d = 1 << (int)U.size();
            const cvec a = embed_into(A.phi_op.mat, A.phi_op.pos, A.phi_op.m, U);
            const cvec adag = adjoint(a, d);
            RevOp m;
            m.phi_op = on_union(U, matmul(embed_into(r.phi_op.mat, r.phi_op.pos, r.phi_op.m, U), a, d));
            m.psi_op = m.phi_op;
            for (const auto &dm : r.dmats)
                m.dmats.push_back(matmul(adag, embed_into(dm, r.phi_op.pos, r.phi_op.m, U), d));
            m.grad_base = r.grad_base;
            m.scale = r.scale;
            out.push_back(std::move(m));
            continue;
        }
        if (r.dmats.empty() && !out.empty() && !out.back().dmats.empty() && foldable(r, out.back())) {
            // B = r runs after P: inv' = B inv, D' = D B^dag
            RevOp &p = out.back();
            const std::vector<int> U = union_of(r.phi_op, p.phi_op);
            const int d = 1 << (int)U.size();
            const cvec b = embed_into(r.phi_op.mat, r.phi_op.pos, r.phi_op.m, U);
            const cvec bdag = adjoint(b, d);
            const Gate inv = on_union(U, matmul(b, embed_into(p.phi_op.mat, p.phi_op.pos,
                                                              p.phi_op.m, U), d));
            std::vector<cvec> dm;
            for (const auto &x : p.dmats)
                dm.push_back(matmul(embed_into(x, p.phi_op.pos, p.phi_op.m, U), bdag, d));
            p.phi_op = inv;
            p.psi_op = inv;
            p.dmats = std::move(dm);
            continue;
        }
        out.push_back(r);
    }
    return out;
}

void run_program(DeviceState *s, const std::vector<Gate> &prog, bool fused) {
    if (fused) {
        run_program_fused(s, prog);
        return;
    }
    for (const auto &g : prog) apply_gate_fast(s->amps, s->pn, g, s->stream);
}

void run_reverse(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                 double *dgrads, bool fused) {
    if (fused) {
        const char *nf = std::getenv("VQB_NO_FOLD");
        if (nf && *nf == '1') {
            run_reverse_fused(phi, psi, prog, dgrads);
        } else {
            std::vector<RevOp> folded;
            {
                HostTimer ht("fold_reverse_program");
                folded = fold_reverse_program(prog);
            }
            run_reverse_fused(phi, psi, folded, dgrads);
        }
        return;
    }
    wait_issue_gate();
    for (const auto &r : prog) {
        if (r.dmats.empty()) {
            apply_gate_fast(phi->amps, phi->pn, r.phi_op, phi->stream);
            apply_gate_fast(psi->amps, psi->pn, r.psi_op, phi->stream);
        } else {
            reverse_step_async(phi->amps, psi->amps, phi->pn, r.phi_op.pos, r.phi_op.m,
                               r.phi_op.mat, r.dmats, phi, nullptr, dgrads + r.grad_base, r.scale);
        }
    }
}

} // namespace vqb
