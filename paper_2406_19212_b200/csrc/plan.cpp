// Operation analysis and greedy stage packing (see plan.hpp).
#include "plan.hpp"

#include <algorithm>

namespace vqb {

namespace {

// Split the m local bits of a set of 2^m x 2^m matrices into mixing and
// condition bits: bit b is a condition bit iff every matrix is block
// diagonal in it (entry (r, c) == 0 whenever r and c differ in bit b).
void split_bits(const std::vector<const cvec *> &mats, int m, std::vector<int> &mix,
                std::vector<int> &cnd) {
    const int d = 1 << m;
    for (int b = 0; b < m; ++b) {
        bool mixing = false;
        for (const cvec *M : mats) {
            for (int c = 0; c < d && !mixing; ++c)
                for (int r = 0; r < d; ++r)
                    if (((r ^ c) >> b & 1) && (*M)[r + size_t(c) * d] != cplx(0)) {
                        mixing = true;
                        break;
                    }
            if (mixing) break;
        }
        (mixing ? mix : cnd).push_back(b);
    }
}

// Extract the 2^nc sub-matrices (each (2^nt)^2, column-major) of M.
cvec sub_blocks(const cvec &M, int m, const std::vector<int> &mix, const std::vector<int> &cnd) {
    const int d = 1 << m, nt = (int)mix.size(), nc = (int)cnd.size();
    const int dt = 1 << nt;
    cvec out(size_t(1) << nc << (2 * nt));
    for (int c = 0; c < (1 << nc); ++c) {
        int cbase = 0;
        for (int i = 0; i < nc; ++i)
            if (c >> i & 1) cbase |= 1 << cnd[i];
        for (int col = 0; col < dt; ++col)
            for (int row = 0; row < dt; ++row) {
                int r = cbase, cc = cbase;
                for (int i = 0; i < nt; ++i) {
                    if (row >> i & 1) r |= 1 << mix[i];
                    if (col >> i & 1) cc |= 1 << mix[i];
                }
                out[size_t(c) * dt * dt + row + size_t(col) * dt] = M[r + size_t(cc) * d];
            }
    }
    return out;
}

FusedOp analyse(const int *pos1, int m, const std::vector<const cvec *> &mats) {
    FusedOp f;
    std::vector<int> mix, cnd;
    split_bits(mats, m, mix, cnd);
    f.nt = (int)mix.size();
    f.nc = (int)cnd.size();
    for (int k = 0; k < m; ++k) f.support |= 1ull << (pos1[k] - 1);
    if (f.nt > kMaxMix || f.nc > kMaxCond) {
        f.fusable = false;
        return f;
    }
    for (int i = 0; i < f.nt; ++i) {
        f.mix[i] = pos1[mix[i]] - 1;
        f.mixmask |= 1ull << f.mix[i];
    }
    for (int i = 0; i < f.nc; ++i) f.cnd[i] = pos1[cnd[i]] - 1;
    f.sub_phi = sub_blocks(*mats[0], m, mix, cnd);
    return f;
}

} // namespace

FusedOp analyse_gate(const Gate &g) {
    FusedOp f = analyse(g.pos, g.m, {&g.mat});
    f.gate = g;
    return f;
}

FusedOp analyse_rev(const RevOp &r) {
    std::vector<const cvec *> mats{&r.phi_op.mat};
    const bool pair = r.psi_op.mat != r.phi_op.mat;
    if (pair) mats.push_back(&r.psi_op.mat);
    for (const auto &d : r.dmats) mats.push_back(&d);
    FusedOp f = analyse(r.phi_op.pos, r.phi_op.m, mats);
    f.rev = &r;
    f.gate = r.phi_op;
    if (!f.fusable) return f;
    std::vector<int> mix, cnd;
    split_bits(mats, r.phi_op.m, mix, cnd);
    f.pair = pair;
    if (pair) f.sub_psi = sub_blocks(r.psi_op.mat, r.phi_op.m, mix, cnd);
    f.np = (int)r.dmats.size();
    for (const auto &d : r.dmats) {
        const cvec s = sub_blocks(d, r.phi_op.m, mix, cnd);
        f.sub_d.insert(f.sub_d.end(), s.begin(), s.end());
    }
    f.grad_base = r.grad_base;
    f.scale = r.scale;
    return f;
}

namespace {

// Embed matrix M over positions P (global bits) into the space of U (global
// bits, local order = listed order); identity on U \ P.
cvec embed(const cvec &M, const std::vector<int> &P, const std::vector<int> &U) {
    const int u = (int)U.size(), du = 1 << u, dp = 1 << (int)P.size();
    std::vector<int> where(P.size());
    for (size_t i = 0; i < P.size(); ++i)
        where[i] = (int)(std::find(U.begin(), U.end(), P[i]) - U.begin());
    int pmask = 0;
    for (int w : where) pmask |= 1 << w;
    cvec out(size_t(du) * du);
    for (int c = 0; c < du; ++c)
        for (int r = 0; r < du; ++r) {
            if ((r & ~pmask) != (c & ~pmask)) continue;
            int rp = 0, cp = 0;
            for (size_t i = 0; i < P.size(); ++i) {
                rp |= ((r >> where[i]) & 1) << i;
                cp |= ((c >> where[i]) & 1) << i;
            }
            out[r + size_t(c) * du] = M[rp + size_t(cp) * dp];
        }
    return out;
}

struct Block {
    std::vector<int> U;  // global bits
    cvec phi, psi;       // psi empty unless a pair block
    bool pair = false;
    bool alive = true;
    bool frozen = false; // parametric or too wide: never merged into
    int src = -1;        // original op index when frozen
};

std::vector<int> gate_bits(const Gate &g) {
    std::vector<int> b(g.m);
    for (int i = 0; i < g.m; ++i) b[i] = g.pos[i] - 1;
    return b;
}

} // namespace

std::vector<FusedOp> fuse_blocks(const std::vector<FusedOp> &ops, const std::vector<int> &order,
                                 int max_support) {
    std::vector<Block> blocks;
    std::vector<int> last(64, -1); // last block per qubit
    for (int idx : order) {
        const FusedOp &f = ops[idx];
        const Gate &g = f.gate;
        const std::vector<int> P = gate_bits(g);
        const bool param = f.rev && !f.rev->dmats.empty();
        const bool pair = f.rev && f.rev->psi_op.mat != f.rev->phi_op.mat;
        if (param || (int)P.size() > max_support || !f.fusable) {
            Block b;
            b.U = P;
            b.frozen = true;
            b.src = idx;
            blocks.push_back(b);
            for (int q : P) last[q] = (int)blocks.size() - 1;
            continue;
        }
        // candidate blocks: the latest block on each touched qubit
        std::vector<int> cands;
        for (int q : P)
            if (last[q] >= 0 && std::find(cands.begin(), cands.end(), last[q]) == cands.end())
                cands.push_back(last[q]);
        std::vector<int> U = P;
        bool ok = !cands.empty();
        for (int c : cands) {
            if (blocks[c].frozen) ok = false;
            for (int q : blocks[c].U)
                if (std::find(U.begin(), U.end(), q) == U.end()) U.push_back(q);
        }
        if (ok && (int)U.size() > max_support) ok = false;
        // every candidate must be the latest block on all of its qubits, so
        // nothing after it acts on them: it can move forward to the merge
        // point, and the candidates have disjoint supports (they commute)
        if (ok)
            for (int c : cands)
                for (int q : blocks[c].U)
                    if (last[q] != c) ok = false;
        if (!ok) {
            Block b;
            b.U = P;
            b.phi = g.mat;
            if (pair) {
                b.pair = true;
                b.psi = f.rev->psi_op.mat;
            }
            blocks.push_back(b);
            for (int q : P) last[q] = (int)blocks.size() - 1;
            continue;
        }
        // product of the candidates (disjoint supports, commuting), then op
        std::sort(U.begin(), U.end());
        const int du = 1 << (int)U.size();
        cvec acc_phi(size_t(du) * du), acc_psi;
        for (int i = 0; i < du; ++i) acc_phi[i + size_t(i) * du] = 1.0;
        bool any_pair = pair;
        for (int c : cands) any_pair |= blocks[c].pair;
        if (any_pair) acc_psi = acc_phi;
        for (int c : cands) {
            const Block &b = blocks[c];
            acc_phi = matmul(embed(b.phi, b.U, U), acc_phi, du);
            if (any_pair) acc_psi = matmul(embed(b.pair ? b.psi : b.phi, b.U, U), acc_psi, du);
        }
        acc_phi = matmul(embed(g.mat, P, U), acc_phi, du);
        if (any_pair) acc_psi = matmul(embed(pair ? f.rev->psi_op.mat : g.mat, P, U), acc_psi, du);
        const int keep = *std::max_element(cands.begin(), cands.end());
        for (int c : cands)
            if (c != keep) blocks[c].alive = false;
        Block &k = blocks[keep];
        k.U = U;
        k.phi = std::move(acc_phi);
        k.pair = any_pair;
        k.psi = std::move(acc_psi);
        for (int q : U) last[q] = keep;
    }
    std::vector<FusedOp> out;
    for (const Block &b : blocks) {
        if (!b.alive) continue;
        if (b.frozen) {
            out.push_back(ops[b.src]);
            continue;
        }
        int pos1[VQB_MAX_POSITIONS];
        for (size_t i = 0; i < b.U.size(); ++i) pos1[i] = b.U[i] + 1;
        std::vector<const cvec *> mats{&b.phi};
        if (b.pair) mats.push_back(&b.psi);
        FusedOp f = analyse(pos1, (int)b.U.size(), mats);
        std::vector<int> mix, cnd;
        split_bits(mats, (int)b.U.size(), mix, cnd);
        if (b.pair) {
            f.pair = true;
            f.sub_psi = sub_blocks(b.psi, (int)b.U.size(), mix, cnd);
        }
        f.gate.kind = VQB_GATE_GENERIC;
        f.gate.m = (int)b.U.size();
        for (size_t i = 0; i < b.U.size(); ++i) f.gate.pos[i] = pos1[i];
        f.gate.mat = b.phi;
        out.push_back(std::move(f));
    }
    return out;
}

std::vector<Stage> plan_stages(const std::vector<FusedOp> &ops, int pn, int k) {
    k = std::min(k, pn);
    const int low = std::min(kLowBits, pn);
    uint64_t lowmask = 0;
    for (int b = 0; b < low; ++b) lowmask |= 1ull << b;

    std::vector<Stage> stages;
    std::vector<int> remaining(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) remaining[i] = (int)i;

    while (!remaining.empty()) {
        if (!ops[remaining[0]].fusable) {
            Stage s;
            s.fused = false;
            s.ops = {remaining[0]};
            stages.push_back(s);
            remaining.erase(remaining.begin());
            continue;
        }
        // Pass 1: greedy tile selection in program order.
        uint64_t S = lowmask, blocked = 0;
        for (int i : remaining) {
            const FusedOp &op = ops[i];
            if ((op.support & blocked) || !op.fusable) {
                blocked |= op.support;
                continue;
            }
            const uint64_t need = S | op.mixmask;
            if (__builtin_popcountll(need) <= k) S = need;
            else blocked |= op.support;
        }
        // Fill the tile to exactly k bits: first the mixing bits the deferred
        // operations need (in program order), then the lowest free bits.
        for (int i : remaining) {
            if (__builtin_popcountll(S) >= k) break;
            const uint64_t need = S | ops[i].mixmask;
            if (ops[i].fusable && (ops[i].mixmask & ~S) && __builtin_popcountll(need) <= k) S = need;
        }
        for (int b = 0; b < pn && __builtin_popcountll(S) < k; ++b) S |= 1ull << b;
        // Pass 2: with the tile fixed, take every op that fits and is not
        // ordered behind a deferred op sharing a qubit.
        Stage st;
        st.k = k;
        int nb = 0;
        for (int b = 0; b < pn; ++b)
            if (S >> b & 1) st.bits[nb++] = b;
        std::vector<int> deferred;
        blocked = 0;
        for (int i : remaining) {
            const FusedOp &op = ops[i];
            if ((int)st.ops.size() < kMaxPlanOps && !(op.support & blocked) && op.fusable &&
                (op.mixmask & ~S) == 0) {
                st.ops.push_back(i);
            } else {
                deferred.push_back(i);
                blocked |= op.support;
            }
        }
        stages.push_back(std::move(st));
        remaining.swap(deferred);
    }
    return stages;
}

} // namespace vqb
