// Operation analysis and greedy stage packing (see plan.hpp).
#include "plan.hpp"

#include <atomic>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unordered_map>

#include <algorithm>
#include <deque>

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

// ---- StageJob: ordered-consumption parallel for over a persistent pool ----
struct StageJob::Impl {
    size_t n = 0;
    std::function<void(size_t)> fn;
    std::atomic<size_t> next{0};
    std::unique_ptr<std::atomic<int>[]> state; // 0 pending, 1 running, 2 done, 3 cancelled
    std::mutex mu;
    std::condition_variable cv;
    // run one index if any is left; false when none
    bool help() {
        const size_t i = next.fetch_add(1);
        if (i >= n) return false;
        int expect = 0;
        if (!state[i].compare_exchange_strong(expect, 1)) return true; // cancelled by the owner
        fn(i); // fn reports its own errors through its captures
        state[i].store(2);
        {
            std::lock_guard<std::mutex> lk(mu);
        }
        cv.notify_all();
        return true;
    }
};

namespace {
class PlanPool {
  public:
    PlanPool() {
        const char *v = std::getenv("VQB_PLAN_THREADS");
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        int nt = v && *v ? std::atoi(v) : (int)std::min(4u, hw > 2 ? (hw - 2) / 2 : 0u);
        for (int t = 0; t < nt; ++t) threads_.emplace_back([this] { loop(); });
    }
    ~PlanPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : threads_) t.join();
    }
    void add(const std::shared_ptr<StageJob::Impl> &job) {
        if (threads_.empty()) return;
        {
            std::lock_guard<std::mutex> lk(mu_);
            jobs_.push_back(job);
        }
        cv_.notify_all();
    }

  private:
    void loop() {
        for (;;) {
            std::shared_ptr<StageJob::Impl> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
                if (stop_) return;
                job = jobs_.front();
                if (job->next.load() >= job->n) {
                    jobs_.pop_front();
                    continue;
                }
            }
            while (job->help()) {
            }
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::shared_ptr<StageJob::Impl>> jobs_;
    std::vector<std::thread> threads_;
    bool stop_ = false;
};
PlanPool &plan_pool() {
    static PlanPool *p = new PlanPool; // never destroyed: workers may outlive static teardown
    return *p;
}
} // namespace

StageJob::StageJob(size_t n, std::function<void(size_t)> fn) : impl_(std::make_shared<Impl>()) {
    impl_->n = n;
    impl_->fn = std::move(fn);
    impl_->state.reset(new std::atomic<int>[n ? n : 1]);
    for (size_t i = 0; i < n; ++i) impl_->state[i].store(0);
    if (n > 1) plan_pool().add(impl_);
}

void StageJob::wait_for(size_t i) {
    Impl &J = *impl_;
    while (J.state[i].load() != 2) {
        if (J.help()) continue; // take part instead of sleeping
        std::unique_lock<std::mutex> lk(J.mu);
        J.cv.wait_for(lk, std::chrono::microseconds(50), [&] { return J.state[i].load() == 2; });
    }
}

StageJob::~StageJob() {
    Impl &J = *impl_;
    // nothing may start after this point, and whatever runs must finish (fn
    // references the caller's frame)
    J.next.store(J.n);
    for (size_t i = 0; i < J.n; ++i) {
        int expect = 0;
        if (J.state[i].compare_exchange_strong(expect, 3)) continue; // never started: cancelled
        while (J.state[i].load() == 1) std::this_thread::yield();
    }
}

void parallel_chunks(size_t n, size_t chunk, const std::function<void(size_t, size_t)> &fn) {
    if (n <= chunk) {
        if (n) fn(0, n);
        return;
    }
    const size_t nchunks = (n + chunk - 1) / chunk;
    std::vector<std::exception_ptr> errs(nchunks);
    {
        StageJob job(nchunks, [&](size_t c) {
            try {
                fn(c * chunk, std::min(n, (c + 1) * chunk));
            } catch (...) {
                errs[c] = std::current_exception();
            }
        });
        for (size_t c = 0; c < nchunks; ++c) job.wait_for(c);
    }
    for (auto &e : errs)
        if (e) std::rethrow_exception(e);
}

std::vector<long long> slot_links(const std::vector<long long> &dst) {
    std::vector<long long> link(dst.size(), -1 * 2);
    std::unordered_map<long long, long long> last;
    for (size_t j = 0; j < dst.size(); ++j) {
        auto it = last.find(dst[j]);
        if (it == last.end()) {
            link[j] = -1 * 2 + 1; // first slot of its destination, end of chain
            last[dst[j]] = (long long)j;
        } else {
            // append to the chain, keeping the predecessor's leader bit
            link[it->second] = (long long)j * 2 + (link[it->second] & 1);
            link[j] = -1 * 2;
            it->second = (long long)j;
        }
    }
    return link;
}

int entry_class(const cplx &v) {
    const double re = v.real(), im = v.imag();
    if (im == 0.0) {
        if (re == 0.0) return 0;
        if (re == 1.0) return 4;
        if (re == -1.0) return 5;
        return 1;
    }
    if (re == 0.0) {
        if (im == 1.0) return 6;
        if (im == -1.0) return 7;
        return 2;
    }
    return 3;
}

double subs_cost(const cplx *sub, int nt, int nc) {
    const int D = 1 << nt, dd = D * D;
    double total = 0;
    for (int c = 0; c < (1 << nc); ++c) {
        const cplx *M = sub + size_t(c) * dd;
        bool ident = true;
        for (int r = 0; r < D && ident; ++r)
            for (int col = 0; col < D; ++col)
                if (M[r + col * D] != (r == col ? cplx(1) : cplx(0))) {
                    ident = false;
                    break;
                }
        if (ident) continue;
        for (int r = 0; r < D; ++r) {
            // emission order: a unit entry first (a copy), then the rest
            bool unit = false, any = false;
            double row = 0;
            for (int col = 0; col < D; ++col) {
                const int k = entry_class(M[r + col * D]);
                if (k == 0) continue;
                any = true;
                unit |= k >= 4;
                row += k == 3 ? 4 : 2;
            }
            if (!any) continue;
            // the unit term is the row's free first term; any other first term
            // multiplies instead of accumulating at the same instruction count
            if (unit) row -= 2;
            total += row;
        }
    }
    return total / double(D << nc);
}

void divide_by(cplx *sub, size_t count, const cplx &s) {
    const double n2 = s.real() * s.real() + s.imag() * s.imag();
    for (size_t i = 0; i < count; ++i) {
        const double a = sub[i].real(), b = sub[i].imag();
        sub[i] = cplx((a * s.real() + b * s.imag()) / n2, (b * s.real() - a * s.imag()) / n2);
    }
}

cplx best_scale(const cplx *sub, int nt, int nc, double *cost) {
    const size_t count = size_t(1) << (2 * nt) << nc;
    double best = subs_cost(sub, nt, nc);
    cplx bs = 1.0;
    std::vector<cplx> tried, tmp(count);
    for (size_t i = 0; i < count; ++i) {
        const cplx s = sub[i];
        if (s == cplx(0) || s == cplx(1)) continue;
        if (std::find(tried.begin(), tried.end(), s) != tried.end()) continue;
        tried.push_back(s);
        std::copy(sub, sub + count, tmp.begin());
        divide_by(tmp.data(), count, s);
        const double c = subs_cost(tmp.data(), nt, nc);
        if (c < best) {
            best = c;
            bs = s;
        }
    }
    if (cost) *cost = best;
    return bs;
}

double op_cost(const FusedOp &f) {
    if (f.cost < 0) {
        if (!f.fusable) f.cost = 1e30;
        else best_scale(f.sub_phi.data(), f.nt, f.nc, &f.cost);
    }
    return f.cost;
}

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

constexpr int kMaxFuse = 4;                  // qubits (pseudo bits) per fused block
constexpr int kMaxFuseDim = 1 << kMaxFuse;   // 16
constexpr int kMaxFuseEnt = kMaxFuseDim * kMaxFuseDim;

// out = embed(M over P into U) * acc, all du x du column-major (du = 2^|U|);
// embed is the identity on U \ P. No temporaries.
void embed_mul(const cplx *M, const int *P, int np, const int *U, int nu, const cplx *acc, cplx *out) {
    const int du = 1 << nu;
    int where[kMaxFuse], pmask = 0;
    for (int i = 0; i < np; ++i) {
        where[i] = 0;
        for (int j = 0; j < nu; ++j)
            if (U[j] == P[i]) where[i] = j;
        pmask |= 1 << where[i];
    }
    const int dp = 1 << np;
    for (int i = 0; i < du * du; ++i) out[i] = cplx(0);
    // (E acc)[r, j] = sum_c E[r, c] acc[c, j]; E[r, c] != 0 only if r, c agree off P
    for (int j = 0; j < du; ++j)
        for (int c = 0; c < du; ++c) {
            const cplx a = acc[c + j * du];
            if (a == cplx(0)) continue;
            int cp = 0;
            for (int i = 0; i < np; ++i) cp |= ((c >> where[i]) & 1) << i;
            const int rest = c & ~pmask;
            for (int rp = 0; rp < dp; ++rp) {
                int r = rest;
                for (int i = 0; i < np; ++i) r |= ((rp >> i) & 1) << where[i];
                out[r + j * du] += M[rp + cp * dp] * a;
            }
        }
}

struct Block {
    int U[kMaxFuse];     // global bits
    int nu = 0;
    cplx phi[kMaxFuseEnt], psi[kMaxFuseEnt]; // psi unused unless a pair block
    bool pair = false;
    bool alive = true;
    bool frozen = false; // parametric or too wide: never merged into
    int src = -1;        // original op index (frozen, or a single unmerged op)
    bool merged = false;
    double cost = -1;    // merged blocks: op_cost of the product (cost model)
};

} // namespace

std::vector<const FusedOp *> fuse_blocks_ref(const std::vector<FusedOp> &ops, const std::vector<int> &order,
                                             int max_support, std::deque<FusedOp> &store, bool cost_model) {
    max_support = std::min(max_support, kMaxFuse);
    std::vector<Block> blocks;
    blocks.reserve(order.size());
    int last[64];
    for (int &x : last) x = -1;
    for (int idx : order) {
        const FusedOp &f = ops[idx];
        const Gate &g = f.gate;
        const int np = g.m;
        int P[VQB_MAX_POSITIONS];
        for (int i = 0; i < np; ++i) P[i] = g.pos[i] - 1;
        const bool param = f.rev && !f.rev->dmats.empty();
        const bool pair = f.rev && f.rev->psi_op.mat != f.rev->phi_op.mat;
        auto fresh = [&](bool frozen) {
            blocks.emplace_back();
            Block &b = blocks.back();
            b.frozen = frozen;
            b.src = idx;
            b.nu = std::min(np, kMaxFuse);
            for (int i = 0; i < b.nu; ++i) b.U[i] = P[i];
            for (int i = 0; i < np; ++i) last[P[i]] = (int)blocks.size() - 1;
        };
        if (param || np > max_support || !f.fusable) {
            fresh(true);
            continue;
        }
        // candidate blocks: the latest block on each touched qubit
        int cands[kMaxFuse], nc = 0;
        for (int i = 0; i < np; ++i) {
            const int c = last[P[i]];
            if (c < 0) continue;
            bool seen = false;
            for (int k = 0; k < nc; ++k) seen |= cands[k] == c;
            if (!seen) cands[nc++] = c;
        }
        int U[2 * kMaxFuse], nu = 0;
        for (int i = 0; i < np; ++i) U[nu++] = P[i];
        bool ok = nc > 0;
        for (int k = 0; k < nc && ok; ++k) {
            const Block &c = blocks[cands[k]];
            if (c.frozen) ok = false;
            for (int i = 0; i < c.nu && ok; ++i) {
                bool in = false;
                for (int j = 0; j < nu; ++j) in |= U[j] == c.U[i];
                if (!in) {
                    if (nu >= max_support) ok = false;
                    else U[nu++] = c.U[i];
                }
            }
        }
        // every candidate must be the latest block on all of its qubits, so
        // nothing after it acts on them: it can move forward to the merge
        // point, and the candidates have disjoint supports (they commute)
        for (int k = 0; k < nc && ok; ++k)
            for (int i = 0; i < blocks[cands[k]].nu; ++i)
                if (last[blocks[cands[k]].U[i]] != cands[k]) ok = false;
        if (!ok) {
            fresh(false);
            continue;
        }
        // product of the candidates (disjoint supports, commuting), then op
        for (int i = 1; i < nu; ++i) // insertion sort (nu <= kMaxFuse)
            for (int j = i; j > 0 && U[j - 1] > U[j]; --j) std::swap(U[j - 1], U[j]);
        const int du = 1 << nu;
        cplx acc_phi[kMaxFuseEnt], acc_psi[kMaxFuseEnt], tmp[kMaxFuseEnt];
        for (int i = 0; i < du * du; ++i) acc_phi[i] = cplx(0);
        for (int i = 0; i < du; ++i) acc_phi[i + i * du] = 1.0;
        bool any_pair = pair;
        for (int k = 0; k < nc; ++k) any_pair |= blocks[cands[k]].pair;
        if (any_pair) std::copy(acc_phi, acc_phi + du * du, acc_psi);
        auto src_mat = [&](const Block &b, bool psi) -> const cplx * {
            if (b.merged) return psi && b.pair ? b.psi : b.phi;
            const FusedOp &o = ops[b.src];
            if (psi && o.rev && o.rev->psi_op.mat != o.rev->phi_op.mat) return o.rev->psi_op.mat.data();
            return o.gate.mat.data();
        };
        for (int k = 0; k < nc; ++k) {
            const Block &b = blocks[cands[k]];
            embed_mul(src_mat(b, false), b.U, b.nu, U, nu, acc_phi, tmp);
            std::copy(tmp, tmp + du * du, acc_phi);
            if (any_pair) {
                embed_mul(src_mat(b, true), b.U, b.nu, U, nu, acc_psi, tmp);
                std::copy(tmp, tmp + du * du, acc_psi);
            }
        }
        embed_mul(g.mat.data(), P, np, U, nu, acc_phi, tmp);
        std::copy(tmp, tmp + du * du, acc_phi);
        if (any_pair) {
            embed_mul(pair ? f.rev->psi_op.mat.data() : g.mat.data(), P, np, U, nu, acc_psi, tmp);
            std::copy(tmp, tmp + du * du, acc_psi);
        }
        double merged_cost = -1;
        if (cost_model && !any_pair) {
            // merge only if the specialised kernel's cost does not grow
            auto block_cost = [&](const cplx *M, const int *Ub, int nub) {
                int pos1[kMaxFuse];
                for (int i = 0; i < nub; ++i) pos1[i] = Ub[i] + 1;
                const int dub = 1 << nub;
                cvec mm(M, M + dub * dub);
                const FusedOp a = analyse(pos1, nub, {&mm});
                if (!a.fusable) return 1e30;
                double c = 0;
                best_scale(a.sub_phi.data(), a.nt, a.nc, &c);
                return c;
            };
            double parts = op_cost(f);
            for (int k = 0; k < nc; ++k) {
                const Block &b = blocks[cands[k]];
                parts += b.merged ? b.cost : op_cost(ops[b.src]);
            }
            merged_cost = block_cost(acc_phi, U, nu);
            if (merged_cost > parts + 1e-9) {
                fresh(false);
                continue;
            }
        }
        const int keep = *std::max_element(cands, cands + nc);
        for (int k = 0; k < nc; ++k)
            if (cands[k] != keep) blocks[cands[k]].alive = false;
        Block &kb = blocks[keep];
        kb.nu = nu;
        std::copy(U, U + nu, kb.U);
        std::copy(acc_phi, acc_phi + du * du, kb.phi);
        kb.pair = any_pair;
        if (any_pair) std::copy(acc_psi, acc_psi + du * du, kb.psi);
        kb.merged = true;
        kb.cost = merged_cost;
        for (int i = 0; i < nu; ++i) last[U[i]] = keep;
    }
    std::vector<const FusedOp *> out;
    out.reserve(blocks.size());
    for (const Block &b : blocks) {
        if (!b.alive) continue;
        if (!b.merged) { // frozen or never merged into: the analysed op as is
            out.push_back(&ops[b.src]);
            continue;
        }
        const int du = 1 << b.nu;
        int pos1[VQB_MAX_POSITIONS];
        for (int i = 0; i < b.nu; ++i) pos1[i] = b.U[i] + 1;
        cvec phi(b.phi, b.phi + du * du), psi;
        std::vector<const cvec *> mats{&phi};
        if (b.pair) {
            psi.assign(b.psi, b.psi + du * du);
            mats.push_back(&psi);
        }
        FusedOp f = analyse(pos1, b.nu, mats);
        std::vector<int> mix, cnd;
        split_bits(mats, b.nu, mix, cnd);
        if (b.pair) {
            f.pair = true;
            f.sub_psi = sub_blocks(psi, b.nu, mix, cnd);
        }
        f.gate.kind = VQB_GATE_GENERIC;
        f.gate.m = b.nu;
        for (int i = 0; i < b.nu; ++i) f.gate.pos[i] = pos1[i];
        f.gate.mat = std::move(phi);
        store.push_back(std::move(f));
        out.push_back(&store.back());
    }
    return out;
}

std::vector<FusedOp> fuse_blocks(const std::vector<FusedOp> &ops, const std::vector<int> &order,
                                 int max_support) {
    std::deque<FusedOp> store;
    std::vector<FusedOp> out;
    for (const FusedOp *f : fuse_blocks_ref(ops, order, max_support, store)) out.push_back(*f);
    return out;
}

// The greedy packing is sensitive to which low bits every tile is made to hold
// (config 1 at 28 qubits: 35 stages with bits 0-2, 29 with bits 0-3; the QAOA
// and noisy sweeps the other way round), and 256-byte runs move ~8 % faster
// than 128-byte ones (64-byte runs are far slower: VQB_LOW_BITS=2 costs 25 %
// per launch). Large states are planned both ways and the plan with the
// smaller estimated time (stages x relative time per stage) runs; planning
// costs tens of microseconds per hundred operations.
//
// A plan depends on the program's structure only (which bits every operation
// touches and mixes), not on matrix values: plans are cached by that
// structure, so a variational loop or a benchmark plans once per circuit
// shape (the search costs ~5 ms for 800 operations).
namespace {
struct PlanCache {
    std::mutex mu;
    std::unordered_map<uint64_t, std::pair<std::vector<uint64_t>, std::vector<Stage>>> map;
};
PlanCache &plan_cache() {
    static PlanCache *c = new PlanCache;
    return *c;
}
// Estimated time of a plan in units of one HBM pass with 128-byte runs: a
// stage costs the larger of its pass (0.92 with 256-byte runs) and its emitted
// FP64 work (config 1: a launch turns FP64-bound at ~127 executed flops per
// amplitude, about 70 op_cost units).
double plan_estimate(const std::vector<Stage> &st, const std::vector<FusedOp> &ops, int low_bits) {
    const double pass = low_bits > kLowBits ? 0.92 : 1.0;
    double t = 0;
    for (const Stage &s : st) {
        if (!s.fused) {
            t += 1.0;
            continue;
        }
        double c = 0;
        for (int i : s.ops) c += op_cost(ops[i]);
        t += std::max(pass, c / 70.0);
    }
    return t;
}

// The packing is greedy and sensitive to its knobs -- which low bits every
// tile holds, how much the tile search favours the operations at the front of
// the program (a ragged frontier leaves a tail of nearly empty stages) -- so a
// small portfolio of settings is planned and the plan with the smallest
// estimate runs. Paid once per circuit structure (plan cache).
std::vector<Stage> plan_stages_uncached(const std::vector<FusedOp> &ops, int pn, int k, int max_ops,
                                        int seeds_hint) {
    const char *v = std::getenv("VQB_LOW_BITS");
    std::vector<int> lows;
    if (v && *v) lows = {std::max(0, std::min(6, std::atoi(v)))};
    else if (pn < 22 || k < kLowBits + 4) lows = {kLowBits}; // small states are launch-bound: 128-byte runs suffice
    else lows = {kLowBits, kLowBits + 1};
    static const int portfolio = [] {
        const char *e = std::getenv("VQB_PLAN_PORTFOLIO");
        return e && *e ? std::atoi(e) : 3;
    }();
    static const int front[3][2] = {{0, 128}, {32, 64}, {128, 200}};
    // starting points of the tile search per stage: 12 for large states (config
    // 3's adjoint: 27 launches without, 23 with, 21 with 24 of them, which
    // costs config 1 two launches: profiles/r2_ab_plan_seeds.txt), 6 for the
    // small, host-bound ones
    std::vector<int> seed_counts;
    if (const char *e = std::getenv("VQB_PLAN_SEEDS"); e && *e) seed_counts = {std::atoi(e)};
    else seed_counts = {seeds_hint > 0 ? seeds_hint : pn < 22 ? 6 : 12};
    // very long programs: the search is linear in the operation count (~0.2 ms
    // per operation with the whole portfolio); keep the one-time cost bounded
    const bool huge = ops.size() > 4000;
    if (huge && seed_counts[0] > 4) seed_counts[0] = 4;
    std::vector<Stage> best;
    double best_t = 0;
    for (int seeds : seed_counts)
    for (int low : lows)
        for (int f = 0; f < std::max(1, std::min(huge ? 1 : 3, portfolio)); ++f) {
            std::vector<Stage> cand =
                plan_stages(ops, pn, k, PlanKnobs{low, front[f][0], front[f][1], max_ops, seeds});
            static const bool by_count = [] {
                const char *e = std::getenv("VQB_PLAN_PICK");
                return e && std::strcmp(e, "count") == 0;
            }();
            double t = plan_estimate(cand, ops, low);
            if (by_count) {
                t = 0;
                for (const Stage &sx : cand) t += sx.fused && low > kLowBits ? 0.92 : 1.0;
            }
            if (best.empty() || t < best_t - 1e-9) {
                best = std::move(cand);
                best_t = t;
            }
        }
    return best;
}
} // namespace

std::vector<Stage> plan_stages(const std::vector<FusedOp> &ops, int pn, int k, int max_ops, int seeds) {
    std::vector<uint64_t> key;
    key.reserve(2 * ops.size() + 2);
    key.push_back((uint64_t)pn);
    key.push_back((uint64_t)k | (uint64_t)max_ops << 32 | (uint64_t)seeds << 48);
    uint64_t h = 1469598103934665603ull ^ (uint64_t)max_ops;
    auto mix = [&](uint64_t w) {
        key.push_back(w);
        h = (h ^ w) * 1099511628211ull;
        h ^= h >> 29;
    };
    for (const FusedOp &f : ops) {
        mix(f.support);
        mix(f.mixmask ^ (f.fusable ? 0 : 1ull << 63));
    }
    // the planner's switches are part of the key (tests flip them in one process)
    for (const char *e : {"VQB_LOW_BITS", "VQB_PLAN_PORTFOLIO", "VQB_PLAN_SEARCH", "VQB_PLAN_PICK", "VQB_PLAN_SEEDS"}) {
        const char *v = std::getenv(e);
        uint64_t w = 0xcbf29ce484222325ull;
        for (; v && *v; ++v) w = (w ^ (unsigned char)*v) * 1099511628211ull;
        mix(w);
    }
    h ^= (uint64_t)pn * 0x9e3779b97f4a7c15ull + (uint64_t)k;
    PlanCache &pc = plan_cache();
    {
        std::lock_guard<std::mutex> lk(pc.mu);
        auto it = pc.map.find(h);
        if (it != pc.map.end() && it->second.first == key) return it->second.second;
    }
    std::vector<Stage> st = plan_stages_uncached(ops, pn, k, max_ops, seeds);
    {
        std::lock_guard<std::mutex> lk(pc.mu);
        if (pc.map.size() >= 64) pc.map.clear();
        pc.map[h] = {std::move(key), st};
    }
    return st;
}

std::vector<Stage> plan_stages(const std::vector<FusedOp> &ops, int pn, int k, const PlanKnobs &knobs) {
    k = std::min(k, pn);
    const int low = std::min(knobs.low_bits, pn);
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
        // Pass 1: greedy tile selection in program order, from the tile bits
        // `seed` (the forced low bits, or those plus one pending operation's
        // mixing bits: several starting points are tried below).
        int tile_score = 0;
        auto build_tile = [&](uint64_t seed) {
        uint64_t S = seed, blocked = 0;
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
        // Hill climbing on the tile: swap one free tile bit for a bit a pending
        // operation mixes while the stage would take more operations (mixing
        // operations weigh 4, diagonal ones 1: the latter ride along anyway).
        // First-fit alone packs config 1 into 29-35 stages and config 4 into
        // 28-30; the climbed tiles need 24 and 18 (VQB_PLAN_SEARCH=0: first fit).
        static const bool search = [] {
            const char *v = std::getenv("VQB_PLAN_SEARCH");
            return !(v && *v == '0');
        }();
        if (search) {
            const int gamma = knobs.gamma, gamma_window = std::max(1, knobs.window);
            const uint64_t all = pn >= 64 ? ~0ull : (1ull << pn) - 1;
            auto taken = [&](uint64_t T) {
                uint64_t bl = 0;
                int n = 0, w = 0, seen = 0;
                for (int i : remaining) {
                    const FusedOp &op = ops[i];
                    if (n < knobs.max_ops && !(op.support & bl) && op.fusable && (op.mixmask & ~T) == 0) {
                        ++n;
                        w += (op.mixmask ? 64 : 16) + (seen < gamma_window ? gamma * (gamma_window - seen) / gamma_window : 0);
                    } else {
                        bl |= op.support;
                        if ((bl & all) == all) break; // every qubit is behind a deferred operation
                    }
                    if (++seen >= 512) break;
                }
                return w;
            };
            uint64_t cand = 0;
            int seen = 0;
            for (int i : remaining) {
                cand |= ops[i].mixmask;
                if (++seen >= 160) break;
            }
            int best = taken(S);
            for (int iter = 0; iter < 12; ++iter) {
                uint64_t bestS = S;
                for (int bo = 0; bo < pn; ++bo) {
                    if (!(S >> bo & 1) || (lowmask >> bo & 1)) continue;
                    for (int bi = 0; bi < pn; ++bi) {
                        if ((S >> bi & 1) || !(cand >> bi & 1)) continue;
                        const uint64_t T = (S & ~(1ull << bo)) | (1ull << bi);
                        const int sc = taken(T);
                        if (sc > best) {
                            best = sc;
                            bestS = T;
                        }
                    }
                }
                if (bestS == S) break;
                S = bestS;
            }
            tile_score = best;
        }
        return S;
        };
        uint64_t S = build_tile(lowmask);
        // Other starting points: the tile seeded with one pending operation's
        // mixing bits. The first pending operations may be stragglers (config
        // 3's reverse sweep starts with one channel per qubit, and a tile grown
        // from four of them takes those four and nothing else); a tile grown
        // from an operation further along may take a whole chain, and the
        // stragglers ride with a later stage that holds their qubits anyway.
        if (knobs.seeds > 0 && tile_score > 0) {
            int best_score = tile_score, tried = 0;
            uint64_t seen_seed = 0;
            for (int i : remaining) {
                if (tried >= knobs.seeds) break;
                const uint64_t m = ops[i].mixmask & ~lowmask;
                if (!ops[i].fusable || !m || (m & ~seen_seed) == 0) continue;
                seen_seed |= m;
                if (__builtin_popcountll(lowmask | m) > k) continue;
                ++tried;
                const uint64_t T = build_tile(lowmask | m);
                if (tile_score > best_score) {
                    best_score = tile_score;
                    S = T;
                }
            }
        }
        uint64_t blocked = 0;
        // Pass 2: with the tile fixed, take every op that fits and is not
        // ordered behind a deferred op sharing a qubit.
        Stage st;
        st.k = k;
        int nb = 0;
        for (int b = 0; b < pn; ++b)
            if (S >> b & 1) st.bits[nb++] = b;
        std::vector<int> deferred;
        for (int i : remaining) {
            const FusedOp &op = ops[i];
            if ((int)st.ops.size() < knobs.max_ops && !(op.support & blocked) && op.fusable &&
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
