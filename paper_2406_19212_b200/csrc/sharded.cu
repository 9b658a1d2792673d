// Single-process multi-device sharded state (see sharded.hpp).
#include "sharded.hpp"

#include <algorithm>
#include <cstring>

#include "plan.hpp"

namespace vqb {

namespace {

constexpr int kMaxSwapBits = 4; // P <= 16

struct SwapArgs {
    int k;
    int l[kMaxSwapBits]; // local bit positions, ascending
};

// mine[i | sel_m] <-> theirs[i | sel_t] for the j-th index i (j in [j0, j1))
// with zero local bits at args.l: one 16-B amplitude each way per thread and
// iteration; `theirs` is the peer shard (another device: NVLink loads and
// stores through peer access).
__global__ void k_swap_peer(double2 *__restrict__ mine, double2 *__restrict__ theirs, uint64_t j0,
                            uint64_t j1, SwapArgs args, uint64_t sel_m, uint64_t sel_t) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = j0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < j1; j += stride) {
        uint64_t i = j;
#pragma unroll
        for (int q = 0; q < kMaxSwapBits; ++q)
            if (q < args.k) i = ((i >> args.l[q]) << (args.l[q] + 1)) | (i & ((1ull << args.l[q]) - 1));
        const double2 a = mine[i | sel_m];
        const double2 b = theirs[i | sel_t];
        mine[i | sel_m] = b;
        theirs[i | sel_t] = a;
    }
}

// rows/cols of the local bits not in `fixed` (bit b fixed to vals bit b);
// the fixed bits must be non-mixing
cvec restrict_matrix(const cvec &M, int m, unsigned fixed, unsigned vals) {
    const int d = 1 << m;
    std::vector<int> keep;
    for (int b = 0; b < m; ++b)
        if (!((fixed >> b) & 1)) keep.push_back(b);
    const int dk = 1 << keep.size();
    std::vector<int> idx(dk);
    for (int k = 0; k < dk; ++k) {
        int i = (int)(vals & fixed);
        for (size_t q = 0; q < keep.size(); ++q)
            if ((k >> q) & 1) i |= 1 << keep[q];
        idx[k] = i;
    }
    cvec out(size_t(dk) * dk);
    for (int c = 0; c < dk; ++c)
        for (int r = 0; r < dk; ++r) out[r + size_t(c) * dk] = M[idx[r] + size_t(idx[c]) * d];
    return out;
}

std::vector<int> mixing_bits(const Gate &phys_gate) {
    const FusedOp f = analyse_gate(phys_gate);
    std::vector<int> out;
    if (!f.fusable) { // wider than the planner's analysis: every position mixes
        for (int q = 0; q < phys_gate.m; ++q) out.push_back(phys_gate.pos[q] - 1);
        return out;
    }
    for (int q = 0; q < f.nt; ++q) out.push_back(f.mix[q]);
    return out;
}

void barrier(Sharded *s) {
    // follower shards' streams first join their main shard's stream
    for (const auto &set : s->followers)
        for (int r = 0; r < s->P; ++r) {
            DevScope on(s->devs[r]);
            VQB_CUDA(cudaEventRecord(s->events[r], set[r]->stream));
            VQB_CUDA(cudaStreamWaitEvent(s->shards[r]->stream, s->events[r], 0));
        }
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        VQB_CUDA(cudaEventRecord(s->events[r], s->shards[r]->stream));
    }
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        for (int q = 0; q < s->P; ++q)
            if (q != r) VQB_CUDA(cudaStreamWaitEvent(s->shards[r]->stream, s->events[q], 0));
        for (const auto &set : s->followers) VQB_CUDA(cudaStreamWaitEvent(set[r]->stream, s->events[r], 0));
    }
}

} // namespace

Sharded *sharded_create(int n, int P, const int *devices) {
    if (P < 1 || (P & (P - 1)) || P > (1 << kMaxSwapBits))
        raise(VQB_ERR_UNSUPPORTED, "sharded state: the device count must be a power of two <= 16");
    int g = 0;
    while ((1 << g) < P) ++g;
    if (n - g < 12) raise(VQB_ERR_SIZE, "sharded state: at least 12 local qubits per shard");
    int ndev = 0;
    VQB_CUDA(cudaGetDeviceCount(&ndev));
    for (int r = 0; r < P; ++r)
        if (devices[r] < 0 || devices[r] >= ndev)
            raise(VQB_ERR_INDEX, "sharded state: device " + std::to_string(devices[r]) + " does not exist");
    // peer access between every pair of distinct devices (NVLink / NVSwitch)
    for (int a = 0; a < P; ++a)
        for (int b = 0; b < P; ++b) {
            if (devices[a] == devices[b]) continue;
            int ok = 0;
            VQB_CUDA(cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]));
            if (!ok)
                raise(VQB_ERR_UNSUPPORTED, "sharded state: no peer access from device " +
                                               std::to_string(devices[a]) + " to " + std::to_string(devices[b]));
            DevScope on(devices[a]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else VQB_CUDA(e);
        }
    auto *s = new Sharded();
    s->n = n;
    s->g = g;
    s->n_loc = n - g;
    s->P = P;
    s->devs.assign(devices, devices + P);
    s->log2phys.resize(n);
    for (int q = 0; q < n; ++q) s->log2phys[q] = q;
    try {
        for (int r = 0; r < P; ++r) {
            DevScope on(devices[r]);
            DeviceState *d = state_create(s->n_loc, 0);
            d->global_offset = uint64_t(r) << s->n_loc;
            d->global_qubits = g;
            s->shards.push_back(d);
            cudaEvent_t ev;
            VQB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            s->events.push_back(ev);
        }
        sharded_set_zero(s);
    } catch (...) {
        sharded_destroy(s);
        throw;
    }
    return s;
}

void sharded_destroy(Sharded *s) {
    if (!s) return;
    for (size_t r = 0; r < s->shards.size(); ++r) state_destroy(s->shards[r]);
    for (size_t r = 0; r < s->events.size(); ++r) {
        DevScope on(s->devs[r]);
        cudaEventDestroy(s->events[r]);
    }
    delete s;
}

void sharded_sync(Sharded *s) {
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        sync(s->shards[r]);
    }
}

void sharded_set_zero(Sharded *s) {
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        state_set_zero(s->shards[r]); // amplitude 0 = 1 only in shard 0 (global_offset 0)
    }
    for (int q = 0; q < s->n; ++q) s->log2phys[q] = q;
}

void sharded_swap(Sharded *s, const std::vector<std::pair<int, int>> &pairs_in) {
    if (pairs_in.empty()) return;
    std::vector<std::pair<int, int>> pairs = pairs_in;
    std::sort(pairs.begin(), pairs.end(), [](auto &x, auto &y) { return x.second < y.second; });
    const int k = (int)pairs.size();
    if (k > s->g) raise(VQB_ERR_INTERNAL, "sharded swap: more pairs than global bits");
    SwapArgs args{};
    args.k = k;
    int G[kMaxSwapBits];
    for (int i = 0; i < k; ++i) {
        G[i] = pairs[i].first - s->n_loc;
        args.l[i] = pairs[i].second;
        if (G[i] < 0 || G[i] >= s->g || args.l[i] < 0 || args.l[i] >= s->n_loc)
            raise(VQB_ERR_INTERNAL, "sharded swap: bad bit pair");
    }
    auto value_at_G = [&](int r) {
        int a = 0;
        for (int i = 0; i < k; ++i) a |= ((r >> G[i]) & 1) << i;
        return a;
    };
    auto sel = [&](int v) {
        uint64_t m = 0;
        for (int i = 0; i < k; ++i)
            if ((v >> i) & 1) m |= 1ull << args.l[i];
        return m;
    };
    barrier(s);
    const uint64_t count = 1ull << (s->n_loc - k);
    const uint64_t half = count / 2;
    for (int r = 0; r < s->P; ++r) {
        const int a = value_at_G(r);
        for (int b = a + 1; b < (1 << k); ++b) {
            int r2 = r;
            for (int i = 0; i < k; ++i) r2 = (r2 & ~(1 << G[i])) | (((b >> i) & 1) << G[i]);
            // shard r's elements with local value b <-> shard r2's with value a;
            // each device moves half of the range
            const struct {
                int who, peer;
                uint64_t j0, j1, sm, st;
            } parts[2] = {{r, r2, 0, half, sel(b), sel(a)}, {r2, r, half, count, sel(a), sel(b)}};
            for (size_t set = 0; set <= s->followers.size(); ++set) {
                const std::vector<DeviceState *> &sh = set == 0 ? s->shards : s->followers[set - 1];
                for (const auto &p : parts) {
                    DevScope on(s->devs[p.who]);
                    DeviceState *me = s->shards[p.who]; // its stream orders every set's swap
                    const ProfMark pf = prof_begin(me->stream);
                    k_swap_peer<<<148 * 4, 256, 0, me->stream>>>(sh[p.who]->amps, sh[p.peer]->amps, p.j0, p.j1,
                                                                 args, p.sm, p.st);
                    check_launch("k_swap_peer", pf);
                }
                s->bytes_moved += 2 * count * sizeof(double2);
            }
        }
    }
    barrier(s);
    for (const auto &pr : pairs) {
        const int x = (int)(std::find(s->log2phys.begin(), s->log2phys.end(), pr.first) - s->log2phys.begin());
        const int y = (int)(std::find(s->log2phys.begin(), s->log2phys.end(), pr.second) - s->log2phys.begin());
        s->log2phys[x] = pr.second;
        s->log2phys[y] = pr.first;
    }
    ++s->rounds;
    s->bits_swapped += k;
}

namespace {

// Bring the global bits `need` local in one round, together with the global
// mixing bits of the upcoming operations while free local bits last; local
// partners avoid `avoid` and the upcoming operations' mixing bits, highest
// first (long contiguous runs for the peer copies).
void bring_local(Sharded *s, const std::vector<int> &need, const std::vector<std::vector<int>> &upcoming,
                 const std::vector<int> &avoid) {
    std::vector<int> soon;
    for (const auto &v : upcoming) soon.insert(soon.end(), v.begin(), v.end());
    auto has = [](const std::vector<int> &v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); };
    std::vector<int> want;
    for (int b : need)
        if (!has(want, b)) want.push_back(b);
    for (const auto &v : upcoming)
        for (int b : v)
            if (b >= s->n_loc && !has(want, b)) want.push_back(b);
    std::vector<int> fresh, rest;
    for (int l = s->n_loc - 1; l >= 0; --l) {
        if (has(avoid, l)) continue;
        (has(soon, l) ? rest : fresh).push_back(l);
    }
    std::vector<std::pair<int, int>> pairs;
    size_t fi = 0, ri = 0;
    for (int gb : want) {
        if (fi < fresh.size()) pairs.push_back({gb, fresh[fi++]});
        else if (has(need, gb) && ri < rest.size()) pairs.push_back({gb, rest[ri++]});
    }
    sharded_swap(s, pairs);
}

Gate physical(const Sharded *s, const Gate &g) {
    Gate p = g;
    for (int q = 0; q < g.m; ++q) p.pos[q] = s->log2phys[g.pos[q] - 1] + 1;
    return p;
}

} // namespace

void sharded_apply_circuit(Sharded *s, const vqb_op *ops, int64_t count) {
    const auto es = build_elements(ops, count);
    std::vector<Gate> gates;
    for (const auto &e : es) {
        if (e.channel)
            raise(VQB_ERR_TYPE, "apply_circuit: a quantum channel cannot act on a pure state; use a MixedState");
        check_fit(e.gate.pos, e.gate.m, s->n);
        gates.push_back(e.gate);
    }
    std::vector<std::vector<Gate>> batch(s->P);
    auto flush = [&] {
        for (int r = 0; r < s->P; ++r) {
            if (batch[r].empty()) continue;
            DevScope on(s->devs[r]);
            run_program(s->shards[r], batch[r], true); // asynchronous on the shard's stream
            batch[r].clear();
        }
    };
    for (size_t i = 0; i < gates.size(); ++i) {
        Gate pg = physical(s, gates[i]);
        std::vector<int> need;
        for (int b : mixing_bits(pg))
            if (b >= s->n_loc) need.push_back(b);
        if (!need.empty()) {
            flush();
            std::vector<std::vector<int>> upcoming;
            for (size_t j = i + 1; j < gates.size() && j <= i + (size_t)s->lookahead; ++j)
                upcoming.push_back(mixing_bits(physical(s, gates[j])));
            std::vector<int> avoid;
            for (int q = 0; q < pg.m; ++q) avoid.push_back(pg.pos[q] - 1);
            bring_local(s, need, upcoming, avoid);
            pg = physical(s, gates[i]);
        }
        // restrict the global (condition) bits to each shard's values
        unsigned fixed = 0;
        for (int q = 0; q < pg.m; ++q)
            if (pg.pos[q] - 1 >= s->n_loc) fixed |= 1u << q;
        for (int r = 0; r < s->P; ++r) {
            Gate lg;
            lg.kind = VQB_GATE_GENERIC;
            if (!fixed) {
                lg = pg;
                lg.np = 0;
            } else {
                unsigned vals = 0;
                for (int q = 0; q < pg.m; ++q)
                    if ((fixed >> q) & 1) vals |= (unsigned)((r >> (pg.pos[q] - 1 - s->n_loc)) & 1) << q;
                const cvec sub = restrict_matrix(pg.mat, pg.m, fixed, vals);
                int nk = 0;
                for (int q = 0; q < pg.m; ++q)
                    if (!((fixed >> q) & 1)) lg.pos[nk++] = pg.pos[q];
                if (nk == 0) { // fully global diagonal: this shard's scalar
                    if (sub[0] == cplx(1)) continue;
                    lg.m = 1;
                    lg.pos[0] = 1;
                    lg.mat = {sub[0], 0.0, 0.0, sub[0]};
                } else {
                    lg.m = nk;
                    lg.mat = sub;
                    bool ident = true;
                    const int d = 1 << nk;
                    for (int a = 0; a < d && ident; ++a)
                        for (int b = 0; b < d; ++b)
                            if (sub[a + size_t(b) * d] != (a == b ? cplx(1) : cplx(0))) {
                                ident = false;
                                break;
                            }
                    if (ident) continue;
                }
            }
            batch[r].push_back(std::move(lg));
        }
    }
    flush();
    sharded_sync(s);
}

void sharded_canonicalize(Sharded *s) {
    auto where = [&](int logical) { return s->log2phys[logical]; };
    // global positions: logical p must sit at physical p
    for (int p = s->n_loc; p < s->n; ++p) {
        int cur = where(p);
        if (cur == p) continue;
        if (cur >= s->n_loc) { // on another global bit: bring it local first
            int l = s->n_loc - 1;
            sharded_swap(s, {{cur, l}});
            cur = where(p);
        }
        sharded_swap(s, {{p, cur}});
    }
    // local positions: transpositions by SWAP gates on every shard
    std::vector<Gate> swaps;
    for (int l = 0; l < s->n_loc; ++l) {
        const int cur = where(l);
        if (cur == l) continue;
        Gate g;
        g.kind = VQB_GATE_SWAP;
        g.m = 2;
        g.pos[0] = l + 1;
        g.pos[1] = cur + 1;
        g.mat.assign(16, cplx(0));
        g.mat[0] = g.mat[1 + 2 * 4] = g.mat[2 + 1 * 4] = g.mat[15] = 1.0;
        swaps.push_back(g);
        const int other = (int)(std::find(s->log2phys.begin(), s->log2phys.end(), l) - s->log2phys.begin());
        s->log2phys[other] = cur;
        s->log2phys[l] = l;
    }
    if (!swaps.empty())
        for (int r = 0; r < s->P; ++r) {
            DevScope on(s->devs[r]);
            run_program(s->shards[r], swaps, true);
        }
    sharded_sync(s);
}

void sharded_save(Sharded *s, const char *path) {
    sharded_canonicalize(s);
    save_segments(path, s->n, s->shards);
}

void sharded_load(Sharded *s, const char *path, int *precision) {
    sharded_sync(s);
    load_segments(path, s->n, s->shards, precision);
    for (int q = 0; q < s->n; ++q) s->log2phys[q] = q;
}

namespace {
// The Pauli sum as seen from destination shard r: terms grouped by the
// global part xg of their X mask (X and Y factors on global qubits). A term
// of group xg maps the amplitudes of shard r ^ xg onto shard r; its Z and Y
// factors on global qubits become the sign (-1)^popc((r ^ xg) & zg) of the
// SOURCE shard and Y's factor i, folded into the coefficient; the local
// factors stay (pack_operator handles them as for an unsharded state).
struct CrossPack {
    int xg;
    PauliPack pack;
};
std::vector<CrossPack> cross_packs(const Sharded *s, int r, const vqb_pauli_term *terms, int64_t nterms) {
    std::vector<int> order;
    std::vector<std::vector<vqb_pauli_term>> lt;
    std::vector<std::vector<int32_t>> qs(nterms);
    std::vector<std::string> ls(nterms);
    static const cplx ipow[4] = {1.0, cplx(0, 1), -1.0, cplx(0, -1)};
    for (int64_t t = 0; t < nterms; ++t) {
        int xg = 0, zg = 0, ny = 0;
        for (int k = 0; k < terms[t].num_factors; ++k) {
            const int q = terms[t].qubits[k];
            if (q < 1 || q > s->n) raise(VQB_ERR_INDEX, "expectation: operator acts on qubit " + std::to_string(q));
            const char l = terms[t].labels[k] | 0x20;
            if (l != 'x' && l != 'y' && l != 'z')
                raise(VQB_ERR_VALIDITY, std::string("unknown Pauli label '") + terms[t].labels[k] + "'");
            const int p = s->log2phys[q - 1];
            if (p >= s->n_loc) {
                const int bit = 1 << (p - s->n_loc);
                if (l == 'x' || l == 'y') xg |= bit;
                if (l == 'y' || l == 'z') zg |= bit;
                if (l == 'y') ++ny;
            } else {
                qs[t].push_back(p + 1);
                ls[t].push_back(terms[t].labels[k]);
            }
        }
        const double sign = (__builtin_popcount((unsigned)((r ^ xg) & zg)) & 1) ? -1.0 : 1.0;
        const cplx c = cplx(terms[t].coeff.re, terms[t].coeff.im) * ipow[ny & 3] * sign;
        vqb_pauli_term u;
        u.coeff.re = c.real();
        u.coeff.im = c.imag();
        u.num_factors = (int32_t)qs[t].size();
        u.qubits = qs[t].data();
        u.labels = ls[t].data();
        size_t g = std::find(order.begin(), order.end(), xg) - order.begin();
        if (g == order.size()) {
            order.push_back(xg);
            lt.emplace_back();
        }
        lt[g].push_back(u);
    }
    std::vector<CrossPack> out;
    for (size_t g = 0; g < order.size(); ++g)
        out.push_back({order[g], pack_operator(lt[g].data(), (int64_t)lt[g].size(), false)});
    return out;
}

// the reverse step of element g restricted to shard r: positions on local
// bits, matrices with the global (condition) bits fixed; false = identity
bool local_step(const Sharded *s, int r, const Gate &pg, const cvec &inv, const std::vector<cvec> &dmats,
                RevOp &out) {
    unsigned fixed = 0, vals = 0;
    for (int q = 0; q < pg.m; ++q) {
        const int b = pg.pos[q] - 1;
        if (b >= s->n_loc) {
            fixed |= 1u << q;
            vals |= (unsigned)((r >> (b - s->n_loc)) & 1) << q;
        }
    }
    int nk = 0;
    Gate g;
    g.kind = VQB_GATE_GENERIC;
    for (int q = 0; q < pg.m; ++q)
        if (!((fixed >> q) & 1)) g.pos[nk++] = pg.pos[q];
    auto sub = [&](const cvec &M) { return fixed ? restrict_matrix(M, pg.m, fixed, vals) : M; };
    if (nk == 0) { // fully global diagonal: scalars, applied as a 1-bit op on bit 0
        g.m = 1;
        g.pos[0] = 1;
        const cplx a = sub(inv)[0];
        g.mat = {a, 0.0, 0.0, a};
        out.phi_op = out.psi_op = g;
        out.dmats.clear();
        for (const cvec &d : dmats) {
            const cplx x = sub(d)[0];
            out.dmats.push_back({x, 0.0, 0.0, x});
        }
        return true;
    }
    g.m = nk;
    g.mat = sub(inv);
    out.phi_op = out.psi_op = g;
    out.dmats.clear();
    for (const cvec &d : dmats) out.dmats.push_back(sub(d));
    if (out.dmats.empty()) {
        const int d = 1 << nk;
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b)
                if (g.mat[a + size_t(b) * d] != (a == b ? cplx(1) : cplx(0))) return true;
        return false;
    }
    return true;
}
} // namespace

ShardedGradient sharded_gradient_pure(Sharded *s, const vqb_op *ops, int64_t count,
                                      const vqb_pauli_term *terms, int64_t nterms) {
    const auto es = build_elements(ops, count);
    std::vector<int64_t> base(count);
    int64_t total = 0;
    for (int64_t i = 0; i < count; ++i) {
        if (es[i].channel) raise(VQB_ERR_TYPE, "gradient_pure: noisy circuits need gradient_mixed");
        check_fit(es[i].gate.pos, es[i].gate.m, s->n);
        base[i] = total;
        total += es[i].gate.num_active();
    }
    ShardedGradient out;
    sharded_apply_circuit(s, ops, count);
    out.loss = sharded_expectation(s, terms, nterms).real();
    out.grads.assign(total, 0.0);
    if (total == 0) return out;
    // Psi = H |Phi>, shard by shard
    std::vector<DeviceState *> psi(s->P, nullptr);
    struct Guard {
        Sharded *s;
        std::vector<DeviceState *> &psi;
        ~Guard() {
            s->followers.clear();
            for (DeviceState *d : psi) state_destroy(d);
        }
    } guard{s, psi};
    std::vector<double *> dgrads(s->P, nullptr);
    static thread_local DevMem gbuf[kMaxDevices * 2];
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        psi[r] = state_create(s->n_loc, 0);
        VQB_CUDA(cudaStreamSynchronize(psi[r]->stream));
        // Psi_r = sum over term groups of H_(r, xg) Phi_(r ^ xg)
        bool first = true;
        for (const CrossPack &cp : cross_packs(s, r, terms, nterms)) {
            apply_operator_from(s->shards[r], s->shards[r ^ cp.xg]->amps, psi[r]->amps, cp.pack, !first);
            first = false;
        }
        // per-shard device gradient vector (shards on one device get their own)
        int slot = 0;
        for (int q = 0; q < r; ++q) slot += s->devs[q] == s->devs[r];
        DevMem &m = gbuf[std::min(slot, kMaxDevices * 2 - 1)];
        m.ensure(sizeof(double) * (size_t)total + 16);
        dgrads[r] = static_cast<double *>(m.p);
        VQB_CUDA(cudaMemsetAsync(dgrads[r], 0, sizeof(double) * (size_t)total, s->shards[r]->stream));
        VQB_CUDA(cudaStreamSynchronize(s->shards[r]->stream)); // psi is read on the shard's stream below
    }
    s->followers.push_back(psi);
    barrier(s); // the costates read partner shards: done before any shard changes
    std::vector<std::vector<RevOp>> batch(s->P);
    auto flush = [&] {
        for (int r = 0; r < s->P; ++r) {
            if (batch[r].empty()) continue;
            DevScope on(s->devs[r]);
            // the adjoint executor's scratch is per thread and device: shards
            // sharing a device (the one-GPU test layout) take turns
            for (int q = 0; q < r; ++q)
                if (s->devs[q] == s->devs[r]) VQB_CUDA(cudaStreamSynchronize(s->shards[q]->stream));
            run_reverse(s->shards[r], psi[r], batch[r], dgrads[r], true);
            batch[r].clear();
        }
    };
    auto step_mix = [&](const Gate &pg, const cvec &inv, const std::vector<cvec> &dm) {
        Gate t = pg;
        std::vector<int> mix;
        t.mat = inv;
        for (int b : mixing_bits(t)) mix.push_back(b);
        for (const cvec &d : dm) {
            t.mat = d;
            for (int b : mixing_bits(t))
                if (std::find(mix.begin(), mix.end(), b) == mix.end()) mix.push_back(b);
        }
        return mix;
    };
    for (int64_t i = count; i-- > 0;) {
        const Gate &g = es[i].gate;
        const cvec inv = gate_inverse(g).mat;
        std::vector<cvec> dm;
        for (int p = 0; p < g.np; ++p)
            if (g.is_param[p]) dm.push_back(gate_derivative(g, p));
        Gate pg = physical(s, g);
        std::vector<int> need;
        for (int b : step_mix(pg, inv, dm))
            if (b >= s->n_loc) need.push_back(b);
        if (!need.empty()) {
            flush();
            std::vector<std::vector<int>> upcoming;
            for (int64_t j = i - 1; j >= 0 && j >= i - s->lookahead; --j) {
                const Gate &h = es[j].gate;
                std::vector<cvec> hd;
                for (int p = 0; p < h.np; ++p)
                    if (h.is_param[p]) hd.push_back(gate_derivative(h, p));
                upcoming.push_back(step_mix(physical(s, h), gate_inverse(h).mat, hd));
            }
            std::vector<int> avoid;
            for (int q = 0; q < pg.m; ++q) avoid.push_back(pg.pos[q] - 1);
            bring_local(s, need, upcoming, avoid);
            pg = physical(s, g);
        }
        for (int r = 0; r < s->P; ++r) {
            RevOp op;
            if (!local_step(s, r, pg, inv, dm, op)) continue;
            if (!op.dmats.empty()) {
                op.grad_base = base[i];
                op.scale = 2.0; // grads = 2 Re(acc) (autodiff.hpp:147-149)
            }
            batch[r].push_back(std::move(op));
        }
    }
    flush();
    std::vector<double> h((size_t)total);
    for (int r = 0; r < s->P; ++r) { // shard order: deterministic
        DevScope on(s->devs[r]);
        VQB_CUDA(cudaMemcpyAsync(h.data(), dgrads[r], sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost,
                                 s->shards[r]->stream));
        VQB_CUDA(cudaStreamSynchronize(s->shards[r]->stream));
        for (int64_t k = 0; k < total; ++k) out.grads[(size_t)k] += h[(size_t)k];
    }
    sharded_sync(s);
    return out;
}

double sharded_norm(Sharded *s) {
    double acc = 0;
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        acc += norm_sq(s->shards[r]); // shard order: deterministic
    }
    return std::sqrt(acc);
}

cplx sharded_expectation(Sharded *s, const vqb_pauli_term *terms, int64_t nterms) {
    // every term group reads its ket from the partner shard r ^ xg (peer
    // memory across devices): no exchange round, the layout is unchanged
    barrier(s);
    cplx acc = 0;
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        for (const CrossPack &cp : cross_packs(s, r, terms, nterms))
            acc += expectation_cross(s->shards[r], s->shards[r ^ cp.xg]->amps, cp.pack); // shard order
    }
    return acc;
}

namespace {
// physical index of the amplitude with logical index L
uint64_t phys_index(const Sharded *s, uint64_t L) {
    uint64_t p = 0;
    for (int q = 0; q < s->n; ++q) p |= ((L >> q) & 1) << s->log2phys[q];
    return p;
}
} // namespace

void sharded_download(Sharded *s, vqb_c128 *host, uint64_t count) {
    if (count != (1ull << s->n)) raise(VQB_ERR_SHAPE, "sharded download: count does not match 2^n");
    std::vector<double2> phys(count);
    const uint64_t ls = 1ull << s->n_loc;
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        VQB_CUDA(cudaMemcpyAsync(phys.data() + r * ls, s->shards[r]->amps, sizeof(double2) * ls,
                                 cudaMemcpyDeviceToHost, s->shards[r]->stream));
        sync(s->shards[r]);
    }
    for (uint64_t L = 0; L < count; ++L) {
        const double2 v = phys[phys_index(s, L)];
        host[L].re = v.x;
        host[L].im = v.y;
    }
}

void sharded_upload(Sharded *s, const vqb_c128 *host, uint64_t count) {
    if (count != (1ull << s->n)) raise(VQB_ERR_SHAPE, "sharded upload: count does not match 2^n");
    for (int q = 0; q < s->n; ++q) s->log2phys[q] = q; // canonical layout
    const uint64_t ls = 1ull << s->n_loc;
    for (int r = 0; r < s->P; ++r) {
        DevScope on(s->devs[r]);
        VQB_CUDA(cudaMemcpyAsync(s->shards[r]->amps, host + r * ls, sizeof(double2) * ls,
                                 cudaMemcpyHostToDevice, s->shards[r]->stream));
        sync(s->shards[r]);
    }
}

} // namespace vqb
