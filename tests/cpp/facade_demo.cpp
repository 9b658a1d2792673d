// Integration demo (TEST INFRASTRUCTURE): the reference's own C++ API next to
// the drop-in binding include/vqcs_b200.hpp. Builds a config-0-shaped ansatz
// and a noisy circuit with the reference builders, runs vqcs:: (CPU, the
// reference) and vqb:: (B200 through libvqcs_b200.so), and checks parity.
// Exit code 0 = parity within tolerance.
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>

#include "vqcs/autodiff.hpp"
#include "vqcs/bench_circuits.hpp"
#include "vqcs/io.hpp"
#include "vqcs/observables.hpp"
#include "vqcs_b200.hpp"

int main() {
    using namespace vqcs;
    const int n = 12;
    Circuit<double> c = bench::generate_rqc<double>(n, 4, 2024); // CNOT ladder + Ry, Rx
    const PauliOperator op = heisenberg_1d(n);
    const PureState<double> s0(n);
    const auto cfg = ThreadConfig::with_threads(4);

    const auto ref = vqcs::gradient_pure(op, c, s0, cfg);
    const auto dev = vqb::gradient_pure(op, c, s0);
    double gmax = 0, dmax = 0;
    for (size_t i = 0; i < ref.grads.size(); ++i) {
        gmax = std::max(gmax, std::abs(ref.grads[i]));
        dmax = std::max(dmax, std::abs(ref.grads[i] - dev.grads[i]));
    }
    const bool g_ok = dev.grads.size() == ref.grads.size() && dmax <= 1e-10 * gmax &&
                      std::abs(dev.loss - ref.loss) <= 1e-10 * std::abs(ref.loss);

    PureState<double> a(n), b(n);
    vqcs::apply_circuit(c, a, cfg);
    vqb::apply_circuit(c, b);
    double amax = 0;
    for (std::uint64_t k = 0; k < a.size(); ++k) amax = std::max(amax, std::abs(a[k] - b[k]));

    Circuit<double> noisy = bench::generate_noisy_rqc<double>(4, 2, 0.05, 11);
    const MixedState<double> dm0(4);
    const auto rn = vqcs::gradient_mixed(heisenberg_1d(4), noisy, dm0, cfg);
    const auto dn = vqb::gradient_mixed(heisenberg_1d(4), noisy, dm0);
    double nmax = 0, ngmax = 0;
    for (size_t i = 0; i < rn.grads.size(); ++i) {
        ngmax = std::max(ngmax, std::abs(rn.grads[i]));
        nmax = std::max(nmax, std::abs(rn.grads[i] - dn.grads[i]));
    }
    bool threw = false;
    try {
        Circuit<double> bad;
        bad.push_back(parametric_gate(GateKind::Rx, {1}, 0.4, true));
        bad.push_back(standard_channel(ChannelKind::AmplitudeDamping, 1, 1.0));
        PauliOperator z;
        z.add_term(PauliTerm({{1, PauliLabel::Z}}, 1.0));
        vqb::gradient_mixed(z, bad, MixedState<double>(1));
    } catch (const NonInvertibleChannelError &) {
        threw = true;
    }
    // fuse_gates (circuit.hpp:199-276): same gate list, same matrices
    const Circuit<double> fr = vqcs::fuse_gates(c), fd = vqb::fuse_gates(c);
    std::vector<GateOp<double>> gr, gd;
    fr.for_each_gate([&](const GateOp<double> &g) { gr.push_back(g); });
    fd.for_each_gate([&](const GateOp<double> &g) { gd.push_back(g); });
    double fmax = gr.size() == gd.size() ? 0 : 1;
    for (size_t i = 0; i < std::min(gr.size(), gd.size()); ++i) {
        if (gr[i].positions != gd[i].positions) fmax = 1;
        for (size_t k = 0; k < gr[i].matrix.size(); ++k)
            fmax = std::max(fmax, std::abs(gr[i].matrix[k] - gd[i].matrix[k]));
    }

    // measure (circuit.hpp:303-385): identical streams give identical outcomes
    std::mt19937_64 r1(77), r2(77);
    PureState<double> m1 = a, m2 = a;
    bool m_ok = true;
    double mmax = 0;
    for (int q = 1; q <= n; ++q) {
        const auto x = vqcs::measure(m1, q, r1);
        const auto y = vqb::measure(m2, q, r2);
        m_ok = m_ok && x.outcome == y.outcome && std::abs(x.probability - y.probability) <= 1e-12;
    }
    for (std::uint64_t k = 0; k < m1.size(); ++k) mmax = std::max(mmax, std::abs(m1[k] - m2[k]));

    // apply_circuit_copy over a batch of host states (one pipelined call)
    std::vector<PureState<double>> ins;
    for (int j = 0; j < 4; ++j) {
        PureState<double> x(n);
        vqcs::apply_circuit(bench::generate_rqc<double>(n, 1, 100 + j), x, cfg);
        ins.push_back(x);
    }
    const auto outs = vqb::apply_circuit_copy(c, ins);
    double bmax = outs.size() == ins.size() ? 0 : 1;
    for (size_t j = 0; j < ins.size() && j < outs.size(); ++j) {
        const PureState<double> r = vqcs::apply_circuit_copy(c, ins[j], cfg);
        for (std::uint64_t k = 0; k < r.size(); ++k) bmax = std::max(bmax, std::abs(r[k] - outs[j][k]));
    }

    // state dumps (io.hpp): a device dump loads back through the reference
    vqb::DeviceState ds(a);
    vqb::save_state(ds, "/tmp/vqb_facade_demo.vqcs");
    const LoadedState ls = vqcs::load_state(std::string("/tmp/vqb_facade_demo.vqcs"));
    double iomax = ls.num_qubits == n ? 0 : 1;
    for (std::uint64_t k = 0; k < a.size(); ++k) iomax = std::max(iomax, std::abs(ls.amplitudes[k] - a[k]));

    // the sharded state (four shards; on a one-GPU box all on device 0):
    // same circuit, same gradient as the unsharded reference
    const int ns = 14;
    Circuit<double> cs = bench::generate_rqc<double>(ns, 4, 77);
    const PauliOperator ops = heisenberg_1d(ns);
    vqb::ShardedState sh(ns, {0, 0, 0, 0});
    vqb::apply_circuit(cs, sh);
    PureState<double> rs(ns);
    vqcs::apply_circuit(cs, rs, cfg);
    std::vector<std::complex<double>> got(rs.size());
    sh.download(got);
    double smax = 0;
    for (std::uint64_t k = 0; k < rs.size(); ++k) smax = std::max(smax, std::abs(rs[k] - got[k]));
    const double se = std::abs(vqb::expectation(ops, sh) - vqcs::expectation(ops, rs, cfg));
    sh.set_zero();
    const auto sg = vqb::gradient_pure(ops, cs, sh);
    const auto rg = vqcs::gradient_pure(ops, cs, PureState<double>(ns), cfg);
    double sgmax = 0, rgmax = 0;
    for (size_t i = 0; i < rg.grads.size() && i < sg.grads.size(); ++i) {
        rgmax = std::max(rgmax, std::abs(rg.grads[i]));
        sgmax = std::max(sgmax, std::abs(rg.grads[i] - sg.grads[i]));
    }
    const bool sh_ok = smax <= 1e-12 && se <= 1e-12 && sg.grads.size() == rg.grads.size() &&
                       sgmax <= 1e-10 * rgmax && std::abs(sg.loss - rg.loss) <= 1e-10 * std::abs(rg.loss);

    std::printf("grad max|d|=%.3e (max|g|=%.3e) state max|d|=%.3e noisy max|d|=%.3e "
                "non-invertible->vqcs::NonInvertibleChannelError:%d fuse max|d|=%.3e "
                "measure outcomes equal:%d max|d|=%.3e dump max|d|=%.3e batch max|d|=%.3e "
                "sharded state max|d|=%.3e expectation |d|=%.3e gradient max|d|=%.3e\n",
                dmax, gmax, amax, nmax, threw, fmax, m_ok, mmax, iomax, bmax, smax, se, sgmax);
    return (g_ok && amax <= 1e-12 && nmax <= 1e-10 * ngmax && threw && fmax <= 1e-15 && m_ok &&
            mmax <= 1e-12 && iomax == 0 && bmax <= 1e-12 && sh_ok)
               ? 0
               : 1;
}
