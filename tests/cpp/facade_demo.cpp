// Integration demo (TEST INFRASTRUCTURE): the reference's own C++ API next to
// the drop-in binding include/vqcs_b200.hpp. Builds a config-0-shaped ansatz
// and a noisy circuit with the reference builders, runs vqcs:: (CPU, the
// reference) and vqb:: (B200 through libvqcs_b200.so), and checks parity.
// Exit code 0 = parity within tolerance.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "vqcs/autodiff.hpp"
#include "vqcs/bench_circuits.hpp"
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
    std::printf("grad max|d|=%.3e (max|g|=%.3e) state max|d|=%.3e noisy max|d|=%.3e "
                "non-invertible->vqcs::NonInvertibleChannelError:%d\n",
                dmax, gmax, amax, nmax, threw);
    return (g_ok && amax <= 1e-12 && nmax <= 1e-10 * ngmax && threw) ? 0 : 1;
}
