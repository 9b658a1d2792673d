// TEST INFRASTRUCTURE ONLY: the reference harness's own emit_report
// (src/bench.cpp, compiled from /root/reference with its JSON library) as a
// small executable, so tests/test_next_rows.py can compare the product's
// vqb_bench_report byte for byte. (A separate process: the harness's
// iostream formatting crashed when its library was dlopen'ed into Python.)
//
// stdin: the format ("json" | "csv") on the first line, then one record per
// line, fields separated by spaces, strings hex-encoded:
//   task n depth threads speedup nsec s1 .. s_nsec ninfo k1 v1 .. (doubles as %a)
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "vqcs/bench.hpp"

static std::string unhex(const std::string &h) {
    std::string s;
    for (size_t i = 0; i + 1 < h.size(); i += 2) s += char(std::stoi(h.substr(i, 2), nullptr, 16));
    return s;
}

int main() {
    std::string fmt, line;
    std::getline(std::cin, fmt);
    std::vector<vqcs::bench::BenchRecord> rs;
    while (std::getline(std::cin, line)) {
        if (line.empty()) continue;
        std::istringstream in(line);
        vqcs::bench::BenchRecord r;
        std::string task, sp;
        size_t ns = 0, ni = 0;
        in >> task >> r.num_qubits >> r.depth >> r.threads >> sp >> ns;
        r.task = unhex(task);
        r.speedup = std::strtod(sp.c_str(), nullptr);
        for (size_t k = 0; k < ns; ++k) {
            std::string v;
            in >> v;
            r.seconds.push_back(std::strtod(v.c_str(), nullptr));
        }
        in >> ni;
        for (size_t k = 0; k < ni; ++k) {
            std::string a, b;
            in >> a >> b;
            r.info[unhex(a)] = unhex(b);
        }
        r.finish_stats();
        rs.push_back(std::move(r));
    }
    vqcs::bench::emit_report(rs, fmt == "csv" ? vqcs::bench::ReportFormat::Csv : vqcs::bench::ReportFormat::Json,
                             std::cout);
    return 0;
}
