// BenchRecord reports (the reference harness's result records,
// src/bench.cpp:296-310 finish_stats and :329-369 emit_report): CSV rows
// "task,n,depth,threads,rep,seconds" with seconds printed like
// std::ostream at precision 12, or a JSON array with the field order task, n,
// depth, threads, seconds, mean_seconds, stddev_seconds, [speedup], params
// (2-space indentation; doubles as their shortest round-trip decimal, written
// like the JSON library the reference uses: fixed notation for decimal
// exponents in (-4, 15], "x.0" for integral values, otherwise d.ddde+XX;
// non-finite values as null). Output is byte-identical to the reference's
// (tests/test_next_rows.py compares the two on the same records).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>

#include "common.hpp"

namespace vqb {

namespace {

std::string g12(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.12g", v);
    return b;
}

// shortest digits d1..dn and exponent e with v = 0.d1..dn x 10^e
void shortest(double v, std::string &digits, int &point) {
    char b[64];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(b, sizeof b, "%.*e", p - 1, v);
        if (std::strtod(b, nullptr) == v) break;
    }
    // b = "d.ddde[+-]XX"
    const char *e = std::strchr(b, 'e');
    digits.clear();
    for (const char *c = b; c < e; ++c)
        if (*c >= '0' && *c <= '9') digits += *c;
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    point = std::atoi(e + 1) + 1; // decimal point after `point` digits
}

std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
    std::string out = v < 0 ? "-" : "";
    std::string d;
    int n;
    shortest(std::fabs(v), d, n);
    const int k = (int)d.size();
    if (k <= n && n <= 15) { // integral: digits, zeros, ".0"
        out += d + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += d.substr(0, size_t(n)) + "." + d.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(size_t(-n), '0') + d;
    } else {
        out += d.substr(0, 1);
        if (k > 1) out += "." + d.substr(1);
        const int ex = n - 1;
        char b[16];
        std::snprintf(b, sizeof b, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
        out += b;
    }
    return out;
}

std::string json_string(const char *s) {
    std::string o = "\"";
    for (const unsigned char *c = reinterpret_cast<const unsigned char *>(s); *c; ++c) {
        switch (*c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        default:
            if (*c < 0x20) {
                char b[8];
                std::snprintf(b, sizeof b, "\\u%04x", *c);
                o += b;
            } else {
                o += char(*c);
            }
        }
    }
    return o + "\"";
}

} // namespace

std::string bench_report(const vqb_bench_record *recs, int64_t count, int format) {
    if (count <= 0) raise(VQB_ERR_USAGE, "emit_report: no records to write");
    std::string out;
    if (format == 1) {
        out = "task,n,depth,threads,rep,seconds\n";
        for (int64_t i = 0; i < count; ++i) {
            const vqb_bench_record &r = recs[i];
            for (int64_t k = 0; k < r.num_seconds; ++k)
                out += std::string(r.task) + "," + std::to_string(r.num_qubits) + "," + std::to_string(r.depth) +
                       "," + std::to_string(r.threads) + "," + std::to_string(k) + "," + g12(r.seconds[k]) + "\n";
        }
        return out;
    }
    out = "[\n";
    for (int64_t i = 0; i < count; ++i) {
        const vqb_bench_record &r = recs[i];
        // finish_stats: mean and population standard deviation
        double mean = 0, sd = 0;
        if (r.num_seconds > 0) {
            double sum = 0;
            for (int64_t k = 0; k < r.num_seconds; ++k) sum += r.seconds[k];
            mean = sum / double(r.num_seconds);
            double sq = 0;
            for (int64_t k = 0; k < r.num_seconds; ++k) sq += (r.seconds[k] - mean) * (r.seconds[k] - mean);
            sd = std::sqrt(sq / double(r.num_seconds));
        }
        out += "  {\n    \"task\": " + json_string(r.task) + ",\n    \"n\": " + std::to_string(r.num_qubits) +
               ",\n    \"depth\": " + std::to_string(r.depth) + ",\n    \"threads\": " + std::to_string(r.threads) +
               ",\n    \"seconds\": ";
        if (r.num_seconds == 0) {
            out += "[]";
        } else {
            out += "[\n";
            for (int64_t k = 0; k < r.num_seconds; ++k)
                out += "      " + json_double(r.seconds[k]) + (k + 1 < r.num_seconds ? ",\n" : "\n");
            out += "    ]";
        }
        out += ",\n    \"mean_seconds\": " + json_double(mean) + ",\n    \"stddev_seconds\": " + json_double(sd);
        if (r.speedup != 0) out += ",\n    \"speedup\": " + json_double(r.speedup);
        // params in key order (std::map)
        std::map<std::string, std::string> info;
        for (int64_t k = 0; k < r.num_info; ++k) info[r.info_keys[k]] = r.info_values[k];
        out += ",\n    \"params\": ";
        if (info.empty()) {
            out += "{}";
        } else {
            out += "{\n";
            size_t j = 0;
            for (const auto &kv : info)
                out += "      " + json_string(kv.first.c_str()) + ": " + json_string(kv.second.c_str()) +
                       (++j < info.size() ? ",\n" : "\n");
            out += "    }";
        }
        out += std::string("\n  }") + (i + 1 < count ? ",\n" : "\n");
    }
    return out + "]\n";
}

} // namespace vqb
