// Raw state dumps in the reference's "VQCS" v1 format (io.hpp:15-20):
//   "VQCS" | u32 version (= 1) | u32 qubit count | u8 precision
//   | 2^n little-endian (re, im) double pairs in flat amplitude order.
// The payload layout is exactly the device layout (double2), so a dump is a
// chunked device->pinned->file stream (and the reverse for a load); the
// whole state never needs a pageable host copy.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "device.hpp"

namespace vqb {

namespace {

constexpr char kMagic[4] = {'V', 'Q', 'C', 'S'};
constexpr uint32_t kVersion = 1;        // io.hpp:38
constexpr uint8_t kPrecisionDouble = 2; // Precision::ComplexDouble
constexpr size_t kChunk = size_t(64) << 20;

struct File {
    FILE *f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// Pinned staging chunk, grown on demand and kept per thread.
struct Pinned {
    void *p = nullptr;
    size_t cap = 0;
    void *get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            VQB_CUDA(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return p;
    }
};
thread_local Pinned g_chunk;

} // namespace

// save_state (io.hpp:56-82) over one or more device segments written back to
// back (a sharded state in canonical layout: shard 0, shard 1, ...)
void save_segments(const char *path, int n, const std::vector<DeviceState *> &segs) {
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) raise(VQB_ERR_IO, std::string("save_state: cannot open '") + path + "' for writing");
    const uint32_t version = kVersion, nq = (uint32_t)n;
    const uint8_t prec = kPrecisionDouble;
    bool ok = std::fwrite(kMagic, 1, 4, out.f) == 4 &&
              std::fwrite(&version, sizeof version, 1, out.f) == 1 &&
              std::fwrite(&nq, sizeof nq, 1, out.f) == 1 && std::fwrite(&prec, 1, 1, out.f) == 1;
    for (DeviceState *s : segs) {
        DevScope on(s->device);
        const size_t total = sizeof(double2) * s->size;
        const size_t chunk = std::min(total, kChunk);
        char *buf = static_cast<char *>(g_chunk.get(chunk));
        VQB_CUDA(cudaStreamSynchronize(s->stream));
        for (size_t off = 0; ok && off < total; off += chunk) {
            const size_t len = std::min(chunk, total - off);
            VQB_CUDA(cudaMemcpyAsync(buf, reinterpret_cast<const char *>(s->amps) + off, len,
                                     cudaMemcpyDeviceToHost, s->stream));
            VQB_CUDA(cudaStreamSynchronize(s->stream));
            ok = std::fwrite(buf, 1, len, out.f) == len;
        }
    }
    if (!ok || std::fflush(out.f) != 0) raise(VQB_ERR_IO, "save_state: write failed");
}

void state_save(DeviceState *s, const char *path) {
    if (s->mixed) raise(VQB_ERR_TYPE, "save_state: only pure states can be dumped");
    save_segments(path, s->n, {s});
}

// load_state (io.hpp:84-128): same checks, same order, same messages
namespace {
struct Header {
    uint32_t n;
    uint8_t prec;
};
Header read_header(std::FILE *f) {
    char magic[4] = {0, 0, 0, 0};
    uint32_t version = 0, n = 0;
    uint8_t prec = 0;
    const bool header = std::fread(magic, 1, 4, f) == 4 && std::fread(&version, sizeof version, 1, f) == 1 &&
                        std::fread(&n, sizeof n, 1, f) == 1 && std::fread(&prec, 1, 1, f) == 1;
    if (!header || std::memcmp(magic, kMagic, 4) != 0)
        raise(VQB_ERR_IO, "load_state: not a state dump (bad magic)");
    if (version != kVersion)
        raise(VQB_ERR_IO, "load_state: unsupported format version " + std::to_string(version));
    if (n < 1 || n > 40) // PureState<double>::kMaxQubits (state.hpp:179)
        raise(VQB_ERR_IO, "load_state: qubit count " + std::to_string(n) + " out of range");
    if (prec != 1 && prec != 2) raise(VQB_ERR_IO, "load_state: unknown precision tag");
    return {n, prec};
}
void read_payload(std::FILE *f, const std::vector<DeviceState *> &segs) {
    for (DeviceState *s : segs) {
        DevScope on(s->device);
        const size_t total = sizeof(double2) * s->size;
        const size_t chunk = std::min(total, kChunk);
        char *buf = static_cast<char *>(g_chunk.get(chunk));
        for (size_t off = 0; off < total; off += chunk) {
            const size_t len = std::min(chunk, total - off);
            if (std::fread(buf, 1, len, f) != len) raise(VQB_ERR_IO, "load_state: truncated amplitude payload");
            VQB_CUDA(cudaMemcpyAsync(reinterpret_cast<char *>(s->amps) + off, buf, len, cudaMemcpyHostToDevice,
                                     s->stream));
            VQB_CUDA(cudaStreamSynchronize(s->stream)); // the chunk is reused
        }
    }
}
} // namespace

DeviceState *state_load(const char *path, int *precision) {
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) raise(VQB_ERR_IO, std::string("load_state: cannot open '") + path + "'");
    const Header h = read_header(in.f);
    DeviceState *s = state_create((int)h.n, 0);
    try {
        read_payload(in.f, {s});
    } catch (...) {
        state_destroy(s);
        throw;
    }
    if (precision) *precision = h.prec;
    return s;
}

// a dump read into existing segments (a sharded state in canonical layout);
// the file's qubit count must equal n
void load_segments(const char *path, int n, const std::vector<DeviceState *> &segs, int *precision) {
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) raise(VQB_ERR_IO, std::string("load_state: cannot open '") + path + "'");
    const Header h = read_header(in.f);
    if ((int)h.n != n)
        raise(VQB_ERR_SHAPE, "load_state: the dump holds " + std::to_string(h.n) + " qubits, the state " +
                                 std::to_string(n));
    read_payload(in.f, segs);
    if (precision) *precision = h.prec;
}

} // namespace vqb
