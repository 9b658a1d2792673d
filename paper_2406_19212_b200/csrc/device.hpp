// Device-side state and launcher declarations.
#pragma once

#include "common.hpp"
#include "gates.hpp"

namespace vqb {

// Reduction workspace owned by a state (one stream per state).
struct Workspace {
    double2 *partials = nullptr;   // [kMaxReduceBlocks * kMaxReduceSlots]
    unsigned *counter = nullptr;   // last-block-done ticket
    double2 *result = nullptr;     // device results [kMaxReduceSlots]
    double2 *host_result = nullptr; // pinned mirror
    void *terms = nullptr;         // packed Pauli groups/terms
    size_t terms_bytes = 0;
};

constexpr int kMaxReduceBlocks = 1184; // 148 SMs x 8
constexpr int kMaxReduceSlots = 8;

struct DeviceState {
    double2 *amps = nullptr;
    int n = 0;          // physical qubits
    int mixed = 0;
    int pn = 0;         // pseudo qubits (n, or 2n for a density matrix)
    uint64_t size = 0;  // 2^pn
    int device = 0;     // CUDA device holding amps (every call runs there)
    bool owned = true;
    uint64_t global_offset = 0;
    int global_qubits = 0;
    cudaStream_t stream = nullptr;
    Workspace ws;
};

DeviceState *state_create(int n, int mixed);
DeviceState *state_wrap(void *ptr, int n, int mixed, uint64_t global_offset, int global_qubits);
void state_destroy(DeviceState *s);
void state_set_zero(DeviceState *s);
void sync(DeviceState *s);

// ---- per-element application (unfused path; kernels.hpp:365-461) ----
// Dense m-qubit matrix on 0-based bit positions (listed order: first = local LSB).
void launch_dense(double2 *a, int pn, const int *bits, int m, const cvec &mat, cudaStream_t st);
// apply_gate_fast semantics on a (pseudo) state of pn qubits; positions are
// 1-based, already validated.
void apply_gate_fast(double2 *a, int pn, const Gate &g, cudaStream_t st);
// rho <- U rho U^dag on a density matrix (kernels.hpp:434-449).
void apply_gate_both_sides(DeviceState *s, const Gate &g);
// Channel through its superoperator (kernels.hpp:453-461).
void apply_superop(DeviceState *s, const Channel &c);

// ---- reductions (results land in s->ws.result on the device) ----
struct PauliPack; // host-side packed observable
double norm_sq(DeviceState *s);                          // state.hpp:236-242
cplx trace(DeviceState *s);                              // state.hpp:329-336
void expectation_async(DeviceState *s, const PauliPack &p, double2 *out_dev, const double2 *ket = nullptr);
cplx expectation(DeviceState *s, const PauliPack &p);    // observables.hpp:176-213
// sum_b conj(bra[b ^ x]) W(b) ket[b]: a term group whose X/Y factors flip
// global qubits of a sharded state reads the ket from the partner shard
cplx expectation_cross(DeviceState *bra, const double2 *ket, const PauliPack &p);
void apply_operator(DeviceState *src, double2 *dst, const PauliPack &p, bool conj_coeffs);
// dst (+)= H src_amps with src's stream and workspace (src_amps may be another
// shard's buffer, on a peer device)
void apply_operator_from(DeviceState *src, const double2 *src_amps, double2 *dst, const PauliPack &p,
                         bool accumulate);
void identity_costate(DeviceState *s, const PauliPack &p); // <<I|H as a ket, in place
cplx dot_async_result(DeviceState *s, const double2 *a, const double2 *b); // <a|b>
void dot_async(DeviceState *s, const double2 *a, const double2 *b, double2 *out_dev);
cplx bilinear_form(DeviceState *bra, DeviceState *ket, const int *pos1, int m, const cvec &local);
// Fused reverse step; results: complex sums to out_c (device, nullable) and
// real_scale * Re(sum) to out_r (device, nullable).
void reverse_step_async(double2 *phi, double2 *psi, int pn, const int *pos1, int m,
                        const cvec &inv, const std::vector<cvec> &dmats, DeviceState *ws_owner,
                        double2 *out_c, double *out_r, double real_scale);
double max_abs_diff(DeviceState *s, const double2 *a, const double2 *b);
// measurement (circuit.hpp:303-375): unclamped P(qubit = 1), and the collapse
double prob_one(DeviceState *s, int qubit);
void collapse(DeviceState *s, int qubit, int outcome, double scale);
// state dumps (io.hpp:40-128), streamed through a pinned chunk buffer
void state_save(DeviceState *s, const char *path);
DeviceState *state_load(const char *path, int *precision);
void save_segments(const char *path, int n, const std::vector<DeviceState *> &segs);
void load_segments(const char *path, int n, const std::vector<DeviceState *> &segs, int *precision);

// ---- Pauli operator packing (observables.hpp:38-110) ----
struct PauliGroupDev {
    unsigned long long xmask;
    int first;
    int count;
};
struct PauliTermDev {
    unsigned long long zmask; // y|z bits
    double2 coeff;            // coeff * i^{#Y}
};
struct PauliPack {
    std::vector<PauliGroupDev> groups;
    std::vector<PauliTermDev> terms;
    int max_qubit = 0;
};
PauliPack pack_operator(const vqb_pauli_term *terms, int64_t nterms, bool conjugate);
void upload_operator(DeviceState *s, const PauliPack &p);

} // namespace vqb
