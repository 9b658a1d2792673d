"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (header-only vqcs compiled from
/root/reference by oracle/Makefile into oracle/_ref/libvqcs_ref.so) on the
seeded generators of paper_2406_19212_b200.circuits and stores its outputs.
The fixtures pin both the oracle restatement (tests/test_oracle.py) and the
CUDA path (tests/test_gpu_golden.py) without needing /root/reference at test
time. Re-run with:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402


def main():
    ref = oracle.reference()
    oracle.set_reference_threads(1)  # serial: segment-order sums identical to a 1-thread run
    out = {"generator": "paper_2406_19212_b200.circuits", "reference": "vqcs (oracle/_ref)",
           "threads": 1}

    # config 0 at full size: loss + 600 gradients (autodiff.hpp:95-156)
    w = circuits.config0()
    loss, g, res = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(w.num_qubits),
                                     with_residual=True)
    s = ref.pure_state(w.num_qubits)
    ref.apply_circuit(w.circuit, s)
    amps = ref.download(s)
    out["config0"] = {"n": 20, "layers": 10, "seed": 0, "loss": loss, "grads": list(map(float, g)),
                      "reverse_residual": res, "amp0": [amps[0].real, amps[0].imag],
                      "norm": ref.norm(s)}

    # config 1 reduced (3x4 grid, 8 cycles): the final state
    w = circuits.config1(rows=3, cols=4, cycles=8)
    s = ref.pure_state(w.num_qubits)
    ref.apply_circuit(w.circuit, s)
    np.save(os.path.join(HERE, "config1_3x4_8cyc_state.npy"), ref.download(s))
    out["config1_3x4_8cyc"] = {"n": 12, "elements": len(w.circuit), "norm": ref.norm(s)}

    # config 2 reduced (10 nodes, p = 3): loss + per-gate and tied gradients
    w = circuits.config2(n=10, p=3)
    loss, g = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(10))
    tied = circuits.qaoa_tied_gradients(g, 10, len(w.extra["edges"]), 3)
    out["config2_10_p3"] = {"loss": loss, "grads": list(map(float, g)), "tied": list(map(float, tied)),
                            "edges": w.extra["edges"]}

    # config 3 reduced (4 qubits, 2 layers): noisy loss + gradients (autodiff.hpp:184-329)
    w = circuits.config3(n=4, layers=2)
    loss, g = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(4))
    dm = ref.mixed_state(4)
    ref.apply_circuit(w.circuit, dm)
    out["config3_4_2l"] = {"loss": loss, "grads": list(map(float, g)),
                           "trace": [ref.trace(dm).real, ref.trace(dm).imag]}
    np.save(os.path.join(HERE, "config3_4_2l_rho.npy"), ref.download(dm))

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
