"""Generate tests/golden/fullsize.json: the REFERENCE's own results for
BASELINE.json's configs 1-4 at their stated sizes.

The unmodified reference (oracle/_ref/libvqcs_ref.so, compiled from
/root/reference by oracle/Makefile) runs on the seeded generators of
paper_2406_19212_b200.circuits on a large host (it needs up to 137 GB of RAM
and about an hour on 16 cores: config 2's gradient holds four 16 GiB states,
config 3's five, config 4's 33-qubit state is 128 GiB), so this script is run
once on the GPU box's host and its output committed:

    python tests/golden/make_fullsize_golden.py [out.json] [config ...]

Stored per config (the GPU tests tests/test_gpu_parity_fullsize.py compare the
CUDA path against these):
  * config1 (28q RQC), config4 (33q RQC): norm, amplitudes at a fixed index
    sample (tests/helpers.sample_indices) and NUM_PROJECTIONS overlaps of the
    whole state with seeded product states
    (tests/helpers.product_projections_host);
  * config2 (30q QAOA, p=8): loss, the 600 per-gate gradients and the 16 tied
    gradients (gradient_pure, autodiff.hpp:95-156);
  * config3 (15q noisy DM): loss and the 270 gradients (gradient_mixed,
    autodiff.hpp:184-329), plus the trace of the forward density matrix.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import product_projections_host, sample_amplitudes, sample_indices  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402


def c2l(z):
    return [[float(np.real(x)), float(np.imag(x))] for x in np.atleast_1d(z)]


def state_record(ref, w, t0):
    s = ref.pure_state(w.num_qubits)
    ref.apply_circuit(w.circuit, s)
    t_apply = time.time() - t0
    idx = sample_indices(w.num_qubits)
    rec = {"name": w.name, "n": w.num_qubits, "elements": len(w.circuit), "seed": w.seed,
           "norm": ref.norm(s), "sample_index": [int(i) for i in idx],
           "sample": c2l(sample_amplitudes(ref, s, idx)),
           "product_projections": c2l(product_projections_host(ref, s, w.num_qubits)),
           "reference_seconds": t_apply}
    s.free()
    return rec


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "fullsize.json")
    which = sys.argv[2:] or ["config1", "config2", "config3", "config4"]
    ref = oracle.reference()
    threads = os.cpu_count() or 1
    oracle.set_reference_threads(threads)
    out = {}
    if os.path.exists(out_path):
        with open(out_path) as f:
            out = json.load(f)
    out["_meta"] = {"generator": "paper_2406_19212_b200.circuits", "reference": "vqcs (oracle/_ref)",
                    "threads": threads, "script": "tests/golden/make_fullsize_golden.py"}

    def save():
        with open(out_path, "w") as f:
            json.dump(out, f, indent=0)

    for name in which:
        t0 = time.time()
        if name == "config1":
            out[name] = state_record(ref, circuits.config1(), t0)
        elif name == "config4":
            out[name] = state_record(ref, circuits.config4(num_gpus=1), t0)
        elif name == "config2":
            w = circuits.config2()
            s0 = ref.pure_state(w.num_qubits)
            loss, g = ref.gradient_pure(w.observable, w.circuit, s0)
            s0.free()
            tied = circuits.qaoa_tied_gradients(g, w.num_qubits, len(w.extra["edges"]), w.extra["p"])
            out[name] = {"name": w.name, "n": w.num_qubits, "loss": loss, "grads": [float(x) for x in g],
                         "tied": [float(x) for x in tied], "reference_seconds": time.time() - t0}
        elif name == "config3":
            w = circuits.config3()
            d0 = ref.mixed_state(w.num_qubits)
            loss, g = ref.gradient_mixed(w.observable, w.circuit, d0)
            d0.free()
            out[name] = {"name": w.name, "n": w.num_qubits, "loss": loss, "grads": [float(x) for x in g],
                         "reference_seconds": time.time() - t0}
        else:
            raise SystemExit(f"unknown config {name}")
        save()
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
