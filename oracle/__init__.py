"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the CUDA path.

Two implementations of the include/vqcs_b200.h C-ABI on the CPU:

* ``reference()`` — the unmodified reference library (header-only C++,
  /root/reference/proj/include/vqcs) compiled by oracle/Makefile from the
  reference sources into oracle/_ref/libvqcs_ref.so via ref_shim.cpp;
* ``restatement()`` — the plain-C restatement oracle/vqcs_oracle.c
  (oracle/_ref/libvqcs_oracle.so), pinned against the former and the golden
  vectors in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline. The product (paper_2406_19212_b200) never imports it.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

from paper_2406_19212_b200.engine import Engine

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libvqcs_ref.so")
ORC_SO = os.path.join(HERE, "_ref", "libvqcs_oracle.so")

_cache: dict = {}


def build(quiet: bool = True) -> None:
    """Compile the checkers (reference shim only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _load(path: str, prefix: str, name: str) -> Engine:
    if name not in _cache:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built; run `make -C oracle`")
        lib = ct.CDLL(path)
        _cache[name] = Engine(lib, prefix, name)
    return _cache[name]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference() -> Engine:
    """The reference vqcs library itself (multi-threaded per VQCS_NUM_THREADS
    or set_num_threads)."""
    return _load(REF_SO, "vqcsref_", "reference")


def restatement() -> Engine:
    return _load(ORC_SO, "vqcsorc_", "restatement")


def checker() -> Engine:
    """The strongest available checker: the reference itself if built, else
    the restatement."""
    return reference() if reference_available() else restatement()


REFBENCH_CLI = os.path.join(HERE, "_ref", "refbench_cli")


def reference_bench_report(records, fmt: str = "json") -> str:
    """The reference harness's own emit_report (src/bench.cpp) on the same
    records (oracle/_ref/refbench_cli, a separate process)."""
    lines = [fmt]
    for r in records:
        secs = [float(x).hex() for x in r["seconds"]]
        items = sorted((str(k), str(v)) for k, v in r.get("params", {}).items())
        f = [str(r["task"]).encode().hex(), str(int(r["n"])), str(int(r["depth"])), str(int(r["threads"])),
             float(r.get("speedup", 0.0)).hex(), str(len(secs))] + secs + [str(len(items))]
        for k, v in items:
            f += [k.encode().hex() or "-", v.encode().hex() or "-"]
        lines.append(" ".join(f))
    out = subprocess.run([REFBENCH_CLI], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True)
    return out.stdout


def set_reference_threads(t: int) -> None:
    reference().lib.vqcsref_set_num_threads(int(t))


def reference_uniform(seed: int, skip: int = 0) -> float:
    """The uniform the reference's measure() draws from std::mt19937_64(seed)
    after `skip` draws (circuit.hpp:287-290)."""
    u = ct.c_double()
    rc = reference().lib.vqcsref_uniform_unit(ct.c_uint64(seed), ct.c_uint64(skip), ct.byref(u))
    reference().check(rc)
    return u.value


def reference_measure(state, qubit: int, seed: int, skip: int = 0):
    """The reference's own measure() on std::mt19937_64(seed) -> (outcome, p)."""
    eng = reference()
    o, p = ct.c_int32(), ct.c_double()
    eng.check(eng.lib.vqcsref_measure_seeded(state.handle, qubit, ct.c_uint64(seed),
                                             ct.c_uint64(skip), ct.byref(o), ct.byref(p)))
    return o.value, p.value
