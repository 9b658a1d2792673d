#!/usr/bin/env python
"""Benchmark of the B200 hot path against BASELINE.json's configurations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config rqc28|hea20|qaoa30|noisy15|rqc33] [--no-extra] [--unfused]

Default at N = 1: config 1 — the 28-qubit random circuit (4x7 grid, 20
cycles, 785 gates, complex128) through ``vqb_apply_circuit``, metric gates/s —
as the headline line, and BASELINE.json's other metrics measured in the same
run under ``"configs"``: config 0 (hea20) and config 2 (qaoa30) adjoint
gradient evals/s, config 3 (noisy15) noisy gradient evals/s and noisy DM
gates/s, config 4 (rqc33, 33 qubits = 128 GiB on one GPU) gates/s — each with
its own roofline, end-to-end number and bounded CPU-reference sample.

Default at N > 1 (torchrun, one rank per GPU): config 4 sharded — 33 + log2 N
qubits, 2^33 amplitudes (128 GiB) per GPU, the top log2 N qubits global,
global<->local swaps as all-to-all rounds over NCCL
(``distributed.ShardedState``), weak scaling. ``--config qaoa30`` at N > 1 runs
config 2's gradient on the sharded layout (strong scaling). A sharded run
processes ONE circuit (or gradient) per step across all ranks, so `value` =
units per step x K / time (no factor N); single-GPU configs at N > 1 run one
replica per rank and `value` counts every rank's units.

A step = reset the device state to |0...0> and run the whole circuit (or one
full adjoint gradient evaluation). `value` is timed with CUDA events on the
state's stream over exactly K steps after W warm-up steps, max over ranks;
`e2e` is the same metric through the C-ABI with host buffers (inputs uploaded
from pinned host memory and results read back every step, inside the timed
region).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libvqcs_ref.so, compiled from /root/reference) on all host cores
with the reference harness's protocol (src/bench.cpp:128-151: the state is
allocated once and reset with std::fill every step), each step a bounded
sample of the same workload; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2406_19212_b200 import circuits  # noqa: E402
from paper_2406_19212_b200.abi import Circuit  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")
FP64_PATH = os.path.join(ROOT, "profiles", "fp64_peak.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
NVLINK_NOMINAL_GBS = 900.0  # per direction per GPU (NVLink 5); no measured figure on a 1-GPU pool
ALL_CONFIGS = ["rqc28", "hea20", "qaoa30", "noisy15", "rqc33"]


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def dfma_peak():
    try:
        with open(FP64_PATH) as f:
            return float(json.load(f)["dfma_tflops"]), "measured (profiles/fp64_peak.json)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal"


# ------------------------------------------------------------------ workloads
class Workload:
    """metric unit per step and the per-step call."""

    def __init__(self, name, args, world=1):
        self.name = name
        self.fused = not getattr(args, "unfused", False)
        self.world = world
        self.sharded = world > 1 and name in ("rqc33", "qaoa30")
        if name == "rqc33":
            self.w = circuits.config4(num_gpus=world)
            self.kind = "apply"
        elif name == "rqc28":
            self.w = circuits.config1()
            self.kind = "apply"
        elif name == "hea20":
            self.w = circuits.config0()
            self.kind = "grad_pure"
        elif name == "qaoa30":
            self.w = circuits.config2()
            self.kind = "grad_pure"
        elif name == "noisy15":
            self.w = circuits.config3()
            self.kind = "grad_mixed"
        else:
            raise SystemExit(f"unknown config {name}")
        self.n = self.w.num_qubits
        self.mixed = self.w.mixed
        self.gates = len(self.w.circuit)
        if self.kind == "apply":
            self.metric, self.unit = "gates/s", "gates/s"
            self.units_per_step = self.gates
        else:
            self.metric, self.unit = "gradient evals/s", "evals/s"
            self.units_per_step = 1

    @property
    def g(self) -> int:
        return int(round(math.log2(self.world))) if self.sharded else 0

    def job_units(self, steps: int) -> float:
        """Units the whole job processed in `steps` steps: a sharded run does
        one circuit per step across all ranks; replicas each do their own."""
        per = self.units_per_step * steps
        return per if self.sharded else per * self.world

    def step(self, eng, state):
        if self.kind == "apply":
            eng.apply_circuit(self.w.circuit, state, fused=self.fused)
        elif self.kind == "grad_pure":
            eng.gradient_pure(self.w.observable, self.w.circuit, state)
        else:
            eng.gradient_mixed(self.w.observable, self.w.circuit, state)

    def algorithmic_bytes(self, world: int = 1) -> float:
        """SURVEY.md §8(d) touched-amplitude rule over the reference schedule
        (per GPU: a sharded state holds 2^(n - log2 N) amplitudes per rank)."""
        pn = 2 * self.n if self.mixed else self.n
        if self.sharded:
            pn -= int(round(math.log2(world)))
        unit = 32.0 * (1 << pn)
        fwd = sum(circuits.touched_fraction(e) for e in self.w.circuit.elements)
        if self.kind == "apply":
            return fwd * unit
        rev = 2 * fwd  # reverse steps touch two states
        return (fwd + 1 + rev) * unit


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    20 ms while the timed region runs (plus one sample at entry and exit, so
    short regions are covered); falls back to `nvidia-smi -lms 200`."""
    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []  # (sm_mhz, sm_max_mhz, set of reasons)
        self.stop = threading.Event()
        self.nv = None
        self.proc = None
        self.mx = None

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        if self.mx is None:  # constant: asked once (every NVML query takes driver locks the launches need too)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = self.mx
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        reasons = {k for k, attr in self.NAMES.items() if r & getattr(nv, attr, 0)}
        self.samples.append((float(sm), float(mx), reasons))

    def _poll(self):
        while not self.stop.wait(0.02):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self._sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read_smi, daemon=True)
                self.t.start()
            except Exception:
                self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                reasons = {k for k, v in zip(self.NAMES, parts[2:6]) if v.lower().startswith("active")}
                self.samples.append((float(parts[0]), float(parts[1]), reasons))
            except (ValueError, IndexError):
                pass

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = set()
        for _, _, r in self.samples:
            reasons |= r
        return {"sm_mhz": statistics.median(x[0] for x in self.samples),
                "sm_max_mhz": max(x[1] for x in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml" if self.nv is not None else "nvidia-smi"}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1 and args.impl == "b200":
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", init_method="env://")
        dist = td
    return world, rank, local, dist


def barrier(dist, local):
    if dist is not None:
        dist.barrier(device_ids=[local])


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ reference arm
def reference_engine():
    import oracle
    if not oracle.reference_available():
        return None, "oracle/_ref/libvqcs_ref.so not built"
    eng = oracle.reference()
    threads = os.cpu_count() or 1
    oracle.set_reference_threads(threads)
    return eng, threads


def numa_note() -> str:
    """BASELINE.md §3 asks for numactl --interleave=all; say what the host has."""
    if shutil.which("numactl") is None:
        try:
            nodes = [d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")]
        except OSError:
            nodes = []
        return (f"numactl absent; host has {len(nodes) or 1} NUMA node(s)"
                + (" (interleave is moot)" if len(nodes) <= 1 else " (not interleaved)"))
    return "numactl present (run bench under numactl --interleave=all)"


class ReferenceSample:
    """A bounded sample of the workload for the CPU reference (about 10-30 s
    of host work), run with the reference harness's protocol
    (src/bench.cpp:128-151): states allocated once by prepare(), every run()
    resets the state with std::fill and applies the sample. `units` = what
    one run is worth in the metric's unit; samples smaller than the workload
    are scaled by the amplitude-count ratio (every reference kernel is a
    linear pass over the state, kernels.hpp:128-176) and say so."""

    def __init__(self, wl: Workload, full: bool = False):
        self.wl = wl
        self.state = None
        k = 160 if full else 80
        if wl.kind == "apply":
            n = min(wl.n, 28)  # config 4 (128 GiB+) does not fit the host
            w = circuits.config1() if n != wl.n else wl.w
            self.circ = Circuit(w.circuit.elements[:k])
            self.n, self.mixed, self.kind = n, False, "apply"
            scale = 2.0 ** (n - wl.n)
            self.units = k * scale
            self.sample = (f"first {k} of {wl.gates} gates at n={wl.n}" if n == wl.n else
                           f"first {k} gates of the 28-qubit member of the same circuit family, gates/s "
                           f"extrapolated to n={wl.n} by 2^(28-{wl.n}) (state does not fit the host)")
        elif wl.name == "hea20":
            self.circ, self.op = wl.w.circuit, wl.w.observable
            self.n, self.mixed, self.kind, self.units = wl.n, False, "grad_pure", 1.0
            self.sample = "one full gradient evaluation (20q, 600 params)"
        elif wl.name == "qaoa30":
            small = circuits.config2(n=22, p=wl.w.extra["p"], seed=wl.w.seed)
            self.circ, self.op = small.circuit, small.observable
            self.n, self.mixed, self.kind = 22, False, "grad_pure"
            self.units = 2.0 ** (22 - wl.n)
            self.sample = ("one gradient evaluation of the same QAOA family (3-regular, p=8) at "
                           f"n=22, evals/s extrapolated to n={wl.n} by 2^(22-{wl.n})")
        elif wl.name == "noisy15":
            small = circuits.config3(n=11)
            self.circ, self.op = small.circuit, small.observable
            self.n, self.mixed, self.kind = 11, True, "grad_mixed"
            self.units = 4.0 ** (11 - wl.n)
            self.sample = ("one noisy gradient evaluation of the same ansatz (6 layers) at n=11 "
                           f"(4^11 entries), evals/s extrapolated to n={wl.n} by 4^(11-{wl.n})")
        else:
            raise ValueError(wl.name)

    def prepare(self, eng):
        self.state = eng.create(self.n, self.mixed)

    def run(self, eng):
        if self.kind == "apply":
            eng.set_zero(self.state)
            eng.apply_circuit(self.circ, self.state)
        elif self.kind == "grad_pure":
            eng.gradient_pure(self.op, self.circ, self.state)  # s0 is const (autodiff.hpp:95-98)
        else:
            eng.gradient_mixed(self.op, self.circ, self.state)

    def free(self):
        if self.state is not None:
            self.state.free()
            self.state = None


def reference_sample(wl: Workload, full: bool = False):
    """(run(eng), units, description) — kept for callers that want a one-shot
    sample (allocates per call)."""
    smp = ReferenceSample(wl, full)

    def run(eng):
        smp.prepare(eng)
        try:
            smp.run(eng)
        finally:
            smp.free()
    return run, smp.units, smp.sample


def run_reference_arm(args, wl, world, rank):
    if rank != 0:
        return 0
    eng, threads = reference_engine()
    line = {"impl": "reference", "metric": wl.metric, "unit": wl.unit, "higher_is_better": True,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "data": "synthetic",
            "dtype": "c128", "scaling": "strong" if (wl.sharded and wl.name == "qaoa30") else "weak",
            "vs_baseline": None, "config": config_block(wl, world)}
    if eng is None:
        line["unavailable"] = threads
        print(json.dumps(line))
        return 0
    smp = ReferenceSample(wl)
    smp.prepare(eng)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        smp.run(eng)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    smp.free()
    total = sum(times)
    value = smp.units * len(times) / total
    mean = total / len(times)
    line.update({"value": value, "ms_per_step": 1e3 * mean,
                 "seconds": times, "stddev_seconds": statistics.pstdev(times),
                 "cpu_baseline": {"value": value, "unit": wl.unit, "cores": threads,
                                  "kind": "reference", "sample": smp.sample,
                                  "protocol": "state allocated once, std::fill reset per step "
                                              "(src/bench.cpp:128-151); " + numa_note()},
                 "e2e": {"value": value, "unit": wl.unit, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line))
    return 0


def cpu_baseline(wl: Workload):
    eng, threads = reference_engine()
    if eng is None:
        return None
    smp = ReferenceSample(wl, full=True)
    smp.prepare(eng)
    t0 = time.perf_counter()
    smp.run(eng)
    dt = time.perf_counter() - t0
    smp.free()
    return {"value": smp.units / dt, "unit": wl.unit, "cores": threads, "kind": "reference",
            "sample": smp.sample + f"; {dt:.2f} s on the GPU box host; " + numa_note()}


# ------------------------------------------------------------------ sharded runs (N > 1)
class ShardedRunner:
    """Config 4 (rqc33: 33 + log2 N qubits, 2^33 amplitudes per rank) and
    config 2 (qaoa30 gradient, 2^(30 - log2 N) per rank) on the sharded layout
    of distributed.ShardedState: the shard is a torch CUDA tensor, local runs
    go through the fused executor (vqb_state_wrap), global<->local swaps
    (all-to-all rounds, bounded chunks) and reductions through
    torch.distributed over NCCL."""

    def __init__(self, eng, wl, dist, rank, world, local):
        import torch
        from paper_2406_19212_b200.distributed import DeviceEngine, ShardedState
        g = int(round(math.log2(world)))
        self.wl = wl
        shard = torch.zeros(1 << (wl.n - g), dtype=torch.complex128, device=f"cuda:{local}")
        self.st = ShardedState(wl.n, dist, DeviceEngine(eng), shard, rank, world)
        self.loss = None

    def reset(self):
        self.st.set_zero()

    def step(self):
        if self.wl.kind == "apply":
            self.st.apply_circuit(self.wl.w.circuit)
        else:
            self.loss, _ = self.st.gradient_pure(self.wl.w.observable, self.wl.w.circuit)

    def norm(self):
        return self.st.norm()

    def stats(self):
        return {"swap_rounds": self.st.swaps, "swapped_bits": self.st.swapped_bits,
                "bytes_exchanged_per_rank": self.st.bytes_exchanged,
                "max_transfer_buffer_amps": self.st.max_buffer_amps}

    def free(self):
        self.st.local = None


# ------------------------------------------------------------------ one config
def config_block(wl: Workload, world: int) -> dict:
    return {"workload": wl.w.name, "qubits": wl.n, "mixed": wl.mixed, "elements": wl.gates,
            "seed": wl.w.seed, "fused": wl.fused,
            "parallelism": (f"sharded top {wl.g} qubits over {world} ranks" if wl.sharded
                            else ("replicas" if world > 1 else "single")),
            "l2": (f"state {16 * (1 << ((2 * wl.n if wl.mixed else wl.n) - wl.g)) / 2**30:.2f} GiB per GPU"
                   " vs 126 MB L2: "
                   + ("inputs larger than L2, no flush" if (2 * wl.n if wl.mixed else wl.n) - wl.g >= 24
                      else "state L2-resident (reported as is)"))}


def roofline_of(eng, wl, prof, launch_recs, step_flops, world):
    """HBM roofline of the step's dominant kernel: algorithmic bytes per launch
    (one read + one write pass of the state; the adjoint kernels stream both
    Phi and Psi) / its average launch time, CUDA events on the launching
    stream; plus the FP64 view and the per-launch binding bound."""
    if not prof:
        return None
    peak, peak_kind = hbm_peak()
    name, (cnt, tot_ms) = max(prof.items(), key=lambda kv: kv[1][1])
    pn = (2 * wl.n if wl.mixed else wl.n) - wl.g
    nstates = 2 if "rev" in name else 1
    bytes_per_launch = 32.0 * nstates * (1 << pn)
    avg_s = tot_ms / cnt / 1e3
    achieved = bytes_per_launch / avg_s / 1e9
    traffic = None
    fp64_pipe = None
    try:
        with open(TRAFFIC_PATH) as f:
            rec = json.load(f).get(wl.name, {})
        traffic = rec.get(name)
        fp64_pipe = rec.get("fp64_pipe_active_pct", {}).get(name)
    except Exception:
        pass
    step_ms = sum(v[1] for v in prof.values())
    roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_kind, "launches_per_step": cnt,
            "avg_launch_us": 1e6 * avg_s, "share_of_step": tot_ms / step_ms if step_ms else None,
            "algorithmic_bytes_per_launch": bytes_per_launch}
    if fp64_pipe:
        # from the committed ncu capture of this kernel (like `traffic`): how
        # busy the FP64 pipe is, [min, max] % over the captured launches
        roof["fp64_pipe_active_pct_ncu"] = fp64_pipe
    dfma, dfma_kind = dfma_peak()
    fused_ms = sum(v[1] for k, v in prof.items() if k.startswith("k_regstage") or k.startswith("k_stage"))
    if step_flops > 0 and fused_ms > 0:
        ach = step_flops / (fused_ms / 1e3) / 1e12
        roof["fp64"] = {"achieved": ach, "peak": dfma, "unit": "TFLOP/s", "frac": ach / dfma,
                        "flops_per_step": step_flops, "peak_source": dfma_kind}
        roof["limiter"] = "fp64" if roof["fp64"]["frac"] > roof["frac"] else "hbm"
    if launch_recs:
        # per launch, the binding roofline is the larger of its HBM time
        # (algorithmic bytes / measured copy peak) and its FP64 time
        # (executed flops / measured DFMA peak); the stage kernels' time
        # against the sum of those floors
        t_meas = sum(r[1] for r in launch_recs) / 1e3
        t_floor = sum(max(r[3] / (peak * 1e9), r[2] / (dfma * 1e12)) for r in launch_recs)
        n_hbm = sum(1 for r in launch_recs if r[3] / (peak * 1e9) >= r[2] / (dfma * 1e12))
        pn = (2 * wl.n if wl.mixed else wl.n) - wl.g
        roof["per_launch"] = [[round(r[1], 4), round(r[2] / float(1 << pn), 1)] for r in launch_recs]
        roof["per_launch_what"] = "[ms, executed FP64 flops per amplitude] of every stage launch of one step"
        roof["per_launch_bound"] = {
            "frac": t_floor / t_meas if t_meas else None, "floor_ms": 1e3 * t_floor,
            "measured_ms": 1e3 * t_meas, "launches": len(launch_recs), "hbm_bound_launches": n_hbm,
            "fp64_peak_tflops": dfma,
            "what": "sum over stage launches of max(bytes / HBM peak, executed flops / measured DFMA peak) "
                    "divided by their measured time"}
    return roof


def measure(wl: Workload, args, eng, world, rank, local, dist, steps=None, warmup=None,
            cpu=True) -> dict:
    import ctypes as ct

    import torch
    steps = steps or args.steps
    warmup = max(warmup or args.warmup, 3)
    if wl.sharded:
        runner = ShardedRunner(eng, wl, dist, rank, world, local)
        state = runner
        stream = torch.cuda.current_stream()
        reset = runner.reset
        step = runner.step
    else:
        state = eng.create(wl.n, wl.mixed)
        stream = torch.cuda.ExternalStream(eng.stream_of(state), device=torch.device("cuda", local))

        def reset():
            eng.set_zero(state)

        def step():
            wl.step(eng, state)
    for _ in range(warmup):
        reset()
        step()
    torch.cuda.synchronize()

    # timed region
    barrier(dist, local)
    torch.cuda.synchronize()
    l0 = eng.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(steps):
            reset()
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(dist, local)
    launches = eng.launch_count() - l0
    ms = max_over_ranks(dist, ev0.elapsed_time(ev1))
    ms_per_step = ms / steps
    value = wl.job_units(steps) / (ms / 1e3)

    check = {}
    if wl.kind == "apply" and not wl.mixed:
        check["norm"] = state.norm() if wl.sharded else eng.norm(state)
    if wl.sharded:
        check.update(runner.stats())
    noisy_fwd = None
    if wl.kind == "grad_mixed":
        # BASELINE.json's "noisy DM gates/s": the circuit's elements (gates and
        # channels) per second of forward evolution of the density matrix
        reset()
        eng.apply_circuit(wl.w.circuit, state)
        torch.cuda.synchronize()
        f0e = torch.cuda.Event(enable_timing=True)
        f1e = torch.cuda.Event(enable_timing=True)
        f0e.record(stream)
        for _ in range(steps):
            reset()
            eng.apply_circuit(wl.w.circuit, state)
        f1e.record(stream)
        f1e.synchronize()
        fms = max_over_ranks(dist, f0e.elapsed_time(f1e)) / steps
        noisy_fwd = {"value": world * wl.gates / (fms / 1e3), "unit": "DM gates/s",
                     "ms_per_forward": fms, "elements": wl.gates,
                     "what": "vqb_apply_circuit on the 2^30-entry vec(rho) (gates as superoperators + channels), "
                             "state reset included"}

    # roofline: per-kernel CUDA-event timing of one more step (untimed)
    reset()
    f0 = eng.flop_count()
    eng.profile_begin()
    step()
    launch_recs = []
    prof = eng.profile_end(launch_recs)
    roof = roofline_of(eng, wl, prof, launch_recs, eng.flop_count() - f0, world)
    peak, _ = hbm_peak()
    ref_sched_gbs = wl.algorithmic_bytes(world) / (ms_per_step / 1e3) / 1e9

    sharded = None
    if wl.sharded:
        # per GPU: the local passes' algorithmic bytes and the swap bytes over
        # NVLink; combined roofline T_roof = local bytes / B_HBM + exchanged
        # bytes / B_NVL, B_NVL nominal (unmeasured here)
        exch = max_over_ranks(dist, float(runner.st.bytes_exchanged)) / (warmup + steps + 1)
        t_s = ms_per_step / 1e3
        # physical floor: the stage launches' passes over the local shard at
        # the HBM peak + the exchanged bytes at the NVLink peak
        stage_bytes = sum(r[3] for r in launch_recs)
        t_roof = stage_bytes / (peak * 1e9) + exch / (NVLINK_NOMINAL_GBS * 1e9)
        sharded = {"hbm_gbs_per_gpu": stage_bytes / t_s / 1e9,
                   "hbm_gbs_per_gpu_reference_schedule": wl.algorithmic_bytes(world) / t_s / 1e9,
                   "nvlink_gbs_per_gpu": exch / t_s / 1e9, "exchanged_bytes_per_step_per_gpu": exch,
                   "combined_roofline_frac": t_roof / t_s,
                   "combined_roofline_what": "(stage-launch bytes / HBM peak + exchanged bytes / NVLink peak) "
                                             "/ measured step time, per GPU",
                   "nvlink_peak_gbs": NVLINK_NOMINAL_GBS, "nvlink_peak_source": "nominal NVLink 5 per direction"}

    # end to end through the C-ABI with host buffers
    e2e = None
    state_bytes = 16 * (1 << ((2 * wl.n if wl.mixed else wl.n) - wl.g))
    if not args.no_e2e and (wl.sharded or state_bytes > (32 << 30)):
        # config 4: the state (128 GiB per GPU) cannot round-trip through host
        # memory every step; the user call is vqb_state_set_zero (the
        # reference's PureState(n) constructor) + vqb_apply_circuit with the
        # circuit packed from host objects + the norm read back to the host
        from paper_2406_19212_b200.abi import vqb_op

        def e2e_step():
            if wl.sharded:
                runner.reset()
                runner.step()
                return state.norm() if wl.kind == "apply" else runner.loss
            reset()
            eng.apply_circuit(wl.w.circuit, state)
            return eng.norm(state)

        e2e_step()
        torch.cuda.synchronize()
        barrier(dist, local)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
        ems = max_over_ranks(dist, e0.elapsed_time(e1))
        grad = wl.kind != "apply"
        e2e = {"value": wl.job_units(steps) / (ems / 1e3), "unit": wl.unit,
               "h2d_bytes_per_step": ct.sizeof(vqb_op) * wl.gates,
               "d2h_bytes_per_step": 8 * (1 + wl.w.circuit.num_active_params()) if grad else 8,
               "ms_per_step": ems / steps,
               "path": ("sharded |0...0> -> ShardedState.gradient_pure (loss + all-reduced gradients to the host)"
                        if grad else
                        "vqb_state_set_zero -> vqb_apply_circuit (ops packed from host objects) -> vqb_norm "
                        "(the 128 GiB state does not round-trip through host memory)")}
    elif not args.no_e2e and wl.kind == "apply":
        # the user call: vqb_apply_circuit_copy_batch over host states (one job
        # per step: upload the input state from pinned memory, run the circuit,
        # download the final state into pinned memory); consecutive jobs'
        # copies overlap the circuits (both PCIe directions + compute)
        nbytes = 16 * state.size
        h_in = torch.zeros(2 * state.size, dtype=torch.float64, pin_memory=True)
        h_in[0] = 1.0
        h_outs = [torch.empty(2 * state.size, dtype=torch.float64, pin_memory=True) for _ in range(3)]
        # at least 16 jobs, so the pipeline's fill (first upload) and drain
        # (last download) do not dominate
        jobs = max(steps, 16)
        ins = [h_in.data_ptr()] * jobs
        outs = [h_outs[j % 3].data_ptr() for j in range(jobs)]
        eng.apply_circuit_copy_batch(wl.w.circuit, wl.n, ins[:2], outs[:2], mixed=wl.mixed)  # warm
        torch.cuda.synchronize()
        barrier(dist, local)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.apply_circuit_copy_batch(wl.w.circuit, wl.n, ins, outs, mixed=wl.mixed)
        e1.record(stream)
        e1.synchronize()
        ems = max_over_ranks(dist, e0.elapsed_time(e1))
        out_norm = float((torch.view_as_complex(h_outs[(jobs - 1) % 3].view(-1, 2)).abs() ** 2).sum())
        e2e = {"value": wl.job_units(jobs) / (ems / 1e3), "unit": wl.unit,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "ms_per_step": ems / jobs, "jobs": jobs,
               "result_norm_sq": out_norm,
               "path": "vqb_apply_circuit_copy_batch (per job: pinned host state -> device, circuit, "
                       "device -> pinned host; jobs pipelined over 3 device states)"}
        del h_in, h_outs
    elif not args.no_e2e:
        nbytes = 16 * state.size
        h_in = torch.zeros(2 * state.size, dtype=torch.float64, pin_memory=True)
        h_in[0] = 1.0
        from paper_2406_19212_b200.abi import c128_p
        pin = ct.cast(ct.c_void_p(h_in.data_ptr()), c128_p)
        up = eng._fn("state_upload_async")  # ordered on the state's stream; the gradient call synchronises

        # gradient_pure / gradient_mixed (autodiff.hpp:95-98,184-188): the
        # input is s0 (uploaded from pinned host memory every step), the
        # result is the loss and the gradient vector, read back to the host by
        # the call itself; s0 is const in the reference API, nothing else
        # comes back
        nparams = wl.w.circuit.num_active_params()
        last = {}

        def e2e_step():
            eng.check(up(state.handle, pin, ct.c_uint64(state.size)))
            if wl.kind == "grad_pure":
                last["loss"], last["grads"] = eng.gradient_pure(wl.w.observable, wl.w.circuit, state)
            else:
                last["loss"], last["grads"] = eng.gradient_mixed(wl.w.observable, wl.w.circuit, state)
            return last["loss"]

        e2e_step()
        torch.cuda.synchronize()
        barrier(dist, local)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
        ems = max_over_ranks(dist, e0.elapsed_time(e1))
        e2e = {"value": wl.job_units(steps) / (ems / 1e3), "unit": wl.unit,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 8 * (1 + nparams),
               "ms_per_step": ems / steps, "loss": last["loss"],
               "path": "vqb_state_upload_async (s0 from pinned host memory) -> vqb_gradient_"
                       + ("pure" if wl.kind == "grad_pure" else "mixed") + " (loss + gradients to host)"}
        del h_in

    if wl.sharded:
        runner.free()
    else:
        state.free()
    eng.release_caches()
    torch.cuda.empty_cache()
    cpu_line = None
    if cpu and rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_line = cpu_baseline(wl)

    return {
        "metric": wl.metric, "value": value, "unit": wl.unit, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if (wl.sharded and wl.name == "qaoa30") else "weak",
        "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded SplitMix64 circuit, |0...0> start)",
        "config": config_block(wl, world),
        "roofline": roof,
        "kernels": {k: {"launches": v[0], "ms": round(v[1], 4)} for k, v in prof.items()},
        # the reference's unfused per-gate schedule's byte count per unit time,
        # as a multiple of the HBM peak: fusion makes it > 1, it is NOT a
        # physical fraction (the physical one is roofline.frac)
        "reference_schedule_bytes_over_hbm_peak": ref_sched_gbs / peak,
        "gpu_launches": launches,
        "noisy_dm_gates": noisy_fwd,
        "sharded": sharded,
        "e2e": e2e,
        "cpu_baseline": cpu_line,
        "clocks": clk.summary(),
        "check": check,
    }


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=ALL_CONFIGS,
                    help="default: rqc28 (+ the other configs under 'configs') at N = 1, rqc33 sharded at N > 1")
    ap.add_argument("--no-extra", action="store_true", help="N = 1 default: skip the other configs")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run rqc33/qaoa30 through the sharded runner even at N = 1 (plumbing check)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    name = args.config or ("rqc33" if world > 1 else "rqc28")
    world, rank, local, dist = dist_setup(args)
    wl = Workload(name, args, world)
    if args.sharded and name in ("rqc33", "qaoa30"):
        wl.sharded = True
    if args.impl == "reference":
        return run_reference_arm(args, wl, world, rank)

    import torch
    import paper_2406_19212_b200 as vqb
    torch.cuda.set_device(local)
    eng = vqb.device()
    line = measure(wl, args, eng, world, rank, local, dist)
    if world == 1 and args.config is None and not args.no_extra:
        # BASELINE.json's other metrics, same run, same protocol
        extra = {}
        for other in ALL_CONFIGS:
            if other == name:
                continue
            ow = Workload(other, args, 1)
            # config 0's 2 ms steps need a longer timed region
            k = max(args.steps, 50) if other == "hea20" else args.steps
            extra[other] = measure(ow, args, eng, 1, rank, local, None, steps=k)
        line["configs"] = extra
        line["gpu_launches_all_configs"] = line["gpu_launches"] + sum(v["gpu_launches"] for v in extra.values())
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
