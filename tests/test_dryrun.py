"""CPU: the whole host side of a gradient -- reverse programs, stage planning on
the planning pool, block fusion, lowering, kernel generation -- in the
planning-only mode (VQB_DRYRUN=1, no CUDA call is made), and that generated
kernels compile for sm_100a with nvcc (cross-compilation needs no GPU).

The mode exists for development on hosts without a GPU (tools/dryrun_dump.py);
here it is the CPU suite's coverage of the generator and of the parallel
planning pipeline. Results of a dry run are garbage by construction and are not
looked at."""
import glob
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2406_19212_b200", "csrc")


def dump(tmp_path, config, threads=None):
    out = tmp_path / ("dump_" + config + ("_t" + threads if threads is not None else ""))
    env = dict(os.environ)
    env.pop("VQB_JIT", None)
    if threads is not None:
        env["VQB_PLAN_THREADS"] = threads
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dryrun_dump.py"), config, str(out)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return out


def compile_kernel(src, tmp_path):
    cub = tmp_path / (os.path.basename(src) + ".cubin")
    r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-I", CSRC, "-Xptxas", "-v", "-o", str(cub), src], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    m = re.search(r"(\d+) bytes spill stores", r.stderr)
    return int(m.group(1)) if m else 0


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_config0_host_path_and_generated_kernels(tmp_path):
    out = dump(tmp_path, "hea20")
    fwd = sorted(glob.glob(str(out / "F_*.cu")))
    rev = sorted(glob.glob(str(out / "R_*.cu")))
    assert fwd and rev, os.listdir(out)
    # the adjoint kernels carry the factored contractions and batched reductions
    text = open(rev[len(rev) // 2]).read()
    assert "vqb_rev" in text and "__shfl_xor_sync" in text
    assert re.search(r"\bw0_\d+_[ri]\d\b", text), "no factored derivative contraction in the adjoint kernel"
    for src in (fwd[0], rev[len(rev) // 2]):
        assert compile_kernel(src, tmp_path) == 0  # no register spills


def test_parallel_planning_generates_the_same_kernels(tmp_path):
    """Stages prepared on the pool (default) and serially (VQB_PLAN_THREADS=0)
    lower to the same programs: identical dumps, file for file."""
    a = dump(tmp_path, "hea20", "0")
    b = dump(tmp_path, "hea20", "3")
    na, nb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert na == nb and na
    for n in na:
        assert open(a / n, "rb").read() == open(b / n, "rb").read(), n


def stage_count(tmp_path, config, **env_extra):
    out = tmp_path / ("plan_" + config + "_" + "_".join(f"{k}{v}" for k, v in env_extra.items()))
    env = dict(os.environ, VQB_PLAN_STATS="1", VQB_PLAN_THREADS="0", **env_extra)
    env.pop("VQB_JIT", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dryrun_dump.py"), config, str(out)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return len(re.findall(r"^\[regstage\] ", r.stderr, re.M)), len(re.findall(r"^\[regstage-rev\] ", r.stderr, re.M))


def test_searched_plan_needs_fewer_launches_than_first_fit(tmp_path):
    """Config 1 at its full size (host side only): the hill-climbed tiles pack
    the 785 gates into far fewer stages (HBM passes) than first fit -- 35 with
    3 forced low bits, 29 with 4 -- and the QAOA gradient of config 2 needs
    fewer forward and adjoint launches too."""
    first_fit, _ = stage_count(tmp_path, "rqc28", VQB_PLAN_SEARCH="0")
    searched, _ = stage_count(tmp_path, "rqc28")
    assert first_fit >= 29 and searched <= 24 and searched < first_fit, (first_fit, searched)
    f0, r0 = stage_count(tmp_path, "qaoa30", VQB_PLAN_SEARCH="0")
    f1, r1 = stage_count(tmp_path, "qaoa30")
    assert f1 <= f0 and r1 <= r0 and f1 + r1 < f0 + r0, (f0, r0, f1, r1)
