"""Regenerate specialised kernels from dumped lowered programs (VQB_JIT_DUMP)
on the host and report what ptxas makes of them: registers, spills, SASS
size, executed FP64 flops per amplitude. No GPU needed.
usage: jit_inspect.py <dump dir> [out dir]"""
import ctypes as ct
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_19212_b200 as vqb  # noqa: E402

lib = ct.CDLL(vqb.library_path())
fn = lib.vqb_debug_jit_source
fn.restype = ct.c_int
fn.argtypes = [ct.c_int32, ct.c_void_p, ct.c_size_t, ct.c_int32, ct.c_char_p, ct.c_size_t,
               ct.POINTER(ct.c_double)]
CSRC = os.path.join(ROOT, "paper_2406_19212_b200", "csrc")


def inspect(path, outdir):
    base = os.path.basename(path)[:-len(".params")]
    rev = base.startswith("R_")
    regs = 8 if "_rs8_" in base else 16
    blob = open(path, "rb").read()
    buf = ct.create_string_buffer(1 << 24)
    fl = ct.c_double()
    rc = fn(regs, blob, len(blob), int(rev), buf, len(buf), ct.byref(fl))
    if rc != 0:
        return base, f"generator rc {rc}: {lib.vqb_last_error()}"
    src = os.path.join(outdir, base + ".cu")
    open(src, "wb").write(buf.value)
    cub = os.path.join(outdir, base + ".cubin")
    r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-I", CSRC, "-Xptxas", "-v", "-o", cub, src], capture_output=True, text=True)
    info = r.stderr
    m_regs = re.search(r"Used (\d+) registers", info)
    m_sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", info)
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    ninst = len(re.findall(r"^\s+/\*[0-9a-f]{4,}\*/", sass, re.M))
    nfp64 = len(re.findall(r"\b(DFMA|DMUL|DADD)\b", sass))
    return base, (f"regs {m_regs.group(1) if m_regs else '?'} spill st/ld "
                  f"{m_sp.group(1) + '/' + m_sp.group(2) if m_sp else '?'} sass {ninst} fp64 {nfp64} "
                  f"flops/amp {fl.value:.1f}" + ("" if r.returncode == 0 else " COMPILE FAILED " + info[-500:]))


if __name__ == "__main__":
    d = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else d + "_regen"
    os.makedirs(out, exist_ok=True)
    for p in sorted(glob.glob(os.path.join(d, "*.params"))):
        b, s = inspect(p, out)
        print(b, s, flush=True)
