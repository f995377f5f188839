"""Build libaca.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with gpurun)."""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libaca.so")
SOURCES = [os.path.join(CSRC, "aca.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("aca_kernels.cuh", "aca_tile.cuh", "aca_misc.cuh", "aca_prim.cuh", "nlog_tables.cuh", "gauss_tables.cuh", "aca_eff.cuh", "aca_agg.cuh", "aca_res.cuh", "aca_qnbr.cuh")] + \
    [os.path.join(ROOT, "include", "aca.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fno-fast-math", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")]


def build(force=False, verbose=False):
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest:
        return SO
    for tab, gen in (("nlog_tables.cuh", "gen_nlog_tables.py"), ("gauss_tables.cuh", "gen_gauss_tables.py")):
        if not os.path.exists(os.path.join(CSRC, tab)):
            subprocess.check_call([sys.executable, os.path.join(CSRC, gen)])
    log = os.path.join(PKG, "build_ptxas.log")
    cmd = [NVCC] + FLAGS + ["-o", SO] + SOURCES + ["-ldl"]
    with open(log, "w") as f:
        r = subprocess.run(cmd, stdout=f, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(open(log).read()[-8000:])
        raise RuntimeError("nvcc failed building libaca.so (see %s)" % log)
    if verbose:
        print(open(log).read())
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
