"""Build the sm_100a C-ABI library in-tree: paper_2603_11953_b200/libmpsvd_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a (B200 only), -lineinfo for ncu
source mapping, -fmad=false so every device FMA is explicit (see
csrc/common.cuh). The CUDA runtime is linked statically; NCCL is dlopen'ed
at first multi-rank use.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmpsvd_b200.so")
SOURCES = ["gram.cu", "gram_ozaki.cu", "gram_ozaki32.cu", "jacobi.cu", "compute_u.cu", "compute_u_tc.cu", "metrics.cu", "onesided.cu", "cholqr.cu", "microbench.cu", "engine.cu", "api.cpp", "textio.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(ROOT, "include", "mpsvd.h")]
    deps += [os.path.join(ROOT, "include", "mpsvd", f) for f in os.listdir(os.path.join(ROOT, "include", "mpsvd"))]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.rsplit(".", 1)[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"[build] {src} failed:\n{' '.join(cmd)}\n{out}\n")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("nvcc failed")
    link = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-ldl", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return OUT


REF_INCLUDE = "/root/reference/proj/include"
C_SRC = os.path.join(ROOT, "tests", "c", "capi_ref.c")
C_BIN = os.path.join(ROOT, "tests", "c", "_bin")


def build_c_consumers() -> list[str]:
    """The C consumer tests/c/capi_ref.c, linked to the library, compiled
    twice: against the reference's own C header (capi_ref; only where
    /root/reference exists - the binary then travels with the repo) and
    against this repo's include/mpsvd.h (capi_own)."""
    os.makedirs(C_BIN, exist_ok=True)
    out = []
    targets = [("capi_own", os.path.join(ROOT, "include"))]
    if os.path.isfile(os.path.join(REF_INCLUDE, "mpsvd.h")):
        targets.insert(0, ("capi_ref", REF_INCLUDE))
    for name, inc in targets:
        exe = os.path.join(C_BIN, name)
        cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", f"-I{inc}", C_SRC, "-o", exe, f"-L{HERE}",
               "-l:libmpsvd_b200.so", "-Wl,-rpath,$ORIGIN/../../../paper_2603_11953_b200", "-lm"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C consumer {name} failed to build:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
        out.append(exe)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
