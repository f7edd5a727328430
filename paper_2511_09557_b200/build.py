"""In-tree build of libnvrar_b200.so for sm_100a (nvcc cross-compiles; no GPU needed).

The library is plain C ABI (include/nvrar.h); it links the CUDA runtime
statically so the same file loads next to torch's own runtime.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.environ.get("NVRAR_BUILD_DIR") or os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libnvrar_b200.so")
SOURCES = ["nvrar_inst_f32.cu", "nvrar_inst_bf16.cu", "nvrar_inst_i32.cu",
           "nvrar_flat_f32.cu", "nvrar_flat_bf16.cu", "nvrar_flat_i32.cu",
           "nvrar_inst_phase_f.cu", "nvrar_inst_phase_i.cu", "nvrar_pull.cu", "nvrar_misc.cu",
           "nvrar_comm.cu"]
HEADERS = ["nvrar_device.cuh", "nvrar_kernels.cuh", os.path.join("..", "..", "include", "nvrar.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--fmad=false", "-cudart", "static", "-I" + os.path.join(ROOT, "include")]
# experiments only: extra nvcc flags (e.g. -DNVRAR_PUT_ST=...) and an output
# directory other than the in-tree lib/ (the product build uses neither)
EXTRA = os.environ.get("NVRAR_NVCC_EXTRA", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS + [os.path.basename(__file__)]:
        p = os.path.join(CSRC, f) if f != os.path.basename(__file__) else __file__
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(LIB_DIR, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        # the per-function "Compile time" lines vary run to run; drop them so a
        # rebuild leaves the tracked register/spill report unchanged
        report = "".join(l for l in r.stderr.splitlines(keepends=True)
                         if "Compile time" not in l)
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(report)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
