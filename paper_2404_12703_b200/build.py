"""Build the in-tree CUDA library ``csrc/libhexdg_b200.so`` for sm_100a.

Three translation units: kernels_exact.cu (-fmad=false: bit-exact vs the
reference), kernels_fast.cu (FMA contraction) and api.cu (the C ABI). Objects
are compiled in parallel and linked with nvcc; the library lands next to its
sources so it travels with the repo snapshot to the GPU box.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# A/B builds: HEXDG_BUILD_DIR puts objects + library elsewhere (load it with HEXDG_B200_LIB)
OUT = os.environ.get("HEXDG_BUILD_DIR") or CSRC
LIB = os.path.join(OUT, "libhexdg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("HEXDG_NVCC_EXTRA", "").split()   # e.g. -DE2_TIMING (A/B builds)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--use_fast_math=false",
          "-Xptxas", "-v"] + ARCH
UNITS = {
    "kernels_exact.cu": ["-fmad=false"],
    "kernels_fast.cu": ["-fmad=true"],
    "api.cu": ["-fmad=false"],
}
HEADERS = ["common.cuh", "physics.cuh", "kernels.cuh", "elem.cuh", "elem2.cuh", "api_kernels.cuh",
           "launch.cuh"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(unit, flags, verbose):
    src = os.path.join(CSRC, unit)
    obj = os.path.join(OUT, unit.replace(".cu", ".o"))
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(HERE, "..", "include", "hexdg_b200.h"), __file__]
    if not _stale(obj, deps):
        return obj, ""
    cmd = [NVCC, "-c", src, "-o", obj] + COMMON + EXTRA + [f for f in flags if f != "--use_fast_math=false"]
    cmd = [c for c in cmd if c != "--use_fast_math=false"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {unit}:\n{res.stderr}")
    return obj, res.stderr if verbose else ""


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile (if stale) and return the path of libhexdg_b200.so."""
    os.makedirs(OUT, exist_ok=True)
    if force:
        for u in UNITS:
            o = os.path.join(OUT, u.replace(".cu", ".o"))
            if os.path.exists(o):
                os.remove(o)
    with ThreadPoolExecutor(len(UNITS)) as ex:
        results = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), UNITS.items()))
    objs = [r[0] for r in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + ["-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
