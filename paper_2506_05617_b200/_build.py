"""Build the sm_100a C-ABI library in-tree (lib/libconvspectra_b200.so).

nvcc cross-compiles for B200 without a GPU.  The library links the CUDA
runtime statically so it does not depend on which libcudart torch loaded;
device pointers and streams are shared through the driver's primary context.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(os.path.dirname(HERE), "build", "obj")
LIBNAME = "libconvspectra_b200.so"
LIBPATH = os.path.join(LIBDIR, LIBNAME)

SOURCES = ["cs_api.cu", "cs_symbol.cu", "cs_jacobi.cu", "cs_jacobi_f32.cu", "cs_jacobi_f64.cu",
           "cs_spectrum.cu", "cs_warm.cu", "cs_tcb.cu",
           "cs_operator.cu", "cs_analysis.cu", "cs_fft.cu"]
# cuFFT (the FFT comparison route only) from the CUDA toolkit of this image
LINK_LIBS = ["-lcufft", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA library cannot be built")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "convspectra_b200.h"))
    cc = nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([cc] + NVCC_FLAGS + ["-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, flush=True)

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIBPATH, objs):
        run([cc] + ARCH + ["-shared", "-cudart", "static", "-o", LIBPATH] + objs + LINK_LIBS)
    return LIBPATH


if __name__ == "__main__":
    print(build(verbose=True))
