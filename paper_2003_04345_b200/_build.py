"""In-tree build of libmb4cu.so (nvcc, sm_100a) and the oracle checkers."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CUDA_SOURCES = ["mb4cu_api.cu", "sweep_tiled.cu", "sweep_march.cu", "sweep_march2.cu", "halo.cu", "krylov.cu",
                "methods.cu", "fft_precond.cu"]
HOST_SOURCES = ["scheme_host.cpp", "inputs_host.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def _sources():
    return [s for s in CUDA_SOURCES + HOST_SOURCES if os.path.exists(os.path.join(CSRC, s))]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


GEN_DIR = os.path.join(ROOT, "build", "gen")


def gen_default_scheme() -> str:
    """Generate build/gen/defscheme.inc: the default MB4 scheme tables as exact
    hex-float constants, from the library's own long-double scheme routine."""
    inc = os.path.join(GEN_DIR, "defscheme.inc")
    srcs = [os.path.join(CSRC, f) for f in ("gen_default_scheme.cpp", "scheme_host.cpp", "mb4cu_internal.hpp")]
    if not _stale(inc, srcs + [os.path.join(ROOT, "include", "mb4cu.h")]):
        return inc
    os.makedirs(GEN_DIR, exist_ok=True)
    exe = os.path.join(GEN_DIR, "gen_default_scheme")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    srcs[0], srcs[1], "-o", exe], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    tmp = inc + ".tmp"
    with open(tmp, "w") as f:
        f.write(out)
    os.replace(tmp, inc)
    return inc


def build_lib(force: bool = False, verbose: bool = False, defines=(), name: str = "libmb4cu.so") -> str:
    """Build libmb4cu.so (or an experiment variant with extra -D defines)."""
    target = os.path.join(HERE, name)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "mb4cu.h")]
    if not force and not _stale(target, deps):
        return target
    objs = []
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    gen_default_scheme()
    procs = []
    for src in _sources():
        obj = os.path.join(ROOT, "build", name + "." + src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", GEN_DIR, "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose and out:
            print(out)
    tmp = target + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lcufft", "-lpthread", "-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


def build_oracle() -> None:
    """Compile oracle/ (the C restatement; and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8", "all"], check=True)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_lib(force=force, verbose=verbose)
    build_oracle()


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
