"""Build libcora_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python paper_2110_10221_b200/build.py [--force] [-v]

The shared library exports the C ABI of include/cora.h.  It links the shared CUDA runtime
(libcudart.so.12, the one torch already loaded when called from Python) and resolves cuTensorMapEncodeTiled through cudaGetDriverEntryPoint, so it has
no link-time dependency on libcuda or on torch.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcora_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-DCORA_CUDA_VERSION_STR=\"12.9\"", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "cora.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out=None, objdir=None) -> str:
    """Compile every csrc/*.cu and link the shared library (extra_flags/out: experiment variants)."""
    lib = out or LIB
    if not force and not extra_flags and out is None and not _stale():
        return LIB
    objdir = objdir or os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra_flags, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + ".tmp"
    # Shared cudart: when torch is already loaded, libcudart.so.12 resolves to torch's copy, so the
    # library and the caller share ONE runtime instance (streams and events interoperate).  The
    # rpath falls back to the toolkit's copy for plain C callers.
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "shared",
                           "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    flags = [a for a in sys.argv[1:] if a.startswith("-D")]
    out = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, extra_flags=flags, out=out,
                objdir=os.path.join(HERE, "build_" + os.path.basename(out)) if out else None))
