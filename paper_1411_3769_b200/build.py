"""Build libpolya.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpolya.so")
SOURCES = ["polya_host.cpp", "kernels.cu", "schur.cu", "ipm.cu", "combine.cpp"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-lcusolver", "-lcublas"]


def _nccl_flags():
    """Link the NCCL that PyTorch itself loads (the pip nvidia-nccl wheel), with an rpath to it: the
    process then holds ONE libnccl.so.2 whichever of torch / libpolya is loaded first (the system
    libnccl.so.2 is an older release whose early load would break torch's NCCL symbols)."""
    import sysconfig
    for base in (sysconfig.get_paths().get("purelib"), sysconfig.get_paths().get("platlib")):
        d = os.path.join(base or "", "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")) and os.path.exists(os.path.join(d, "include", "nccl.h")):
            return ["-I" + os.path.join(d, "include"), "-L" + os.path.join(d, "lib"),
                    "-Xlinker", "-rpath=" + os.path.join(d, "lib"), "-l:libnccl.so.2"]
    return ["-lnccl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "polya.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile the library.  `out`/`defines` build experiment variants (tools/schur_exp.py)."""
    if out == LIB and not defines and not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *FLAGS, *_nccl_flags(), *[f"-D{d}" for d in defines], "-o", out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
