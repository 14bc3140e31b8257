"""Build libdbfft.so in-tree for sm_100a (nvcc; no torch JIT, the .so travels with the repo)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdbfft.so")
SOURCES = ["passes.cu", "cg.cu", "monitors.cu", "peer.cu", "dbfft.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-diag-suppress", "128,177,550"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC)] + [os.path.join(HERE, "..", "include", "dbfft.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, lib=None, defines=()):
    """Compile csrc/*.cu for sm_100a into `lib` (default: the in-tree libdbfft.so)."""
    global LIB
    target = lib or LIB
    if lib is None and not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "..", "build", "obj" + ("_" + "_".join(defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)

    def comp(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-Xptxas", "-v", "-c", os.path.join(SRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(objdir, src + ".log"), "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} (rc={r.returncode}):\n{r.stderr[-4000:]}")
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(comp, SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print("built", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
