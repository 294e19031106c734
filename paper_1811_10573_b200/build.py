"""Build libcppp.so in-tree with nvcc for sm_100a (no torch JIT cache: the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcppp.so")
SOURCES = ["engine.cu", "ttm.cu", "ttv.cu", "ppupdate.cu", "solve.cu", "gen.cu", "diag.cu", "tucker.cu"]
HEADERS = ["internal.h", os.path.join("..", "..", "include", "cppp.h"),
           os.path.join("..", "..", "include", "cppp_tucker.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-gencode", "arch=compute_100a,code=sm_100a", "-I", os.path.join(ROOT, "include"),
         "-Xptxas", "-warn-spills"]
OBJDIR = os.path.join(HERE, "build_obj")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return LIB
    # one nvcc per translation unit, in parallel (no relocatable device code: the units call
    # each other only through host-side launchers), then one shared-library link
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJDIR, exist_ok=True)
    objs = [os.path.join(OBJDIR, os.path.splitext(s)[0] + ".o") for s in SOURCES]

    def compile_one(i):
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, SOURCES[i]), "-o", objs[i]]
        if verbose:
            print("[cppp build]", " ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, range(len(SOURCES))))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a"] + objs + ["-o", tmp, "-ldl"]
    if verbose:
        print("[cppp build]", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build_library(force="--force" in sys.argv)
    print(LIB)
