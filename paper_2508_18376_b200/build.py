"""Build libdsmoe_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2508_18376_b200.build        (or __graft_entry__.build())

Each .cu / .cpp under csrc/ is compiled to an object in build/ (parallel),
then linked into paper_2508_18376_b200/libdsmoe_b200.so with the CUDA runtime
linked statically.  The router translation unit is compiled with -fmad=false
so its float/double arithmetic rounds exactly like the reference's
(-ffp-contract=off, /root/reference/proj/CMakeLists.txt:8).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(os.path.dirname(HERE), "build", "dsmoe_b200")
LIB = os.path.join(HERE, "libdsmoe_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I" + CSRC, "-I" + os.path.join(os.path.dirname(HERE), "include")]
PER_FILE = {"router.cu": ["-fmad=false"], "reconstruct.cu": ["-fmad=false"]}


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _obj(src):
    return os.path.join(BUILD, src + ".o")


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)) if os.path.isdir(CSRC) else 0


def _compile(src, verbose=False):
    out = _obj(src)
    cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(src, []), "-c", os.path.join(CSRC, src), "-o", out]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build_variant(name: str, defines: list[str]) -> str:
    """Same library with extra -D flags into build/variants/lib<name>.so (A/B runs)."""
    out_dir = os.path.join(os.path.dirname(HERE), "build", "variants", name)
    os.makedirs(out_dir, exist_ok=True)
    srcs = sources()

    def comp(src):
        o = os.path.join(out_dir, src + ".o")
        cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(src, []), *defines, "-c", os.path.join(CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return o

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(comp, srcs))
    lib = os.path.join(out_dir, "libdsmoe_b200.so")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    newest = max(_deps_mtime(), os.path.getmtime(os.path.join(os.path.dirname(HERE), "include", "dsmoe_b200.h")))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        logs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if verbose:
        for s, l in zip(srcs, logs):
            if l.strip():
                print(f"--- {s}\n{l}", file=sys.stderr)
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *[_obj(s) for s in srcs]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_dropin(ref_include="/root/reference/proj/include") -> str | None:
    """C++ drop-in test (tests/cpp/test_dropin.cpp) against the reference's own
    headers + generators (oracle/_ref/core.a).  Only where the reference
    sources exist (this container); the binary travels to the GPU box."""
    root = os.path.dirname(HERE)
    core = os.path.join(root, "oracle", "_ref", "core.a")
    if not (os.path.isdir(ref_include) and os.path.exists(core)):
        return None
    json_dir = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
    out = os.path.join(root, "build", "test_dropin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I" + ref_include, "-I" + os.path.join(root, "include"),
           "-I/usr/local/cuda/include", "-I" + json_dir, os.path.join(root, "tests", "cpp", "test_dropin.cpp"), core,
           "-L" + HERE, "-l:libdsmoe_b200.so", "-L/usr/local/cuda/lib64", "-lcudart_static", "-ldl", "-lrt",
           "-lpthread", "-Wl,-rpath,$ORIGIN/../paper_2508_18376_b200", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"drop-in test build failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":  # --variant NAME -DX=1 ...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
