"""In-tree build of libparl_gpu.so (nvcc, sm_100a) — no JIT cache, no setup.py.

    python -m paper_2511_18871_b200._build        # incremental
The .so lands next to this file so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libparl_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
FLAGS += os.environ.get("PARL_NVCC_EXTRA", "").split()  # A/B builds (e.g. -DATTN_POLY_MASK=0x11)
SOURCES = ["abi.cu", "k_elem.cu", "k_grpo.cu", "k_gemm_simt.cu", "k_attn.cu", "k_gemm_tc.cu", "k_attn_tc.cu"]


def _deps(src: str):
    hdrs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    return [os.path.join(CSRC, src), os.path.join(ROOT, "include", "parl_gpu.h")] + hdrs


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    if _stale(obj, _deps(src)):
        cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(BUILD, src + ".log")
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError(f"nvcc failed for {src} (see {log})")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        subprocess.check_call(cmd)
    if verbose:
        print("built", LIB)
    return LIB


def build_cpp_tests() -> str:
    """C++ drop-in parity suite: header-only layer + libparl_gpu.so + the C oracle."""
    build()
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    out = os.path.join(BUILD, "test_dropin")
    deps = [src, os.path.join(ROOT, "include", "parl_gpu.hpp"), os.path.join(ROOT, "include", "parl_gpu.h"), LIB]
    if _stale(out, deps):
        oracle_o = os.path.join(BUILD, "parl_oracle.o")
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-c", os.path.join(ROOT, "oracle", "parl_oracle.c"),
                               "-o", oracle_o])
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                               "-I/usr/local/cuda/include", src, oracle_o, "-L" + PKG, "-lparl_gpu",
                               "-Wl,-rpath," + PKG, "-lm", "-o", out])
    return out


REF_PROJ = os.environ.get("PARL_REF_PROJ", "/root/reference/proj")
REF_SUITES = {  # suite -> reference sources compiled against the drop-in headers (unmodified)
    "test_packing": [],
    "test_grpo": [],
    "test_model": ["src/gradcheck.cpp"],
    "test_pipeline": ["src/pipeline.cpp", "src/rollout.cpp", "src/tasks.cpp"],
}


def build_ref_suites() -> list:
    """The reference's own hot-path test suites (proj/tests/test_*.cpp), compiled UNMODIFIED
    from where they lie against the drop-in headers (include/parl/*.hpp shadow the reference's
    model / packing / grpo / errors headers; the rest of its include tree is used as is) with a
    doctest shim (tests/cpp/doctest), linked with libparl_gpu.so.  The reference caller code the
    suites need (pipeline.cpp, rollout.cpp, tasks.cpp, gradcheck.cpp) is compiled the same way.
    Binaries go to build/ref_suites/ (git-ignored; shipped to the GPU box); nothing is copied.
    Only where /root/reference exists (this container)."""
    if not os.path.isdir(REF_PROJ):
        return []
    build()
    out_dir = os.path.join(BUILD, "ref_suites")
    os.makedirs(out_dir, exist_ok=True)
    inc = ["-I" + os.path.join(ROOT, "tests", "cpp", "doctest"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(REF_PROJ, "include")]
    hdrs = [os.path.join(ROOT, "include", "parl", h) for h in os.listdir(os.path.join(ROOT, "include", "parl"))]
    hdrs += [os.path.join(ROOT, "include", "parl_gpu.h"), os.path.join(ROOT, "tests", "cpp", "doctest", "doctest.h")]

    def one(name):
        srcs = [os.path.join(REF_PROJ, "tests", name + ".cpp"), os.path.join(REF_PROJ, "tests", "doctest_main.cpp")]
        srcs += [os.path.join(REF_PROJ, s) for s in REF_SUITES[name]]
        exe = os.path.join(out_dir, name)
        if _stale(exe, srcs + hdrs + [LIB]):
            cmd = ["g++", "-std=c++20", "-O2", *inc, *srcs, "-L" + PKG, "-lparl_gpu", "-Wl,-rpath,$ORIGIN/../..",
                   "-lpthread", "-o", exe]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stderr[-4000:])
                raise RuntimeError(f"reference suite {name} failed to compile against the drop-in")
        return exe

    with ThreadPoolExecutor(max_workers=len(REF_SUITES)) as ex:
        return list(ex.map(one, REF_SUITES))


if __name__ == "__main__":
    build(verbose=True)
