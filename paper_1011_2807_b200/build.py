"""Build libknnjoin.so in-tree: nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a), -lineinfo,
one object per translation unit (compiled in parallel), static cudart, hidden visibility except the C ABI."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libknnjoin.so")
BUILD = os.path.join(HERE, "build")
SOURCES = ["index_build.cu", "query.cu", "merge.cu", "accumulate_ks1.cu", "accumulate_ks4.cu", "accumulate_ks8.cu", "iiib.cu", "wide.cu"]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
# checked builds (tools/checked_build.sh): KJ_EXTRA_NVCC_FLAGS="-DKJ_CHECKS" adds the device-side bounds checks
FLAGS += os.environ.get("KJ_EXTRA_NVCC_FLAGS", "").split()


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    log = obj + ".ptxas.txt"
    cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


def newest_source_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "knnjoin.h")]
    return max(os.path.getmtime(f) for f in files if os.path.exists(f))


def up_to_date() -> bool:
    return os.path.exists(OUT) and os.path.getmtime(OUT) >= newest_source_mtime()


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = OUT + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xlinker", "--no-undefined",
                           "-o", tmp, *objs])
    os.replace(tmp, OUT)
    if verbose:
        print(f"built {OUT}", file=sys.stderr)
    return OUT


if __name__ == "__main__":
    # --src DIR --out FILE: build a variant library from another source tree (A/B experiments, tools/ab.py)
    if "--src" in sys.argv:
        CSRC = os.path.abspath(sys.argv[sys.argv.index("--src") + 1])
        OUT = os.path.abspath(sys.argv[sys.argv.index("--out") + 1])
        BUILD = OUT + ".build"
        build(force=True)
    else:
        build(force="--force" in sys.argv)
