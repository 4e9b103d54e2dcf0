"""Build libtwc.so in-tree with nvcc for sm_100a (the only target).

    python -m paper_2412_12382_b200.build [--verbose]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtwc.so")
# the checked build: the same sources with -DTWC_CHECKED, i.e. device-side asserts on every
# shared-memory ring / staging index, every computed global index and every capacity the kernels
# rely on (twc_common.cuh TWC_ASSERT).  compute-sanitizer is not available on this GPU pool, so
# the test suite runs against this library instead (TWC_LIB=checked, scripts/gpu_checked.sh).
LIB_CHECKED = os.path.join(HERE, "libtwc_checked.so")
SOURCES = ["twc_scan.cu", "twc_score.cu", "twc_cluster.cu", "twc_similarity.cu", "twc_stats.cu",
           "twc_k4.cu", "twc_dist.cu", "twc_api.cu"]
HEADERS = ["twc_common.cuh", "twc_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-Wall",
    "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "twc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, checked=False, variant=None, defines=()):
    """variant: an A/B build libtwc_<variant>.so of the same sources with extra -D defines
    (loaded with TWC_LIB=<variant>; measurement only, never the default library)."""
    lib = LIB_CHECKED if checked else LIB
    if variant:
        lib = os.path.join(HERE, f"libtwc_{variant}.so")
    if not force and not _stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-DTWC_CHECKED"] if checked else []), *defines,
           *(["-Xptxas", "-v"] if verbose else []), "-o", tmp,
           *[os.path.join(CSRC, f) for f in SOURCES]]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    _variant = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else None
    print(build(force=True, verbose="--verbose" in sys.argv, checked="--checked" in sys.argv,
                variant=_variant, defines=[a for a in sys.argv[1:] if a.startswith("-D")]))
