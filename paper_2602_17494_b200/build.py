"""Build the in-tree C-ABI library ``libtvstokes.so`` for sm_100a with nvcc (no GPU needed)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libtvstokes.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("tvs_kernels.cu", "tvs_gemm_tc.cu", "tvs_czt.cu", "tvs_api.cu")]
HEADERS = [os.path.join(HERE, "csrc", "tvs_internal.h"), os.path.join(ROOT, "include", "tvstokes.h")]

NCCL_DIR = None
for _cand in [os.path.join(os.path.dirname(os.__file__), "site-packages", "nvidia", "nccl"),
              "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"]:
    if os.path.exists(os.path.join(_cand, "include", "nccl.h")):
        NCCL_DIR = _cand
        break

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]
if NCCL_DIR:   # the torch-bundled NCCL (same library torch loads); rpath so no LD_LIBRARY_PATH needed
    NVCC_FLAGS += ["-I", os.path.join(NCCL_DIR, "include"), "-L", os.path.join(NCCL_DIR, "lib"),
                   "-Xlinker", "-rpath=" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2"]
else:
    NVCC_FLAGS += ["-lnccl"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in SOURCES + HEADERS)


def build(force=False, verbose=False, defines=(), out=None):
    """Compile every CUDA source into libtvstokes.so (sm_100a).  Returns the library path.
    defines / out: a build-time variant into another file (A/B experiments via TVS_LIB_PATH)."""
    out = out or LIB
    if not force and not defines and out == LIB and up_to_date():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-o", out] + SOURCES
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
