"""Build libnnls_b200.so in-tree with nvcc for sm_100a (no JIT, no torch types)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnnls_b200.so")
SOURCES = ["api.cu", "ingest_gram.cu", "pivot.cu", "cholesky.cu", "lsqr.cu", "batched.cu", "condest.cu", "gram_dense.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "nnls.h")]
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        # NNLS_EXTRA_NVCC_FLAGS: development A/B switches (e.g. -DNAME), empty by default
        extra = os.environ.get("NNLS_EXTRA_NVCC_FLAGS", "").split()
        cmd = [nvcc, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    # static CUDA runtime: the headers we compile against (12.9) and the
    # runtime must match; a dynamic libcudart.so.12 would resolve to whatever
    # the process loaded first (e.g. torch's 12.8 wheel)
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                           *objs, "-cudart", "static", "-Xcompiler", "-fvisibility=hidden"])
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
