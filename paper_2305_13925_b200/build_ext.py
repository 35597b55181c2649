"""Build libxlmimo_b200.so in-tree with nvcc for sm_100a (no torch types)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_native", "libxlmimo_b200.so")
SOURCES = ["xl_abi.cu", "simt_gemm.cu", "simt_solve.cu", "chan_gen.cu", "fused_tc.cu", "link_ber.cu", "gemm_tc.cu", "cluster_pcg.cu", "stream_tc.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
         "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-lcublas", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]


def build(verbose=False, force=False, out=None, extra=()):
    """Compile the library (mtime-checked).  ``out``/``extra`` build a
    development variant (e.g. ``-DXL_...``) elsewhere for A/B timing."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "xlmimo_b200.h"))
    lib = out or LIB
    if (not force and out is None and os.path.exists(lib)
            and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps)):
        return lib
    os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)
    cmd = [NVCC, *FLAGS, *extra, "-o", lib, *srcs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        out = args[args.index("--out") + 1]
    build(verbose=True, force="--force" in args, out=out,
          extra=[a for a in args if a.startswith("-D")])
