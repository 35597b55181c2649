"""Build libxlmimo_b200.so in-tree with nvcc for sm_100a (no torch types).

Every translation unit is compiled to an object in parallel (``build/obj``),
then linked once; a unit is recompiled only when it or a header changed."""

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_native", "libxlmimo_b200.so")
SOURCES = ["xl_abi.cu", "simt_gemm.cu", "simt_solve.cu", "chan_gen.cu", "fused_tc.cu", "link_ber.cu",
           "gemm_tc.cu", "cluster_pcg.cu", "stream_tc.cu", "large_k.cu", "dmma.cu", "fused_c128.cu",
           "fused_c64s.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
          "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills"]
LDFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-lcublas",
           "-Xlinker", "-rpath=/usr/local/cuda/lib64"]


def _sources():
    return [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def build(verbose=False, force=False, out=None, extra=()):
    """Compile the library (mtime-checked).  ``out``/``extra`` build a
    development variant (e.g. ``-DXL_...``) elsewhere for A/B timing."""
    srcs = [os.path.join(CSRC, s) for s in _sources()]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "xlmimo_b200.h"))
    lib = out or LIB
    hdr_t = max(os.path.getmtime(d) for d in hdrs)
    if (not force and out is None and os.path.exists(lib)
            and os.path.getmtime(lib) >= max([hdr_t] + [os.path.getmtime(s) for s in srcs])):
        return lib
    tag = "dev" if (out or extra) else "prod"
    objdir = os.path.join(os.path.dirname(HERE), "build", "obj_" + tag)
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if (not force and not extra and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(hdr_t, os.path.getmtime(src))):
            return obj
        cmd = [NVCC, *CFLAGS, *extra, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.stdout or r.stderr:
            print(r.stdout + r.stderr, end="", flush=True)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd)
        return obj

    with cf.ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = [NVCC, *LDFLAGS, "-o", lib, *objs]
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
