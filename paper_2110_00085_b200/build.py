"""Builds the in-tree CUDA library paper_2110_00085_b200/libpathrec_gpu.so for sm_100a.

nvcc cross-compiles without a GPU.  The whole library is compiled with --fmad=false so
that fp64 voxel indexing (DDA, pixel_of, voxel_of) is bit-identical to the reference's
FMA-free x86-64 code; FMA is used only where written out as fma().
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpathrec_gpu.so")
SOURCES = ["prc_kernels.cu", "prc_wavefront.cu", "prc_materialized.cu", "prc_nvls.cu", "prc_capi.cu", "prc_host_api.cu"]
HEADERS = ["prc_device.cuh", "prc_kernels.cuh", "prc_eval.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """The NCCL that torch loads (the nvidia-nccl wheel, 2.28).  Linking the engine against
    the same library matters: both bind the soname libnccl.so.2, so whichever loads first
    serves the process, and torch's libtorch_cuda needs 2.28 symbols the system 2.27
    lacks (ncclDevCommCreate)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    return ""


NCCL_DIR = _nccl_dir()
CHECKED_OUT = os.path.join(HERE, "libpathrec_gpu_checked.so")  # -DPRC_CHECKED (tests/test_checked.py)

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden,-O2",
    "-Xptxas", "-v",
] + (["-I", os.path.join(NCCL_DIR, "include")] if NCCL_DIR else [])


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(SRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "pathrec_gpu.h"))
    deps.append(os.path.join(HERE, "..", "include", "pathrec.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """defines/out: A/B experiment builds (-D overrides into a separate .so)."""
    if out == OUT and not defines and not force and not _stale():
        return OUT
    tag = "" if out == OUT else "." + os.path.basename(out).replace(".so", "")
    objs, procs = [], []
    for s in SOURCES:  # the translation units compile in parallel
        obj = os.path.join(SRC if not tag else os.path.dirname(out), s.replace(".cu", tag + ".o"))
        cmd = [NVCC, *FLAGS, *("-D" + d for d in defines), "-c", os.path.join(SRC, s), "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for s, p in procs:
        so, se = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(se)
        if not tag:  # register / spill report (compile times dropped: the file is tracked)
            with open(os.path.join(SRC, s.replace(".cu", ".ptxas.txt")), "w") as f:
                f.write("".join(l for l in se.splitlines(True) if "Compile time" not in l))
    tmp = out + ".tmp"
    if NCCL_DIR:
        nccl = ["-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker",
                "-rpath," + os.path.join(NCCL_DIR, "lib")]
    else:
        nccl = ["-lnccl", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, *nccl,
           "-Xlinker", "-soname," + os.path.basename(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DNAME=VALUE ...]
    args = sys.argv[1:]
    out = OUT
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, defines=defs, out=out))
