"""Build libgs.so in-tree with nvcc for sm_100a (no torch JIT, no CPU fallback)."""
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgs.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    site = sysconfig.get_paths()["purelib"]
    d = os.path.join(site, "nvidia", "nccl")
    if not os.path.exists(os.path.join(d, "include", "nccl.h")):
        raise RuntimeError(f"NCCL headers not found under {d}")
    return d


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def up_to_date(lib=LIB):
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force=False, verbose=False, defines=(), lib=LIB):
    """Compile every source for sm_100a and link `lib`.  `defines` (e.g. "GS_ATTN_ALT=1") build a
    development variant of the library for A/B runs (tools/kbench.py --lib); numerics-changing
    choices are compile-time constants, never environment variables."""
    if not force and up_to_date(lib):
        return lib
    nd = nccl_dir()
    tag = "_".join(d.replace("=", "") for d in defines)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objs = []
    bdir = os.path.join(HERE, "build" + ("_" + tag if tag else ""))
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
               "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
               *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose and out:
            sys.stderr.write(out.decode())
    link = [nvcc, *ARCH, "-shared", "-o", lib, *objs,
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode())
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), LIB)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, lib=out))
