"""Build libprotea.so in-tree (nvcc, sm_100a).  Called by __graft_entry__.build()."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libprotea.so")


def nccl_dir():
    import nvidia.nccl  # torch's bundled NCCL 2.28
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def sources():
    return [os.path.join(CSRC, f) for f in ("engine.cu", "layout.cpp", "planner.cpp")]


def deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "protea.h")]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    nd = nccl_dir()
    dbg = ["-DPROTEA_DBG=1"] if os.environ.get("PROTEA_DBG") == "1" else []  # kernel cycle counters (tools)
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", *dbg,
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           *sources(), "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"), "-o", OUT + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(OUT)
