"""Build the in-tree C-ABI library libgorila.so for sm_100a (nvcc cross-compiles without a GPU)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libgorila.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")


def nccl_dir():
    import nvidia.nccl  # torch's bundled NCCL (the copy the process already loads)
    return os.path.dirname(os.path.abspath(nvidia.nccl.__file__)) if nvidia.nccl.__file__ else \
        list(nvidia.nccl.__path__)[0]


def sources():
    out = [os.path.join(INCLUDE, "gorila.h")]
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cuh")):
            out.append(os.path.join(CSRC, f))
    return out


def stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force=False, verbose=False, trace=False):
    so = SO.replace("libgorila.so", "libgorila_trace.so") if trace else SO
    if not force and not trace and not stale():
        return SO
    nd = nccl_dir()
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I" + os.path.join(nd, "include"),
           os.path.join(CSRC, "gorila.cu"), "-o", so + ".tmp",
           "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    if trace:
        cmd.insert(1, "-DGORILA_TRACE")
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force=True, verbose=True)
