# build libgorila_old.so from a git revision (default HEAD) for same-box A/B runs (tools/ab_lib.sh)
REV=${1:-HEAD}
rm -rf /tmp/oldsrc && mkdir -p /tmp/oldsrc && git -C /root/repo archive $REV paper_1507_04296_b200/csrc include | tar -x -C /tmp/oldsrc
python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, '/root/repo')
from paper_1507_04296_b200 import _build
nd = _build.nccl_dir()
subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-shared",
                       "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I" + os.path.join(nd, "include"),
                       "/tmp/oldsrc/paper_1507_04296_b200/csrc/gorila.cu", "-o",
                       "/root/repo/paper_1507_04296_b200/libgorila_old.so", "-L" + os.path.join(nd, "lib"),
                       "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")],
                      stderr=subprocess.DEVNULL)
print("built libgorila_old.so from", os.environ.get("REV", "HEAD"))
PY
