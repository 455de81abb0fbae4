"""Build a phase-instrumented copy of the library (IGS_PHASE_TIMING) and
print where the fused apply's cycles go (thread 0 of every CTA, summed)."""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1809_05471_b200 import build as B  # noqa: E402

src = os.path.join(B.CSRC, "apply3d.cu")
obj = "/tmp/apply3d_timing.o"
r = subprocess.run([B.NVCC, *B.ARCH, *B.COMMON, "-DIGS_PHASE_TIMING", "-c", src, "-o", obj],
                   capture_output=True, text=True)
assert r.returncode == 0, r.stderr[-3000:]
objs = [os.path.join(B.BUILD, os.path.splitext(n)[0] + ".o") for n in B.SOURCES if n != "apply3d.cu"]
lib = "/tmp/libigs_timing.so"
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, obj, *objs, "-lcudart", "-lgomp"],
                   capture_output=True, text=True)
assert r.returncode == 0, r.stderr[-3000:]
from paper_1809_05471_b200 import _lib  # noqa: E402

_lib.LIB_PATH = lib
from paper_1809_05471_b200 import matfree, workloads  # noqa: E402

L = _lib.load()
fn = L.igs_debug_phase_cycles
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["elem-end+barrier", "Z+Z^T", "Y", "X+Y^T", "-"]
for name in sys.argv[1:] or ["C4", "C5"]:
    c = workloads.CONFIGS[name]
    prob = workloads.make_problem(c["d"], c["p"], c["K"], c["kind"])
    op = matfree.MatrixFreeOperator(prob)
    x = torch.randn(prob.shape[1], dtype=torch.float64, device="cuda")
    op.apply_device(x)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    fn(buf, 1)
    op.apply_device(x)
    torch.cuda.synchronize()
    fn(buf, 1)
    tot = sum(buf[i] for i in range(5))
    print(name, " ".join(f"{names[i]}={100.0 * buf[i] / tot:.1f}%" for i in range(5)), f"total={tot:.3e} cycles",
          f"X-phase TMA wait (warp 0)={100.0 * buf[5] / tot:.1f}%")
