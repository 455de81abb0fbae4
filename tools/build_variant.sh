#!/bin/bash
# Build library variants of one translation unit with extra -D flags into ab/
# (development A/B timing; the production build never sets these):
#   tools/build_variant.sh NAME "-DFLAG=1 ..." [source.cu]
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; src=${3:-assemble3d.cu}
mkdir -p variants/$name
python - "$name" "$flags" "$src" <<'PY'
import os, subprocess, sys, glob
sys.path.insert(0, ".")
from paper_1809_05471_b200 import build as B
name, flags, src = sys.argv[1], sys.argv[2].split(), sys.argv[3]
obj = f"variants/{name}/{os.path.splitext(src)[0]}.o"
subprocess.run([B.NVCC, *B.ARCH, *B.COMMON, *flags, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True,
               capture_output=True)
objs = [os.path.join(B.BUILD, os.path.splitext(n)[0] + ".o") for n in B.SOURCES if n != src] + [obj]
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", f"variants/{name}/libigs_b200.so", *objs, "-lcudart", "-lcuda",
                "-lgomp", "-ldl"], check=True)
print("built", f"variants/{name}/libigs_b200.so")
PY
