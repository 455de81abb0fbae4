"""The C-ABI alone (no Python, no torch) drives the whole path: a C program
(tools/capi_example.c) builds a 3D mass+stiffness problem with igs_gauss_rule,
igs_tabulate, igs_fill_synthetic and the 1D/tensor patterns, applies it
(igs_apply), assembles it (igs_assemble_values), and checks 1ᵀA1 = Σ w·c and
CSR·x = apply·x to 1e-12."""

import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.mark.gpu
def test_c_program_through_the_c_abi(cuda, tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    lib = os.path.join(REPO, "paper_1809_05471_b200")
    exe = tmp_path / "capi_example"
    subprocess.run(["gcc", "-O2", os.path.join(REPO, "tools", "capi_example.c"), "-I", os.path.join(REPO, "include"),
                    "-I", os.path.join(CUDA, "include"), "-L", lib, "-ligs_b200", "-L", os.path.join(CUDA, "lib64"),
                    "-lcudart", "-lm", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=lib + ":" + os.path.join(CUDA, "lib64") + ":" +
               os.environ.get("LD_LIBRARY_PATH", ""))
    out = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "capi example ok" in out.stdout
