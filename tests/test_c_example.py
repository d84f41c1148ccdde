"""The C ABI used from plain C (examples/c_abi_step.c, no Python / PyTorch in
the process): it compiles against include/attn_softmax.h with gcc (CPU) and
runs one stage step on the GPU with a sane loss and a documented error path."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1909_00562_b200", "lib")
CUDA = "/usr/local/cuda"


def _compile(tmp_path, built_lib):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "c_abi_step")
    cmd = [gcc, "-std=c99", "-Wall", "-Werror", "-o", exe, os.path.join(ROOT, "examples", "c_abi_step.c"),
           "-I" + os.path.join(ROOT, "include"), "-I" + CUDA + "/include", "-L" + LIBDIR, "-lattnsm",
           "-L" + CUDA + "/lib64", "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles(built_lib, tmp_path):
    _compile(tmp_path, built_lib)


@pytest.mark.gpu
def test_c_example_runs(cuda_lib, tmp_path):
    exe = _compile(tmp_path, cuda_lib)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sm_100a" in r.stdout and "status 1" in r.stdout
