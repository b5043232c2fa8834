"""The boundary from plain C: compile tests/c/abi_smoke.c with gcc against
include/ds.h, link libds.so (no Python, no torch), run the host-only part on
the CPU and the device part on the GPU."""
import os
import subprocess

import pytest

import paper_1103_4881_b200 as ds
from conftest import ROOT


def _build(tmp_path):
    lib = ds.lib_path()
    ds.lib()                                   # builds libds.so if needed
    exe = str(tmp_path / "abi_smoke")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror",
                           "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_smoke.c"),
                           lib, f"-Wl,-rpath,{os.path.dirname(lib)}",
                           # the program's own CUDA runtime for cudaMalloc/cudaMemcpy (libds.so
                           # links cudart statically and exports only ds_*)
                           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64",
                           "-o", exe])
    return exe


def test_c_program_host_part(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "host part ok" in out.stdout


@pytest.mark.gpu
def test_c_program_gpu_part(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu part ok (kernel 1)" in out.stdout
