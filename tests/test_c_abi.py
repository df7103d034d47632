"""The C ABI from plain C99 (examples/c_abi_demo.c): the header compiles as C, the
demo links against libhfb200.so alone (+ the CUDA runtime), and on a GPU it solves
L columns through hf_pcg_multi and hf_pcg_stream with bit-identical results."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1811_07717_b200", "_lib")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime_api.h")):
        pytest.skip("gcc or the CUDA headers are missing")
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "c_abi_demo.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"), "-L", LIBDIR, "-lhfb200",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_header_is_c99_and_demo_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_demo_runs_on_the_gpu(tmp_path, cuda):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "mismatches 0" in res.stdout
