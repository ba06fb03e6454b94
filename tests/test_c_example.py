"""The C ABI from plain C (examples/ams_example.c): it compiles against include/ams.h and
links libams.so on CPU; on the GPU it records 4096 fp32 contexts, looks up 8 perturbed and
8 random queries, and must replay (hit, top-1 = source) exactly the perturbed ones."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "ams_example")
    lib_dir = os.path.join(ROOT, "paper_2508_10259_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", os.path.join(ROOT, "examples", "ams_example.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"), "-L", lib_dir, "-l:libams.so",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{lib_dir}", "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


def test_c_example_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("no CUDA toolkit headers")
    _build(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().endswith("ok")
