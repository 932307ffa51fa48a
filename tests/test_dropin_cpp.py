"""The reference's C++ API (include/h2mmp) compiles against the B200 library
and, on a GPU, runs the reference's call sequence end to end."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1908_05218_b200", "lib")


def _compile(out):
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L" + LIB, "-lh2mmp_b200",
           "-Wl,-rpath," + LIB, "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_api_compiles_and_links(tmp_path):
    _compile(str(tmp_path / "dropin"))
    assert (tmp_path / "dropin").exists()


@pytest.mark.gpu
def test_cpp_dropin_runs_on_gpu(tmp_path):
    exe = str(tmp_path / "dropin")
    _compile(exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0 and "DROPIN OK" in res.stdout, res.stdout + res.stderr
