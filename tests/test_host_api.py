"""The C++ host API (include/pathrec_gpu.hpp) compiles here and passes its GPU test."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def build_host_test(tmp_path):
    from paper_2110_00085_b200.build import build
    lib = build()
    from pyoracle import build_port
    port = build_port()
    exe = str(tmp_path / "host_api_test")
    subprocess.check_call([
        "g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
        os.path.join(ROOT, "tests", "cpp", "host_api_test.cpp"), "-o", exe,
        lib, port, f"-Wl,-rpath,{os.path.dirname(lib)}:{os.path.dirname(port)}"])
    return exe


def test_host_api_compiles(tmp_path):
    assert os.path.exists(build_host_test(tmp_path))


@pytest.mark.gpu
def test_host_api_on_gpu(tmp_path):
    exe = build_host_test(tmp_path)
    r = subprocess.run([exe], cwd=str(tmp_path), capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
