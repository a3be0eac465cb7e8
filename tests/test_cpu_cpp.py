"""CPU: the C++ layer (include/zcomm_b200.hpp) compiles with g++ against the C-ABI library and its
host-side entry points behave like the reference's C++ API (tests/cpp/host_api_test.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_12396_b200")


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_cpp_host_api(tmp_path):
    exe = tmp_path / "host_api_test"
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_api_test.cpp"), "-L", LIBDIR, "-lzcomm_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
