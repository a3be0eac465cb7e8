"""GPU: the C++ layer (include/zcomm_b200.hpp) driven on the device — coder plugins,
profile_sample, frame_commit_raw, and LocalCommunicator::run with point-to-point and collectives
(tests/cpp/device_api_test.cpp, built with g++ against libzcomm_b200.so only)."""
import os
import shutil
import subprocess

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_12396_b200")


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_cpp_device_api(tmp_path, zc):
    exe = tmp_path / "device_api_test"
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-pthread", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "device_api_test.cpp"), "-L", LIBDIR, "-lzcomm_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
