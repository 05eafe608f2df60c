"""The C++ host mirror (include/hexbp_b200.hpp) driven like the reference's
own callers (tests/cpp/test_host_api.cpp), on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_host_api")


def build_cpp_test() -> str:
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                        "-L", os.path.join(ROOT, "paper_2109_05072_b200"), "-lhexbp_b200",
                        "-Wl,-rpath,$ORIGIN/../../paper_2109_05072_b200", "-o", BIN], check=True)
    return BIN


def test_cpp_header_compiles_and_links():
    assert os.path.exists(build_cpp_test())


@pytest.mark.gpu
def test_cpp_host_api_on_device():
    out = subprocess.run([build_cpp_test()], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
