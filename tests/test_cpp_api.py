"""The C++ host mirror (include/hexbp_b200.hpp) driven like the reference's
own callers (tests/cpp/test_host_api.cpp), on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_host_api")
HDR = os.path.join(ROOT, "include", "hexbp_b200.hpp")


def build_cpp_test(name: str = "test_host_api") -> str:
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    out = os.path.join(ROOT, "tests", "cpp", name)
    if not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(src), os.path.getmtime(HDR)):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src,
                        "-L", os.path.join(ROOT, "paper_2109_05072_b200"), "-lhexbp_b200",
                        "-Wl,-rpath,$ORIGIN/../../paper_2109_05072_b200", "-o", out], check=True)
    return out


def test_cpp_header_compiles_and_links():
    assert os.path.exists(build_cpp_test())
    assert os.path.exists(build_cpp_test("test_dist_api"))


@pytest.mark.gpu
def test_cpp_host_api_on_device():
    out = subprocess.run([build_cpp_test()], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout


@pytest.mark.gpu
def test_cpp_distributed_api_on_device():
    """hexbp::b200::DistributedOperator (hexbp_dist_*, library-owned NCCL
    communicator) against the single-GPU operator and CG."""
    out = subprocess.run([build_cpp_test("test_dist_api")], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
