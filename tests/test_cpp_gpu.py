"""The reference's unit-test scenarios in C++ against include/latsum_b200/latsum.hpp
(reference names and exception types over the C ABI), run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_header_builds():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])


@pytest.mark.gpu
def test_cpp_dropin_scenarios():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    out = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_latsum_hpp")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK (0 failures)" in out.stdout
