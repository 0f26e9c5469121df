"""The C++ drop-in headers (include/sphemu/*.hpp over the C-ABI): CPU — they
compile with -Wall -Wextra and link against the library; GPU — the test
program mirroring the reference's C++ test cases passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "build.sh")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_cpp_api")


def build():
    r = subprocess.run([BUILD], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "warning" not in r.stderr, r.stderr
    return BIN


def test_headers_compile_and_link(sph):
    sph._sphemu.lib()  # the library exists (built by __graft_entry__.build())
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cpp_api_on_gpu(sph):
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
