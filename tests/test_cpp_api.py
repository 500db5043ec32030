"""Builds and runs the C++ API test program (tests/cpp/test_host_api.cpp)
against include/parsol/*.hpp + libparsol_b200.so + libpsg.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_0912_3678_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_host_api")
EXE_LF = os.path.join(ROOT, "tests", "cpp", "test_localfact")


def _compile(src, exe):
    subprocess.run(["g++", "-O1", "-std=c++20", "-I" + os.path.join(ROOT, "include"), "-o", exe, src, "-L" + PKG,
                    "-lparsol_b200", "-lpsg", "-Wl,-rpath," + PKG], check=True)


@pytest.fixture(scope="module")
def exe():
    from paper_0912_3678_b200 import build
    build.build(verbose=False)
    _compile(os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp"), EXE)
    _compile(os.path.join(ROOT, "tests", "cpp", "test_localfact.cpp"), EXE_LF)
    return EXE


def test_cpp_api_host(exe):
    r = subprocess.run([exe, "--cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_api_gpu(exe, cuda):
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_localfact_gpu(exe, cuda):
    """The reference's LocalFactorization suite (proj/tests/test_localfact.cpp,
    minus ARCE) against this library, factorizations on the GPU."""
    r = subprocess.run([EXE_LF, "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert " 0 failures" in r.stdout
