"""The C++ drop-in headers (include/tilefuse/*.hpp) compile against the
reference's API surface and, on a B200, pass the conformance program
(tests/cpp/conformance.cpp) through libtfg."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "conformance")


def build_exe():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["/usr/bin/g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "conformance.cpp"),
           "-L", os.path.join(ROOT, "paper_2407_00243_b200"), "-ltfg",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2407_00243_b200"), "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return EXE


def test_headers_compile_and_link():
    build_exe()


@pytest.mark.gpu
def test_conformance_program_passes(cuda):
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
