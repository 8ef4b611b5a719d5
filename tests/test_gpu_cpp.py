"""Builds tests/cpp/test_cpp_api.cpp against include/psattn/*.hpp + libpsattn_b200.so and runs it
(C++ API source compatibility with the reference's psattn:: entry points)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    lib = os.path.join(ROOT, "paper_2503_00392_b200", "_lib")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", lib, "-lpsattn_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    """Compile-only check (CPU): the headers are self-contained C++20 and the library links."""
    _build(tmp_path)


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = _build(tmp_path)
    golden = os.path.join(ROOT, "tests", "golden", "attention_cases.txt")  # compiled-reference values
    r = subprocess.run([exe, golden], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    print(r.stdout)
    assert r.stdout.strip().splitlines()[-1].startswith("OK")
