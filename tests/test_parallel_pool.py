"""The host ThreadPool (csrc/host/parallel.cpp) against its contract: tests/cpp/test_parallel.cpp
compiled with g++ and run (CPU only)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ absent")
def test_thread_pool_contract(tmp_path):
    exe = tmp_path / "test_parallel"
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/test_parallel.cpp",
                    f"{ROOT}/paper_1502_00355_b200/csrc/host/parallel.cpp", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "ok"
