"""Builds tests/cpp/test_cxx_api.cpp against the C++ drop-in API
(include/tpo/*.hpp, libtpo_b200.so) and the oracle; the link check runs on
CPU, the program itself on the GPU."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "tests" / "cpp" / "build" / "test_cxx_api"


def build_exe(orc):
    EXE.parent.mkdir(parents=True, exist_ok=True)
    pkg = ROOT / "paper_2506_13523_b200"
    cmd = ["g++", "-std=c++20", "-O1", str(ROOT / "tests" / "cpp" / "test_cxx_api.cpp"),
           f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle'}", f"-L{pkg}", "-ltpo_b200",
           f"-L{ROOT / 'oracle' / 'build'}", "-ltpo_oracle",
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{ROOT / 'oracle' / 'build'}", "-o", str(EXE)]
    subprocess.run(cmd, check=True)
    return EXE


def test_cxx_api_links(orc):
    assert build_exe(orc).exists()


@pytest.mark.gpu
def test_cxx_api_runs_on_gpu(orc):
    exe = build_exe(orc)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, env=dict(os.environ))
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
