"""The C++ mirror of the reference API (include/hypercurves_b200.hpp): it
compiles against the reference's own hc:: types (CPU) and returns
NeighborLists identical to the oracle on a B200 (GPU)."""
import os
import subprocess

import pytest

from hcg_testutil import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
REF_INC = "/root/reference/proj/include"
BIN = os.path.join(ROOT, "tests", "cpp", "test_wrapper.bin")


def _build_demo():
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(CPP, "test_wrapper.cpp"),
           "-L", os.path.join(ROOT, "paper_1209_0410_b200"), "-lhcg", "-L", os.path.join(ROOT, "oracle"), "-loracle",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1209_0410_b200')}:{os.path.join(ROOT, 'oracle')}", "-o", BIN]
    subprocess.run(cmd, check=True)


def test_wrapper_compiles_and_links():
    _build_demo()
    assert os.path.exists(BIN)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent (GPU box)")
def test_wrapper_accepts_reference_types():
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                    os.path.join(CPP, "ref_types_compile.cpp")], check=True)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_wrapper_matches_oracle_on_gpu():
    if not os.path.exists(BIN):
        _build_demo()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "wrapper ok" in out.stdout
