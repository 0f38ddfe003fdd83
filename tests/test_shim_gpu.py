"""The reference-side C++ shim (include/cbm_b200_shim.hpp) with the
reference's own CbmMatrix/DenseMatrix types, builder and test cases
(tests/cpp/test_shim.cpp, built into oracle/_ref/test_shim)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_shim")


@pytest.mark.gpu
def test_reference_shim_bitwise_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_shim not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_shim_header_compiles_against_reference_types():
    src = "/root/reference/proj/include"
    if not os.path.isdir(src):
        pytest.skip("reference headers absent (GPU box)")
    code = '#include "cbm_b200_shim.hpp"\nint main() { return 0; }\n'
    r = subprocess.run(["g++", "-std=c++20", "-DCBM_SINGLE_PRECISION", "-fsyntax-only",
                        f"-I{src}", f"-I{os.path.join(ROOT, 'include')}", "-x", "c++", "-"],
                       input=code, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
