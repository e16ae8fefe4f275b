"""The reference-typed C++ adapter (include/sconv_b200.hpp) compiled against the
reference's own headers: compile check here (CPU), full run on the GPU."""
import os
import subprocess

import pytest

from oracle_lib import ROOT

EXE = os.path.join(ROOT, "tests", "cpp", "test_adapter")
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers only exist on the build machine")
def test_adapter_compiles_against_reference_headers(tmp_path):
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-DSCONV_ORACLE_USE_REFERENCE", f"-I{REF_INC}",
                        f"-I{ROOT}/include", f"-I{ROOT}/oracle",
                        os.path.join(ROOT, "tests", "cpp", "test_adapter.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_adapter_runs_on_gpu():
    if not os.path.exists(EXE):
        pytest.skip("adapter binary not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "threw=1" in r.stdout and "failures 0" in r.stdout
