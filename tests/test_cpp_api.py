"""The C++ host API (include/swinflow/b200.hpp) as a drop-in for the reference signatures: the
reference's golden-probe test (test_swin_core.cpp:415-422) written against it compiles with plain
g++, links the sm_100a library, fails loudly without a GPU and reproduces the golden value on one."""
import os
import subprocess

import pytest

import paper_2509_13523_b200 as swf
from tests.util import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden_bin(tmp_path_factory):
    if not os.path.exists(swf.LIB_PATH):
        swf.build()
    out = str(tmp_path_factory.mktemp("cpp") / "golden_probe")
    libdir = os.path.dirname(swf.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "golden_probe.cpp"), "-o", out, "-L" + libdir,
                    "-lswinflow_b200", "-Wl,-rpath," + libdir], check=True)
    return out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU error path")
def test_cpp_no_gpu_exit_code(golden_bin):
    r = subprocess.run([golden_bin], capture_output=True, text=True)
    assert r.returncode == 4 and "device error" in r.stderr


@pytest.mark.gpu
def test_cpp_golden_probe_on_gpu(golden_bin):
    r = subprocess.run([golden_bin, "1"], capture_output=True, text=True, timeout=300)  # FP32 validation mode
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.strip()) == pytest.approx(1.2440901490316572, rel=1e-4)
