"""The C++ host API (include/swinflow/b200.hpp) as a drop-in for the reference signatures: the
reference's golden-probe test (test_swin_core.cpp:415-422) written against it compiles with plain
g++, links the sm_100a library, fails loudly without a GPU and reproduces the golden value on one."""
import os
import subprocess

import pytest

import paper_2509_13523_b200 as swf
from tests.util import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path_factory, name):
    if not os.path.exists(swf.LIB_PATH):
        swf.build()
    out = str(tmp_path_factory.mktemp("cpp") / name)
    libdir = os.path.dirname(swf.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", out, "-L" + libdir,
                    "-lswinflow_b200", "-Wl,-rpath," + libdir, "-lpthread"], check=True)
    return out


@pytest.fixture(scope="module")
def golden_bin(tmp_path_factory):
    return _compile(tmp_path_factory, "golden_probe")


@pytest.fixture(scope="module")
def group_bin(tmp_path_factory):
    return _compile(tmp_path_factory, "group_probe")


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU error path")
def test_cpp_no_gpu_exit_code(golden_bin):
    r = subprocess.run([golden_bin], capture_output=True, text=True)
    assert r.returncode == 4 and "device error" in r.stderr


@pytest.mark.gpu
def test_cpp_golden_probe_on_gpu(golden_bin):
    r = subprocess.run([golden_bin, "1"], capture_output=True, text=True, timeout=300)  # FP32 validation mode
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.strip()) == pytest.approx(1.2440901490316572, rel=1e-4)


def test_cpp_group_probe_compiles(group_bin):
    assert os.path.exists(group_bin)


@pytest.mark.gpu
def test_cpp_group_probe_on_gpu(group_bin):
    """Single-process multi-device forward() (device_ids {0,0} on a 1-GPU box, {0,1} on two) bitwise
    equal to one device; in-place parameter updates re-uploaded; block_window_forward."""
    import torch
    devs = ["0", "1"] if torch.cuda.device_count() >= 2 else ["0", "0"]
    r = subprocess.run([group_bin] + devs, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "GROUP_PROBE PASS" in r.stdout, r.stdout + r.stderr
