"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads, exports every
symbol include/swinflow_capi.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import subprocess

import pytest

import paper_2509_13523_b200 as swf
from tests.util import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(swf.LIB_PATH):
        swf.build()
    return swf.lib()


def test_exports_every_declared_symbol(built):
    names = swf.exported_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(built, n)]
    assert not missing, missing


def test_param_count_formula_matches_reference_golden(built):
    # parameter_count_formula (model.hpp:118-129); golden 1,324,144,198 (test_swin_core.cpp:157-173)
    c = swf.ModelConfig(1536, 12, 9216, 10, 2, 30, 144, 70)
    assert swf.param_count(c) == 1324144198


def test_library_is_sm100a_only(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", swf.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", swf.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # tcgen05.mma + TMA present


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly(built):
    with pytest.raises(swf.SwfError) as ei:
        swf.Denoiser(swf.ModelConfig(128, 4, 256, 2, 1, 8, 8, 3), 32, 64)
    assert ei.value.rc in (swf.ERR_CUDA, swf.ERR_CONFIG)


def test_config_errors_before_device(built):
    # ConfigError (rc 2) for shape problems, like the reference's require() (common.hpp:53-55)
    with pytest.raises(swf.ConfigError):
        swf.Denoiser(swf.ModelConfig(128, 4, 256, 2, 1, 8, 8, 3), 30, 64)  # 30 % 8 != 0
    with pytest.raises(swf.ConfigError):
        swf.Denoiser(swf.ModelConfig(130, 5, 256, 2, 1, 8, 8, 3), 32, 64)  # head_dim 26 % 4 != 0
