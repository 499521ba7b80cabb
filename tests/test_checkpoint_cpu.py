"""Weight ingestion from the reference checkpoint format (checkpoint.hpp:29-89): strict manifest
and fnv1a64 checks on the host (no GPU)."""
import os

import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o

TINY = dict(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=4, out_channels=2,
            time_dim=16)


@pytest.fixture()
def ckpt(tmp_path):
    oc = o.ModelConfig(**TINY)
    p = o.init_params(oc, 2024, random=True)
    base = str(tmp_path / "params")
    o.save_named_arrays(base, oc, p)
    return base, p


def test_fnv1a64_known_values():
    assert o.fnv1a64(b"") == 0xcbf29ce484222325
    assert o.fnv1a64(b"a") == 0xaf63dc4c8601ec8c  # published FNV-1a 64 test vector


def test_verify_ok(ckpt):
    swf.verify_checkpoint(swf.ModelConfig(**TINY), ckpt[0])


def test_corrupt_byte_is_io_error(ckpt):
    base, _ = ckpt
    with open(base + ".bin", "r+b") as f:
        f.seek(100)
        b = f.read(1)
        f.seek(100)
        f.write(bytes([b[0] ^ 0x40]))
    with pytest.raises(swf.IoError, match="checksum"):
        swf.verify_checkpoint(swf.ModelConfig(**TINY), base)


def test_layout_mismatch_is_io_error(ckpt):
    base, _ = ckpt
    with pytest.raises(swf.IoError, match="layout mismatch"):
        swf.verify_checkpoint(swf.ModelConfig(**dict(TINY, ffn_dim=48)), base)


def test_missing_and_truncated(ckpt, tmp_path):
    base, _ = ckpt
    with pytest.raises(swf.IoError):
        swf.verify_checkpoint(swf.ModelConfig(**TINY), str(tmp_path / "nope"))
    with open(base + ".bin", "r+b") as f:
        f.truncate(os.path.getsize(base + ".bin") // 2)
    with pytest.raises(swf.IoError, match="truncated"):
        swf.verify_checkpoint(swf.ModelConfig(**TINY), base)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_save_checkpoint_matches_reference_format(tmp_path, dtype):
    """save_checkpoint writes the bytes the reference's save_named_arrays writes (restated by the
    oracle), and param_arrays lists parameter_arrays' names and shapes."""
    oc, sc = o.ModelConfig(**TINY), swf.ModelConfig(**TINY)
    assert swf.param_arrays(sc) == [(n, r, c) for n, r, c in o.param_shapes(oc)]
    p = o.init_params(oc, 9, random=True, dtype=dtype)
    o.save_named_arrays(str(tmp_path / "ref"), oc, p)
    swf.save_checkpoint(str(tmp_path / "ours"), sc, o.split_params(oc, p))
    for ext in (".manifest", ".bin"):
        assert (tmp_path / ("ref" + ext)).read_bytes() == (tmp_path / ("ours" + ext)).read_bytes()
    swf.verify_checkpoint(sc, str(tmp_path / "ours"))
    assert swf.fnv1a64(b"") == 0xcbf29ce484222325


def test_save_checkpoint_rejects_wrong_shapes(tmp_path):
    sc = swf.ModelConfig(**TINY)
    arrays = [np.zeros(r * c, np.float32) for _, r, c in swf.param_arrays(sc)]
    arrays[3] = np.zeros(arrays[3].size + 1, np.float32)
    with pytest.raises(swf.ConfigError):
        swf.save_checkpoint(str(tmp_path / "bad"), sc, arrays)
    c = swf._Cfg(*swf.astuple(sc))
    buf, r, k = swf.C.create_string_buffer(64), swf.C.c_longlong(), swf.C.c_longlong()
    n = len(swf.param_arrays(sc))
    assert swf.lib().swf_param_array(swf.C.byref(c), n, buf, 64, swf.C.byref(r), swf.C.byref(k)) == swf.ERR_CONFIG
