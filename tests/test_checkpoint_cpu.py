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
