"""Chunked field container (f4 input format): the reference's test_grid_data.cpp:150-245 cases through
the C-ABI, plus byte compatibility with the numpy restatement in oracle/pyoracle.py (no GPU needed)."""
import itertools
import os

import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as orc


def _field(C, H, W, seed):
    return np.random.default_rng(seed).standard_normal((H * W, C)).astype(np.float32)


def test_full_grid_rect_equals_field_bitwise(tmp_path):  # test_grid_data.cpp:150-162
    f = _field(3, 16, 32, 11)
    p = str(tmp_path / "full.chk")
    swf.write_chunked(p, f, 16, 32, 8, 8)
    rd = swf.ChunkedReader(p)
    assert (rd.channels, rd.height, rd.width, rd.chunk_h, rd.chunk_w) == (3, 16, 32, 8, 8)
    assert np.array_equal(rd.read_full(), f)


def test_quadrant_reads_partition_exactly(tmp_path):  # :164-190
    f = _field(2, 16, 32, 13)
    p = str(tmp_path / "quad.chk")
    swf.write_chunked(p, f, 16, 32, 8, 8)
    rd = swf.ChunkedReader(p)
    re = np.zeros((16, 32, 2), np.float32)
    for qy, qx in itertools.product(range(2), range(2)):
        rd.reset_chunk_reads()
        part = rd.read_window_slice(qy * 8, qx * 16, 8, 16)
        assert rd.chunk_reads() == 2 == rd.chunk_cover(qy * 8, qx * 16, 8, 16)
        re[qy * 8:qy * 8 + 8, qx * 16:qx * 16 + 16] = part.reshape(8, 16, 2)
    assert np.array_equal(re.reshape(-1, 2), f)


def test_chunk_counter_equals_bruteforce_cover(tmp_path):  # :192-216 (non-dividing chunk dims)
    H, W = 24, 40
    f = np.arange(H * W, dtype=np.float32).reshape(-1, 1)
    p = str(tmp_path / "cover.chk")
    swf.write_chunked(p, f, H, W, 7, 9)
    rd = swf.ChunkedReader(p)
    rng = np.random.default_rng(17)
    for _ in range(50):
        y0, x0 = int(rng.integers(0, H)), int(rng.integers(0, W))
        h, w = int(rng.integers(1, H - y0 + 1)), int(rng.integers(1, W - x0 + 1))
        touched = {(y // 7, x // 9) for y in range(y0, y0 + h) for x in range(x0, x0 + w)}
        rd.reset_chunk_reads()
        part = rd.read_window_slice(y0, x0, h, w)
        assert rd.chunk_reads() == len(touched)
        assert part[0, 0] == float(y0 * W + x0)
        assert np.array_equal(part.reshape(h, w), f.reshape(H, W)[y0:y0 + h, x0:x0 + w])


def test_out_of_bounds_and_corruption_fail_loudly(tmp_path):  # :218-245
    f = np.ones((16 * 16, 1), np.float32)
    p = str(tmp_path / "corrupt.chk")
    swf.write_chunked(p, f, 16, 16, 8, 8)
    rd = swf.ChunkedReader(p)
    with pytest.raises(swf.ConfigError):  # std::out_of_range
        rd.read_window_slice(0, 0, 17, 4)
    with pytest.raises(swf.ConfigError):
        rd.read_window_slice(-1, 0, 4, 4)
    rd.close()
    with open(p, "r+b") as fh:  # flip one payload byte
        fh.seek(-3, os.SEEK_END)
        b = fh.read(1)
        fh.seek(-3, os.SEEK_END)
        fh.write(bytes([b[0] ^ 0x40]))
    with pytest.raises(swf.IoError):  # IntegrityError
        swf.ChunkedReader(p).read_full()
    with open(p, "r+b") as fh:
        fh.write(b"XXXXXXXX")
    with pytest.raises(swf.IoError):
        swf.ChunkedReader(p)


@pytest.mark.parametrize("C,H,W,ch,cw", [(3, 16, 32, 8, 8), (2, 24, 40, 7, 9), (70, 60, 120, 30, 60)])
def test_byte_compatible_with_oracle_restatement(tmp_path, C, H, W, ch, cw):
    f = _field(C, H, W, C * 7 + H)
    a, b = str(tmp_path / "cpp.chk"), str(tmp_path / "np.chk")
    swf.write_chunked(a, f, H, W, ch, cw)
    orc.write_chunked_np(b, f, H, W, ch, cw)
    assert open(a, "rb").read() == open(b, "rb").read()
    rd = swf.ChunkedReader(b)
    rng = np.random.default_rng(C)
    for _ in range(10):
        y0, x0 = int(rng.integers(0, H)), int(rng.integers(0, W))
        h, w = int(rng.integers(1, H - y0 + 1)), int(rng.integers(1, W - x0 + 1))
        ref, reads = orc.read_chunked_np(a, y0, x0, h, w)
        rd.reset_chunk_reads()
        assert np.array_equal(rd.read_window_slice(y0, x0, h, w), ref)
        assert rd.chunk_reads() == reads
