"""Index-map KATs: window partition / shift / seam mask / RoPE / SP bands / ownership.

Restates proj/tests/test_swin_core.cpp:76-144,265-276 and test_topology.cpp:128-235.
"""
import numpy as np
import pytest

from oracle import pyoracle as o


def test_window_arithmetic():
    # test_swin_core.cpp:76-89
    assert len(o.window_perm(24, 48, 6, 0)) == 24 * 48
    assert (720 // 60) * (1440 // 60) == 288


@pytest.mark.parametrize("shift", [0, 3])
def test_partition_merge_inverse_bitwise(shift):
    # test_swin_core.cpp:91-101
    x = o.random_field(5, 144, 42)
    g = o.window_gather(12, 12, 6, shift, x)
    assert np.array_equal(o.window_scatter(12, 12, 6, shift, g), x)


@pytest.mark.parametrize("shift", [0, 3])
def test_every_pixel_in_one_window(shift):
    # test_swin_core.cpp:103-113
    perm = o.window_perm(12, 18, 6, shift)
    assert np.array_equal(np.sort(perm), np.arange(12 * 18))


def test_pixel_of_formula_c2():
    H, W, w = 720, 1440, 60
    for s in (0, 30):
        perm = o.window_perm(H, W, w, s)
        idx = np.arange(H * W)
        win, tok = idx // (w * w), idx % (w * w)
        wy, wx, r, c = win // (W // w), win % (W // w), tok // w, tok % w
        exp = ((wy * w + s + r) % H) * W + (wx * w + s + c) % W
        assert np.array_equal(perm, exp)


def test_seam_mask_entries():
    # test_swin_core.cpp:265-276
    m = o.seam_mask(12, 12, 6, 3, 1)
    assert m is not None
    assert m[0 * 6 + 0, 2 * 6 + 5] == 0.0
    assert m[0 * 6 + 0, 3 * 6 + 0] == -np.inf
    assert m[4 * 6 + 1, 5 * 6 + 2] == 0.0
    assert o.seam_mask(12, 12, 6, 3, 0) is None
    assert o.seam_mask(12, 12, 6, 0, 1) is None


def test_rope_identity_and_isometry():
    # test_swin_core.cpp:115-130: zero position is the identity (angles all zero)
    assert np.all(o.rope_angles(8, 0, 0) == 0)
    a = o.rope_angles(128, 3, 5)
    om = 10000.0 ** (-np.arange(32) / 32)
    assert np.allclose(a[:32], 3 * om) and np.allclose(a[32:], 5 * om)


def test_sp_bands_shift_invariant():
    # test_topology.cpp:170-191
    for gy in range(24):
        r0 = gy % 6
        r3 = (gy - 3 + 24) % 24 % 6
        assert o.band_of_row(24, 48, 6, 0, r0, 3) == o.band_of_row(24, 48, 6, 3, r3, 3)


def test_window_owner_round_robin():
    # test_topology.cpp:128-150
    assert o.window_owner(3, 5, 2, 2) == (1, 1)


def test_shift_transfer_plan_balance():
    # test_topology.cpp:193-235: brute-force displaced count, equal per WP rank
    tot, per = o.shift_transfer_total(24, 48, 6, 0, 3, 2, 2, 2)
    expect = 0
    for y in range(24):
        for x in range(48):
            own0 = o.window_owner(y // 6, x // 6, 2, 2)
            sy, sx = (y - 3) % 24, (x - 3) % 48
            if own0 != o.window_owner(sy // 6, sx // 6, 2, 2):
                expect += 1
    # plan direction here is 0 -> 3 (owner under shift 0 = source)
    assert tot == expect
    assert len(set(per)) == 1
    assert o.shift_transfer_total(24, 48, 6, 0, 0, 2, 2, 1)[0] == 0


def test_noise_field_keying():
    # test_trigflow.cpp:352-370: field assembled per (window, token) key
    z = o.noise_field(99, 5, 3, 12, 24, 6)
    zfk = o.key_derive(99, 0x7A, 5)
    for wid in (7, 2, 0):
        wy, wx = wid // 4, wid % 4
        for tok in (0, 13, 35):
            key = o.key_derive(zfk, wid, tok)
            pix = o.pixel_of(12, 24, 6, 0, wy, wx, tok // 6, tok % 6)
            for c in range(3):
                assert z[pix, c] == o.gaussian(key, c)
    assert abs(z.mean()) < 0.1 and abs((z ** 2).mean() - 1) < 0.15
