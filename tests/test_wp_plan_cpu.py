"""Window-parallel planning on the host (no GPU): ownership partitions and the owner-changed
token exchange at block boundaries, checked against the oracle's restatement of the reference's
window_owner / shift_transfer_plan (topology.hpp:107-188) -- bit-exact integer index maps."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o


@pytest.mark.parametrize("wp", [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4)])
@pytest.mark.parametrize("own", [swf.OWN_CONTIGUOUS, swf.OWN_ROUND_ROBIN])
def test_owners_partition_balanced(wp, own):
    H, W, w = 720, 1440, 60
    owners = swf.plan_owners(H, W, w, *wp, own)
    counts = np.bincount(owners, minlength=wp[0] * wp[1])
    assert (counts == counts[0]).all() and counts.sum() == 288


def test_round_robin_matches_reference_window_owner():
    H, W, w, a, b = 720, 1440, 60, 2, 4
    owners = swf.plan_owners(H, W, w, a, b, swf.OWN_ROUND_ROBIN)
    for wid in range(288):
        wy, wx = divmod(wid, 24)
        oa, ob = o.window_owner(wy, wx, a, b)
        assert owners[wid] == oa * b + ob


@pytest.mark.parametrize("wp", [(1, 2), (2, 2), (2, 4)])
def test_exchange_matches_reference_shift_transfer_plan(wp):
    # round-robin is the reference map: totals and per-source counts must equal the brute-force plan
    H, W, w = 24, 48, 6
    sent = swf.plan_exchange(H, W, w, *wp, swf.OWN_ROUND_ROBIN, 0, 3)
    tot, per_src = o.shift_transfer_total(H, W, w, 0, 3, *wp, 1)
    assert sent.sum() == tot
    assert list(sent.sum(axis=1)) == per_src
    assert np.all(np.diag(sent) == 0)


def test_contiguous_exchange_fractions_c2():
    # contiguous ownership moves 4.2% (1x2), 12.2% (2x2), 16.0% (2x4) of tokens;
    # the reference round-robin map moves 50% / 75% / 75%.
    N = 720 * 1440
    for wp, frac_c, frac_rr in (((1, 2), 0.042, 0.50), ((2, 2), 0.122, 0.75), ((2, 4), 0.160, 0.75)):
        c = swf.plan_exchange(720, 1440, 60, *wp, swf.OWN_CONTIGUOUS).sum() / N
        r = swf.plan_exchange(720, 1440, 60, *wp, swf.OWN_ROUND_ROBIN).sum() / N
        assert abs(c - frac_c) < 0.002, (wp, c)
        assert abs(r - frac_rr) < 0.002, (wp, r)


def test_exchange_is_symmetric_inverse():
    # the 0 -> w/2 boundary and the w/2 -> 0 boundary move the same token counts, transposed
    a = swf.plan_exchange(720, 1440, 60, 2, 2, swf.OWN_CONTIGUOUS, 0, 30)
    b = swf.plan_exchange(720, 1440, 60, 2, 2, swf.OWN_CONTIGUOUS, 30, 0)
    assert np.array_equal(a, b.T)


@pytest.mark.parametrize("wp,sp", [((1, 1), 2), ((1, 2), 2), ((1, 1), 4), ((1, 2), 4), ((2, 2), 2)])
def test_sp_token_partition_and_bands(wp, sp):
    # SP bands by global row phase (window.hpp:67-79): every pixel owned exactly once; a rank's
    # tokens all sit in its band under the reference band_of_row, for both shifts (shift-invariant)
    H, W, w = 48, 96, 12
    world = wp[0] * wp[1] * sp
    allp = []
    for r in range(world):
        pix = swf.plan_tokens(H, W, w, *wp, sp, r)
        allp.append(pix)
        band = r % sp
        ys = pix // W
        # row phase y mod w decides the band, independent of the layout shift
        for shift in (0, 6):
            rr = (ys - shift) % H % w
            assert all(o.band_of_row(H, W, w, shift, int(x), sp) == band for x in np.unique(rr))
    allp = np.concatenate(allp)
    assert np.array_equal(np.sort(allp), np.arange(H * W))


def test_sp1_order_is_canonical_window_order():
    H, W, w = 48, 96, 12
    pix = swf.plan_tokens(H, W, w, 1, 1, 1, 0)
    assert np.array_equal(pix, o.window_perm(H, W, w, 0))
