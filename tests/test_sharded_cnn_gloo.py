"""Output-channel sharded CNN (config 4's layout, sharded_cnn.py) over gloo.

World sizes 1, 2 and 3 run the same small degree-3 CNN with the float test
engine; every rank must produce the float64 forward pass.  World 3 does not
divide the channel counts, so uneven shards and padded ring payloads are
covered.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_16834_b200.featuremajor import Activation, CnnSpec

SPEC = CnnSpec(channels=(3, 4, 5), H=4, W=4, act=Activation((0.5, 0.5, 0.0, 0.0625)), pool_after=(0, 1))
SAMPLES = 6


def _images():
    rng = np.random.default_rng(3)
    return rng.uniform(0.0, 1.0, size=(SAMPLES, 3, SPEC.H, SPEC.W))


def _run(rank, world):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from toy_engine import ToyEngine

    from paper_2604_16834_b200.sharded_cnn import TorchRing, run_cnn_sharded

    wts = SPEC.make_weights(7)
    eng = ToyEngine(SAMPLES)
    imgs = _images()
    x = eng.encrypt_batch(imgs.reshape(SAMPLES, -1).T)          # feature-major: ct f = pixel f of every sample
    out = run_cnn_sharded(eng, x, SPEC, wts, rank, world, ring=TorchRing(rank, world))
    got = np.stack(eng.decrypt_batch(out)).T                     # [samples, classes]
    eng.release(*out)
    return got, eng.live


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got, live = _run(rank, world)
        q.put((rank, got, live))
    finally:
        dist.destroy_process_group()


def test_sharded_cnn_world1_matches_float_forward():
    got, live = _run(0, 1)
    ref = SPEC.forward_plain(SPEC.make_weights(7), _images())
    assert np.max(np.abs(got - ref)) < 1e-9
    assert live == 0                          # every intermediate released


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cnn_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = SPEC.forward_plain(SPEC.make_weights(7), _images())
    for rank, got, live in res:
        assert np.max(np.abs(got - ref)) < 1e-9, rank
        assert live == 0, rank


def test_window_groups_equal_full_map_groups():
    """conv3x3_window_groups over a row window == featuremajor.conv3x3_groups on
    the full map, with column indices translated into the window."""
    from paper_2604_16834_b200.featuremajor import conv3x3_groups
    from paper_2604_16834_b200.sharded_cnn import conv3x3_window_groups

    p, H, W = 3, 8, 6
    for r0, r1 in [(0, 2), (2, 4), (6, 8), (3, 4), (0, 8)]:
        ya, yb = max(0, r0 - 1), min(H, r1 + 1)
        tp, col, tap, n = conv3x3_groups(p, H, W, range(r0, r1))
        wtp, wcol, wtap, wn = conv3x3_window_groups(p, H, W, r0, r1, ya, yb)
        assert n == wn and np.array_equal(tp, wtp) and np.array_equal(tap, wtap)
        i, rest = col // (H * W), col % (H * W)
        y, x = rest // W, rest % W
        assert np.array_equal(wcol, i * (yb - ya) * W + (y - ya) * W + x)
    with pytest.raises(ValueError):
        conv3x3_window_groups(p, H, W, 2, 4, 2, 5)   # row 1 missing


def test_streamed_rows_bound_resident_ciphertexts():
    """Row streaming: on a 24x4, three-block network the peak number of live
    ciphertexts stays well below one full activation map, and the result still
    equals the float64 forward pass for every tile size."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from toy_engine import ToyEngine

    from paper_2604_16834_b200.sharded_cnn import run_cnn_sharded

    spec = CnnSpec(channels=(2, 4, 4, 3), H=24, W=4, act=Activation((0.5, 0.5, 0.0, 0.0625)), pool_after=(1, 2))
    wts = spec.make_weights(9)
    imgs = np.random.default_rng(4).uniform(0.0, 1.0, size=(5, 2, 24, 4))
    ref = spec.forward_plain(wts, imgs)
    for tile in (1, 2, 4):
        eng = ToyEngine(5)
        peak = [0]
        ct0 = eng._ct

        def _ct(*a, **k):
            c = ct0(*a, **k)
            peak[0] = max(peak[0], eng.live)
            return c

        eng._ct = _ct
        x = eng.encrypt_batch(imgs.reshape(5, -1).T)
        out = run_cnn_sharded(eng, x, spec, wts, 0, 1, tile_rows=tile)
        got = np.stack(eng.decrypt_batch(out)).T
        eng.release(*out)
        assert np.max(np.abs(got - ref)) < 1e-9, tile
        assert eng.live == 0
        inputs, full_map = 2 * 24 * 4, 4 * 24 * 4   # block 1's whole output map: 384 ciphertexts
        assert peak[0] - inputs < full_map, (tile, peak[0])   # windows + one tile's temporaries only


def test_window_fulltaps_equal_full_map_fulltaps():
    """The tensor-core gather table of a row window == featuremajor.conv3x3_fulltaps
    on the full map with indices translated into the window; and the split-scale
    weights reproduce round(w * mult) within F / 2 with |W| < 2^23."""
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import conv3x3_fulltaps
    from paper_2604_16834_b200.sharded_cnn import conv3x3_window_fulltaps

    p, H, W = 3, 8, 6
    for r0, r1 in [(0, 2), (2, 4), (6, 8), (3, 4), (0, 8)]:
        ya, yb = max(0, r0 - 1), min(H, r1 + 1)
        full = conv3x3_fulltaps(p, H, W, range(r0, r1))
        win = conv3x3_window_fulltaps(p, H, W, r0, r1, ya, yb)
        i, rest = full // (H * W), full % (H * W)
        y, x = rest // W, rest % W
        want = np.where(full >= 0, i * (yb - ya) * W + (y - ya) * W + x, -1)
        assert np.array_equal(win, want)
    rng = np.random.default_rng(8)
    w = rng.normal(0, 0.3, (32, 144))
    for mult in (2.0 ** 50, 2.0 ** 30, 1000.0):
        wi, F = GpuEngine.split_scale_weights(w, mult)
        assert np.abs(wi).max() < 2 ** 23 and F & (F - 1) == 0
        assert np.max(np.abs(wi * float(F) - w * mult)) <= F / 2 + 1e-6 * F
        if mult < 2 ** 22:
            assert F == 1 and np.array_equal(wi, np.rint(w * mult).astype(np.int64))
