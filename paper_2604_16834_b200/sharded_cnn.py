"""Row-streamed, output-channel-sharded CNN (config 4).

Config 4 (four conv3x3 blocks 16 -> 32 -> 64 -> 64 on 32x32 maps, degree-3
activations, 24 x 50-bit limbs) does not fit one GPU as whole activation maps:
block 1's output alone is 16 x 1024 ciphertexts at 12 limbs = 197 GB.  So the
network runs as a PULL PIPELINE OVER IMAGE ROWS: every block is a stage that
produces its output rows on demand, in tiles of a few conv rows, from the
rows of the stage before it, and frees an input row as soon as no later tile
reads it (a 3x3 conv of rows [r0, r1) reads input rows [r0-1, r1+1)).  Only a
window of about four rows per block is ever resident, plus the encrypted
inputs; the last block's rows go straight into the GAP sums.

Across ranks the OUTPUT CHANNELS are sharded (reference counterpart: the
per-output-channel loop of /root/reference/pkg/src/hebatch/conv.py:149-156):
rank r owns ``channel_shards(q, G)[r]`` of every block's outputs, for every
pixel.  A conv tile needs every input channel of its input rows, which the
previous block left spread over the ranks, so each tile runs a RING over the
input-channel shards of those rows:

    round k (k = 0 .. G-1): the row window of rank (r - k) mod G is resident;
        post its send to rank r+1 and the receive of the next one from r-1
        (NCCL over NVLink on the GPU box, gloo in the CPU tests), convolve it
        into rank r's OWN output accumulators as exact un-rescaled partial
        sums (lincomb_grouped(skip_rescale=True)), wait for the exchange.

After the ring every owned output channel of the tile holds its full sum; one
rescale, the bias, the activation and the (per-channel, hence local) pool
follow.  Partial sums mod q added in any order equal the full sum, so world
size 1 is bit-identical to featuremajor.run_cnn(lazy_relin=False) and world G
reproduces it as well.  GAP sums are per channel (local); the q_last GAP
ciphertexts are all-gathered for the dense head.

Per-rank peak HBM at config 4 (levels 14 -> 11 -> 8 -> 5 -> 2 of 50-bit
limbs, N = 2^16, ciphertext = 2 x limbs x 512 KB): the replicated inputs
(3072 x 15 MB = 46 GB) + per block a window of <= 4 output rows of its own
channel shard (block 1: 16/G x 32 x 12 MB = 6.3/G GB per row; block 2: 32/G x
16 x 9 MB; block 3: 64/G x 16 x 6 MB; block 4: 64/G x 16 x 3 MB) + one tile's
temporaries (the tile's conv outputs and the activation's three products) +
two ring buffers of one window.  About 90 GB at G = 1.

The engine is any object with the methods used below (GpuEngine, or the
float test engine of tests/toy_engine.py).
"""

from __future__ import annotations

import numpy as np

from .featuremajor import apply_activation, dense_csr, fm_dense, gap_csr, pool2x2_csr  # noqa: F401
from .sharding import channel_shards


class TorchRing:
    """Ring neighbour exchange over torch.distributed (send to r+1, receive from r-1)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def start(self, t):
        """Post the send of ``t`` and the receive of an equally shaped tensor; returns a handle."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return t
        buf = torch.empty_like(t)
        ops = [dist.P2POp(dist.isend, t.contiguous(), (self.rank + 1) % self.world),
               dist.P2POp(dist.irecv, buf, (self.rank - 1) % self.world)]
        reqs = dist.batch_isend_irecv(ops)
        return reqs, buf

    def finish(self, h):
        if self.world == 1:
            return h
        reqs, buf = h
        for r in reqs:
            r.wait()
        return buf

    def all_gather(self, t):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return [t]
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t.contiguous())
        return parts


def conv3x3_window_groups(p: int, H: int, W: int, r0: int, r1: int, ya: int, yb: int):
    """Term lists of a pad-1 3x3 conv over output rows [r0, r1) whose inputs are
    a row WINDOW [ya, yb) of a p-channel H x W map, held as p*(yb-ya)*W
    ciphertexts indexed i*(yb-ya)*W + (y-ya)*W + x.  Padding is applied at the
    true image border only.  Returns (term_ptr, col, tap, n_pixels) like
    featuremajor.conv3x3_groups; tap = i*9 + (dy+1)*3 + (dx+1)."""
    if not (0 <= ya <= max(0, r0 - 1) and min(H, r1 + 1) <= yb <= H):
        raise ValueError(f"window [{ya}, {yb}) does not cover the taps of rows [{r0}, {r1})")
    nw = yb - ya
    y = np.arange(r0, r1)[:, None, None, None]
    x = np.arange(W)[None, :, None, None]
    k = np.arange(9)[None, None, None, :]
    dy, dx = k // 3 - 1, k % 3 - 1
    i = np.arange(p)[None, None, :, None]
    yy, xx = y + dy, x + dx
    shape = (r1 - r0, W, p, 9)
    valid = np.broadcast_to((yy >= 0) & (yy < H) & (xx >= 0) & (xx < W), shape)
    col = np.broadcast_to(i * nw * W + (yy - ya) * W + xx, shape)[valid]
    tap = np.broadcast_to(i * 9 + k, shape)[valid]
    counts = valid.reshape((r1 - r0) * W, -1).sum(axis=1)
    term_ptr = np.zeros(len(counts) + 1, np.int64)
    term_ptr[1:] = np.cumsum(counts)
    return term_ptr.astype(np.int32), col.astype(np.int32), tap.astype(np.int32), len(counts)


def conv3x3_window_fulltaps(p: int, H: int, W: int, r0: int, r1: int, ya: int, yb: int) -> np.ndarray:
    """[pixels][9p] window index of every tap slot of output rows [r0, r1) (-1 outside
    the image), tap order i*9 + (dy+1)*3 + (dx+1): the gather table of he_conv_mma."""
    nw = yb - ya
    y = np.arange(r0, r1)[:, None, None, None]
    x = np.arange(W)[None, :, None, None]
    k = np.arange(9)[None, None, None, :]
    yy, xx = y + k // 3 - 1, x + k % 3 - 1
    i = np.arange(p)[None, None, :, None]
    valid = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
    col = np.where(valid, i * nw * W + (yy - ya) * W + xx, -1)
    return np.ascontiguousarray(col.reshape((r1 - r0) * W, p * 9).astype(np.int32))


def conv3x3_partial(engine, window, weights, H, W, r0, r1, ya, yb, out_scale, tensor_cores: bool = True):
    """Exact (un-rescaled) contribution of one input-channel block (its rows
    [ya, yb) in ``window``) to output rows [r0, r1) of every output channel of
    ``weights`` [q_local][p_block*9], outputs indexed (o, y, x), declared scale
    q_l * out_scale.  With ``tensor_cores`` (GpuEngine.conv_exact_partial) the
    sums run as exact int8-digit GEMMs with split-scale integer weights W * 2^k;
    otherwise (or when the tensor-core bounds fail) he_lincomb_grouped with the
    weights round(w q_l out_scale / s_in)."""
    w = np.asarray(weights, np.float64)
    q = w.shape[0]
    p = w.shape[1] // 9
    tc = getattr(engine, "conv_exact_partial", None) if tensor_cores else None
    gcol = conv3x3_window_fulltaps(p, H, W, r0, r1, ya, yb) if tc is not None else None
    tp = col = tap = None
    npix = (r1 - r0) * W
    out = []
    for c0 in range(0, q, 32):  # <= 32 outputs per pixel group and launch
        m = min(32, q - c0)
        part = tc(window, gcol, w[c0:c0 + m], m * npix, out_scale) if tc is not None else None
        if part is None:
            if tp is None:
                tp, col, tap, npix = conv3x3_window_groups(p, H, W, r0, r1, ya, yb)
            part = engine.lincomb_grouped(window, tp, col, tap, np.arange(npix), npix, w[c0:c0 + m], m * npix,
                                          out_scale=out_scale, skip_rescale=True)
        out.extend(part)
    return out


def _accumulate(engine, acc, part):
    """acc += part (mod q); ``part`` is released.  In place on the GPU engine."""
    if acc is None:
        return part
    f = getattr(engine, "add_inplace", None)
    if f is not None:
        f(acc, part)
        engine.release(*part)
        return acc
    s = engine.add_batch(acc, part)
    engine.release(*acc, *part)
    return s


class _InputRows:
    """The replicated layer-0 input (every channel on every rank)."""

    replicated = True

    def __init__(self, cts, p, H, W, engine=None):
        """``engine``: release input rows as soon as no later tile reads them
        (run_cnn_sharded(release_inputs=True)); None keeps them for the caller."""
        self.cts, self.p, self.H, self.W, self.engine = list(cts), p, H, W, engine
        self.released = 0

    def ensure(self, upto):
        pass

    def window(self, ya, yb):
        """All channels' rows [ya, yb) in window order i*(yb-ya)*W + (y-ya)*W + x."""
        H, W = self.H, self.W
        return [self.cts[i * H * W + y * W + x] for i in range(self.p) for y in range(ya, yb) for x in range(W)]

    def release_below(self, y):
        if self.engine is None:
            return
        H, W = self.H, self.W
        for r in range(self.released, min(y, H)):
            self.engine.release(*[self.cts[i * H * W + r * W + x] for i in range(self.p) for x in range(W)])
        self.released = max(self.released, min(y, H))

    def release_all(self, engine):
        if self.engine is not None:
            self.release_below(self.H)
        self.cts = []


class _BlockStage:
    """One conv3x3 -> (folded affine) -> activation -> [2x2 pool] block, producing
    its output rows on demand.  ``rows[y]`` holds this rank's channels of output
    row y, indexed o_local*Wo + x."""

    replicated = False

    def __init__(self, engine, up, w, bias, act, fold, pool, H, W, rank, world, ring, tile_rows, trace, blk,
                 max_outputs=512, tensor_cores=True):
        self.engine, self.up = engine, up
        self.q, self.p = w.shape[:2]
        self.mine = list(channel_shards(self.q, world)[rank])
        self.in_shards = None if up.replicated else channel_shards(self.p, world)
        a, b = fold
        self.wm = a * np.asarray(w, np.float64)[self.mine].reshape(len(self.mine), self.p * 9)
        self.bias = a * np.asarray(bias, np.float64)[self.mine] + b
        self.act, self.pool = act, pool
        self.H, self.W = H, W
        self.Ho, self.Wo = (H // 2, W // 2) if pool else (H, W)
        self.rank, self.world, self.ring = rank, world, ring
        R = max(1, int(tile_rows))
        self.R = R + (R % 2) if pool else R
        self.trace, self.blk = trace, blk
        self.max_outputs = max_outputs
        self.tensor_cores = tensor_cores
        self.rows = {}
        self.done = 0          # conv rows produced so far
        self.released = 0      # output rows below this index are freed

    @property
    def produced(self):
        return self.done // 2 if self.pool else self.done

    def ensure(self, upto):
        """Produce output rows < upto."""
        while self.produced < min(upto, self.Ho):
            self._tile(self.done, min(self.H, self.done + self.R))

    def window(self, ya, yb):
        """This rank's channels of output rows [ya, yb), window order o*(yb-ya)*Wo + (y-ya)*Wo + x."""
        return [self.rows[y][o * self.Wo + x] for o in range(len(self.mine)) for y in range(ya, yb)
                for x in range(self.Wo)]

    def release_below(self, y):
        for r in range(self.released, min(y, self.produced)):
            self.engine.release(*self.rows.pop(r))
            self.released = r + 1

    def release_all(self, engine):
        for r in list(self.rows):
            engine.release(*self.rows.pop(r))

    def _tile(self, r0, r1):
        eng, H, W = self.engine, self.H, self.W
        ya, yb = max(0, r0 - 1), min(H, r1 + 1)
        self.up.ensure(yb)
        s_out = eng.context.scale
        acc = None
        local = self.up.window(ya, yb)         # this rank's input channels of rows [ya, yb)
        if self.up.replicated or self.world == 1:   # every input channel is resident: one local round
            acc = conv3x3_partial(eng, local, self.wm, H, W, r0, r1, ya, yb, s_out, self.tensor_cores)
        else:
            t, level, scale = eng.pack_batch(local)
            pad = max(len(sh) for sh in self.in_shards) * (yb - ya) * W
            if t.shape[0] < pad:                      # equal-size ring payloads (uneven shards)
                import torch

                t = torch.cat([t, torch.zeros((pad - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                                              device=t.device)])
            for k in range(self.world):
                src = (self.rank - k) % self.world
                h = self.ring.start(t) if k + 1 < self.world else None
                chans = list(self.in_shards[src])
                n = len(chans) * (yb - ya) * W
                blk_cts = eng.unpack_batch(t[:n], level, scale)
                cols = (np.asarray(chans)[:, None] * 9 + np.arange(9)[None, :]).reshape(-1)
                part = conv3x3_partial(eng, blk_cts, self.wm[:, cols], H, W, r0, r1, ya, yb, s_out, self.tensor_cores)
                eng.release(*blk_cts)
                acc = _accumulate(eng, acc, part)
                if h is not None:
                    t = self.ring.finish(h)
            del t
        if self.trace is not None:
            self.trace("acc", acc, {"blk": self.blk, "rows": (r0, r1), "window": (ya, yb), "inputs": local,
                                    "weights": self.wm})
        del local
        self.up.release_below(r1 - 1)          # rows below r1 - 1 are not read by later tiles
        nr, nq = r1 - r0, len(self.mine)
        Wo, nro, y0 = (W // 2, nr // 2, r0 // 2) if self.pool else (W, nr, r0)
        outs = [None] * (nq * nro * Wo)
        # rescale, bias, activation and pool in chunks of output channels: the
        # activation holds three or four batches of its inputs' size at once, which
        # bounds one tile's temporaries to ~max_outputs ciphertexts per batch
        cc = max(1, self.max_outputs // (nr * W))
        for c0 in range(0, nq, cc):
            c1 = min(nq, c0 + cc)
            a_ch = acc[c0 * nr * W:c1 * nr * W]
            z = eng.rescale_batch(a_ch, out_scale=s_out)
            eng.release(*a_ch)
            if np.any(self.bias[c0:c1] != 0):
                zb = eng.add_const_batch(z, np.repeat(self.bias[c0:c1], nr * W))
                eng.release(*z)
                z = zb
            y = apply_activation(eng, z, self.act, lazy=False)
            if self.trace is not None:
                self.trace("act", y, {"blk": self.blk, "rows": (r0, r1), "pre": z, "channels": (c0, c1)})
            eng.release(*z)
            if self.pool:
                rp, cols = pool2x2_csr(c1 - c0, nr, W)
                yp = eng.lincomb_int(y, rp, cols, np.ones(len(cols), np.int64), out_scale=4.0 * y[0].scale)
                eng.release(*y)
                y = yp
            outs[c0 * nro * Wo:c1 * nro * Wo] = y
        for r in range(nro):
            self.rows[y0 + r] = [outs[(o * nro + r) * Wo + x] for o in range(nq) for x in range(Wo)]
        self.done = r1


def run_cnn_sharded(engine, x_cts, spec, wts, rank: int, world: int, ring=None, release_inputs: bool = True,
                    tile_rows: int = 2, trace=None, max_outputs: int = 512, tensor_cores: bool = True):
    """Encrypted forward pass of ``spec`` with output channels sharded over
    ``world`` ranks, streamed over image rows (module docstring).

    x_cts: the C0*H*W input ciphertexts (channel-major), replicated on every rank.
    ``tile_rows``: conv rows per tile (even for pooled blocks); ``max_outputs``:
    ciphertexts per batch of a tile's rescale / activation / pool.  ``tensor_cores``:
    the conv sums as exact int8-digit GEMMs (split-scale weights, conv3x3_partial);
    False keeps featuremajor.run_cnn's CUDA-core weight encoding (bit-identical
    to run_cnn(lazy_relin=False)).  ``trace``
    (tests): trace(stage, cts, info) with stage "acc" (a tile's exact conv sums
    before the rescale), "act" (the activation outputs, info["pre"] its inputs),
    "gap" and "dense".  Returns the n_classes output ciphertexts on every rank."""
    ring = ring or TorchRing(rank, world)
    H, W = spec.H, spec.W
    fold = spec.act.fold()
    nblk = len(wts.convs)
    src = _InputRows(x_cts, wts.convs[0][0].shape[1], H, W, engine if release_inputs else None)
    stages = []
    for blk, (w, bias) in enumerate(wts.convs):
        # (as run_cnn: a pool right before the GAP is skipped -- GAP of the pooled
        # sums is the same sum over every pixel)
        pool = blk in spec.pool_after and blk != nblk - 1
        st = _BlockStage(engine, src, w, bias, spec.act, fold, pool, H, W, rank, world, ring, tile_rows, trace, blk,
                         max_outputs, tensor_cores)
        stages.append(st)
        src = st
        if pool:
            H, W = H // 2, W // 2
    last = stages[-1]
    # GAP over the last block's rows as they are produced: per-channel row sums, accumulated
    nq = len(last.mine)
    hw = last.Ho * last.Wo
    gap = None
    for y in range(last.Ho):
        last.ensure(y + 1)
        row = last.rows[y]
        rp, cols = gap_csr(nq, last.Wo)
        part = engine.lincomb_int(row, rp, cols, np.ones(len(cols), np.int64), out_scale=hw * row[0].scale)
        gap = _accumulate(engine, gap, part)
        last.release_below(y + 1)
    for st in stages:
        st.release_all(engine)
    stages[0].up.release_all(engine)
    q = wts.convs[-1][0].shape[0]
    if world > 1:
        shards = channel_shards(q, world)
        pad = max(len(sh) for sh in shards)
        t, level, scale = engine.pack_batch(gap)
        if t.shape[0] < pad:
            import torch

            t = torch.cat([t, torch.zeros((pad - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)])
        parts = ring.all_gather(t)
        engine.release(*gap)
        gap = []
        for r, sh in enumerate(shards):
            gap.extend(engine.unpack_batch(parts[r][: len(sh)], level, scale))
    if trace is not None:
        trace("gap", gap, {})
    out = fm_dense(engine, gap, wts.dense[0], wts.dense[1])
    engine.release(*gap)
    if trace is not None:
        trace("dense", out, {})
    return out


def plan_input_level(spec) -> int:
    """Input level at which the streamed non-lazy plan ends with 2 limbs for
    decryption: 1 (conv rescale) + 1 or 2 (activation products) per block, 1 for
    the dense head, 1 left over (config 4: 4 x 3 + 1 + 1 = 14, i.e. 15 of 24 limbs)."""
    per_block = 1 + (1 if spec.act.degree == 2 else 2)
    return per_block * (len(spec.channels) - 1) + 1 + 1
