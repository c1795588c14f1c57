"""Output-channel-sharded CNN across ranks (config 4).

Rank r of G owns the output channels ``channel_shards(q, G)[r]`` of every conv
layer, for every pixel.  A 3x3 conv needs every input channel, but the
previous layer left them spread over the ranks, and config 4's activation
maps do not fit one GPU (16384 ciphertexts at >= 11 limbs after block 1).
So each layer runs a RING over the input-channel shards:

    round k (k = 0 .. G-1): the shard of rank (r - k) mod G is resident;
        start sending it to rank r+1 and receiving the next one from r-1,
        convolve it into rank r's OWN output accumulators (exact partial
        sums, no rescale), wait for the exchange.

After the ring every output channel of the rank holds the full sum; one
rescale, the bias, the activation and the (per-channel, hence local) pooling
follow.  No rank ever holds more than its own shards plus two ring buffers.
GAP is per channel (local); the 64 GAP ciphertexts are all-gathered for the
dense head.  With G = 1 the ring is a single local round and the result is
bit-identical to featuremajor.run_cnn(lazy_relin=False): partial sums mod q
added in any order equal the full sum, then the same rescale and bias.

The exchange moves ``engine.pack_batch`` tensors (int64 [k, 2, limbs, N]);
``TorchRing`` carries them with torch.distributed point-to-point ops (NCCL
over NVLink on the GPU box, gloo in the CPU tests).  The engine is any object
with the methods used below (GpuEngine, or the float test engine).
"""

from __future__ import annotations

import numpy as np

from .featuremajor import apply_activation, conv3x3_groups, fm_avgpool2x2, fm_dense, gap_csr
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


def conv3x3_partial(engine, inputs, weights, H, W, out_scale):
    """Exact (un-rescaled) contribution of one input-channel block to every
    output channel of ``weights`` [q_local][p_block][3][3]: lincomb_grouped
    with skip_rescale, outputs indexed (o, y, x), declared scale q_l * out_scale."""
    w = np.asarray(weights, np.float64)
    q, p = w.shape[:2]
    tp, col, tap, npix = conv3x3_groups(p, H, W)
    out = []
    for c0 in range(0, q, 32):  # he_lincomb_grouped takes <= 32 outputs per pixel group
        m = min(32, q - c0)
        out.extend(engine.lincomb_grouped(inputs, tp, col, tap, np.arange(npix), npix,
                                          w[c0:c0 + m].reshape(m, p * 9), m * npix, out_scale=out_scale,
                                          skip_rescale=True))
    return out


def _ring_shapes(n_items_per_rank):
    """Every rank's shard padded to the largest (the ring moves equal tensors)."""
    return max(n_items_per_rank)


def run_cnn_sharded(engine, x_cts, spec, wts, rank: int, world: int, ring=None, release_inputs: bool = True):
    """Encrypted forward pass of ``spec`` with output channels sharded over ``world`` ranks.

    x_cts: the C0*H*W input ciphertexts (channel-major), replicated on every rank.
    Returns the n_classes output ciphertexts on every rank."""
    ring = ring or TorchRing(rank, world)
    H, W = spec.H, spec.W
    a, b = spec.act.fold()
    s_out = engine.context.scale
    cur = list(x_cts)          # layer input held by this rank
    cur_chans = None           # None: all input channels (replicated layer-0 input)
    for blk, (w, bias) in enumerate(wts.convs):
        q, p = w.shape[:2]
        mine = list(channel_shards(q, world)[rank])
        wm = a * np.asarray(w, np.float64)[mine]                 # folded activation affine
        acc = None
        if cur_chans is None:   # replicated input: one local round over all channels
            acc = conv3x3_partial(engine, cur, wm, H, W, s_out)
        else:
            shards = channel_shards(p, world)
            hw = H * W
            pad = _ring_shapes([len(sh) * hw for sh in shards])
            level, scale = cur[0].level, cur[0].scale
            t, _, _ = engine.pack_batch(cur)
            if t.shape[0] < pad:                                # equal-size ring payloads
                import torch

                t = torch.cat([t, torch.zeros((pad - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                                              device=t.device)])
            for k in range(world):
                src = (rank - k) % world
                h = ring.start(t) if k + 1 < world else None
                chans = list(shards[src])
                blk_cts = engine.unpack_batch(t[: len(chans) * hw], level, scale)
                part = conv3x3_partial(engine, blk_cts, wm[:, chans], H, W, s_out)
                engine.release(*blk_cts)
                if acc is None:
                    acc = part
                else:
                    nsum = engine.add_batch(acc, part)
                    engine.release(*acc, *part)
                    acc = nsum
                if h is not None:
                    t = ring.finish(h)
        if release_inputs or blk > 0:
            engine.release(*cur)
        z = engine.rescale_batch(acc, out_scale=s_out)
        engine.release(*acc)
        bias_ch = a * np.asarray(bias, np.float64)[mine] + b
        if np.any(bias_ch != 0):
            zb = engine.add_const_batch(z, np.repeat(bias_ch, H * W))
            engine.release(*z)
            z = zb
        y = apply_activation(engine, z, spec.act, lazy=False)
        engine.release(*z)
        # (as run_cnn: a pool right before the GAP is skipped -- GAP of the
        # pooled sums is the same sum over every pixel)
        if blk in spec.pool_after and blk != len(wts.convs) - 1:
            yp = fm_avgpool2x2(engine, y, len(mine), H, W)
            engine.release(*y)
            y = yp
            H, W = H // 2, W // 2
        cur, cur_chans = y, mine
    # GAP over this rank's channels, gather all channels, dense head
    q = wts.convs[-1][0].shape[0]
    mine = cur_chans
    rp, cols = gap_csr(len(mine), H * W)
    gap = engine.lincomb_int(cur, rp, cols, np.ones(len(cols), np.int64), out_scale=H * W * cur[0].scale)
    engine.release(*cur)
    if world > 1:
        shards = channel_shards(q, world)
        pad = max(len(sh) for sh in shards)
        level, scale = gap[0].level, gap[0].scale
        t, _, _ = engine.pack_batch(gap)
        if t.shape[0] < pad:
            import torch

            t = torch.cat([t, torch.zeros((pad - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)])
        parts = ring.all_gather(t)
        engine.release(*gap)
        gap = []
        for r, sh in enumerate(shards):
            gap.extend(engine.unpack_batch(parts[r][: len(sh)], level, scale))
    out = fm_dense(engine, gap, wts.dense[0], wts.dense[1])
    engine.release(*gap)
    return out
