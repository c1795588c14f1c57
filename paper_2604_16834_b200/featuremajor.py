"""Feature-major batched layers and the BASELINE networks (configs 1, 3, 4, 5).

Feature-major packing puts ONE feature (pixel of one channel) of n samples in
each ciphertext, so every linear layer is a plaintext-weighted linear
combination of whole ciphertexts and needs no rotation:

  conv3x3 (pad 1): out[o,y,x] = sum_{i,dy,dx valid} W[o,i,dy,dx] in[i,y+dy,x+dx]
  2x2 avg pool   : out[c,y,x] = 1/4 sum_{a,b} in[c,2y+a,2x+b]
  GAP            : out[c]     = 1/HW sum_p in[c,p]
  dense          : out[o]     = sum_c W[o,c] in[c] + b[o]

The reference expresses the k=1 case through conv_forward (conv.py:109-173,
PackingLayout(H=1, W=1, b=n, p=features)); it has no feature-major spatial
conv, but one is exactly reproduced with its own constant / mult_plain / add
primitives.  Here each layer is one he_lincomb launch.

Level plan (frozen; the CPU oracle follows the same one):
  * conv / dense: one rescale; weights encoded at q_last * s_out / s_in so the
    output scale is exactly the context scale.
  * degree-2 activation c2 x^2 + c1 x + c0 = (a x + b)^2 + c with
    a = sqrt(c2), b = c1 / (2 sqrt(c2)), c = c0 - c1^2 / (4 c2): (a, b) are
    folded into the preceding layer's weights / bias, leaving one ct x ct
    multiply (relinearise + rescale) and one constant add -> 1 level.
  * degree-3 activation c3 x^3 + c1 x + c0 with y = a x, a = cbrt(c3):
    y (y^2 + c1/a) + c0 -> 2 levels, 2 relinearisations.
  * average pools: unit-weight sums without rescale, the 1/k factor is moved
    into the ciphertext scale (k * s) and cancelled by the next layer's
    weight encoding -> 0 levels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import HebatchError, LevelExhausted, ShapeMismatch


# ---------------------------------------------------------------- term builders (CSR)
def conv3x3_csr(p: int, out_channels, H: int, W: int):
    """CSR of a pad-1 3x3 conv for the listed output channels.

    Inputs are indexed i*H*W + y*W + x; outputs (o in out_channels, y, x) in
    that order.  Returns (row_ptr, col, widx) with widx indexing
    weights.reshape(-1) of a (q, p, 3, 3) tensor.
    """
    oc = np.asarray(list(out_channels), dtype=np.int64)
    q = len(oc)
    y = np.arange(H)[:, None, None, None]
    x = np.arange(W)[None, :, None, None]
    dy = (np.arange(9) // 3 - 1)[None, None, None, :]
    dx = (np.arange(9) % 3 - 1)[None, None, None, :]
    i = np.arange(p)[None, None, :, None]
    yy, xx = y + dy, x + dx
    valid = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)                      # [H, W, 1, 9]
    valid = np.broadcast_to(valid, (H, W, p, 9))
    col = (i * H * W + yy * W + xx)                                          # [H, W, p, 9]
    col = np.broadcast_to(col, (H, W, p, 9))
    tap = np.broadcast_to(i * 9 + np.arange(9)[None, None, None, :], (H, W, p, 9))
    counts = valid.reshape(H * W, -1).sum(axis=1)                            # terms per pixel
    cols_px = col[valid]                                                     # pixel-major order
    taps_px = tap[valid]
    row_ptr = np.zeros(q * H * W + 1, np.int64)
    row_ptr[1:] = np.cumsum(np.tile(counts, q))
    cols = np.tile(cols_px, q)
    widx = (oc[:, None] * (p * 9) + taps_px[None, :]).reshape(-1)
    return row_ptr.astype(np.int32), cols.astype(np.int32), widx


def conv3x3_groups(p: int, H: int, W: int, rows=None):
    """Pixel groups of a pad-1 3x3 conv restricted to output ``rows``.

    Group g = pixel (y, x) in row-major order over the selected rows; its terms
    are the valid taps (i, dy, dx) with input col = i*H*W + (y+dy)*W + (x+dx)
    and tap index i*9 + (dy+1)*3 + (dx+1) into a (q, p, 3, 3) weight tensor.
    Returns (term_ptr, col, tap, n_pixels)."""
    rows = np.arange(H) if rows is None else np.asarray(list(rows))
    y = rows[:, None, None, None]
    x = np.arange(W)[None, :, None, None]
    k = np.arange(9)[None, None, None, :]
    dy, dx = k // 3 - 1, k % 3 - 1
    i = np.arange(p)[None, None, :, None]
    yy, xx = y + dy, x + dx
    shape = (len(rows), W, p, 9)
    valid = np.broadcast_to((yy >= 0) & (yy < H) & (xx >= 0) & (xx < W), shape)
    col = np.broadcast_to(i * H * W + yy * W + xx, shape)[valid]
    tap = np.broadcast_to(i * 9 + k, shape)[valid]
    counts = valid.reshape(len(rows) * W, -1).sum(axis=1)
    term_ptr = np.zeros(len(counts) + 1, np.int64)
    term_ptr[1:] = np.cumsum(counts)
    return term_ptr.astype(np.int32), col.astype(np.int32), tap.astype(np.int32), len(counts)


def pool2x2_csr(C: int, H: int, W: int):
    """CSR of a 2x2 / stride-2 sum pool: out (c, y, x) at H/2 x W/2."""
    if H % 2 or W % 2:
        raise ShapeMismatch(f"{H}x{W} not divisible by 2")
    Hp, Wp = H // 2, W // 2
    c = np.arange(C)[:, None, None, None]
    y = np.arange(Hp)[None, :, None, None]
    x = np.arange(Wp)[None, None, :, None]
    a = np.array([0, 0, 1, 1])[None, None, None, :]
    b = np.array([0, 1, 0, 1])[None, None, None, :]
    cols = (c * H * W + (2 * y + a) * W + (2 * x + b)).reshape(-1)
    row_ptr = np.arange(C * Hp * Wp + 1) * 4
    return row_ptr.astype(np.int32), cols.astype(np.int32)


def gap_csr(C: int, HW: int, channel_offset: int = 0):
    """CSR of per-channel sums over HW positions (inputs c*HW + p)."""
    row_ptr = np.arange(C + 1) * HW
    cols = (np.arange(C)[:, None] * HW + np.arange(HW)[None, :]).reshape(-1) + channel_offset
    return row_ptr.astype(np.int32), cols.astype(np.int32)


def dense_csr(n_out: int, n_in: int):
    row_ptr = np.arange(n_out + 1) * n_in
    cols = np.tile(np.arange(n_in), n_out)
    return row_ptr.astype(np.int32), cols.astype(np.int32)


# ---------------------------------------------------------------- activations
@dataclass(frozen=True)
class Activation:
    """Polynomial activation sum_k coeffs[k] x^k (degree 2, or 3 with no x^2 term)."""

    coeffs: tuple

    @property
    def degree(self) -> int:
        return len(self.coeffs) - 1

    @property
    def depth(self) -> int:
        return 1 if self.degree == 2 else 2

    def fold(self):
        """(a, b): the affine map folded into the preceding linear layer."""
        if self.degree == 2:
            c0, c1, c2 = self.coeffs
            if c2 <= 0:
                raise ValueError("degree-2 activation needs a positive x^2 coefficient")
            a = math.sqrt(c2)
            return a, c1 / (2 * a)
        c0, c1, c2, c3 = self.coeffs
        if c2 != 0 or c3 == 0:
            raise ValueError("degree-3 activation must have c2 = 0 and c3 != 0")
        return float(np.cbrt(c3)), 0.0

    def __call__(self, x):
        return sum(c * x ** k for k, c in enumerate(self.coeffs))


def apply_activation(engine, cts, act: Activation, lazy: bool = False):
    """Evaluate ``act`` on ciphertexts that already carry the folded affine map.

    lazy=True leaves the LAST ciphertext product unrelinearised and unrescaled
    (3 components at scale s^2): the caller sums such outputs (pool / GAP)
    and relinearises + rescales only the sums (engine.relin_rescale_batch).
    Relinearisation and rescale are linear up to their rounding, so this is
    the standard lazy-relinearisation / lazy-rescale rewrite; the CPU oracle
    replays exactly the same sequence."""
    if act.degree == 2:
        c0, c1, c2 = act.coeffs
        c = c0 - c1 * c1 / (4 * c2)
        sq = engine.tensor_batch(cts, cts) if lazy else engine.mult_ct_batch(cts, cts)
        if c == 0:
            return sq
        out = engine.add_const_batch(sq, [c] * len(sq))
        engine.release(*sq)
        return out
    c0, c1, c2, c3 = act.coeffs
    a = float(np.cbrt(c3))
    d = c1 / a
    sq = engine.mult_ct_batch(cts, cts)                  # y^2
    sqd = engine.add_const_batch(sq, [d] * len(sq)) if d else sq
    if sqd is not sq:
        engine.release(*sq)
    cub = engine.tensor_batch(cts, sqd) if lazy else engine.mult_ct_batch(cts, sqd)   # y (y^2 + d)
    engine.release(*sqd)
    if c0 == 0:
        return cub
    out = engine.add_const_batch(cub, [c0] * len(cub))
    engine.release(*cub)
    return out


# ---------------------------------------------------------------- layer calls
def fm_conv3x3(engine, inputs, weights, bias, H, W, out_channels=None, fold=(1.0, 0.0), out_scale=None,
               rows=None, weight_scale=None):
    """Feature-major 3x3 / pad-1 convolution (+ folded affine).

    inputs: p*H*W ciphertexts indexed i*H*W + y*W + x.  Returns the outputs
    for ``out_channels`` (default all; at most 32 per launch) and output
    ``rows`` (default all), indexed (o, y, x) over the selection.  Each
    launch is one he_lincomb_grouped: a pixel's taps are gathered once and
    multiplied into every selected channel."""
    w = np.asarray(weights, np.float64)
    q, p = w.shape[:2]
    if len(inputs) != p * H * W:
        raise ShapeMismatch(f"{len(inputs)} inputs for {p}x{H}x{W}")
    oc = list(range(q)) if out_channels is None else list(out_channels)
    a, b = fold
    tp, col, tap, npix = conv3x3_groups(p, H, W, rows)
    use_tc = weight_scale is not None and getattr(engine, "use_tensor_cores", False) and engine.N % 128 == 0
    gcol = conv3x3_fulltaps(p, H, W, rows) if use_tc else None
    out = []
    for c0 in range(0, len(oc), 32):
        ch = oc[c0:c0 + 32]
        wm = a * w[ch].reshape(len(ch), p * 9)
        bias_ch = a * np.asarray(bias, np.float64)[ch] + b             # one value per output channel
        res = None
        if use_tc:   # exact int8-digit tensor-core path (bit-identical results)
            res = engine.conv_mma(inputs, gcol, np.arange(npix), npix, wm, len(ch) * npix, weight_scale,
                                  bias=bias_ch)
        if res is None:
            res = engine.lincomb_grouped(inputs, tp, col, tap, np.arange(npix), npix, wm, len(ch) * npix,
                                         bias=bias_ch, out_scale=out_scale or engine.context.scale,
                                         weight_scale=weight_scale)
        out.extend(res)
    return out


def fm_conv_square_sum(engine, inputs, weights, bias, H, W, fold=(1.0, 0.0), rows=None, weight_scale=None,
                       const=0.0, pool=True, scale_mult=None, planar_out=None):
    """Deferred-rescale conv fused with the lazy square activation and the
    2x2-pool (pool=True) or GAP (pool=False) unit sum: one he_conv_square_sum
    launch per <= 32 output channels.  Returns the window sums indexed
    (o, r/2, x/2) / (o,), or None when the fused kernel does not apply.
    ``planar_out`` (engine.planar_carry): the pooled sums are written into the
    planar carry instead (returns [])."""
    w = np.asarray(weights, np.float64)
    q, p = w.shape[:2]
    a, b = fold
    out = []
    for c0 in range(0, q, 32):
        ch = list(range(c0, min(q, c0 + 32)))
        wm = a * w[ch].reshape(len(ch), p * 9)
        bias_ch = a * np.asarray(bias, np.float64)[ch] + b
        kw = {"planar_out": planar_out} if planar_out is not None else {}
        res = engine.conv_square_sum(inputs, p, H, W, wm, weight_scale, bias_ch, const, pool, rows=rows,
                                     scale_mult=scale_mult, **kw)
        if res is None:
            engine.release(*out)
            return None
        out.extend(res)
    return out


def conv3x3_fulltaps(p: int, H: int, W: int, rows=None) -> np.ndarray:
    """[pixels][9p] input index of every tap slot (-1 where the window leaves
    the image), tap order i*9 + (dy+1)*3 + (dx+1), pixels row-major over rows."""
    rows = np.arange(H) if rows is None else np.asarray(list(rows))
    y = rows[:, None, None, None]
    x = np.arange(W)[None, :, None, None]
    k = np.arange(9)[None, None, None, :]
    yy, xx = y + k // 3 - 1, x + k % 3 - 1
    i = np.arange(p)[None, None, :, None]
    valid = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
    col = np.where(valid, i * H * W + yy * W + xx, -1)
    return np.ascontiguousarray(col.reshape(len(rows) * W, p * 9).astype(np.int32))


def deferred_weight_scale(engine, cts, drops: int = 2) -> float:
    """Weight scale for a deferred-rescale conv feeding a degree-2 activation:
    (s_in * dw)^2 / (q_{l-1} ... q_{l-drops}) = Delta, so after the activation's
    relinearisation `drops` dropped primes bring the scale back to Delta."""
    limbs = cts[0].level + 1
    prod = 1.0
    for k in range(drops):
        prod *= engine.moduli[limbs - 1 - k]
    return math.sqrt(engine.context.scale * prod) / cts[0].scale


def _ncomp(engine, cts) -> int:
    f = getattr(engine, "_ncomp", None)
    return f(cts) if f is not None else 2


def carried_drops(engine, cts, min_scale: float = 2.0 ** 16) -> int:
    """Primes the 5-component relinearisation drops after a conv whose inputs are
    unrelinearised squares (scale ~ Delta^3): the fewest that give the conv an
    integer weight scale >= min_scale (2^18 for config 3: six 40-bit primes)."""
    limbs = cts[0].level + 1
    for d in range(2, limbs):
        if deferred_weight_scale(engine, cts, d) >= min_scale:
            return d
    raise LevelExhausted("no level budget for the carried activation")


def min_input_level(engine, spec: CnnSpec) -> int:
    """Lowest input level at which run_cnn's fused carry plan (two blocks, the
    first pooled, degree-2 activations, N = 2^16) completes with >= 2 limbs left
    for decryption: the plan consumes no level before the carried activation's
    5-component relinearisation (which drops carried_drops primes) and one for
    the dense head.  Limbs above that level would be carried through every layer
    and never used, so inputs are encrypted at it (he_encrypt_level) -- config 3:
    9 of the chain's 14 limbs (6 dropped at the relinearisation, 1 by the dense
    rescale, 2 decrypted).  Other plans: the top level."""
    top = engine.context.n_q - 1
    fused = (spec.act.degree == 2 and len(spec.pool_after) == 1 and 0 in spec.pool_after
             and len(getattr(spec, "channels", (0, 0, 0))) == 3 and getattr(engine, "N", 0) == 1 << 16
             and getattr(engine, "use_fused_conv", False) and getattr(engine, "joint_moddown", False))
    if not fused:
        return top

    class _S:  # scale/level stand-in for the plan arithmetic
        def __init__(self, level, scale):
            self.level, self.scale = level, scale

    for level in range(2, top + 1):
        x = _S(level, engine.context.scale)
        dw = deferred_weight_scale(engine, [x], 2)
        carried = _S(level, (x.scale * dw) ** 2 * 4.0)
        try:
            d = carried_drops(engine, [carried])
        except LevelExhausted:
            continue
        if level + 1 - d - 1 >= 2:
            return level
    return top


def fm_avgpool2x2(engine, inputs, C, H, W):
    """2x2 average pool as unit-weight sums (no level): scale x4."""
    rp, cols = pool2x2_csr(C, H, W)
    s = inputs[0].scale
    return engine.lincomb_int(inputs, rp, cols, np.ones(len(cols), np.int64), out_scale=4.0 * s)


def fm_gap(engine, inputs, C, HW):
    rp, cols = gap_csr(C, HW)
    s = inputs[0].scale
    return engine.lincomb_int(inputs, rp, cols, np.ones(len(cols), np.int64), out_scale=HW * s)


def fm_dense(engine, inputs, weights, bias, fold=(1.0, 0.0), out_scale=None):
    w = np.asarray(weights, np.float64)
    rp, cols = dense_csr(w.shape[0], w.shape[1])
    a, b = fold
    return engine.lincomb(inputs, rp, cols, a * w.reshape(-1), bias=a * np.asarray(bias, np.float64) + b,
                          out_scale=out_scale or engine.context.scale)


# ---------------------------------------------------------------- networks
@dataclass
class CnnWeights:
    convs: list            # [(W (q,p,3,3), b (q,))]
    dense: tuple           # (W (10, C), b (10,))


@dataclass(frozen=True)
class CnnSpec:
    """A feature-major CNN: conv blocks, pools after listed blocks, GAP, dense."""

    channels: tuple        # (3, 16, 32) -> convs 3->16, 16->32
    H: int
    W: int
    act: Activation
    pool_after: tuple      # block indices followed by a 2x2 avg pool
    n_classes: int = 10

    def make_weights(self, seed: int) -> CnnWeights:
        """N(0, 1/fan_in) weights, zero biases (BASELINE.json configs 3-4)."""
        rng = np.random.default_rng(seed)
        convs = []
        for p, q in zip(self.channels[:-1], self.channels[1:]):
            convs.append((rng.normal(0.0, math.sqrt(1.0 / (9 * p)), (q, p, 3, 3)), np.zeros(q)))
        C = self.channels[-1]
        dense = (rng.normal(0.0, math.sqrt(1.0 / C), (self.n_classes, C)), np.zeros(self.n_classes))
        return CnnWeights(convs, dense)

    def levels_needed(self) -> int:
        return len(self.channels[:-1]) * (1 + self.act.depth) + 1

    def forward_plain(self, wts: CnnWeights, images: np.ndarray) -> np.ndarray:
        """float64 reference forward pass. images [samples, C, H, W] -> [samples, classes]."""
        x = np.asarray(images, np.float64)
        H, W = self.H, self.W
        for blk, (w, b) in enumerate(wts.convs):
            xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
            out = np.zeros((x.shape[0], w.shape[0], H, W))
            for dy in range(3):
                for dx in range(3):
                    out += np.einsum("oi,sihw->sohw", w[:, :, dy, dx], xp[:, :, dy:dy + H, dx:dx + W])
            x = self.act(out + b[None, :, None, None])
            if blk in self.pool_after:
                x = x.reshape(x.shape[0], x.shape[1], H // 2, 2, W // 2, 2).mean(axis=(3, 5))
                H, W = H // 2, W // 2
        g = x.mean(axis=(2, 3))
        return g @ wts.dense[0].T + wts.dense[1]


def _free_planar(engine, pc, unpack=True):
    """Drop a planar carry; with ``unpack`` return its ciphertexts first."""
    cts = engine.unpack_planar(pc) if unpack else None
    pc.data = None
    return cts


def run_cnn(engine, x_cts, spec: CnnSpec, wts: CnnWeights, stream: bool = True, release_inputs: bool = True,
            tile_outputs: int = 1024, lazy_relin: bool = True, carry: bool = True,
            fused_tile_outputs: int = 1024, trace=None):
    """Encrypted forward pass of ``spec`` over feature-major input ciphertexts.

    x_cts: C0*H*W ciphertexts (channel-major).  Each block is streamed over
    tiles of output rows: one grouped conv launch per tile covers every output
    channel (<= 32 per launch), then the tile is activated and pooled (or
    GAP-summed) before the next tile starts, so the full pre-pool activation
    map is never resident (config 3's conv1 output alone would be 223 GB).
    ``tile_outputs`` bounds ciphertexts per launch (``fused_tile_outputs`` the
    pooled window sums per fused conv launch: config 3's conv1 runs as 4 launches
    of 1024; one launch of 4096 measured the same).  Releases its inputs
    unless ``release_inputs`` is False.  Returns the n_classes output
    ciphertexts.

    ``carry`` (fused degree-2 plan, N = 2^16): the pooled 3-component squares of
    the block before the last are NOT relinearised; the last block's fused conv
    takes them as they are (5-component squares, he_conv_square_sum_n), and only
    its global sums -- one per output channel -- are relinearised (keys s^2, s^3,
    s^4, engine.relin_rescale_batch) with `carried_drops` primes dropped.  For
    config 3 that replaces 4096 + 32 relinearisations by 32.

    ``trace`` (tests): called as trace(stage, cts, info) with every layer's
    outputs before they are released -- ("block", tile outputs, {"blk", "rows"})
    per row tile, ("planar", engine.PlanarCarry, {"blk"}) once a planar carry
    is complete, ("gap", ...) before the last relinearisation, ("relin", ...)
    after it and ("dense", ...) at the end.
    """
    H, W = spec.H, spec.W
    cur = list(x_cts)
    nblk = len(wts.convs)
    a, b = spec.act.fold()
    fused_ok = (lazy_relin and spec.act.degree == 2 and getattr(engine, "use_fused_conv", False)
                and getattr(engine, "N", 0) == 1 << 16 and getattr(engine, "joint_moddown", False))
    for blk, (w, bias) in enumerate(wts.convs):
        q = w.shape[0]
        pool = blk in spec.pool_after
        last = blk == nblk - 1
        # this block's pooled squares stay unrelinearised for the last block
        carry_out = (carry and fused_ok and pool and blk == nblk - 2 and (W // 2) % 2 == 0)
        # ... and, where both tcgen05 kernels take the shapes, in the planar layout
        # (5 bytes per residue, conv2's ring layout) instead of as ciphertexts
        planar = (carry_out and hasattr(engine, "planar_ok")
                  and engine.planar_ok(w.shape[1], H, W, q, wts.convs[blk + 1][0].shape[0], cur[0].level))
        planar_in = not isinstance(cur, list)
        ref = [cur] if planar_in else cur  # level / scale of the block's inputs
        drops = 2
        if planar_in or _ncomp(engine, cur) == 3:  # carried squares: one 5-component relin after the GAP
            drops = carried_drops(engine, ref)
            p_in = w.shape[1]
            wmax = np.abs(a * w).max() * deferred_weight_scale(engine, ref, drops)
            if not (last and p_in <= 16 and W % 2 == 0 and np.rint(wmax) < 2 ** 23
                    and min(engine.moduli[:ref[0].level + 1]) >= 2 ** 36):
                if planar_in:
                    cur = _free_planar(engine, cur)
                z = engine.relin_rescale_batch(cur, drops=2)  # outside the fused kernel's bounds
                engine.release(*cur)
                cur, drops = z, 2
                planar_in, ref = False, z
        R = max(2 if pool else 1, (tile_outputs // (q * W)) // 2 * 2 if pool else tile_outputs // (q * W))
        R = min(R, H) if stream else H
        Ho, Wo = (H // 2, W // 2) if pool else (H, W)
        nxt = [None] * (q * Ho * Wo) if not last else None
        pc = engine.planar_carry(q, Ho, Wo, cur[0].level) if planar else None
        gap = None
        lazy = lazy_relin and (pool or last)
        # deferred rescale: the conv output keeps its level (weights at ~2^20),
        # the activation's summed products drop two primes after relinearising
        defer = lazy and spec.act.degree == 2
        dw = deferred_weight_scale(engine, ref, drops) if defer else None
        # conv + square + pool/GAP in one kernel: no conv map in HBM, so the
        # tiles only bound the 3-component window sums (about tile_outputs)
        fused = defer and getattr(engine, "use_fused_conv", False) and (last or pool)
        if fused and stream:
            R = H if last else min(H, 2 * max(1, fused_tile_outputs // (q * (W // 2))))
        for r0 in range(0, H, R):
            rows = list(range(r0, min(H, r0 + R)))
            nr = len(rows)
            if lazy and spec.act.degree == 2:
                c0, c1, c2 = spec.act.coeffs
                cst = c0 - c1 * c1 / (4 * c2)
                part = (fm_conv_square_sum(engine, cur, w, bias, H, W, fold=(a, b), rows=rows, weight_scale=dw,
                                           const=cst, pool=not last, scale_mult=H * W if last else 4.0,
                                           planar_out=pc)
                        if fused else None)
                if part is None and (planar_in or pc is not None or _ncomp(engine, cur) == 3):
                    raise HebatchError("fused conv declined carried 3-component inputs")
                if pc is not None:
                    continue  # the pooled rows are in the planar carry
                if part is None:
                    # conv, then square (no relin) + constant + pool / GAP sum in one pass
                    y = fm_conv3x3(engine, cur, w, bias, H, W, fold=(a, b), rows=rows, weight_scale=dw)
                    if last:
                        rp, cols = gap_csr(q, nr * W)
                        part = engine.square_sum_batch(y, rp, cols, cst, H * W)
                    else:
                        rp, cols = pool2x2_csr(q, nr, W)
                        part = engine.square_sum_batch(y, rp, cols, cst, 4.0)
                    engine.release(*y)
                if trace is not None:
                    trace("block", part, {"blk": blk, "rows": rows, "fused": fused})
                if last:
                    if gap is None:
                        gap = part
                    else:
                        nsum = engine.add_batch(gap, part)
                        engine.release(*gap, *part)
                        gap = nsum
                    continue
                if carry_out:
                    z = part  # stays 3-component: the last block squares it unrelinearised
                else:
                    z = engine.relin_rescale_batch(part, drops=2 if defer else 1)
                    engine.release(*part)
                nr //= 2
                y0 = rows[0] // 2
                for o in range(q):
                    for r in range(nr):
                        for x in range(Wo):
                            nxt[o * Ho * Wo + (y0 + r) * Wo + x] = z[(o * nr + r) * Wo + x]
                continue
            y = fm_conv3x3(engine, cur, w, bias, H, W, fold=(a, b), rows=rows, weight_scale=dw)   # [o][r][x]
            z = apply_activation(engine, y, spec.act, lazy=lazy)
            engine.release(*y)
            if last:
                # GAP of the (pooled) map = mean over every pixel of the block
                hw = H * W
                rp, cols = gap_csr(q, nr * W)
                part = engine.lincomb_int(z, rp, cols, np.ones(len(cols), np.int64), out_scale=hw * z[0].scale)
                engine.release(*z)
                if gap is None:
                    gap = part
                else:
                    nsum = engine.add_batch(gap, part)
                    engine.release(*gap, *part)
                    gap = nsum
                continue
            if pool:
                zp = fm_avgpool2x2(engine, z, q, nr, W)                         # [o][r/2][x/2]
                engine.release(*z)
                z = zp
                nr //= 2
            if lazy:
                zr = engine.relin_rescale_batch(z, drops=2 if defer else 1)
                engine.release(*z)
                z = zr
            y0 = rows[0] // 2 if pool else rows[0]
            for o in range(q):
                for r in range(nr):
                    for x in range(Wo):
                        nxt[o * Ho * Wo + (y0 + r) * Wo + x] = z[(o * nr + r) * Wo + x]
        if planar_in:
            _free_planar(engine, cur, unpack=False)
        elif blk > 0 or release_inputs:
            engine.release(*cur)
        if pc is not None:
            if trace is not None:
                trace("planar", pc, {"blk": blk})
            nxt = pc
        if last and lazy_relin:
            if trace is not None:
                trace("gap", gap, {"blk": blk, "drops": drops if defer else 1})
            g2 = engine.relin_rescale_batch(gap, drops=drops if defer else 1)
            engine.release(*gap)
            gap = g2
            if trace is not None:
                trace("relin", gap, {"blk": blk})
        cur = gap if last else nxt
        H, W = Ho, Wo
    out = fm_dense(engine, cur, wts.dense[0], wts.dense[1])
    engine.release(*cur)
    if trace is not None:
        trace("dense", out, {})
    return out


# ---------------------------------------------------------------- config 1: MLP
@dataclass(frozen=True)
class MlpSpec:
    sizes: tuple = (64, 32, 10)
    act: Activation = Activation((0.0, 0.0, 1.0))

    def make_weights(self, seed: int):
        rng = np.random.default_rng(seed)
        return [(rng.normal(0.0, math.sqrt(1.0 / p), (q, p)), np.zeros(q))
                for p, q in zip(self.sizes[:-1], self.sizes[1:])]

    def forward_plain(self, wts, x):
        h = np.asarray(x, np.float64)
        for k, (w, b) in enumerate(wts):
            h = h @ w.T + b
            if k < len(wts) - 1:
                h = self.act(h)
        return h


def run_mlp(engine, x_cts, spec: MlpSpec, wts):
    cur = list(x_cts)
    a, bb = spec.act.fold()
    for k, (w, b) in enumerate(wts):
        last = k == len(wts) - 1
        y = fm_dense(engine, cur, w, b, fold=(1.0, 0.0) if last else (a, bb))
        engine.release(*cur)
        if not last:
            z = apply_activation(engine, y, spec.act)
            engine.release(*y)
            y = z
        cur = y
    return cur
