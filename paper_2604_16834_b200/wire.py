"""Ciphertext / evaluation-key wire format: the client/server boundary of the
paper's threat model (/root/reference/PAPER.md:210-214 -- the client encrypts
locally, sends ciphertexts, the server evaluates with its plaintext model and
the client's EVALUATION keys, and returns an encrypted prediction; the secret
key never leaves the client).  SURVEY.md 8f rank 4.

Format (little-endian), one blob per message:

    header  : magic b"HEBW", u16 version (1), u16 kind (1 = ciphertexts, 2 = keys),
              u32 N, u16 L, u16 K, u16 dnum, u16 reserved, u64 moduli[L + K]
              (the receiver rejects a blob whose parameters differ from its context:
              ContextMismatch)
    kind 1  : u32 count, u16 n_comp, u16 limbs, u32 level, u32 reserved,
              f64 scale[count], then the residues [count][n_comp][limbs][N] in the
              NTT domain (bit-reversed order), limb i packed
              to w_i = ceil(bits(q_i) / 8) bytes per residue (5 bytes for a 40-bit
              prime instead of 8)
    kind 2  : u32 n_keys, then per key: u32 code (0 = relinearisation s^2, 2 / 4 =
              s^3 / s^4, odd = Galois element 5^k mod 2N), the key
              [dnum][2][L + K][N] in canonical form, modulus m packed to w_m bytes

Packing and unpacking run on the device (byte slices of the uint64 residues);
only the packed bytes cross PCIe.  Imported residues are checked to be < q_i.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from .errors import ContextMismatch, HebatchError

MAGIC = b"HEBW"
VERSION = 1
KIND_CTS, KIND_KEYS = 1, 2
_HDR = struct.Struct("<4sHHIHHHH")
_CTS = struct.Struct("<IHHII")


def _torch():
    import torch

    return torch


def _widths(moduli):
    return [(int(q).bit_length() + 7) // 8 for q in moduli]


def _header(engine, kind: int) -> bytes:
    ctx = engine.context
    L, K = ctx.n_q, len(ctx.p_chain_bits)
    mods = np.asarray(engine.moduli[: L + K], np.uint64)
    return _HDR.pack(MAGIC, VERSION, kind, engine.N, L, K, engine._dnum, 0) + mods.tobytes()


def _check_header(engine, blob: bytes, kind: int) -> int:
    if len(blob) < _HDR.size or blob[:4] != MAGIC:
        raise HebatchError("not a hebatch wire blob (bad magic)")
    magic, ver, k, N, L, K, dnum, _ = _HDR.unpack_from(blob, 0)
    if ver != VERSION:
        raise HebatchError(f"wire version {ver} (expected {VERSION})")
    if k != kind:
        raise HebatchError(f"wire blob of kind {k}, expected {kind}")
    off = _HDR.size
    mods = np.frombuffer(blob, np.uint64, L + K, off)
    ctx = engine.context
    mine = np.asarray(engine.moduli[: ctx.n_q + len(ctx.p_chain_bits)], np.uint64)
    if N != engine.N or L != ctx.n_q or K != len(ctx.p_chain_bits) or dnum != engine._dnum \
            or not np.array_equal(mods, mine):
        raise ContextMismatch(f"wire blob for N={N}, L={L}, K={K}, dnum={dnum} does not match this context")
    return off + 8 * (L + K)


def _pack(t, widths) -> bytes:
    """int64 device tensor [..., M, N] -> bytes, modulus m packed to widths[m] bytes per residue."""
    torch = _torch()
    b = t.contiguous().view(torch.uint8).reshape(t.shape + (8,))
    parts = [b[..., m, :, :w].contiguous().reshape(b.shape[:-3] + (-1,)) for m, w in enumerate(widths)]
    return torch.cat(parts, dim=-1).cpu().numpy().tobytes()


def _unpack(buf, shape, widths, device):
    """Inverse of _pack: bytes -> int64 device tensor of ``shape`` [..., M, N]."""
    torch = _torch()
    lead, (M, N) = tuple(shape[:-2]), shape[-2:]
    src = torch.frombuffer(bytearray(buf), dtype=torch.uint8).to(device).reshape(lead + (-1,))
    out = torch.zeros(lead + (M, N, 8), dtype=torch.uint8, device=device)
    o = 0
    for m, w in enumerate(widths):
        out[..., m, :, :w] = src[..., o:o + N * w].reshape(lead + (N, w))
        o += N * w
    return out.view(torch.int64).reshape(tuple(shape))


def export_ciphertexts(engine, cts) -> bytes:
    """Serialise ciphertexts of one level and component count (all on ``engine``)."""
    torch = _torch()
    cts = list(cts)
    if not cts:
        raise HebatchError("export_ciphertexts: nothing to export")
    for c in cts:
        engine._check(c)
    nc, level = engine._ncomp(cts), cts[0].level
    if any(c.level != level for c in cts):
        raise HebatchError("export_ciphertexts needs one level")
    limbs = level + 1
    t = torch.stack([c.data for c in cts])
    scales = np.array([c.scale for c in cts], np.float64)
    return (_header(engine, KIND_CTS) + _CTS.pack(len(cts), nc, limbs, level, 0) + scales.tobytes()
            + _pack(t, _widths(engine.moduli[:limbs])))


def import_ciphertexts(engine, blob: bytes):
    """Deserialise ciphertexts into ``engine`` (which must share the parameters)."""
    torch = _torch()
    off = _check_header(engine, blob, KIND_CTS)
    count, nc, limbs, level, _ = _CTS.unpack_from(blob, off)
    off += _CTS.size
    if limbs != level + 1 or not 1 <= limbs <= engine.context.n_q or nc < 2:
        raise HebatchError(f"bad ciphertext header: {count} x {nc} components, {limbs} limbs, level {level}")
    scales = np.frombuffer(blob, np.float64, count, off)
    off += 8 * count
    widths = _widths(engine.moduli[:limbs])
    need = count * nc * engine.N * sum(widths)
    if len(blob) - off != need:
        raise HebatchError(f"ciphertext payload is {len(blob) - off} bytes, expected {need}")
    t = _unpack(memoryview(blob)[off:], (count, nc, limbs, engine.N), widths, engine.device)
    q = torch.as_tensor(np.asarray(engine.moduli[:limbs], np.int64), device=engine.device).view(1, 1, limbs, 1)
    if bool(((t < 0) | (t >= q)).any()):
        raise HebatchError("imported ciphertext holds residues outside [0, q)")
    batch = engine._alloc(count, nc, limbs)
    batch.copy_(t)
    return engine._wrap_batch(batch, level, [float(s) for s in scales])


def _key_codes(engine, offsets=None):
    codes = []
    for code in (0, 2, 4):
        if engine._L.he_has_switch_key(engine._h, code):
            codes.append(code)
    offs = engine.keys.resident if offsets is None else {engine.keys.canonical(o) for o in offsets}
    for c in sorted(offs):
        if c:
            codes.append(pow(5, c, 2 * engine.N))
    return codes


def export_eval_keys(engine, offsets=None) -> bytes:
    """The evaluation keys a server needs: relinearisation (and power) keys plus
    the Galois keys of ``offsets`` (default: every resident rotation offset)."""
    torch = _torch()
    ctx = engine.context
    M = ctx.n_q + len(ctx.p_chain_bits)
    widths = _widths(engine.moduli[:M])
    codes = _key_codes(engine, offsets)
    out = [_header(engine, KIND_KEYS), struct.pack("<I", len(codes))]
    for code in codes:
        k = torch.empty((engine._dnum, 2, M, engine.N), dtype=torch.int64, device=engine.device)
        _lib.check(engine._L.he_export_switch_key(engine._h, code, k.data_ptr(), engine.stream), "export key")
        out.append(struct.pack("<I", code))
        out.append(_pack(k, widths))
    return b"".join(out)


def import_eval_keys(engine, blob: bytes) -> list:
    """Install keys from ``export_eval_keys``; rotation offsets become resident
    (engine.keys) without key generation.  Returns the installed key codes."""
    off = _check_header(engine, blob, KIND_KEYS)
    (n,) = struct.unpack_from("<I", blob, off)
    off += 4
    ctx = engine.context
    M = ctx.n_q + len(ctx.p_chain_bits)
    widths = _widths(engine.moduli[:M])
    per = engine._dnum * 2 * engine.N * sum(widths)
    twoN = 2 * engine.N
    log5 = {pow(5, k, twoN): k for k in range(engine.context.n)}
    codes = []
    for _ in range(n):
        (code,) = struct.unpack_from("<I", blob, off)
        off += 4
        if len(blob) < off + per:
            raise HebatchError("truncated key blob")
        k = _unpack(memoryview(blob)[off:off + per], (engine._dnum, 2, M, engine.N), widths, engine.device)
        off += per
        _lib.check(engine._L.he_import_switch_key(engine._h, code, k.data_ptr(), engine.stream), "import key")
        if code % 2 == 1:
            if code not in log5:
                raise HebatchError(f"key code {code} is not a rotation 5^k mod 2N")
            engine.keys.register([log5[code]])
        elif code == 0:
            engine._relin = True
        codes.append(code)
    if off != len(blob):
        raise HebatchError("trailing bytes after the last key")
    return codes
