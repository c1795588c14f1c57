"""B200 RNS-CKKS engine behind the reference's VectorEngine protocol.

Drop-in for ``hebatch.engine`` (reference /root/reference/pkg/src/hebatch/
engine.py).  ``EngineContext``, ``CipherVec``, ``PlainVec``,
``RotationKeySet``, ``OpCounters`` and the ``VectorEngine`` protocol keep the
reference's names, fields and semantics; ``GpuEngine`` replaces
``SimulatorEngine`` (engine.py:229-420): the float64 slot arithmetic becomes
real RNS-CKKS executed by the sm_100a kernels of libhe_sm100.so.

Semantics preserved from the reference (and tested):
  * rotate(ct, k): output slot i holds input slot i+k (engine.py:13-15);
    k = 0 mod n returns the same handle uncounted (engine.py:278-279); a
    missing key raises MissingRotationKey(k) before anything is counted.
  * every mult_plain / mult_ct costs ``mult_level_cost`` levels and raises
    LevelExhausted when the level would go negative (engine.py:297-313);
    add/mult_ct results sit at the lower operand level (engine.py:289).
  * counters, live-handle tracking, window peaks and double-release errors
    behave as in _Accounting (engine.py:180-227).
A ciphertext at ``level`` has ``level + 1`` Q-limbs; a fresh one is at
``max_level``.  There is no CPU fallback: without the CUDA library or a GPU
the engine raises.
"""

from __future__ import annotations

import itertools
import math
import threading
from dataclasses import dataclass, field
from typing import Iterable, Protocol, Sequence

import numpy as np

from . import _lib
from .errors import (
    ContextMismatch,
    HebatchError,
    LengthExceedsSlots,
    LevelExhausted,
    MissingRotationKey,
    ScaleMismatch,
    ShapeMismatch,
)

# relative scale difference tolerated by add() (error contribution <= 2^-20 * |x|)
SCALE_RTOL = 2.0 ** -20


@dataclass(frozen=True)
class EngineContext:
    """CKKS parameter set (reference EngineContext, engine.py:36-63).

    The reference carries ``first_modulus_bits``, ``rescale_bits`` and
    ``key_switch_digits`` "for configuration fidelity only"; here they are
    live: q_0 has ``first_modulus_bits`` bits, q_1..q_max_level have
    ``rescale_bits`` bits, and key switching uses ``key_switch_digits`` digits
    (alpha = ceil((max_level+1)/digits) limbs each).  Additions:
    ``special_prime_bits`` (default: alpha primes of first_modulus_bits bits),
    ``scale_bits`` (encoding scale, default rescale_bits), ``q_bits`` (explicit
    Q chain override), ``device`` and ``secret_hamming`` (0: dense ternary
    secret; h > 0: sparse secret of expected Hamming weight h, which keeps the
    bootstrap's ModRaise overflow small).  ``noise_sigma`` is the simulator's
    slot perturbation and has no meaning for real encryption (ignored).
    """

    n: int
    max_level: int = 25
    mult_level_cost: int = 1
    noise_sigma: float = 0.0
    bootstrap_reserve: int = 10
    first_modulus_bits: int = 50
    rescale_bits: int = 46
    key_switch_digits: int = 4
    noise_seed: int = 0
    special_prime_bits: tuple = ()
    scale_bits: int | None = None
    q_bits: tuple | None = None
    device: int = 0
    secret_hamming: int = 0

    def __post_init__(self) -> None:
        if self.n < 1 or (self.n & (self.n - 1)) != 0:
            raise ValueError(f"slot count must be a power of two, got {self.n}")
        if not (0 < self.bootstrap_reserve < self.max_level):
            raise ValueError("bootstrap_reserve must lie in (0, max_level)")
        if self.mult_level_cost < 1:
            raise ValueError("mult_level_cost must be >= 1")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be nonnegative")
        if self.key_switch_digits < 1:
            raise ValueError("key_switch_digits must be >= 1")
        if self.q_bits is not None and len(self.q_bits) != self.max_level + 1:
            raise ValueError("q_bits must list max_level + 1 prime sizes")

    # -- derived RNS parameters
    @property
    def ring_degree(self) -> int:
        return 2 * self.n

    @property
    def log_n(self) -> int:
        return int(math.log2(self.ring_degree))

    @property
    def n_q(self) -> int:
        return self.max_level + 1

    @property
    def alpha(self) -> int:
        return -(-self.n_q // self.key_switch_digits)

    @property
    def q_chain_bits(self) -> tuple:
        if self.q_bits is not None:
            return tuple(self.q_bits)
        return (self.first_modulus_bits,) + (self.rescale_bits,) * self.max_level

    @property
    def p_chain_bits(self) -> tuple:
        if self.special_prime_bits:
            return tuple(self.special_prime_bits)
        return (self.first_modulus_bits,) * self.alpha

    @property
    def scale(self) -> float:
        return 2.0 ** (self.scale_bits if self.scale_bits is not None else self.rescale_bits)

    def he_params(self) -> "_lib.HeParams":
        p = _lib.HeParams()
        p.log_n = self.log_n
        qb, pb = self.q_chain_bits, self.p_chain_bits
        p.n_q, p.n_p, p.alpha = len(qb), len(pb), self.alpha
        for i, b in enumerate(qb):
            p.q_bits[i] = b
        for i, b in enumerate(pb):
            p.p_bits[i] = b
        p.seed = self.noise_seed & 0xFFFFFFFFFFFFFFFF
        p.scale = self.scale
        p.sk_hamming = int(self.secret_hamming)
        return p


@dataclass(frozen=True, eq=False)
class CipherVec:
    """Handle to one device-resident RNS-CKKS ciphertext.

    ``data`` is a torch int64 tensor [n_comp][level+1][N] (NTT domain, the
    uint64 residues reinterpreted); ``scale`` is the exact CKKS scale;
    ``scale_bits`` its rounded log2 (reference field, engine.py:66-80).
    Immutable: every engine operation returns a fresh handle.
    """

    data: object
    level: int
    scale_bits: int
    id: int
    scale: float = 1.0
    n_slots: int = 0
    owner: int = 0

    def __len__(self) -> int:
        return self.n_slots

    @property
    def limbs(self) -> int:
        return self.level + 1

    @property
    def ptr(self) -> int:
        if self.data is None:
            raise HebatchError(f"ciphertext {self.id} was released")
        return self.data.data_ptr()


@dataclass(eq=False)
class PlanarCarry:
    """The pooled, unrelinearised 3-component squares of the block before the
    last (run_cnn's carry), held in the conv2 kernel's shared-memory ring layout
    instead of as C*H*W ciphertexts: [limb][N/8 coefficient chunks][y][x]
    [component][byte plane][8 coefficients x 16 channels], one byte per residue
    byte, 5 bytes per 40-bit residue (include/he_sm100.h he_conv_square_sum_pl).
    conv1's epilogue writes it, conv2 fills its ring with one bulk copy per row.
    Every residue is canonical, so he_planar_unpack recovers the ciphertexts
    bit for bit."""

    data: object          # torch uint8 [limbs * N/8 * H * W * 1920]
    channels: int
    H: int
    W: int
    level: int
    scale: float
    owner: int

    BYTES_PER_PIXEL = 3 * 5 * 128

    @property
    def limbs(self) -> int:
        return self.level + 1


@dataclass(frozen=True)
class PlainVec:
    """A plaintext slot vector, full slot width (engine.py:83-90).

    Host data: encoding happens inside mult_plain / add_plain, at the scale
    the operation needs.  A vector whose slots are all equal takes the scalar
    fast path (a constant polynomial: the same residue at every NTT point).
    """

    slots: np.ndarray

    def __len__(self) -> int:
        return self.slots.shape[0]


class RotationKeySet:
    """Resident rotation offsets, canonical mod n (engine.py:93-136).

    Offset 0 is never stored; ``generation_count`` counts every key ever
    registered.  The key material itself lives on the device (he_ctx).
    """

    def __init__(self, n: int):
        self._n = n
        self._offsets: set[int] = set()
        self.generation_count = 0

    def canonical(self, offset: int) -> int:
        return offset % self._n

    def register(self, offsets: Iterable[int]) -> int:
        """Add keys; returns how many became newly resident (idempotent), as
        the reference does (engine.py:108-119)."""
        added = 0
        for off in offsets:
            c = self.canonical(off)
            if c and c not in self._offsets:
                self._offsets.add(c)
                added += 1
        self.generation_count += added
        return added

    def unload(self, offsets: Iterable[int]) -> None:
        for off in offsets:
            self._offsets.discard(self.canonical(off))

    def unload_all(self) -> None:
        self._offsets.clear()

    def holds(self, offset: int) -> bool:
        return self.canonical(offset) in self._offsets

    @property
    def resident(self) -> frozenset:
        return frozenset(self._offsets)

    def __len__(self) -> int:
        return len(self._offsets)


@dataclass(frozen=True)
class OpCounters:
    """Cumulative operation counts plus the live-ciphertext peak."""

    rotations: int = 0
    plain_mults: int = 0
    ct_mults: int = 0
    adds: int = 0
    bootstraps: int = 0
    key_loads: int = 0
    peak_live_ciphertexts: int = 0

    def delta(self, earlier: "OpCounters") -> "OpCounters":
        """Difference since ``earlier``; the peak is reported as-is."""
        return OpCounters(
            rotations=self.rotations - earlier.rotations,
            plain_mults=self.plain_mults - earlier.plain_mults,
            ct_mults=self.ct_mults - earlier.ct_mults,
            adds=self.adds - earlier.adds,
            bootstraps=self.bootstraps - earlier.bootstraps,
            key_loads=self.key_loads - earlier.key_loads,
            peak_live_ciphertexts=self.peak_live_ciphertexts,
        )


class VectorEngine(Protocol):
    """Operation surface every backend provides (engine.py:164-177)."""

    context: EngineContext

    def encrypt(self, values) -> CipherVec: ...
    def decrypt(self, ct: CipherVec) -> np.ndarray: ...
    def rotate(self, ct: CipherVec, k: int) -> CipherVec: ...
    def add(self, a: CipherVec, b: CipherVec) -> CipherVec: ...
    def add_plain(self, a: CipherVec, p: PlainVec) -> CipherVec: ...
    def mult_plain(self, ct: CipherVec, p: PlainVec) -> CipherVec: ...
    def mult_ct(self, a: CipherVec, b: CipherVec) -> CipherVec: ...
    def bootstrap(self, ct: CipherVec) -> CipherVec: ...
    def release(self, *cts: CipherVec) -> None: ...


class _Ledger:
    """Lock-protected counters and live-handle set (engine.py:180-227)."""

    _FIELDS = ("rotations", "plain_mults", "ct_mults", "adds", "bootstraps", "key_loads")

    def __init__(self) -> None:
        self.lock = threading.Lock()
        self.counts = dict.fromkeys(self._FIELDS, 0)
        self.live: set[int] = set()
        self.peak = 0
        self.window_peak = 0

    def bump(self, name: str, by: int = 1) -> None:
        with self.lock:
            self.counts[name] += by

    def track(self, ids: Sequence[int]) -> None:
        with self.lock:
            self.live.update(ids)
            k = len(self.live)
            self.peak = max(self.peak, k)
            self.window_peak = max(self.window_peak, k)

    def drop(self, handle: int) -> None:
        with self.lock:
            if handle not in self.live:
                raise HebatchError(f"release of unknown or already-released handle {handle}")
            self.live.discard(handle)

    def snapshot(self) -> OpCounters:
        with self.lock:
            return OpCounters(peak_live_ciphertexts=self.peak, **self.counts)


def _storage_uses(t) -> int:
    """References to ``t``'s storage (tensors and views sharing it + the
    temporary wrapper).  Uses torch's storage use count when this torch build
    exposes it; otherwise reports every cached batch as in use (no slab reuse:
    correct, only slower)."""
    torch = _torch()
    f = getattr(torch._C, "_storage_Use_Count", None)
    if f is None:
        return 1 << 30
    return f(t.untyped_storage()._cdata)


def _torch():
    import torch

    return torch


class GpuEngine:
    """RNS-CKKS on one B200: the sm_100a replacement of SimulatorEngine.

    Per-ciphertext protocol methods (encrypt, add, mult_plain, ...) each launch
    a handful of kernels; the ``*_batch`` methods and ``lincomb`` are the
    batched hot path used by the layer calls (conv_forward, fm_* in
    featuremajor.py): one launch sequence for a whole layer.
    """

    def __init__(self, context: EngineContext):
        torch = _torch()
        if not torch.cuda.is_available():
            raise HebatchError("GpuEngine needs a CUDA device (sm_100a); there is no CPU fallback")
        if context.mult_level_cost != 1:
            raise HebatchError("GpuEngine implements mult_level_cost == 1 (one rescale per multiplication)")
        self.context = context
        self.device = torch.device("cuda", context.device)
        self._L = _lib.load()
        import ctypes as C

        self._params = context.he_params()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.he_ctx_create(C.byref(self._params), context.device, C.byref(h)), "he_ctx_create")
        self._h = h
        M = context.n_q + len(context.p_chain_bits)
        mods = np.zeros(M, np.uint64)
        psi = np.zeros(M, np.uint64)
        _lib.check(self._L.he_ctx_moduli(self._h, _lib.addr(mods), _lib.addr(psi)))
        self.moduli = [int(x) for x in mods]
        self.psi = [int(x) for x in psi]
        self.N = context.ring_degree
        self.keys = RotationKeySet(context.n)
        self._acct = _Ledger()
        self._ids = itertools.count(1)
        self._enc_counter = 0
        self._enc_lock = threading.Lock()
        self.registration_log: list[frozenset] = []
        self._relin = False
        self._dnum = -(-context.n_q // context.alpha)  # key-switch digits (key layout [dnum][2][L+K][N])
        self._timing = None  # {category: [(start_event, end_event, units)]} when enabled
        self._slab: dict = {}  # shape -> cached ciphertext batches (see _alloc)
        self.pool_releases = 0  # out-of-memory retries (_release_pool)
        # exact int8-digit tensor-core convolutions (he_conv_mma); False = CUDA-core kernel
        self.use_tensor_cores = True
        self.joint_moddown = True  # relin + rescales as one ModDown (N = 2^16)
        self.use_fused_conv = True  # conv + square + pool/GAP in one kernel (he_conv_square_sum)

    # ------------------------------------------------------------ timing hooks (bench.py)
    def enable_timing(self, on: bool = True) -> None:
        """Record CUDA events around every C-ABI call, on the launching stream."""
        self._timing = {} if on else None

    def timing_summary(self) -> dict:
        """{category: (calls, total_ms, units)} for the recorded calls (synchronises)."""
        torch = _torch()
        torch.cuda.synchronize(self.device)
        out = {}
        for cat, evs in (self._timing or {}).items():
            ms = sum(s.elapsed_time(e) for s, e, _ in evs)
            units = np.sum(np.array([u for _, _, u in evs], dtype=np.float64), axis=0)
            out[cat] = (len(evs), ms, units)
        return out

    def _call(self, cat: str, fn, *args, units=(0.0, 0.0)):
        """Run one C-ABI call; with timing on, bracket it with CUDA events.
        ``units`` = (algorithmic HBM bytes, algorithmic modular MACs)."""
        if self._timing is None:
            rc = fn(*args)
            if rc == _lib.HE_ENOMEM:   # the library's scratch did not fit: return parked batches, once
                self._release_pool()
                rc = fn(*args)
            return rc
        torch = _torch()
        st = torch.cuda.current_stream(self.device)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        rc = fn(*args)
        if rc == _lib.HE_ENOMEM:
            self._release_pool()
            rc = fn(*args)
        e.record(st)
        self._timing.setdefault(cat, []).append((s, e, units))
        return rc

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "_L", None) is not None:
            try:
                self._L.he_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------ plumbing
    @property
    def stream(self) -> int:
        return _torch().cuda.current_stream(self.device).cuda_stream

    # Batches of at least this many bytes are kept by the engine after their last
    # ciphertext is released and handed out again for the next batch of the same
    # shape.  A pass allocates the same sequence of 21 GB batches every time; a
    # fresh stream-ordered allocation of that size can cost 25-500 ms of host time
    # (the pool remaps physical pages into a new virtual range), which a pass
    # started right after a device synchronize cannot hide.
    SLAB_MIN_BYTES = 1 << 30
    # At most this many bytes of FREE cached batches are kept when a new batch
    # shape is allocated (a pass whose shapes vary -- the row-streamed config-4
    # runner -- would otherwise park released batches of every shape it ever
    # used; the library's own scratch comes from the same pool).  A pass that
    # repeats its shapes (config 3) always finds its own free batch and never
    # triggers the cap.  Config 4 on one B200: 37.8 s per group with 16 GB parked,
    # 31.4 s with 4 GB, 29.3 s with none (fewer out-of-memory retries and remaps).
    SLAB_FREE_CAP = 0

    def _alloc(self, count: int, n_comp: int, limbs: int):
        torch = _torch()
        shape = (count, n_comp, limbs, self.N)
        big = count * n_comp * limbs * self.N * 8 >= self.SLAB_MIN_BYTES
        if big:
            # free = no ciphertext view left: the storage is referenced only by the
            # cached batch and the temporary storage wrapper.  Reuse is stream-ordered
            # like torch's own allocator (every op runs on the current stream).
            for t in self._slab.get(shape, ()):
                if _storage_uses(t) == 2:
                    return t
            self._cap_free_slabs()
        try:
            t = torch.empty(shape, dtype=torch.int64, device=self.device)
        except torch.OutOfMemoryError:
            # drop the cached batches and hand the pool's unused pages back, so a
            # large request is not refused for want of one contiguous free range
            self._release_pool()
            t = torch.empty(shape, dtype=torch.int64, device=self.device)
        if big:
            self._slab.setdefault(shape, []).append(t)
        return t

    def _cap_free_slabs(self) -> None:
        """Drop free cached batches (largest first) until at most SLAB_FREE_CAP bytes stay parked."""
        free = [(t.numel() * t.element_size(), shape, t) for shape, ts in self._slab.items() for t in ts
                if _storage_uses(t) == 2]
        total = sum(b for b, _, _ in free)
        for b, shape, t in sorted(free, key=lambda x: -x[0]):
            if total <= self.SLAB_FREE_CAP:
                break
            self._slab[shape] = [u for u in self._slab[shape] if u is not t]
            if not self._slab[shape]:
                del self._slab[shape]
            total -= b

    def _release_pool(self) -> None:
        """Drop the cached batches and hand the pool's unused pages back to the
        device, so a large request is not refused for want of one free range."""
        torch = _torch()
        self.pool_releases += 1
        self.trim()
        torch.cuda.synchronize(self.device)
        torch.cuda.empty_cache()

    def trim(self) -> None:
        """Return the engine's cached (released) ciphertext batches to the pool."""
        for shape in list(self._slab):
            keep = [t for t in self._slab[shape] if _storage_uses(t) > 2]
            if keep:
                self._slab[shape] = keep
            else:
                del self._slab[shape]

    def _wrap(self, tensors, level: int, scales) -> list[CipherVec]:
        ids = [next(self._ids) for _ in range(len(tensors))]
        out = []
        for t, i, s in zip(tensors, ids, scales):
            out.append(CipherVec(data=t, level=level, scale_bits=int(round(math.log2(s))), id=i, scale=float(s),
                                 n_slots=self.context.n, owner=id(self)))
        self._acct.track(ids)
        return out

    def _wrap_batch(self, batch, level: int, scales) -> list[CipherVec]:
        return self._wrap([batch[i] for i in range(batch.shape[0])], level, scales)

    @staticmethod
    def _ptrs(cts: Sequence[CipherVec]) -> np.ndarray:
        return _lib.ptr_array([c.ptr for c in cts])

    @staticmethod
    def _tptrs(batch) -> np.ndarray:
        base, stride = batch.data_ptr(), batch.stride(0) * 8
        return _lib.ptr_array([base + i * stride for i in range(batch.shape[0])])

    def _check(self, ct: CipherVec) -> None:
        if not isinstance(ct, CipherVec) or ct.n_slots != self.context.n or ct.owner != id(self):
            width = getattr(ct, "n_slots", None)
            raise ContextMismatch(f"ciphertext (width {width}) does not belong to this context (slots {self.context.n})")
        if ct.data is None:
            raise HebatchError(f"ciphertext {ct.id} was released")

    def _check_plain(self, p: PlainVec) -> np.ndarray:
        v = np.asarray(p.slots, dtype=np.float64)
        if v.shape != (self.context.n,):
            raise ContextMismatch(f"plaintext width {v.shape[0] if v.ndim else 0} != context slots {self.context.n}")
        return v

    def _res(self, value_int: int, limbs: int) -> list[int]:
        return [value_int % q for q in self.moduli[:limbs]]

    def _at_level(self, cts: Sequence[CipherVec], level: int) -> list:
        """Tensors of `cts` truncated to level (+1 limbs); copies only if needed."""
        out = []
        for c in cts:
            if c.level == level:
                out.append(c.data)
            else:
                out.append(c.data[:, : level + 1].contiguous())
        return out

    # ------------------------------------------------------------ encryption
    def _next_enc(self, count: int) -> int:
        with self._enc_lock:
            base = self._enc_counter
            self._enc_counter += count
        return base

    def encrypt(self, values) -> CipherVec:
        return self.encrypt_batch(np.asarray(values, dtype=np.float64).ravel()[None, :])[0]

    def encrypt_batch(self, values, level: int | None = None) -> list[CipherVec]:
        """Encode + encrypt each row of a [count, <=n] array (one launch sequence),
        at ``level`` (default: the top level max_level).  A lower level is a
        direct encryption with level + 1 limbs, equal to the first limbs of the
        top-level encryption (he_encrypt_level)."""
        torch = _torch()
        if isinstance(values, torch.Tensor):
            v = values.to(device=self.device, dtype=torch.float64)
        else:
            v = torch.as_tensor(np.asarray(values, dtype=np.float64), device=self.device)
        if v.dim() != 2:
            raise HebatchError("encrypt_batch expects a 2-D [count, values] array")
        count, nvals = v.shape
        if nvals > self.context.n:
            raise LengthExceedsSlots(f"{nvals} values > {self.context.n} slots")
        v = v.contiguous()
        L = self.context.n_q if level is None else int(level) + 1
        if not 1 <= L <= self.context.n_q:
            raise LevelExhausted(f"encryption level {level} outside 0..{self.context.n_q - 1}")
        out = self._alloc(count, 2, L)
        ptrs = self._tptrs(out)
        base = self._next_enc(count)
        _lib.check(self._call("encrypt", self._L.he_encrypt_level, self._h, v.data_ptr(), count, nvals,
                              self.context.scale, base, L, _lib.addr(ptrs), self.stream,
                              units=(count * (2.0 * L * self.N + nvals) * 8, 0.0)), "encrypt")
        return self._wrap_batch(out, L - 1, [self.context.scale] * count)

    def decrypt(self, ct: CipherVec) -> np.ndarray:
        return self.decrypt_batch([ct])[0]

    def decrypt_batch(self, cts: Sequence[CipherVec], as_tensor: bool = False):
        """Decrypt + decode to float64 slots; levels may differ."""
        torch = _torch()
        for c in cts:
            self._check(c)
        self._need_two(cts, "decrypt")
        out = torch.empty((len(cts), self.context.n), dtype=torch.float64, device=self.device)
        by_level: dict[int, list[int]] = {}
        for i, c in enumerate(cts):
            by_level.setdefault(c.level, []).append(i)
        for level, idx in by_level.items():
            sub = [cts[i] for i in idx]
            tmp = out if len(idx) == len(cts) else torch.empty((len(idx), self.context.n), dtype=torch.float64,
                                                              device=self.device)
            ptrs = self._ptrs(sub)
            scales = np.array([c.scale for c in sub], np.float64)
            _lib.check(self._call("decrypt", self._L.he_decrypt, self._h, _lib.addr(ptrs), len(sub), level + 1,
                                  _lib.addr(scales), tmp.data_ptr(), self.stream,
                                  units=(len(sub) * 4.0 * self.N * 8, 0.0)), "decrypt")
            if tmp is not out:
                out[torch.as_tensor(idx, device=self.device)] = tmp
        if as_tensor:
            return out
        return out.cpu().numpy()

    def decrypt_coeffs(self, ct: CipherVec) -> np.ndarray:
        torch = _torch()
        self._check(ct)
        self._need_two([ct], "decrypt_coeffs")
        out = torch.empty((1, self.N), dtype=torch.float64, device=self.device)
        ptrs = self._ptrs([ct])
        _lib.check(self._L.he_decrypt_coeffs(self._h, _lib.addr(ptrs), 1, ct.level + 1, out.data_ptr(), self.stream))
        return out.cpu().numpy()[0]

    def release(self, *cts: CipherVec) -> None:
        for ct in cts:
            self._acct.drop(ct.id)
            object.__setattr__(ct, "data", None)

    # ------------------------------------------------------------ arithmetic
    def rotate(self, ct: CipherVec, k: int) -> CipherVec:
        self._check(ct)
        self._need_two([ct], "rotate")
        if k % self.context.n == 0:
            return ct
        if not self.keys.holds(k):
            raise MissingRotationKey(k)
        self._acct.bump("rotations")
        return self._rotate_batch([ct], k)[0]

    def rotate_hoisted(self, cts: Sequence[CipherVec], ks: Sequence[int]) -> list[list[CipherVec]]:
        """Rotate every ciphertext by every offset in ``ks`` with hoisted key
        switching (he_rotate_hoisted): one basis extension of each c1 serves all
        offsets -- the rotation set of the CBC convolution (conv.py:78-99,
        PAPER.md:309-346).  Returns out[j][i] = rotate(cts[i], ks[j]) up to the
        hoisted limb contract (same decryption).  Offsets k = 0 (mod n) return
        the input handle (engine.py:278-279); others need a registered key
        (MissingRotationKey, raised before any work) and count as rotations."""
        for c in cts:
            self._check(c)
        self._need_two(cts, "rotate_hoisted")
        if not cts:
            return [[] for _ in ks]
        if len({(c.level, c.data.shape[0]) for c in cts}) != 1:
            raise HebatchError("rotate_hoisted needs 2-component inputs at one level")
        live = []
        for k in ks:
            if k % self.context.n and not self.keys.holds(k):
                raise MissingRotationKey(k)
            if k % self.context.n and k % self.context.n not in live:
                live.append(k % self.context.n)
        outs = self._rotate_hoisted_internal(cts, ks)
        for k in ks:
            if k % self.context.n:
                self._acct.bump("rotations", len(cts))
        return outs

    def _rotate_hoisted_internal(self, cts: Sequence[CipherVec], ks: Sequence[int]) -> list[list[CipherVec]]:
        """rotate_hoisted without key-set checks or counters (the keys must exist in the library)."""
        live = []
        for k in ks:
            if k % self.context.n and k % self.context.n not in live:
                live.append(k % self.context.n)
        res = {}
        if live:
            level = cts[0].level
            gs = np.array([pow(5, k, 2 * self.N) for k in live], np.uint32)
            out = self._alloc(len(live) * len(cts), 2, level + 1)
            src = self._ptrs(cts)
            dst = self._tptrs(out)
            _lib.check(self._L.he_rotate_hoisted(self._h, _lib.addr(gs), len(live), _lib.addr(src), _lib.addr(dst),
                                                 len(cts), level + 1, self.stream), "rotate_hoisted")
            wrapped = self._wrap_batch(out, level, [c.scale for c in cts] * len(live))
            for j, k in enumerate(live):
                res[k] = wrapped[j * len(cts):(j + 1) * len(cts)]
        return [list(cts) if k % self.context.n == 0 else res[k % self.context.n] for k in ks]

    def _rotate_batch(self, cts: Sequence[CipherVec], k: int) -> list[CipherVec]:
        return self._automorph_batch(cts, pow(5, k % self.context.n, 2 * self.N))

    def _automorph_batch(self, cts: Sequence[CipherVec], g: int) -> list[CipherVec]:
        """X -> X^g plus key switch with the Galois key of g (5^k: rotation by k; 2N - 1: conjugation)."""
        level = cts[0].level
        out = self._alloc(len(cts), 2, level + 1)
        src = self._ptrs(cts)
        dst = self._tptrs(out)
        _lib.check(self._L.he_rotate(self._h, g, _lib.addr(src), _lib.addr(dst), len(cts), level + 1, self.stream),
                   "rotate")
        return self._wrap_batch(out, level, [c.scale for c in cts])

    def add(self, a: CipherVec, b: CipherVec) -> CipherVec:
        self._check(a)
        self._check(b)
        self._acct.bump("adds")
        return self._add_batch([a], [b])[0]

    def _add_batch(self, A: Sequence[CipherVec], B: Sequence[CipherVec], sub: bool = False) -> list[CipherVec]:
        level = min(min(c.level for c in A), min(c.level for c in B))
        for a, b in zip(A, B):
            if abs(a.scale / b.scale - 1.0) > SCALE_RTOL:
                raise ScaleMismatch(f"scales {a.scale:.6g} and {b.scale:.6g} differ")
        nc = self._ncomp(list(A) + list(B))
        ta, tb = self._at_level(A, level), self._at_level(B, level)
        out = self._alloc(len(A), nc, level + 1)
        pa = _lib.ptr_array([t.data_ptr() for t in ta])
        pb = _lib.ptr_array([t.data_ptr() for t in tb])
        po = self._tptrs(out)
        fn = self._L.he_sub if sub else self._L.he_add
        _lib.check(fn(self._h, _lib.addr(pa), _lib.addr(pb), _lib.addr(po), len(A), level + 1, nc, self.stream), "add")
        return self._wrap_batch(out, level, [a.scale for a in A])

    def add_batch(self, A: Sequence[CipherVec], B: Sequence[CipherVec]) -> list[CipherVec]:
        for c in list(A) + list(B):
            self._check(c)
        self._acct.bump("adds", len(A))
        return self._add_batch(A, B)

    def add_inplace(self, A: Sequence[CipherVec], B: Sequence[CipherVec]) -> None:
        """A[i] += B[i] (mod q) in place: accumulators of partial sums (sharded_cnn).
        Equal levels, scales and component counts; B is left untouched."""
        for c in list(A) + list(B):
            self._check(c)
        if len(A) != len(B):
            raise ShapeMismatch(f"add_inplace: {len(A)} accumulators, {len(B)} addends")
        if not A:
            return
        level = A[0].level
        nc = self._ncomp(list(A) + list(B))
        for a, b in zip(A, B):
            if a.level != level or b.level != level:
                raise HebatchError("add_inplace needs one level")
            if abs(a.scale / b.scale - 1.0) > SCALE_RTOL:
                raise ScaleMismatch(f"scales {a.scale:.6g} and {b.scale:.6g} differ")
        self._acct.bump("adds", len(A))
        pa, pb = self._ptrs(A), self._ptrs(B)
        _lib.check(self._L.he_add(self._h, _lib.addr(pa), _lib.addr(pb), _lib.addr(pa), len(A), level + 1, nc,
                                  self.stream), "add_inplace")

    def add_plain(self, a: CipherVec, p: PlainVec) -> CipherVec:
        self._check(a)
        v = self._check_plain(p)
        self._acct.bump("adds")
        if np.all(v == v[0]):
            return self.add_const_batch([a], [float(v[0])], count=False)[0]
        torch = _torch()
        limbs = a.level + 1
        pt = torch.empty((limbs, self.N), dtype=torch.int64, device=self.device)
        vv = torch.as_tensor(v, device=self.device)
        _lib.check(self._L.he_encode_plain(self._h, vv.data_ptr(), self.context.n, a.scale, limbs, pt.data_ptr(),
                                           self.stream), "encode_plain")
        nc = a.data.shape[0]
        out = self._alloc(1, nc, limbs)
        out[0, 1:].copy_(a.data[1:])
        pa = _lib.ptr_array([a.ptr])
        pp = _lib.ptr_array([pt.data_ptr()])
        po = self._tptrs(out)
        _lib.check(self._L.he_add(self._h, _lib.addr(pa), _lib.addr(pp), _lib.addr(po), 1, limbs, 1, self.stream))
        return self._wrap_batch(out, a.level, [a.scale])[0]

    def add_const_batch(self, cts: Sequence[CipherVec], values: Sequence[float], count: bool = True) -> list[CipherVec]:
        """ct_i + values[i] in every slot (no level consumed)."""
        for c in cts:
            self._check(c)
        if count:
            self._acct.bump("adds", len(cts))
        level = cts[0].level
        if any(c.level != level for c in cts):
            raise HebatchError("add_const_batch needs equal levels")
        limbs = level + 1
        nc = self._ncomp(cts)
        res = np.array([self._res(int(np.rint(v * c.scale)), limbs) for v, c in zip(values, cts)], np.uint64)
        out = self._alloc(len(cts), nc, limbs)
        pi, po = self._ptrs(cts), self._tptrs(out)
        _lib.check(self._call("add_const", self._L.he_add_const, self._h, _lib.addr(pi), _lib.addr(po), len(cts),
                              limbs, nc, _lib.addr(res), self.stream,
                              units=(len(cts) * 2.0 * nc * limbs * self.N * 8, 0.0)), "add_const")
        return self._wrap_batch(out, level, [c.scale for c in cts])

    @staticmethod
    def _ncomp(cts: Sequence[CipherVec]) -> int:
        nc = cts[0].data.shape[0]
        if any(c.data.shape[0] != nc for c in cts):
            raise HebatchError("mixed 2- and 3-component ciphertexts in one batch")
        return nc

    @staticmethod
    def _need_two(cts: Sequence[CipherVec], op: str) -> None:
        """Operations defined only on relinearised (2-component) ciphertexts:
        rotation (the Galois key switches c1 alone) and decryption.  An
        unrelinearised product (3 or 5 components, tensor_batch /
        conv_square_sum) must be relinearised first (relin_rescale_batch)."""
        for c in cts:
            if c.data.shape[0] != 2:
                raise HebatchError(f"{op} needs a relinearised 2-component ciphertext, got {c.data.shape[0]} "
                                   f"components (relinearise it first)")

    def tensor_batch(self, A: Sequence[CipherVec], B: Sequence[CipherVec]) -> list[CipherVec]:
        """ct x ct WITHOUT relinearisation or rescale: 3-component results at the
        common level, scale s_a * s_b (lazy relinearisation / rescaling: sums of
        such products -- pooling, GAP -- are relinearised and rescaled once)."""
        for c in list(A) + list(B):
            self._check(c)
        if any(c.level < self.context.mult_level_cost for c in list(A) + list(B)):
            raise LevelExhausted("operand level below multiplication cost")
        self._acct.bump("ct_mults", len(A))
        level = min(min(c.level for c in A), min(c.level for c in B))
        limbs = level + 1
        ta, tb = self._at_level(A, level), self._at_level(B, level)
        out = self._alloc(len(A), 3, limbs)
        pa = _lib.ptr_array([t.data_ptr() for t in ta])
        pb = _lib.ptr_array([t.data_ptr() for t in tb])
        po = self._tptrs(out)
        _lib.check(self._call("tensor", self._L.he_tensor, self._h, _lib.addr(pa), _lib.addr(pb), _lib.addr(po),
                              len(A), limbs, self.stream, units=(len(A) * 7.0 * limbs * self.N * 8, 0.0)), "tensor")
        return self._wrap_batch(out, level, [a.scale * b.scale for a, b in zip(A, B)])

    def square_sum_batch(self, inputs: Sequence[CipherVec], row_ptr, col, const: float,
                         scale_mult: float) -> list[CipherVec]:
        """out[o] = sum_{t in row o} (in[col_t]^2 + const), unrelinearised (3
        components), not rescaled; declared scale s_in^2 * scale_mult (pool: 4,
        GAP: pixel count).  Equals tensor_batch + add_const_batch + lincomb_int."""
        for c in inputs:
            self._check(c)
        s = inputs[0].scale
        if any(c.scale != s for c in inputs):
            raise ScaleMismatch("square_sum_batch needs inputs at one scale")
        level = min(c.level for c in inputs)
        limbs = level + 1
        rp = np.ascontiguousarray(row_ptr, np.int32)
        cl = np.ascontiguousarray(col, np.int32)
        n_out = len(rp) - 1
        cnt = np.diff(rp)
        C = int(np.rint(const * (s * s)))                 # add_const_batch's residue per square
        res = np.array([self._res(int(k) * C, limbs) for k in cnt], np.uint64) if const else None
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        out = self._alloc(n_out, 3, limbs)
        pout = self._tptrs(out)
        _lib.check(self._call("square_sum", self._L.he_square_sum, self._h, _lib.addr(pin), len(inputs),
                              _lib.addr(pout), n_out, _lib.addr(rp), _lib.addr(cl),
                              _lib.addr(res) if res is not None else None, limbs, self.stream,
                              units=((len(np.unique(cl)) * 2 + n_out * 3) * limbs * self.N * 8.0,
                                     4.0 * len(cl) * limbs * self.N)), "square_sum")
        self._acct.bump("ct_mults", int(len(cl)))
        self._acct.bump("adds", int(len(cl)) + max(0, int(len(cl)) - n_out))
        return self._wrap_batch(out, level, [s * s * scale_mult] * n_out)

    def _ks_modmuls(self, limbs: int, drops: int, nk: int = 1) -> float:
        """Algorithmic modular multiplications of one relinearisation of ``nk``
        switched components with a joint ModDown over P and ``drops`` limbs
        (SURVEY.md 8d key-switch row): NTT butterflies + ModUp / ModDown BConv
        MACs + inner-product MACs (ModUp and inner product once per component)."""
        K, alpha, N = len(self.context.p_chain_bits), self.context.alpha, self.N
        digits = [min(alpha, limbs - j * alpha) for j in range(-(-limbs // alpha))]
        ext = limbs + K
        n_ntt = nk * (limbs + sum(ext - a for a in digits)) + 2 * (K + drops) + 2 * (limbs - drops)
        bconv = nk * sum(a * (ext - a) for a in digits) + 2 * (K + drops) * (limbs - drops)
        ip = nk * 2 * len(digits) * ext
        return float(n_ntt * (N // 2) * int(math.log2(N)) + (bconv + ip) * N)

    def relin_rescale_batch(self, cts: Sequence[CipherVec], drops: int = 1) -> list[CipherVec]:
        """3-component ciphertexts -> relinearise (key switch of c2) -> rescale
        ``drops`` times (2 after a deferred-rescale linear layer).  5-component
        ciphertexts (squares of 3-component ones) switch c2, c3, c4 with the
        s^2, s^3, s^4 keys into one accumulator and need the joint ModDown
        (N = 2^16; oracle oc_relin_rescale_n)."""
        for c in cts:
            self._check(c)
        nc = self._ncomp(cts)
        if nc not in (3, 5):
            raise HebatchError("relin_rescale_batch expects 3- or 5-component ciphertexts")
        self._ensure_relin()
        level = cts[0].level
        if nc == 5:
            if not (self.joint_moddown and self.N == 1 << 16) or drops < 1:
                raise HebatchError("5-component relinearisation needs the joint ModDown (N = 2^16, drops >= 1)")
            self._ensure_power_keys()
            if any(c.level != level for c in cts) or level < drops:
                raise LevelExhausted(f"relin_rescale_batch needs equal levels >= {drops}")
            limbs = level + 1
            pi = self._ptrs(cts)
            out = self._alloc(len(cts), 2, limbs - drops)
            po = self._tptrs(out)
            _lib.check(self._call("relin", self._L.he_relin_rescale_n, self._h, _lib.addr(pi), _lib.addr(po),
                                  len(cts), limbs, drops, 5, self.stream,
                                  units=(len(cts) * (9.0 * limbs - 2 * drops) * self.N * 8,
                                         len(cts) * self._ks_modmuls(limbs, drops, 3))), "relin_rescale_n")
            scales = [c.scale for c in cts]
            for k in range(drops):
                ql = self.moduli[limbs - 1 - k]
                scales = [s_ / ql for s_ in scales]
            return self._wrap_batch(out, level - drops, scales)
        if any(c.level != level for c in cts) or level < drops:
            raise LevelExhausted(f"relin_rescale_batch needs equal levels >= {drops}")
        limbs = level + 1
        pi = self._ptrs(cts)
        scales = [c.scale for c in cts]
        if drops >= 1 and self.joint_moddown and self.N == 1 << 16:
            # one ModDown over P u {dropped limbs} (oracle oc_relin_rescale)
            out = self._alloc(len(cts), 2, limbs - drops)
            po = self._tptrs(out)
            _lib.check(self._call("relin", self._L.he_relin_rescale, self._h, _lib.addr(pi), _lib.addr(po), len(cts),
                                  limbs, drops, self.stream,
                                  units=(len(cts) * (5.0 * limbs - 2 * drops) * self.N * 8,
                                         len(cts) * self._ks_modmuls(limbs, drops))), "relin_rescale")
            for k in range(drops):
                ql = self.moduli[limbs - 1 - k]
                scales = [s / ql for s in scales]
            return self._wrap_batch(out, level - drops, scales)
        cur = self._alloc(len(cts), 2, limbs)
        pm = self._tptrs(cur)
        _lib.check(self._call("relin", self._L.he_relin, self._h, _lib.addr(pi), _lib.addr(pm), len(cts), limbs,
                              self.stream, units=(len(cts) * 5.0 * limbs * self.N * 8, 0.0)), "relin")
        for _ in range(drops):
            ql = self.moduli[limbs - 1]
            out = self._alloc(len(cts), 2, limbs - 1)
            po = self._tptrs(out)
            _lib.check(self._call("rescale", self._L.he_rescale, self._h, _lib.addr(pm), _lib.addr(po), len(cts),
                                  limbs, 2, self.stream, units=(len(cts) * (2 * limbs - 1) * 2 * self.N * 8.0, 0.0)),
                       "rescale")
            cur, pm, limbs = out, po, limbs - 1
            scales = [s / ql for s in scales]
        return self._wrap_batch(cur, level - drops, scales)

    def mult_plain(self, ct: CipherVec, p: PlainVec) -> CipherVec:
        self._check(ct)
        v = self._check_plain(p)
        cost = self.context.mult_level_cost
        if ct.level < cost:
            raise LevelExhausted(f"level {ct.level} < multiplication cost {cost}")
        self._acct.bump("plain_mults")
        if np.all(v == v[0]):
            return self.mul_const_batch([ct], [float(v[0])], count=False)[0]
        torch = _torch()
        limbs = ct.level + 1
        ql = self.moduli[limbs - 1]
        pt = torch.empty((limbs, self.N), dtype=torch.int64, device=self.device)
        vv = torch.as_tensor(v, device=self.device)
        _lib.check(self._L.he_encode_plain(self._h, vv.data_ptr(), self.context.n, float(ql), limbs, pt.data_ptr(),
                                           self.stream), "encode_plain")
        nc = ct.data.shape[0]
        tmp = self._alloc(1, nc, limbs)
        pi, pt_, pm = self._ptrs([ct]), pt.data_ptr(), self._tptrs(tmp)
        _lib.check(self._L.he_mul_plain(self._h, _lib.addr(pi), pt_, _lib.addr(pm), 1, limbs, nc, self.stream))
        return self._rescale_tensor(tmp, limbs, [ct.scale])[0]

    def mul_const_batch(self, cts: Sequence[CipherVec], values: Sequence[float], count: bool = True,
                        out_scales: Sequence[float] | None = None) -> list[CipherVec]:
        """ct_i * values[i] then rescale (one level).  The constant is encoded at
        q_last * out_scale / in_scale so the result lands exactly on out_scale
        (default: the input scale)."""
        for c in cts:
            self._check(c)
        level = cts[0].level
        if any(c.level != level for c in cts):
            raise HebatchError("mul_const_batch needs equal levels")
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        if count:
            self._acct.bump("plain_mults", len(cts))
        limbs = level + 1
        ql = self.moduli[limbs - 1]
        outs = list(out_scales) if out_scales is not None else [c.scale for c in cts]
        res = np.array([self._res(int(np.rint(v * ql * (o / c.scale))), limbs) for v, c, o in zip(values, cts, outs)],
                       np.uint64)
        nc = self._ncomp(cts)
        tmp = self._alloc(len(cts), nc, limbs)
        pi, pm = self._ptrs(cts), self._tptrs(tmp)
        _lib.check(self._L.he_mul_const(self._h, _lib.addr(pi), _lib.addr(pm), len(cts), limbs, nc, _lib.addr(res),
                                        self.stream), "mul_const")
        return self._rescale_tensor(tmp, limbs, outs)

    def _mul_monomial_batch(self, cts: Sequence[CipherVec], power: int) -> list[CipherVec]:
        """ct_i * X^power (exact, no rescale, no level): an element-wise product
        with the NTT of the monomial (X^n multiplies every slot by i)."""
        torch = _torch()
        level = cts[0].level
        limbs = level + 1
        key = (power % (2 * self.N), limbs)
        cache = self.__dict__.setdefault("_mono", {})
        if key not in cache:
            e = torch.zeros((limbs, self.N), dtype=torch.int64, device=self.device)
            p = power % (2 * self.N)
            for l in range(limbs):
                e[l, p % self.N] = 1 if p < self.N else self.moduli[l] - 1  # X^N = -1
            _lib.check(self._L.he_ntt(self._h, e.data_ptr(), 1, limbs, 0, self.stream), "monomial ntt")
            cache[key] = e
        pt = cache[key]
        nc = self._ncomp(cts)
        out = self._alloc(len(cts), nc, limbs)
        pi, po = self._ptrs(cts), self._tptrs(out)
        _lib.check(self._L.he_mul_plain(self._h, _lib.addr(pi), pt.data_ptr(), _lib.addr(po), len(cts), limbs, nc,
                                        self.stream), "mul_monomial")
        return self._wrap_batch(out, level, [c.scale for c in cts])

    def _mul_int_batch(self, cts: Sequence[CipherVec], ks: Sequence[int], out_scales: Sequence[float]) -> list[CipherVec]:
        """ct_i * ks[i] (an exact integer constant) then rescale; declared scales out_scales (no counters)."""
        level = cts[0].level
        limbs = level + 1
        res = np.array([self._res(int(k), limbs) for k in ks], np.uint64)
        nc = self._ncomp(cts)
        tmp = self._alloc(len(cts), nc, limbs)
        pi, pm = self._ptrs(cts), self._tptrs(tmp)
        _lib.check(self._L.he_mul_const(self._h, _lib.addr(pi), _lib.addr(pm), len(cts), limbs, nc, _lib.addr(res),
                                        self.stream), "mul_const")
        return self._rescale_tensor(tmp, limbs, list(out_scales))

    def rescale_batch(self, cts: Sequence[CipherVec], out_scale: float | None = None) -> list[CipherVec]:
        """Divide-and-round by the last prime (one level); the declared output
        scale is ``out_scale`` when given (callers that encoded weights for an
        exact target scale), else scale / q_last."""
        for c in cts:
            self._check(c)
        level = cts[0].level
        if any(c.level != level for c in cts) or level < 1:
            raise LevelExhausted("rescale_batch needs equal levels >= 1")
        limbs = level + 1
        nc = self._ncomp(cts)
        out = self._alloc(len(cts), nc, limbs - 1)
        pi, po = self._ptrs(cts), self._tptrs(out)
        _lib.check(self._call("rescale", self._L.he_rescale, self._h, _lib.addr(pi), _lib.addr(po), len(cts), limbs,
                              nc, self.stream, units=(len(cts) * (2 * limbs - 1) * nc * self.N * 8.0, 0.0)),
                   "rescale")
        ql = self.moduli[limbs - 1]
        return self._wrap_batch(out, level - 1, [out_scale if out_scale is not None else c.scale / ql for c in cts])

    def pack_batch(self, cts: Sequence[CipherVec]):
        """Ciphertexts of one level and scale -> (int64 tensor [k, n_comp, limbs, N], level, scale):
        the payload a collective moves between ranks (sharded_cnn)."""
        torch = _torch()
        level, scale = cts[0].level, cts[0].scale
        if any(c.level != level or c.scale != scale for c in cts):
            raise HebatchError("pack_batch needs one level and one scale")
        return torch.stack([c.data for c in cts]), level, scale

    def unpack_batch(self, t, level: int, scale: float) -> list[CipherVec]:
        """Inverse of pack_batch: fresh handles over the rows of ``t`` (owned by the engine)."""
        return self._wrap_batch(t, level, [scale] * t.shape[0])

    def _rescale_tensor(self, t, limbs: int, scales) -> list[CipherVec]:
        nc = t.shape[1]
        out = self._alloc(t.shape[0], nc, limbs - 1)
        pi, po = self._tptrs(t), self._tptrs(out)
        _lib.check(self._L.he_rescale(self._h, _lib.addr(pi), _lib.addr(po), t.shape[0], limbs, nc, self.stream),
                   "rescale")
        return self._wrap_batch(out, limbs - 2, scales)

    def mult_ct(self, a: CipherVec, b: CipherVec) -> CipherVec:
        self._check(a)
        self._check(b)
        cost = self.context.mult_level_cost
        if a.level < cost or b.level < cost:
            raise LevelExhausted(f"levels ({a.level}, {b.level}) < multiplication cost {cost}")
        self._acct.bump("ct_mults")
        return self._mult_ct_batch([a], [b])[0]

    def mult_ct_batch(self, A: Sequence[CipherVec], B: Sequence[CipherVec]) -> list[CipherVec]:
        for c in list(A) + list(B):
            self._check(c)
        if any(c.level < self.context.mult_level_cost for c in list(A) + list(B)):
            raise LevelExhausted("operand level below multiplication cost")
        self._acct.bump("ct_mults", len(A))
        return self._mult_ct_batch(A, B)

    def _ensure_relin(self) -> None:
        if not self._relin:
            _lib.check(self._L.he_gen_switch_key(self._h, 0, self.stream), "relin keygen")
            self._relin = True

    def _ensure_power_keys(self) -> None:
        """s^3 and s^4 switching keys (codes 2, 4) for 5-component relinearisation."""
        for code in (2, 4):
            if not self._L.he_has_switch_key(self._h, code):
                _lib.check(self._L.he_gen_switch_key(self._h, code, self.stream), "power keygen")

    def _mult_ct_batch(self, A, B) -> list[CipherVec]:
        self._ensure_relin()
        level = min(min(c.level for c in A), min(c.level for c in B))
        limbs = level + 1
        ta, tb = self._at_level(A, level), self._at_level(B, level)
        out = self._alloc(len(A), 2, limbs - 1)
        pa = _lib.ptr_array([t.data_ptr() for t in ta])
        pb = _lib.ptr_array([t.data_ptr() for t in tb])
        po = self._tptrs(out)
        _lib.check(self._call("mult_ct", self._L.he_mult_ct, self._h, _lib.addr(pa), _lib.addr(pb), _lib.addr(po),
                              len(A), limbs, self.stream, units=(len(A) * 6.0 * limbs * self.N * 8, 0.0)), "mult_ct")
        ql = self.moduli[limbs - 1]
        return self._wrap_batch(out, level - 1, [a.scale * b.scale / ql for a, b in zip(A, B)])

    def drop_level_batch(self, cts: Sequence[CipherVec], level: int) -> list[CipherVec]:
        """Discard limbs down to ``level`` (no rescale, scale unchanged)."""
        for c in cts:
            self._check(c)
            if c.level < level:
                raise LevelExhausted(f"cannot raise level {c.level} to {level}")
        out = self._alloc(len(cts), self._ncomp(cts), level + 1)
        for i, c in enumerate(cts):
            out[i].copy_(c.data[:, : level + 1])
        return self._wrap_batch(out, level, [c.scale for c in cts])

    def boot_plan(self):
        """The bootstrap circuit's parameters for this ring (bootstrap.BootPlan)."""
        from .bootstrap import BootPlan

        if getattr(self, "_bplan", None) is None:
            self._bplan = BootPlan(N=self.N, q0=self.moduli[0], hamming=self.context.secret_hamming)
        return self._bplan

    def _ensure_boot_keys(self, plan) -> None:
        self._ensure_relin()
        gs = [pow(5, k, 2 * self.N) for k in plan.rotation_offsets()] + [2 * self.N - 1]
        for g in gs:
            if not self._L.he_has_switch_key(self._h, g):
                _lib.check(self._L.he_gen_switch_key(self._h, g, self.stream), "bootstrap keygen")

    def bootstrap(self, ct: CipherVec) -> CipherVec:
        """Real CKKS bootstrapping (bootstrap.py: ModRaise, CoeffToSlot, EvalMod,
        SlotToCoeff) with the reference's contract (engine.py:315-319): the
        result holds the same slots (up to the circuit's approximation error,
        ~2e-5 with q_0 / scale = 2^10 and a 2^50 scale) at level
        max_level - bootstrap_reserve, and only the ``bootstraps`` counter
        moves.  The circuit needs bootstrap_reserve >= its depth
        (BootPlan.depth: 20 at N = 2^12 with the dense secret); its Galois keys
        (BSGS steps of the factored DFT and conjugation) are generated on
        first use."""
        return self.bootstrap_batch([ct])[0]

    def bootstrap_batch(self, cts: Sequence[CipherVec]) -> list[CipherVec]:
        """bootstrap() for several ciphertexts at once: every step of the circuit
        is one batched launch sequence for the whole batch (inputs of one level
        and scale).  Counts one bootstrap per ciphertext."""
        from .bootstrap import Bootstrapper, GpuBootOps

        cts = list(cts)
        if not cts:
            return []
        for c in cts:
            self._check(c)
        self._need_two(cts, "bootstrap")
        if len({(c.level, c.scale) for c in cts}) != 1:
            raise HebatchError("bootstrap_batch needs ciphertexts of one level and scale")
        plan = self.boot_plan()
        target = self.context.max_level - self.context.bootstrap_reserve
        if self.context.max_level - plan.depth < target:
            raise HebatchError(f"bootstrap_reserve {self.context.bootstrap_reserve} is below the bootstrap circuit's "
                               f"depth {plan.depth}")
        self._ensure_boot_keys(plan)
        s_in = cts[0].scale
        booters = self.__dict__.setdefault("_booters", {})  # per input scale (SlotToCoeff folds 1 / scale)
        if s_in not in booters:
            if len(booters) >= 4:
                booters.pop(next(iter(booters)))
            booters[s_in] = Bootstrapper(GpuBootOps(self), plan, s_in)
        with self._acct.lock:
            saved = (dict(self._acct.counts), self._acct.peak, self._acct.window_peak, set(self._acct.live))
        out = booters[s_in].run(cts, self.context.n_q)
        if out[0].level > target:
            out = self.drop_level_batch(out, target)
        with self._acct.lock:  # circuit temporaries are not user-visible ciphertexts
            counts, peak, wpeak, live = saved
            self._acct.counts = counts
            self._acct.live = live | {o.id for o in out}
            self._acct.peak = max(peak, len(self._acct.live))
            self._acct.window_peak = max(wpeak, len(self._acct.live))
        self._acct.bump("bootstraps", len(out))
        return out

    def ensure_level(self, ct: CipherVec, needed: int) -> CipherVec:
        if ct.level >= needed:
            return ct
        fresh = self.bootstrap(ct)
        self.release(ct)
        return fresh

    # ------------------------------------------------------------ feature-major linear layer
    def lincomb(self, inputs: Sequence[CipherVec], row_ptr, col, weights, bias=None,
                out_scale: float | None = None, count_as_conv: bool = True) -> list[CipherVec]:
        """out[o] = sum_t weights[t] * inputs[col[t]] (+ bias[o]), then rescale.

        The batched form of conv_forward's k=1 fold loop (conv.py:137-166) and
        of feature-major conv / pool / dense.  Each real weight is encoded as
        the integer round(w * q_last * out_scale / scale(input)), so the output
        scale after the rescale is exactly ``out_scale`` (default: the scale of
        inputs[0]) even when the inputs' scales differ.  Counters advance as
        the reference loop would: one plain_mult and one add per term.
        """
        for c in inputs:
            self._check(c)
        level = min(c.level for c in inputs)
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        limbs = level + 1
        row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        w = np.asarray(weights, np.float64)
        n_out = len(row_ptr) - 1
        ql = self.moduli[limbs - 1]
        s_out = float(out_scale) if out_scale is not None else inputs[0].scale
        in_scale = np.array([c.scale for c in inputs], np.float64)
        wf = w * (ql * s_out) / in_scale[col]
        if np.any(np.abs(wf) >= 2.0 ** 62):
            raise HebatchError("lincomb weight too large for the int64 encoding (|w * q| >= 2^62)")
        wi = np.rint(wf).astype(np.int64)
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        acc = self._alloc(n_out, 2, limbs)
        pacc = self._tptrs(acc)
        n_used = len(np.unique(col))
        poly = 2 * limbs * self.N
        _lib.check(self._call("lincomb", self._L.he_lincomb, self._h, _lib.addr(pin), len(inputs), _lib.addr(pacc),
                              n_out, _lib.addr(row_ptr), _lib.addr(col), _lib.addr(wi), limbs, 2, self.stream,
                              units=((n_used + n_out) * poly * 8.0, float(len(col)) * poly)), "lincomb")
        out = self._alloc(n_out, 2, limbs - 1)
        pout = self._tptrs(out)
        _lib.check(self._call("rescale", self._L.he_rescale, self._h, _lib.addr(pacc), _lib.addr(pout), n_out, limbs,
                              2, self.stream, units=(n_out * (2 * limbs - 1) * 2 * self.N * 8.0, 0.0)), "rescale")
        del acc
        if bias is not None and np.any(np.asarray(bias) != 0):  # adding zero residues is a no-op
            b = np.asarray(bias, np.float64)
            res = np.array([self._res(int(np.rint(bv * s_out)), limbs - 1) for bv in b], np.uint64)
            _lib.check(self._call("add_const", self._L.he_add_const, self._h, _lib.addr(pout), _lib.addr(pout), n_out,
                                  limbs - 1, 2, _lib.addr(res), self.stream,
                                  units=(n_out * 2.0 * (limbs - 1) * self.N * 8, 0.0)), "bias")
        if count_as_conv:
            self._acct.bump("plain_mults", int(len(col)))
            self._acct.bump("adds", int(len(col)))
        return self._wrap_batch(out, level - 1, [s_out] * n_out)

    def lincomb_grouped(self, inputs: Sequence[CipherVec], term_ptr, term_col, term_tap, out_base, out_stride: int,
                        weights, n_out: int, bias=None, out_scale: float | None = None,
                        weight_scale: float | None = None, skip_rescale: bool = False) -> list[CipherVec]:
        """Grouped linear combination (he_lincomb_grouped) + rescale + bias.

        ``skip_rescale`` keeps the ordinary weight encoding round(w q_l s_out /
        s_in) but returns the exact sums before the rescale (and without the
        bias), at declared scale q_l * s_out: partial sums over input-channel
        blocks that are added and then rescaled once (rescale_batch with
        out_scale=s_out) equal the unsplit call bit for bit (sharded_cnn).

        Group g (an output pixel) gathers inputs col[t] (t in its term range)
        and produces M = weights.shape[0] outputs
        out[out_base[g] + m * out_stride] = sum_t weights[m, tap[t]] * in[col[t]].
        All inputs must share one scale; weights are encoded like lincomb().

        With ``weight_scale`` the rescale is DEFERRED: weights are encoded as
        round(w * weight_scale), nothing is rescaled, and the outputs keep the
        input level at scale s_in * weight_scale (the caller drops the extra
        prime later -- run_cnn does it after the activation's relinearisation).
        """
        for c in inputs:
            self._check(c)
        s_in = inputs[0].scale
        if any(abs(c.scale / s_in - 1.0) > 0 for c in inputs):
            raise ScaleMismatch("lincomb_grouped needs inputs at one scale")
        level = min(c.level for c in inputs)
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        limbs = level + 1
        w = np.asarray(weights, np.float64)
        M, T = w.shape
        ql = self.moduli[limbs - 1]
        deferred = weight_scale is not None
        if deferred:
            s_out = s_in * float(weight_scale)
            wf = w * float(weight_scale)
        else:
            s_out = float(out_scale) if out_scale is not None else s_in
            wf = w * (ql * s_out) / s_in
        if np.any(np.abs(wf) >= 2.0 ** 62):
            raise HebatchError("lincomb weight too large for the int64 encoding (|w * q| >= 2^62)")
        wi = np.ascontiguousarray(np.rint(wf).astype(np.int64))
        tp = np.ascontiguousarray(term_ptr, np.int32)
        tc = np.ascontiguousarray(term_col, np.int32)
        tt = np.ascontiguousarray(term_tap, np.int32)
        ob = np.ascontiguousarray(out_base, np.int32)
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        acc = self._alloc(n_out, 2, limbs)
        pacc = self._tptrs(acc)
        poly = 2 * limbs * self.N
        n_used = len(np.unique(tc))
        # bias: one value per output channel m; zero residues are a no-op
        b = None if bias is None else np.asarray(bias, np.float64).reshape(M)
        has_bias = b is not None and bool(np.any(b != 0))
        out_limbs = limbs if deferred else limbs - 1
        ch_res = (np.array([self._res(int(np.rint(bv * s_out)), out_limbs) for bv in b], np.uint64)
                  if has_bias else None)
        fused_res = ch_res if (deferred and has_bias) else None     # added inside the lincomb store
        _lib.check(self._call("lincomb", self._L.he_lincomb_grouped, self._h, _lib.addr(pin), len(inputs),
                              _lib.addr(pacc), n_out, len(ob), _lib.addr(tp), _lib.addr(tc), _lib.addr(tt),
                              _lib.addr(ob), int(out_stride), M, T, _lib.addr(wi),
                              _lib.addr(fused_res) if fused_res is not None else None, limbs, 2, self.stream,
                              units=((n_used + n_out) * poly * 8.0, float(len(tc)) * M * poly)), "lincomb_grouped")
        if skip_rescale:
            if deferred or has_bias:
                raise HebatchError("skip_rescale excludes weight_scale and bias (add the bias after rescale_batch)")
            self._acct.bump("plain_mults", int(len(tc)) * M)
            self._acct.bump("adds", int(len(tc)) * M)
            return self._wrap_batch(acc, limbs - 1, [ql * s_out] * n_out)
        if deferred:
            out, pout = acc, pacc
        else:
            out = self._alloc(n_out, 2, limbs - 1)
            pout = self._tptrs(out)
            _lib.check(self._call("rescale", self._L.he_rescale, self._h, _lib.addr(pacc), _lib.addr(pout), n_out,
                                  limbs, 2, self.stream, units=(n_out * (2 * limbs - 1) * 2 * self.N * 8.0, 0.0)),
                       "rescale")
            del acc
            if has_bias:  # after the rescale, at the output scale
                res = np.zeros((n_out, out_limbs), np.uint64)
                for m in range(M):
                    res[ob + m * int(out_stride)] = ch_res[m]
                _lib.check(self._call("add_const", self._L.he_add_const, self._h, _lib.addr(pout), _lib.addr(pout),
                                      n_out, out_limbs, 2, _lib.addr(res), self.stream,
                                      units=(n_out * 2.0 * out_limbs * self.N * 8, 0.0)), "bias")
        self._acct.bump("plain_mults", int(len(tc)) * M)
        self._acct.bump("adds", int(len(tc)) * M)
        return self._wrap_batch(out, out_limbs - 1, [s_out] * n_out)

    # plaintext bytes one he_lincomb_plain launch may hold (larger folds are split over outputs)
    PLAIN_CHUNK_BYTES = 4 << 30

    def lincomb_plain(self, inputs: Sequence[CipherVec], plains, n_out: int, pt_scale: float = 1.0) -> list[CipherVec]:
        """The batched channel-by-channel fold (conv.py:137-156 as one kernel):
        out[o] = rescale(sum_j inputs[j] (.) encode(plains[o, j], q_last)) for
        full-width float64 plaintext slot vectors plains [n_out][n_in][<= n].
        Every plaintext is encoded at q_last exactly as mult_plain encodes it
        (he_encode_plain_batch), the products are summed exactly
        (he_lincomb_plain) and each output is rescaled ONCE, so the output
        scale is the input scale and the level drops by one, as for the
        reference's per-term mult_plain + add fold.  Counters are the caller's.
        ``pt_scale`` != 1 encodes the plaintexts at q_last * pt_scale (more
        precision for small plaintext values) and declares the outputs at
        scale(input) * pt_scale."""
        torch = _torch()
        for c in inputs:
            self._check(c)
        self._need_two(inputs, "lincomb_plain")
        n_in = len(inputs)
        level, s_in = inputs[0].level, inputs[0].scale
        if any(c.level != level or c.scale != s_in for c in inputs):
            raise HebatchError("lincomb_plain needs inputs at one level and scale")
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        if not isinstance(plains, torch.Tensor):
            plains = np.asarray(plains)
        cplx = plains.is_complex() if isinstance(plains, torch.Tensor) else np.iscomplexobj(plains)
        P = torch.as_tensor(plains, dtype=torch.complex128 if cplx else torch.float64, device=self.device)
        if P.dim() != 3 or P.shape[0] != n_out or P.shape[1] != n_in or P.shape[2] > self.context.n:
            raise ShapeMismatch(f"plains {tuple(P.shape)} for {n_out} outputs x {n_in} inputs x <= {self.context.n}")
        limbs = level + 1
        ql = float(self.moduli[limbs - 1]) * pt_scale
        pin = self._ptrs(inputs)
        acc = self._alloc(n_out, 2, limbs)
        per_out = n_in * limbs * self.N * 8
        step = max(1, min(n_out, self.PLAIN_CHUNK_BYTES // per_out))
        for o0 in range(0, n_out, step):
            o1 = min(n_out, o0 + step)
            vals = P[o0:o1].reshape((o1 - o0) * n_in, P.shape[2]).contiguous()
            pt = torch.empty(((o1 - o0) * n_in, limbs, self.N), dtype=torch.int64, device=self.device)
            if cplx:  # complex slot vectors (bootstrap DFT diagonals)
                vr, vi = vals.real.contiguous(), vals.imag.contiguous()
                _lib.check(self._call("encode_plain", self._L.he_encode_plain_batch_c, self._h, vr.data_ptr(),
                                      vi.data_ptr(), vals.shape[0], vals.shape[1], ql, limbs, pt.data_ptr(),
                                      self.stream, units=(vals.numel() * 16.0 + pt.numel() * 8.0, 0.0)),
                           "encode_plain_batch_c")
                del vr, vi
            else:
                _lib.check(self._call("encode_plain", self._L.he_encode_plain_batch, self._h, vals.data_ptr(),
                                      vals.shape[0], vals.shape[1], ql, limbs, pt.data_ptr(), self.stream,
                                      units=(vals.numel() * 8.0 + pt.numel() * 8.0, 0.0)), "encode_plain_batch")
            ppt = self._tptrs(pt)
            pout = _lib.ptr_array([acc.data_ptr() + o * acc.stride(0) * 8 for o in range(o0, o1)])
            poly = 2 * limbs * self.N
            _lib.check(self._call("lincomb_plain", self._L.he_lincomb_plain, self._h, _lib.addr(pin), n_in,
                                  _lib.addr(ppt), _lib.addr(pout), o1 - o0, limbs, self.stream,
                                  units=(((o1 - o0) * n_in * limbs * self.N + (n_in + o1 - o0) * poly) * 8.0,
                                         float((o1 - o0) * n_in) * poly)), "lincomb_plain")
            del pt
        return self._rescale_tensor(acc, limbs, [s_in * pt_scale] * n_out)

    def encode_plains(self, plains, limbs: int, pt_scale: float = 1.0):
        """Slot vectors [count][<= n] (real or complex) -> NTT-domain plaintexts
        [count][limbs][N] at q_last * pt_scale (the encoding lincomb_plain uses)."""
        torch = _torch()
        cplx = np.iscomplexobj(plains)
        P = torch.as_tensor(np.asarray(plains), dtype=torch.complex128 if cplx else torch.float64, device=self.device)
        ql = float(self.moduli[limbs - 1]) * pt_scale
        pt = torch.empty((P.shape[0], limbs, self.N), dtype=torch.int64, device=self.device)
        if cplx:
            vr, vi = P.real.contiguous(), P.imag.contiguous()
            _lib.check(self._call("encode_plain", self._L.he_encode_plain_batch_c, self._h, vr.data_ptr(),
                                  vi.data_ptr(), P.shape[0], P.shape[1], ql, limbs, pt.data_ptr(), self.stream),
                       "encode_plain_batch_c")
        else:
            P = P.contiguous()
            _lib.check(self._call("encode_plain", self._L.he_encode_plain_batch, self._h, P.data_ptr(), P.shape[0],
                                  P.shape[1], ql, limbs, pt.data_ptr(), self.stream), "encode_plain_batch")
        return pt

    def lincomb_plain_encoded(self, inputs: Sequence[CipherVec], pt, n_out: int, pt_scale: float = 1.0):
        """lincomb_plain over plaintexts already encoded by encode_plains (pt
        [n_out * n_in][limbs >= level + 1][N], read at the inputs' level)."""
        for c in inputs:
            self._check(c)
        n_in = len(inputs)
        level, s_in = inputs[0].level, inputs[0].scale
        if any(c.level != level or c.scale != s_in for c in inputs):
            raise HebatchError("lincomb_plain needs inputs at one level and scale")
        limbs = level + 1
        if pt.shape[0] != n_out * n_in or pt.shape[1] != limbs:
            raise ShapeMismatch(f"encoded plaintexts {tuple(pt.shape)} for {n_out} x {n_in} at {limbs} limbs")
        pin = self._ptrs(inputs)
        acc = self._alloc(n_out, 2, limbs)
        ppt = self._tptrs(pt)
        pout = self._tptrs(acc)
        poly = 2 * limbs * self.N
        _lib.check(self._call("lincomb_plain", self._L.he_lincomb_plain, self._h, _lib.addr(pin), n_in,
                              _lib.addr(ppt), _lib.addr(pout), n_out, limbs, self.stream,
                              units=((n_out * n_in * limbs * self.N + (n_in + n_out) * poly) * 8.0,
                                     float(n_out * n_in) * poly)), "lincomb_plain")
        return self._rescale_tensor(acc, limbs, [s_in * pt_scale] * n_out)

    def conv_mma(self, inputs: Sequence[CipherVec], gcol, out_base, out_stride: int, weights, n_out: int,
                 weight_scale: float, bias=None) -> list[CipherVec] | None:
        """Tensor-core (int8-digit, mma.sync) form of a deferred-rescale
        lincomb_grouped with full tap slots: gcol [G][T] input index or -1.
        Weights are encoded as round(w * weight_scale) exactly as in
        lincomb_grouped(weight_scale=...), so the results are bit-identical.
        Returns None when the tensor-core bounds do not hold (caller falls
        back to the CUDA-core kernel)."""
        for c in inputs:
            self._check(c)
        s_in = inputs[0].scale
        if any(c.scale != s_in for c in inputs):
            raise ScaleMismatch("conv_mma needs inputs at one scale")
        level = min(c.level for c in inputs)
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        limbs = level + 1
        w = np.asarray(weights, np.float64)
        M, T = w.shape
        wi = np.ascontiguousarray(np.rint(w * float(weight_scale)).astype(np.int64))
        if np.abs(wi).max(initial=0) >= 2 ** 31:
            return None
        s_out = s_in * float(weight_scale)
        gc = np.ascontiguousarray(gcol, np.int32)
        ob = np.ascontiguousarray(out_base, np.int32)
        b = None if bias is None else np.asarray(bias, np.float64).reshape(M)
        res = (np.array([self._res(int(np.rint(bv * s_out)), limbs) for bv in b], np.uint64)
               if b is not None and np.any(b != 0) else None)
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        out = self._alloc(n_out, 2, limbs)
        pout = self._tptrs(out)
        poly = 2 * limbs * self.N
        nnz = int((gc >= 0).sum())
        rc = self._call("lincomb", self._L.he_conv_mma, self._h, _lib.addr(pin), len(inputs), _lib.addr(pout), n_out,
                        gc.shape[0], _lib.addr(gc), _lib.addr(ob), int(out_stride), M, T, _lib.addr(wi),
                        _lib.addr(res) if res is not None else None, limbs, 2, self.stream,
                        units=((len(np.unique(gc[gc >= 0])) + n_out) * poly * 8.0, float(nnz) * M * poly))
        if rc == _lib.HE_EINVAL:
            return None
        _lib.check(rc, "conv_mma")
        self._acct.bump("plain_mults", nnz * M)
        self._acct.bump("adds", nnz * M)
        return self._wrap_batch(out, level, [s_out] * n_out)

    @staticmethod
    def split_scale_weights(w, mult: float, bits: int = 23):
        """Integer weights of conv_exact_partial: round(w * mult / F) with F = 2^k the
        smallest power of two that brings every |weight| within the 3-signed-digit
        range of the tensor-core kernel (<= 127 (256^3 - 1) / 255 < 2^23).  The
        effective integer weight is W * F (relative precision 2^-23 of the largest)."""
        w = np.asarray(w, np.float64)
        cap = 127 * (256 ** 3 - 1) // 255
        top = float(np.abs(w).max(initial=0.0)) * float(mult)
        k = 0
        while top / (1 << k) > cap - 1:
            k += 1
        wi = np.rint(w * float(mult) / float(1 << k)).astype(np.int64)
        while np.abs(wi).max(initial=0) > cap:
            k += 1
            wi = np.rint(w * float(mult) / float(1 << k)).astype(np.int64)
        return np.ascontiguousarray(wi), 1 << k

    def conv_exact_partial(self, inputs: Sequence[CipherVec], gcol, weights, n_out: int, out_scale: float):
        """Tensor-core form of lincomb_grouped(skip_rescale=True) for config 4's
        standard (rescaled) weight encoding: the exact sums
            out[g + m * G] = sum_t (W[m, t] * F) * in[gcol[g, t]]   mod q
        with (W, F) = split_scale_weights(w, q_l * out_scale / s_in): the int8-digit
        GEMM (he_conv_mma) computes sum W x exactly and one he_mul_const multiplies
        by F.  Declared scale q_l * out_scale, level unchanged (rescale once after
        the partial sums are added).  None when the tensor-core bounds do not hold."""
        for c in inputs:
            self._check(c)
        s_in = inputs[0].scale
        if any(c.scale != s_in for c in inputs):
            raise ScaleMismatch("conv_exact_partial needs inputs at one scale")
        level = min(c.level for c in inputs)
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        limbs = level + 1
        w = np.asarray(weights, np.float64)
        M, T = w.shape
        if M > 32 or self.N % 128:
            return None
        ql = self.moduli[limbs - 1]
        wi, F = self.split_scale_weights(w, ql * float(out_scale) / s_in)
        gc = np.ascontiguousarray(gcol, np.int32)
        G = gc.shape[0]
        ob = np.ascontiguousarray(np.arange(G), np.int32)
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        out = self._alloc(n_out, 2, limbs)
        pout = self._tptrs(out)
        poly = 2 * limbs * self.N
        nnz = int((gc >= 0).sum())
        rc = self._call("lincomb", self._L.he_conv_mma, self._h, _lib.addr(pin), len(inputs), _lib.addr(pout), n_out,
                        G, _lib.addr(gc), _lib.addr(ob), G, M, T, _lib.addr(wi), None, limbs, 2, self.stream,
                        units=((len(np.unique(gc[gc >= 0])) + n_out) * poly * 8.0, float(nnz) * M * poly))
        if rc == _lib.HE_EINVAL:
            return None
        _lib.check(rc, "conv_exact_partial")
        if F != 1:
            res = np.array([self._res(F, limbs)] * n_out, np.uint64)
            _lib.check(self._call("lincomb", self._L.he_mul_const, self._h, _lib.addr(pout), _lib.addr(pout), n_out,
                                  limbs, 2, _lib.addr(res), self.stream, units=(n_out * 2.0 * poly * 8, 0.0)),
                       "conv_exact_partial (x F)")
        self._acct.bump("plain_mults", nnz * M)
        self._acct.bump("adds", nnz * M)
        return self._wrap_batch(out, level, [ql * float(out_scale)] * n_out)

    def conv_square_sum(self, inputs: Sequence[CipherVec], p: int, H: int, W: int, weights, weight_scale: float,
                        bias, const: float, pool: bool, rows=None, scale_mult: float | None = None,
                        planar_out: PlanarCarry | None = None) -> list[CipherVec] | None:
        """Fused deferred-rescale 3x3 conv + lazy degree-2 activation + window
        sum (he_conv_square_sum): equals conv_mma(weight_scale) -> tensor_batch
        -> add_const_batch(const) -> 2x2-pool / GAP unit sum, bit for bit, but
        the conv output map is never written.  inputs: p*H*W ciphertexts
        (channel-major); weights [M][p*9] (already folded); conv output rows
        ``rows`` (a contiguous range, default all).  Returns pool: M*(nr/2)*(W/2)
        outputs indexed (m, r/2, x/2); GAP: M outputs.  3 components (5 when
        the inputs are unrelinearised 3-component squares), scale
        s_out^2 * scale_mult (default 4 for pool, pixel count for GAP).
        None when a tensor-core bound does not hold (caller falls back)."""
        planar_in = isinstance(inputs, PlanarCarry)
        if planar_in:
            if inputs.owner != id(self) or inputs.data is None:
                raise ContextMismatch("planar carry does not belong to this engine (or was released)")
            if (inputs.channels, inputs.H, inputs.W) != (p, H, W):
                raise ShapeMismatch(f"planar carry {inputs.channels}x{inputs.H}x{inputs.W} for {p}x{H}x{W}")
            nci, s_in, level = 3, inputs.scale, inputs.level
        else:
            for c in inputs:
                self._check(c)
            nci = self._ncomp(inputs)
            if nci == 3 and W % 2:
                return None
            s_in = inputs[0].scale
            if any(c.scale != s_in for c in inputs):
                raise ScaleMismatch("conv_square_sum needs inputs at one scale")
            if len(inputs) != p * H * W:
                raise ShapeMismatch(f"{len(inputs)} inputs for {p}x{H}x{W}")
            level = min(c.level for c in inputs)
        if level < self.context.mult_level_cost:
            raise LevelExhausted(f"level {level} < multiplication cost {self.context.mult_level_cost}")
        limbs = level + 1
        rows = list(range(H)) if rows is None else list(rows)
        y0, y1 = rows[0], rows[-1] + 1
        if rows != list(range(y0, y1)):
            raise HebatchError("conv_square_sum needs a contiguous row range")
        w = np.asarray(weights, np.float64)
        M, T = w.shape
        wi = np.ascontiguousarray(np.rint(w * float(weight_scale)).astype(np.int64))
        if M > 32 or T != 9 * p or np.abs(wi).max(initial=0) >= 2 ** 23:
            return None
        s_out = s_in * float(weight_scale)
        b = None if bias is None else np.asarray(bias, np.float64).reshape(M)
        bres = (np.array([self._res(int(np.rint(bv * s_out)), limbs) for bv in b], np.uint64)
                if b is not None and np.any(b != 0) else None)
        npix_win = 4 if pool else (y1 - y0) * W
        C = int(np.rint(const * (s_out * s_out)))
        cres = np.array(self._res(npix_win * C, limbs), np.uint64) if const else None
        nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
        n_out = M * nwin
        nco = 2 * nci - 1
        if planar_out is not None:
            if (planar_out.owner != id(self) or planar_out.level != level or planar_out.channels != M or not pool
                    or (planar_out.H, planar_out.W) != (H // 2, W // 2)):
                raise ShapeMismatch("planar carry output does not match this pooled conv")
            if planar_out.scale is None:
                planar_out.scale = s_out * s_out * (scale_mult if scale_mult is not None else 4.0)
        pin = None if planar_in else _lib.ptr_array([t.data_ptr() for t in self._at_level(inputs, level)])
        out = pout = None
        if planar_out is None:
            out = self._alloc(n_out, nco, limbs)
            pout = self._tptrs(out)
        from .featuremajor import conv3x3_fulltaps

        nnz = int((conv3x3_fulltaps(p, H, W, rows) >= 0).sum())
        poly = limbs * self.N
        # tensor-core work: each modular MAC is nb x E exact int8 products (nb byte
        # planes of the residue: 5 below 2^40, else 8; E signed weight bytes)
        wmax = int(np.abs(wi).max(initial=0))
        E = 1 if wmax < 128 else 2 if wmax < 32768 else 3
        nbs = sum(5 if q < (1 << 40) else 8 for q in self.moduli[:limbs])
        i8 = 1.0 * nci * nnz * M * self.N * nbs * E
        # algorithmic bytes: inputs once (+ the halo rows that exist), outputs once; a planar carry
        # moves 5 bytes per residue instead of 8
        rows_read = min(H, y1 + 1) - max(0, y0 - 1)   # the tile's rows plus the halo inside the image
        in_b = p * rows_read * W * nci * poly * (5.0 if planar_in else 8.0)
        out_b = n_out * nco * poly * (5.0 if planar_out is not None else 8.0)
        args = (self._h, _lib.addr(pin) if pin is not None else None, nci, p, H, W,
                _lib.addr(pout) if pout is not None else None, M, int(bool(pool)), y0, y1, _lib.addr(wi),
                _lib.addr(bres) if bres is not None else None, _lib.addr(cres) if cres is not None else None, limbs)
        # FP64 modular products of the epilogue: one per window / GAP product (3 for 2-component
        # inputs, 6 for 3-component inputs; the recombination runs on the integer pipe)
        fmul = 1.0 * (y1 - y0) * W * M * poly * (nci * (nci + 1) // 2)
        # tensor-pipe cycles of the tcgen05 kernels at the measured standalone cost of their MMAs
        # (tests/test_gpu_tc5.py: 47 cycles for N <= 32, 50 for N = 96, 64 for N = 128); the FP64
        # pipe shares this resource (bench.py roofline.shared_pipe).  One work item = (limb,
        # 8-coefficient chunk[, channel half]); 5 K steps per (16-pixel row step, component)
        items = limbs * (self.N // 8)
        if nci == 2:    # P1: N = 128
            mma_cyc = 1.0 * items * (y1 - y0) * (W // 16) * nci * 5 * 64
        else:           # P16: 5 byte planes x 4 K steps (the very first zero-extended to N = 96) + tap 8 of the
            # plane pairs (0, 1), (2, 3) at N = 48 and of plane 4 at N = 32: 23 MMAs per (row step, component)
            mma_cyc = 1.0 * items * ((M + 15) // 16) * (y1 - y0) * (W // 16) * nci * (50 + 20 * 47 + 2 * 48)
        units = (in_b + out_b, 1.0 * nci * nnz * M * poly, i8, fmul, mma_cyc)
        if planar_in or planar_out is not None:
            rc = self._call("conv_sqsum", self._L.he_conv_square_sum_pl, *args,
                            inputs.data.data_ptr() if planar_in else None,
                            planar_out.data.data_ptr() if planar_out is not None else None, self.stream, units=units)
            _lib.check(rc, "conv_square_sum (planar carry)")
        else:
            rc = self._call("conv_sqsum", self._L.he_conv_square_sum_n, *args, self.stream, units=units)
            if rc == _lib.HE_EINVAL:
                return None
            _lib.check(rc, "conv_square_sum")
        npx = (y1 - y0) * W
        self._acct.bump("plain_mults", nnz * M)
        self._acct.bump("adds", nnz * M)
        self._acct.bump("ct_mults", M * npx)
        self._acct.bump("adds", M * npx + max(0, M * npx - n_out))
        sm = scale_mult if scale_mult is not None else float(npix_win)
        if planar_out is not None:
            return []
        return self._wrap_batch(out, level, [s_out * s_out * sm] * n_out)

    def planar_carry(self, channels: int, H: int, W: int, level: int) -> PlanarCarry:
        """An empty planar carry for `channels` pooled H x W maps at `level`
        (filled by conv_square_sum(planar_out=...); scale set by the first fill)."""
        if channels != 16 or W != 16:
            raise ShapeMismatch("the planar carry holds 16 channels of 16-pixel rows (config 3's conv1 -> conv2)")
        n = (level + 1) * (self.N // 8) * H * W * PlanarCarry.BYTES_PER_PIXEL
        return PlanarCarry(self._alloc_bytes(n), channels, H, W, level, None, id(self))

    def _alloc_bytes(self, n: int):
        """A uint8 device buffer of n bytes through the same slab cache as the
        ciphertext batches (config 3's planar carry is 36 GB per pass)."""
        torch = _torch()
        shape = ("u8", n)
        if n >= self.SLAB_MIN_BYTES:
            for t in self._slab.get(shape, ()):
                if _storage_uses(t) == 2:
                    return t
            self._cap_free_slabs()
        try:
            t = torch.empty(n, dtype=torch.uint8, device=self.device)
        except torch.OutOfMemoryError:
            self._release_pool()
            t = torch.empty(n, dtype=torch.uint8, device=self.device)
        if n >= self.SLAB_MIN_BYTES:
            self._slab.setdefault(shape, []).append(t)
        return t

    def planar_ok(self, p_in: int, H: int, W: int, q: int, q_next: int, level: int) -> bool:
        """Whether run_cnn's carry can go through the planar layout: conv1 on the
        tcgen05 P1 kernel (p_in <= 3, 16 output channels, W % 16 == 0, pooled) feeding
        conv2 on the P16 kernel (16 input channels, 16-pixel rows), primes in (2^40 - 2^25, 2^40)."""
        return (self.use_tensor_cores and self.N == 1 << 16 and p_in <= 3 and q == 16 and W == 32 and H % 2 == 0
                and q_next <= 32 and all((1 << 40) - (1 << 25) < m < (1 << 40) for m in self.moduli[:level + 1]))

    def unpack_planar(self, pc: PlanarCarry) -> list[CipherVec]:
        """The planar carry as channel-major 3-component ciphertexts (tests, tracing)."""
        n = pc.channels * pc.H * pc.W
        out = self._alloc(n, 3, pc.limbs)
        po = self._tptrs(out)
        _lib.check(self._L.he_planar_unpack(self._h, pc.data.data_ptr(), pc.channels, pc.H, pc.W, pc.limbs,
                                            _lib.addr(po), self.stream), "planar_unpack")
        return self._wrap_batch(out, pc.level, [pc.scale] * n)

    def lincomb_int(self, inputs: Sequence[CipherVec], row_ptr, col, int_weights, out_scale: float,
                    count_adds: bool = True) -> list[CipherVec]:
        """out[o] = sum_t int_weights[t] * inputs[col[t]] with NO rescale (level kept).

        Used for average pooling / global average pooling: with unit weights
        the sum of k ciphertexts at scale s encodes the mean at scale k*s,
        so the 1/k factor costs no level (it is folded into the next layer's
        weight encoding).  ``out_scale`` is the scale the caller declares.
        """
        for c in inputs:
            self._check(c)
        level = min(c.level for c in inputs)
        limbs = level + 1
        row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        wi = np.ascontiguousarray(int_weights, np.int64)
        n_out = len(row_ptr) - 1
        nc = self._ncomp(inputs)
        tins = self._at_level(inputs, level)
        pin = _lib.ptr_array([t.data_ptr() for t in tins])
        out = self._alloc(n_out, nc, limbs)
        pout = self._tptrs(out)
        poly = nc * limbs * self.N
        _lib.check(self._call("lincomb_int", self._L.he_lincomb, self._h, _lib.addr(pin), len(inputs),
                              _lib.addr(pout), n_out, _lib.addr(row_ptr), _lib.addr(col), _lib.addr(wi), limbs, nc,
                              self.stream, units=((len(np.unique(col)) + n_out) * poly * 8.0, float(len(col)) * poly)),
                   "lincomb_int")
        if count_adds:
            self._acct.bump("adds", max(0, int(len(col)) - n_out))
        return self._wrap_batch(out, level, [float(out_scale)] * n_out)

    # ------------------------------------------------------------ keys
    def register_rotation_keys(self, offsets: Iterable[int]) -> None:
        offsets = list(offsets)
        before = self.keys.resident
        added = self.keys.register(offsets)
        for c in sorted(self.keys.resident - before):
            _lib.check(self._L.he_gen_switch_key(self._h, pow(5, c, 2 * self.N), self.stream), "galois keygen")
        if added:
            self._acct.bump("key_loads", added)
        self.registration_log.append(
            frozenset(self.keys.canonical(o) for o in offsets if self.keys.canonical(o) != 0))

    def unload_rotation_keys(self, offsets: Iterable[int]) -> None:
        before = self.keys.resident
        self.keys.unload(offsets)
        for c in sorted(before - self.keys.resident):
            self._L.he_drop_switch_key(self._h, pow(5, c, 2 * self.N))

    def unload_all_rotation_keys(self) -> None:
        before = self.keys.resident
        self.keys.unload_all()
        for c in sorted(before):
            self._L.he_drop_switch_key(self._h, pow(5, c, 2 * self.N))

    @property
    def resident_key_count(self) -> int:
        return len(self.keys)

    # ------------------------------------------------------------ accounting
    def snapshot_counters(self) -> OpCounters:
        return self._acct.snapshot()

    @property
    def live_ciphertexts(self) -> int:
        with self._acct.lock:
            return len(self._acct.live)

    def begin_live_window(self) -> None:
        with self._acct.lock:
            self._acct.window_peak = len(self._acct.live)

    @property
    def window_peak_live(self) -> int:
        with self._acct.lock:
            return self._acct.window_peak

    def synchronize(self) -> None:
        _lib.check(self._L.he_sync(self.stream))

    # ------------------------------------------------------------ plaintext helpers
    def plain(self, values) -> PlainVec:
        values = np.asarray(values, dtype=np.float64).ravel()
        n = self.context.n
        if values.shape[0] > n:
            raise LengthExceedsSlots(f"{values.shape[0]} values > {n} slots")
        slots = np.zeros(n, dtype=np.float64)
        slots[: values.shape[0]] = values
        return PlainVec(slots=slots)

    def constant(self, value: float) -> PlainVec:
        return PlainVec(slots=np.full(self.context.n, float(value)))


__all__ = [
    "CipherVec",
    "EngineContext",
    "GpuEngine",
    "OpCounters",
    "PlainVec",
    "RotationKeySet",
    "VectorEngine",
]
