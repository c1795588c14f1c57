"""Client/server over the wire format (paper threat model):
the client (secret key) exports ciphertexts and evaluation keys; a server
engine created WITHOUT the client's secret key (different key seed) imports
them, evaluates mult_ct and rotations, and returns ciphertexts the client
decrypts.  The imported keys are bit-identical to the client's, so the
server's results equal the client computing locally, limb for limb."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import engine_context, to_np

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg3"])
def test_wire_client_server_roundtrip(name):
    import torch

    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.errors import ContextMismatch, HebatchError
    from paper_2604_16834_b200.wire import export_ciphertexts, export_eval_keys, import_ciphertexts, import_eval_keys

    client = GpuEngine(engine_context(name, seed=11))
    server = GpuEngine(engine_context(name, seed=99))
    n = client.context.n
    client._ensure_relin()
    client.register_rotation_keys([1, 5])
    keys = export_eval_keys(client)
    bits = sum((q.bit_length() + 7) // 8 for q in client.moduli)
    assert len(keys) > client._dnum * 2 * client.N * bits * 3            # relin + 2 Galois keys, packed
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (2, n))
    cts = client.encrypt_batch(x)
    blob = export_ciphertexts(client, cts)
    full = 2 * 2 * client.context.n_q * client.N * 8
    assert len(blob) < full                                                  # 5/6-byte residues, not 8
    codes = import_eval_keys(server, keys)
    assert 0 in codes and server.keys.holds(1) and server.keys.holds(5)
    sc = import_ciphertexts(server, blob)
    for a, b in zip(sc, cts):
        assert np.array_equal(to_np(a.data), to_np(b.data)) and a.scale == b.scale and a.level == b.level
    m, r = server.mult_ct(sc[0], sc[1]), server.rotate(sc[0], 5)
    back = import_ciphertexts(client, export_ciphertexts(server, [m, r][:1]))
    back_r = import_ciphertexts(client, export_ciphertexts(server, [r]))
    assert np.array_equal(to_np(back[0].data), to_np(client.mult_ct(cts[0], cts[1]).data))
    assert np.array_equal(to_np(back_r[0].data), to_np(client.rotate(cts[0], 5).data))
    assert np.max(np.abs(client.decrypt(back[0]) - x[0] * x[1])) < 1e-5
    assert np.max(np.abs(client.decrypt(back_r[0]) - np.roll(x[0], -5))) < 1e-5
    # the server cannot decrypt: its own secret key is not the client's
    assert np.max(np.abs(server.decrypt(sc[0]) - x[0])) > 1.0
    # wrong parameters / corrupted payloads are refused
    other = GpuEngine(engine_context("cfg1" if name == "cfg3" else "cfg3", seed=1))
    with pytest.raises(ContextMismatch):
        import_ciphertexts(other, blob)
    bad = bytearray(blob)
    w = (client.moduli[client.context.n_q - 1].bit_length() + 7) // 8
    bad[-w:] = b"\xff" * w                                                  # last residue := 2^(8w) - 1 >= q
    with pytest.raises(HebatchError):
        import_ciphertexts(server, bytes(bad))
    torch.cuda.synchronize()
