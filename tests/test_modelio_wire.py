"""model-io and the wire format's host logic (CPU)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2604_16834_b200 import modelio as MI
from paper_2604_16834_b200.errors import NonFiniteValue, NonPositiveVariance, ParseError, ShapeMismatch


def test_tensor_csv_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    w = rng.normal(size=(2, 3, 3, 3))
    p = tmp_path / "conv0.weight.csv"
    MI.write_tensor_csv(str(p), w)
    assert p.read_text().splitlines()[0] == "shape: 2 3 3 3"
    assert np.array_equal(MI.load_tensor_csv(str(p)), w)          # lossless (repr: 17 digits)
    k = tmp_path / "k.csv"
    k.write_text("shape: 1 1 3 3\n" + ",".join(str(i) for i in range(9)) + "\n")
    assert MI.load_tensor_csv(str(k)).shape == (1, 1, 3, 3)       # 9 cells -> 3x3 kernel
    bad = tmp_path / "bad.csv"
    bad.write_text("shape: 2 3 3 3\n" + ",".join("1" for _ in range(53)) + "\n")
    with pytest.raises(ShapeMismatch):
        MI.load_tensor_csv(str(bad))
    bad.write_text("dims: 2\n1,2\n")
    with pytest.raises(ParseError):
        MI.load_tensor_csv(str(bad))
    bad.write_text("shape: 2\n1,x\n")
    with pytest.raises(ParseError):
        MI.load_tensor_csv(str(bad))
    bad.write_text("shape: 2\n1,nan\n")
    with pytest.raises(NonFiniteValue):
        MI.load_tensor_csv(str(bad))


def test_fold_batch_norm_spec_examples():
    eps = 1e-5
    W, b = np.array([[1.5, -2.0]]), np.array([0.25])
    W2, b2 = MI.fold_batch_norm(W, b, [1.0], [0.0], [0.0], [1.0 - eps], eps)    # identity normalisation
    assert np.allclose(W2, W) and np.allclose(b2, b)
    W2, b2 = MI.fold_batch_norm(np.array([[2.0]]), [0.0], [2.0], [1.0], [3.0], [4.0 - eps], eps)
    assert np.allclose(W2, [[2.0]]) and np.allclose(b2, [-2.0])                 # SPEC worked example
    rng = np.random.default_rng(1)
    q, p, H, Wd = 4, 3, 5, 5
    w, bias = rng.normal(size=(q, p, 3, 3)), rng.normal(size=q)
    g, be, mu, var = rng.uniform(0.5, 2, q), rng.normal(size=q), rng.normal(size=q), rng.uniform(0.1, 2, q)
    x = rng.normal(size=(p, H, Wd))
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1)))

    def conv(w, b):
        return sum(np.einsum("oi,ihw->ohw", w[:, :, dy, dx], xp[:, dy:dy + H, dx:dx + Wd])
                   for dy in range(3) for dx in range(3)) + b[:, None, None]

    y = conv(w, bias)
    bn = g[:, None, None] * (y - mu[:, None, None]) / np.sqrt(var[:, None, None] + eps) + be[:, None, None]
    wf, bf = MI.fold_batch_norm(w, bias, g, be, mu, var, eps)
    assert np.max(np.abs(conv(wf, bf) - bn)) < 1e-9                               # folding correctness
    with pytest.raises(NonPositiveVariance):
        MI.fold_batch_norm(w, bias, g, be, mu, np.full(q, -1.0), eps)


def test_cnn_weights_dir_roundtrip_with_bn(tmp_path):
    from paper_2604_16834_b200 import configs

    spec = configs.CNN3
    wts = spec.make_weights(4)
    MI.save_cnn_weights(str(tmp_path), wts)
    got = MI.load_cnn_weights(str(tmp_path), spec)
    for (a, b), (c, d) in zip(wts.convs, got.convs):
        assert np.array_equal(a, c) and np.array_equal(b, d)
    assert np.array_equal(got.dense[0], wts.dense[0])
    q = spec.channels[1]
    for name, v in (("gamma", np.full(q, 2.0)), ("beta", np.ones(q)), ("mean", np.zeros(q)),
                    ("var", np.full(q, 4.0 - 1e-5))):
        MI.write_tensor_csv(str(tmp_path / f"conv0.bn.{name}.csv"), v)
    f = MI.load_cnn_weights(str(tmp_path), spec)
    assert np.allclose(f.convs[0][0], wts.convs[0][0]) and np.allclose(f.convs[0][1], 1.0)
    (tmp_path / "conv1.weight.csv").write_text("shape: 1 1 3 3\n" + ",".join("0" for _ in range(9)) + "\n")
    with pytest.raises(ShapeMismatch):
        MI.load_cnn_weights(str(tmp_path), spec)


def test_inputs_and_scores_files(tmp_path):
    rng = np.random.default_rng(2)
    x = rng.uniform(size=(3, 2, 2, 2))
    p = tmp_path / "in.csv"
    p.write_text("\n".join(",".join(repr(float(v)) for v in row) for row in x.reshape(3, -1)) + "\n")
    assert np.array_equal(MI.load_inputs(str(p), (2, 2, 2)), x)
    with pytest.raises(ShapeMismatch):
        MI.load_inputs(str(p), (3, 2, 2))
    s = rng.normal(size=(3, 10))
    MI.write_scores(str(tmp_path / "s.csv"), s)
    assert np.array_equal(np.loadtxt(str(tmp_path / "s.csv"), delimiter=","), s)


def test_wire_residue_packing_roundtrip_cpu():
    """The wire format's byte packing (run on the device in production; torch
    CPU tensors here): limb i keeps ceil(bits(q_i)/8) bytes per residue."""
    import torch

    from paper_2604_16834_b200.wire import _pack, _unpack, _widths

    moduli = [(1 << 40) - 87, (1 << 42) - 11, (1 << 60) - 93]
    assert _widths(moduli) == [5, 6, 8]
    rng = np.random.default_rng(3)
    a = np.stack([rng.integers(0, q, size=(2, 3, 64), dtype=np.uint64) for q in moduli], axis=2)  # [2][3][M][N]
    t = torch.from_numpy(a.view(np.int64))
    blob = _pack(t, _widths(moduli))
    assert len(blob) == 2 * 3 * 64 * (5 + 6 + 8)
    back = _unpack(blob, tuple(t.shape), _widths(moduli), "cpu")
    assert torch.equal(back, t)
