"""Model I/O ("model-io"):
CSV weight tensors, batch-norm folding, input batches and score files.

The paper trains in PyTorch, folds batch norm into the conv kernels and
exports every tensor as CSV.  The SPEC fixes
the layout the paper leaves open: first line ``shape: d1 d2 ...``, then the
values in row-major order, comma separated; one file per tensor, named
``<layer>.<param>.csv``.  Round trips are lossless (17 significant digits).
"""

from __future__ import annotations

import math
import os

import numpy as np

from .errors import NonFiniteValue, NonPositiveVariance, ParseError, ShapeMismatch


def write_tensor_csv(path: str, arr, per_line: int | None = None) -> None:
    a = np.asarray(arr, np.float64)
    if not np.all(np.isfinite(a)):
        raise NonFiniteValue(f"{path}: non-finite value")
    flat = a.reshape(-1)
    per_line = per_line or (a.shape[-1] if a.ndim else 1)
    with open(path, "w") as f:
        f.write("shape: " + " ".join(str(d) for d in a.shape) + "\n")
        for i in range(0, flat.size, max(1, per_line)):
            f.write(",".join(repr(float(v)) for v in flat[i:i + per_line]) + "\n")


def load_tensor_csv(path: str) -> np.ndarray:
    """SPEC load_weights_csv for one file: ShapeMismatch if the cell count differs
    from the header, ParseError on a bad header or cell, NonFiniteValue on NaN/inf."""
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines or not lines[0].startswith("shape:"):
        raise ParseError(f"{path}:1: expected 'shape: d1 d2 ...'")
    try:
        shape = tuple(int(t) for t in lines[0][len("shape:"):].split())
    except ValueError as e:
        raise ParseError(f"{path}:1: bad shape ({e})") from None
    if any(d < 0 for d in shape):
        raise ParseError(f"{path}:1: negative dimension")
    vals = []
    for ln, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        for cell in line.split(","):
            try:
                vals.append(float(cell))
            except ValueError:
                raise ParseError(f"{path}:{ln}: bad cell {cell!r}") from None
    want = int(np.prod(shape)) if shape else 1
    if len(vals) != want:
        raise ShapeMismatch(f"{path}: header {list(shape)} needs {want} cells, found {len(vals)}")
    a = np.asarray(vals, np.float64).reshape(shape)
    if not np.all(np.isfinite(a)):
        raise NonFiniteValue(f"{path}: non-finite value")
    return a


def fold_batch_norm(W, bias, gamma, beta, mean, var, eps: float = 1e-5):
    """SPEC fold_batch_norm: per output channel o, s_o = gamma_o / sqrt(var_o + eps),
    W'[o] = s_o W[o], bias'_o = s_o (bias_o - mean_o) + beta_o."""
    W = np.asarray(W, np.float64)
    q = W.shape[0]
    bias = np.zeros(q) if bias is None else np.asarray(bias, np.float64)
    gamma, beta, mean, var = (np.asarray(v, np.float64).reshape(q) for v in (gamma, beta, mean, var))
    d = var + eps
    if np.any(d <= 0):
        raise NonPositiveVariance(f"var + eps <= 0 for channels {np.nonzero(d <= 0)[0].tolist()}")
    s = gamma / np.sqrt(d)
    return W * s.reshape((q,) + (1,) * (W.ndim - 1)), s * (bias - mean) + beta


def save_cnn_weights(directory: str, wts) -> None:
    """featuremajor.CnnWeights -> conv<k>.weight.csv / conv<k>.bias.csv / fc.weight.csv / fc.bias.csv."""
    os.makedirs(directory, exist_ok=True)
    for k, (w, b) in enumerate(wts.convs):
        write_tensor_csv(os.path.join(directory, f"conv{k}.weight.csv"), w)
        write_tensor_csv(os.path.join(directory, f"conv{k}.bias.csv"), b)
    write_tensor_csv(os.path.join(directory, "fc.weight.csv"), wts.dense[0])
    write_tensor_csv(os.path.join(directory, "fc.bias.csv"), wts.dense[1])


def load_cnn_weights(directory: str, spec, fold_bn: bool = True, eps: float = 1e-5):
    """Load a CnnSpec's weights from ``<layer>.<param>.csv`` files; when
    conv<k>.bn.{gamma,beta,mean,var}.csv exist they are folded into the kernel
    (fold_batch_norm).  A missing conv bias defaults to zero (SPEC open question)."""
    from .featuremajor import CnnWeights

    convs = []
    ch = spec.channels
    for k in range(len(ch) - 1):
        w = load_tensor_csv(os.path.join(directory, f"conv{k}.weight.csv"))
        if w.shape != (ch[k + 1], ch[k], 3, 3):
            raise ShapeMismatch(f"conv{k}.weight: {list(w.shape)} != {[ch[k + 1], ch[k], 3, 3]}")
        bpath = os.path.join(directory, f"conv{k}.bias.csv")
        b = load_tensor_csv(bpath) if os.path.exists(bpath) else np.zeros(ch[k + 1])
        bn = [os.path.join(directory, f"conv{k}.bn.{p}.csv") for p in ("gamma", "beta", "mean", "var")]
        if fold_bn and all(os.path.exists(p) for p in bn):
            w, b = fold_batch_norm(w, b, *(load_tensor_csv(p) for p in bn), eps=eps)
        convs.append((w, b.reshape(ch[k + 1])))
    fw = load_tensor_csv(os.path.join(directory, "fc.weight.csv"))
    fb = load_tensor_csv(os.path.join(directory, "fc.bias.csv"))
    if fw.shape[1] != ch[-1] or fb.shape != (fw.shape[0],):
        raise ShapeMismatch(f"fc: weight {list(fw.shape)} / bias {list(fb.shape)} for {ch[-1]} inputs")
    return CnnWeights(convs=convs, dense=(fw, fb))


def load_inputs(path: str, shape) -> np.ndarray:
    """Input batch CSV: one row per image, channel-major p*H*W values -> [b, p, H, W]."""
    shape = tuple(shape)
    per = int(math.prod(shape))
    rows = []
    with open(path) as f:
        for ln, line in enumerate(f, start=1):
            if not line.strip():
                continue
            try:
                r = [float(c) for c in line.split(",")]
            except ValueError:
                raise ParseError(f"{path}:{ln}: bad cell") from None
            if len(r) != per:
                raise ShapeMismatch(f"{path}:{ln}: {len(r)} values, expected {per} = {'x'.join(map(str, shape))}")
            rows.append(r)
    a = np.asarray(rows, np.float64).reshape((len(rows),) + shape)
    if not np.all(np.isfinite(a)):
        raise NonFiniteValue(f"{path}: non-finite value")
    return a


def write_scores(path: str, scores) -> None:
    """Scores CSV: one row per image (17 significant digits)."""
    s = np.asarray(scores, np.float64)
    with open(path, "w") as f:
        for row in s.reshape(s.shape[0], -1):
            f.write(",".join(repr(float(v)) for v in row) + "\n")
