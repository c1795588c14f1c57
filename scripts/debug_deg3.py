"""Layer-by-layer decrypt check of the non-lazy degree-3 CNN plan (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import engine_context  # noqa: E402
from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402
from paper_2604_16834_b200.featuremajor import Activation, CnnSpec, apply_activation, fm_conv3x3  # noqa: E402
from paper_2604_16834_b200.packing import pack_features  # noqa: E402

spec = CnnSpec(channels=(3, 4, 4), H=8, W=8, act=Activation((0.5, 0.5, 0.0, 0.0625)), pool_after=(0, 1))
wts = spec.make_weights(5)
eng = GpuEngine(engine_context(sys.argv[1] if len(sys.argv) > 1 else "cfg4s", seed=3))
n = eng.context.n
rng = np.random.default_rng(2)
images = rng.uniform(0.0, 1.0, size=(n, 3 * 64))
x = pack_features(eng, images)
print("moduli bits", [int(q).bit_length() for q in eng.moduli], "scale", eng.context.scale)
a, b = spec.act.fold()
w, bias = wts.convs[0]
y = fm_conv3x3(eng, x, w, bias, 8, 8, fold=(a, b))
img = images.reshape(n, 3, 8, 8)
xp = np.pad(img, ((0, 0), (0, 0), (1, 1), (1, 1)))
ref = np.zeros((n, 4, 8, 8))
for dy in range(3):
    for dx in range(3):
        ref += np.einsum("oi,sihw->sohw", w[:, :, dy, dx], xp[:, :, dy:dy + 8, dx:dx + 8])
ref = a * ref + b
got = np.stack(eng.decrypt_batch(y[:4])).T
print("conv1 (folded) err", np.max(np.abs(got - ref[:, 0].reshape(n, 64)[:, :4])), "level", y[0].level, "scale", y[0].scale)
z = apply_activation(eng, y[:4], spec.act, lazy=False)
act = spec.act(ref[:, 0].reshape(n, 64)[:, :4] / a - b / a) if False else None
c0, c1, c2, c3 = spec.act.coeffs
yr = ref[:, 0].reshape(n, 64)[:, :4]
t = a * 0 + yr  # y already folded
refz = yr * (yr ** 2 + c1 / np.cbrt(c3)) + c0
gz = np.stack(eng.decrypt_batch(z)).T
print("act1 err", np.max(np.abs(gz - refz)), "level", z[0].level, "scale", z[0].scale, "max|ref|", np.max(np.abs(refz)))
