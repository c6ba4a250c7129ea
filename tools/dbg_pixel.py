"""Debug: trace one pixel of the config-2 step's render (GPU vs oracle)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_fullsize as T  # noqa: E402
from parity import oracle  # noqa: E402


class Req:
    param = int(sys.argv[1])


s = T.step3.__wrapped__(Req())
o = oracle()
W, H = s["cam"].width, s["cam"].height
ot = o.composite(s["pg"], s["off"], s["screen"], W, H)
err = np.abs(s["color"].astype(np.float64) - ot["color"]).max(axis=2)
for y, x in np.argwhere(err > 1e-6):
    print("pixel", y, x, "gpu", s["color"][y, x], "oracle", ot["color"][y, x], "nc", s["n_contrib"][y, x], ot["n_contrib"][y, x])
    tiles_x = (W + 15) // 16
    t = (y // 16) * tiles_x + x // 16
    sc = s["screen"]
    Tr = 1.0
    for k, g in enumerate(s["pg"][s["off"][t]:s["off"][t + 1]]):
        mx, my = sc["mean2d"][g]
        r = sc["radius_cut"][g]
        if not (np.ceil(mx - r) <= x <= np.floor(mx + r) and np.ceil(my - r) <= y <= np.floor(my + r)):
            continue
        inv = sc["inv_cov2d"][g].astype(np.float32)
        dx, dy = np.float32(x) - mx, np.float32(y) - my
        q32 = np.float32(inv[0, 0] * dx * dx + np.float32(2) * inv[0, 1] * dy * dx + inv[1, 1] * dy * dy)
        qc = np.float32(sc["q_cut"][g] + np.float32(1 / 64))
        if q32 > qc:
            continue
        ar = float(sc["opacity"][g]) * np.exp(-0.5 * float(q32))
        a = min(ar, 0.99)
        if a < 1 / 255:
            print("  k", k, "g", g, "cutoff alpha_raw", ar)
            continue
        print("  k", k, "g", g, "q", q32, "qc", qc, "alpha_raw", ar, "T", Tr, "col", sc["color"][g])
        Tr *= 1 - a
        if Tr < 1e-4:
            print("  terminated T", Tr)
            break
