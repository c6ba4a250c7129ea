import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from parity import *
import paper_2404_06926_b200 as sb
o = oracle()
for name in ("slim128_f32", "view160_f32", "sky200_f32"):
    g = load_golden(name)
    fx, fy, cx, cy, w, h = g["intr"]
    pose = sb.CameraPose(g["W"], g["t"]); intr = sb.CameraIntrinsics(fx, fy, cx, cy, int(w), int(h))
    rs = sb.SplatScreen(**screen_from(g))
    grid = sb.bin_and_sort(rs, intr)
    if "refrender_color" in g:
        t = sb.render(grid, rs, intr, early_termination=False)
        c = t.color.cpu().numpy()
        d1 = np.abs(c - g["refrender_color"]); d2 = np.abs(c - g["noterm_color"])
        print(name, "noterm vs refrender", d1.max(), "vs noterm", d2.max(), np.unravel_index(d2.argmax(), d2.shape))
        ot = o.composite(g["pair_gaussian"], g["offsets"], screen_from(g), int(w), int(h), early_termination=False)
        print("   oracle noterm vs golden noterm", np.abs(ot["color"] - g["noterm_color"]).max(), " gpu vs oracle", np.abs(c - ot["color"]).max())
    t = sb.render(grid, rs, intr)
    gm = sb.GaussianMap(dtype=np.float32)
    gm.append_arrays(g["positions"], g["log_scales"], g["rotations"], g["opacity_logits"], g["sh_coeffs"], g["is_sky"])
    buf = sb.backward_per_gaussian(t, torch.as_tensor(g["d_rendered"]).cuda(), rs, grid, gm, pose, intr)
    # f64 truth: oracle f64 on f64-cast reference screen + grid + targets + dC
    s64 = {k: (v.astype(np.float64) if v.dtype == np.float32 else v) for k, v in screen_from(g).items()}
    adj = o.backward_tiles(g["pair_gaussian"], g["offsets"], s64, g["d_rendered"].astype(np.float64), g["color"].astype(np.float64), int(w), int(h))
    gm64 = {k: v.astype(np.float64) if v.dtype == np.float32 else v for k, v in gmap_from(g).items()}
    tr = o.chain(adj, s64, gm64, camera_from(g))
    for f in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        gg = buf.__dict__[f].cpu().numpy().astype(np.float64); rr = g["grad_" + f].astype(np.float64); tt = tr[f]
        sc = np.abs(tt).max()
        print(f"  {f}: gpu-vs-truth {np.abs(gg-tt).max()/sc:.2e}  ref32-vs-truth {np.abs(rr-tt).max()/sc:.2e}  gpu-vs-ref {np.abs(gg-rr).max()/np.abs(rr).max():.2e}")
