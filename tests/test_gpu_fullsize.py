"""Parity of the BENCHMARKED path at full size.

Config 3 (1M Gaussians = 900k foreground + 100k sky, 1280x720, exposure on)
and config 2 (100k, 640x480), each stepped exactly as bench.py times it:
Mapper.optimize_keyframe, CUDA-graph replay, warm per-keyframe tile depth
limits (truncated lists: at config 3 ~1.8M of ~10.6M pairs kept), the fused
chain rule + sparse Adam.  After five warm-up iterations one more iteration
is captured stage by stage from the engine's own buffers and every stage is
re-computed by the CPU oracle on the GPU's own inputs (mapper.py:299-328):

* a1  frustum mask: bit-exact (scene.py:283-298);
* a4  render on the GPU's (depth-limited) pair lists: colour within 1e-4,
      every pixel over 1e-6 explained by a hard decision flip
      (forward.py:277-333, parity.explain_pixels) -- the step's forward takes
      alpha from the hardware exp (2 ulp), the oracle from the correctly
      rounded one;
* a5  loss parts and dE on the GPU's render (loss.py:143-177);
* a6  screen adjoints on the GPU's screen, pairs, render and dC
      (backward.py:91-213): 1e-3 rel / 1e-5 abs per element, normwise,
      f64-calibrated (parity.assert_grads_calibrated);
* a7  chain rule (backward.py:415-500) on the GPU's adjoints: the gradient
      the engine kept (pre-Adam, active rows) against the oracle's chain;
      and end to end against the oracle's own adjoints;
* a8  sparse Adam (adam.py:76-122) on the GPU's gradient: BITWISE, step
      counters exact;
* a9  exposure ScalarAdam (adam.py:125-140) on the GPU's dE.

The oracle needs ~1 min of host time for this; the scene is built once.
"""

import numpy as np
import pytest

from parity import (COLOR_TOL, assert_grads_calibrated, assert_image_close, explain_pixels,
                    explained_pixel_budget, oracle)

pytestmark = pytest.mark.gpu

GRADS = ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")
GROUP_OF = {"d_position": "positions", "d_log_scale": "log_scales", "d_rotation": "rotations",
            "d_opacity_logit": "opacity_logits", "d_sh": "sh_coeffs"}
WIDTHS = (("d_position", (3,)), ("d_log_scale", (3,)), ("d_rotation", (4,)),
          ("d_opacity_logit", ()), ("d_sh", (16, 3)))


def _np(t):
    return t.detach().cpu().numpy()


def _a256(x):
    return (x + 255) & ~255


@pytest.fixture(scope="module", params=[3, 2], ids=["config3", "config2"])
def step3(request):
    """One warm, graph-replayed iteration of the config, its inputs and every
    intermediate the engine kept."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    scene = synthetic.config(request.param)
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=scene.n)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*scene.arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs())
    pose = sb.CameraPose(scene.W, scene.t)
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    entry = mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=scene.image),
                         cfg.lr_exposure, torch.float32)
    entry.exposure.matrix = scene.E
    mp.collect([mp.optimize_keyframe(entry) for _ in range(5)])
    eng = mp.engine
    assert eng.graphs, "the checked iteration must be a graph replay"
    n = mp.map.count
    before = {k: _np(v).copy() for k, v in mp.map.arrays().items()}
    m0 = {g: _np(t).copy() for g, t in mp.adam.m.items()}
    v0 = {g: _np(t).copy() for g, t in mp.adam.v.items()}
    steps0 = _np(mp.adam.steps).copy()
    E0 = entry.exposure.matrix.copy()
    Es0 = _np(entry.exposure.state).copy()
    log = mp.collect([mp.optimize_keyframe(entry)])[0]
    assert mp.reruns == 0
    torch.cuda.synchronize()
    caps_finite = sum(int(torch.isfinite(c).sum()) for c in eng.caps.values())
    b = eng.bufs
    rec = _np(b["records"][:n]).astype(np.float32)
    P = int(eng.binout["offsets"][-1].item())
    ws = b["ws_chain_adam"]
    grad, off = {}, 0
    for name, shape in WIDTHS:
        w = int(np.prod(shape)) if shape else 1
        grad[name] = _np(ws[off:off + 4 * w * n].view(torch.float32)).reshape((n,) + shape).copy()
        off += _a256(w * 4 * n)
    # the element pass's per-row flags: bit 1 = the row has a gradient (some
    # pixel reached it), bit 0 = updated (touched-row skip, adam.cu apply_flags)
    flags = (_np(ws[off:off + n]) & 2) != 0
    out = {
        "scene": scene, "n": n, "log": log, "before": before, "m0": m0, "v0": v0,
        "steps0": steps0, "E0": E0, "Es0": Es0, "rec": rec, "valid": _np(b["valid"][:n]) != 0,
        "frustum": _np(b["frustum"][:n]) != 0, "P": P,
        "pg": _np(eng.binout["a_pg"][:P]).astype(np.int64),
        "off": _np(eng.binout["offsets"]).astype(np.int64),
        "color": _np(eng.fwd["color"]).copy(), "n_contrib": _np(eng.fwd["n_contrib"]).copy(),
        "d_rendered": _np(eng.loss["d_rendered"]).copy(), "d_E": _np(eng.loss["d_E"]).copy(),
        # the merged adjoints of the rows the gather listed (the engine does
        # not zero the others: sb_gather_adjoints' reached list);
        # an unlisted row's adjoints are zero by definition
        "adj": {k: np.where(flags.reshape((-1,) + (1,) * (b[k].dim() - 1)),
                            _np(b[k][:n]), 0).astype(np.float32)
                for k in ("d_mean2d", "d_conic", "d_opacity", "d_color")},
        "grad": grad, "flags": flags, "lrs": mp._lrs(),
        "after": {k: _np(v).copy() for k, v in mp.map.arrays().items()},
        "steps_after": _np(mp.adam.steps).copy(), "E_after": entry.exposure.matrix.copy(),
        "gt": _np(entry.gt).copy(), "caps_finite": caps_finite, "config": request.param,
    }
    o = oracle()
    out["cam"] = o.Camera(W=scene.W, t=scene.t, fx=scene.fx, fy=scene.fy, cx=scene.cx,
                          cy=scene.cy, width=scene.width, height=scene.height)
    # the GPU's own screen (map-indexed records: pair ids are map rows)
    r = rec
    inv = np.stack([np.stack([r[:, 2], r[:, 3]], 1), np.stack([r[:, 3], r[:, 4]], 1)], 1)
    out["screen"] = {"mean2d": r[:, 0:2].copy(), "inv_cov2d": inv, "opacity": r[:, 5].copy(),
                     "q_cut": r[:, 6].copy(), "radius_cut": r[:, 7].copy(),
                     "color": r[:, 8:11].copy(), "depth": r[:, 11].copy()}
    del mp, entry, eng
    torch.cuda.empty_cache()
    return out


def test_c3_limits_were_warm(step3):
    """The checked iteration is the bench's: depth-limited lists (config 3:
    ~1.8M kept pairs; full lists hold ~10.6M)."""
    assert step3["caps_finite"] > 100
    if step3["config"] == 3:
        assert 1_000_000 < step3["P"] < 4_000_000


def test_c3_frustum_mask_bitexact(step3):
    o = oracle()
    want = o.frustum_mask(step3["cam"], step3["before"]["positions"])
    np.testing.assert_array_equal(step3["frustum"], want)


def test_c3_render_on_gpu_lists(step3):
    o = oracle()
    s = step3
    W, H = s["cam"].width, s["cam"].height
    ot = o.composite(s["pg"], s["off"], s["screen"], W, H)
    # the same arithmetic as the oracle but a 2-ulp exp: any pixel off by
    # more than 1e-6 must be explained by a hard decision flip
    err = np.abs(s["color"].astype(np.float64) - ot["color"]).max(axis=2)
    bad = np.argwhere(err > 1e-6)
    unexplained = explain_pixels(bad, s["pg"], s["off"], s["screen"], W)
    assert not unexplained, f"{len(unexplained)} unexplained pixels of {len(bad)}"
    # within 1e-4 everywhere except explained flips (a termination or cutoff
    # decided the other way: a whole contributor more or less)
    assert_image_close(s["color"], ot["color"], tol=COLOR_TOL,
                       budget=min(len(bad), explained_pixel_budget(W * H)))
    assert float(np.mean(s["n_contrib"] != ot["n_contrib"])) <= 1e-5


def test_c3_loss_and_exposure_gradient(step3):
    o = oracle()
    s = step3
    loss, _, d_E, parts = o.photometric_loss(s["color"], s["gt"], s["E0"], 0.2)
    assert s["log"]["loss"] == pytest.approx(loss, rel=1e-6)
    assert s["log"]["l1"] == pytest.approx(parts["l1"], rel=1e-6)
    np.testing.assert_allclose(s["d_E"].reshape(3, 4), d_E, rtol=1e-5,
                               atol=1e-6 * np.abs(d_E).max())


def test_c3_exposure_adam(step3):
    o = oracle()
    s = step3
    ex = o.ScalarAdam((3, 4), 1e-2)
    st = s["Es0"]
    ex.m, ex.v, ex.t = st[:12].reshape(3, 4).copy(), st[12:24].reshape(3, 4).copy(), int(st[24])
    E = s["E0"].copy()
    ex.step(E, s["d_E"].reshape(3, 4))
    np.testing.assert_allclose(s["E_after"], E, rtol=0, atol=1e-14)


def _truth_adjoints(s):
    o = oracle()
    up = {k: v.astype(np.float64) for k, v in s["screen"].items()}
    W, H = s["cam"].width, s["cam"].height
    return o.backward_tiles(s["pg"], s["off"], up, s["d_rendered"].astype(np.float64),
                            s["color"].astype(np.float64), W, H)


@pytest.fixture(scope="module")
def oracle_adj(step3):
    o = oracle()
    s = step3
    W, H = s["cam"].width, s["cam"].height
    a32 = o.backward_tiles(s["pg"], s["off"], s["screen"], s["d_rendered"], s["color"], W, H)
    return a32, _truth_adjoints(s)


def test_c3_screen_adjoints(step3, oracle_adj):
    """K8 at full size on the GPU's own inputs (depth-limited lists)."""
    s = step3
    a32, a64 = oracle_adj
    rows = np.nonzero(s["valid"])[0]
    for k in ("d_mean2d", "d_conic", "d_opacity", "d_color"):
        assert_grads_calibrated(s["adj"][k][rows], a32[k][rows], a64[k][rows], k)


def _chain(s, adj_map, dtype=np.float32):
    """oracle chain (a7) on the oracle's projection of the pre-step map, fed
    with map-indexed adjoints."""
    o = oracle()
    gm = {k: v.astype(dtype) for k, v in s["before"].items()}
    gm["is_sky"] = None
    scr = o.project(gm["positions"], gm["log_scales"], gm["rotations"], gm["opacity_logits"],
                    gm["sh_coeffs"], s["cam"])
    src = scr["source_index"]
    adj = {k: v[src].astype(dtype) for k, v in adj_map.items()}
    return o.chain(adj, scr, gm, s["cam"])


@pytest.fixture(scope="module")
def oracle_grads(step3, oracle_adj):
    s = step3
    a32, a64 = oracle_adj
    return {"on_gpu_adj": _chain(s, s["adj"]), "full": _chain(s, a32),
            "truth": _chain(s, a64, np.float64)}


def test_c3_chain_rule_on_gpu_adjoints(step3, oracle_grads):
    """The engine's pre-Adam gradient (active rows; a row no pixel reached
    has an exactly zero gradient) against the oracle's chain rule fed the
    GPU's own adjoints."""
    s = step3
    act = s["frustum"]
    og = oracle_grads["on_gpu_adj"]
    for k in GRADS:
        got = np.where(s["flags"].reshape((-1,) + (1,) * (s["grad"][k].ndim - 1)), s["grad"][k], 0)
        assert_grads_calibrated(got[act], og[k][act], oracle_grads["truth"][k][act], k)
        # unreached active rows: exactly zero in the oracle too
        un = act & ~s["flags"]
        assert float(np.abs(og[k][un]).max(initial=0)) == 0.0, k


def test_c3_gradients_end_to_end(step3, oracle_grads):
    """The engine's gradient against the oracle's whole backward (its own
    adjoints + chain), f64-calibrated."""
    s = step3
    act = s["frustum"]
    for k in GRADS:
        got = np.where(s["flags"].reshape((-1,) + (1,) * (s["grad"][k].ndim - 1)), s["grad"][k], 0)
        assert_grads_calibrated(got[act], oracle_grads["full"][k][act],
                                oracle_grads["truth"][k][act], k)


def test_c3_sparse_adam_bitwise(step3):
    """K10 at full size: the oracle's adam_step on the GPU's own gradient
    reproduces the GPU's updated map bit for bit."""
    o = oracle()
    s = step3
    params = {g: s["before"][f].copy() for g, f in zip(o.GROUPS, ("positions", "log_scales",
                                                                  "rotations", "opacity_logits",
                                                                  "sh_coeffs"))}
    grads = {}
    for g, k in zip(o.GROUPS, GRADS):
        fl = s["flags"].reshape((-1,) + (1,) * (s["grad"][k].ndim - 1))
        grads[g] = np.ascontiguousarray(np.where(fl, s["grad"][k], 0).astype(np.float32))
    m = {g: s["m0"][g].copy() for g in o.GROUPS}
    v = {g: s["v0"][g].copy() for g in o.GROUPS}
    steps = s["steps0"].copy()
    o.adam_step(params, grads, m, v, steps, s["lrs"], active=s["frustum"])
    np.testing.assert_array_equal(s["steps_after"], steps)
    for g, f in zip(o.GROUPS, ("positions", "log_scales", "rotations", "opacity_logits",
                               "sh_coeffs")):
        np.testing.assert_array_equal(s["after"][f], params[g], err_msg=f)


# ---------------------------------------------------------------------------
# config 5: the keyframe batch through DeviceBatchCompute
# ---------------------------------------------------------------------------
def test_config5_two_views_batched_vs_oracle():
    """BASELINE configs[4] at full size -- the 4M ring map + sky, 1280x720 --
    with 2 of its views in one batched step through DeviceBatchCompute (world
    1, the same calls BatchStep.step makes): the summed flat gradient against
    the batched oracle (the sum over views of the oracle's backward + chain on
    each view's GPU screen, pairs, render and dC; f64-calibrated), and the one
    sparse Adam step over the union of the frustum masks bit for bit."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    from paper_2404_06926_b200.batch import DeviceBatchCompute, group_views
    o = oracle()
    scene, views = synthetic.config5()
    views = views[:2]
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=scene.n)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*scene.arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs())
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    entries = []
    for k, v in enumerate(views):
        e = mp.store.add(sb.CameraFrame(pose=sb.CameraPose(v.W, v.t), intrinsics=intr,
                                        image=v.image, frame_index=k), cfg.lr_exposure)
        e.exposure.matrix = v.E
        entries.append(e)
    comp = DeviceBatchCompute(mp)
    lrs = mp._lrs()
    n = mp.map.count
    before = {k: _np(t).copy() for k, t in mp.map.arrays().items()}
    flat, union = comp.begin()
    per_view = []
    for e, v in zip(entries, views):
        comp.accumulate(e, flat, union)
        torch.cuda.synchronize()
        b = comp.bufs
        P = int(comp.binout["offsets" if "offsets" in comp.binout else "a_off"][-1].item())
        pg = comp.binout["pair_gaussian"][:P] if "pair_gaussian" in comp.binout else \
            comp.binout["a_pg"][:P]
        rec = _np(b["records"][:n])
        inv = np.stack([np.stack([rec[:, 2], rec[:, 3]], 1),
                        np.stack([rec[:, 3], rec[:, 4]], 1)], 1)
        per_view.append({
            "pg": _np(pg).astype(np.int64),
            "off": _np(comp.binout["offsets"]).astype(np.int64),
            "screen": {"mean2d": rec[:, 0:2].copy(), "inv_cov2d": inv,
                       "opacity": rec[:, 5].copy(), "q_cut": rec[:, 6].copy(),
                       "radius_cut": rec[:, 7].copy(), "color": rec[:, 8:11].copy(),
                       "depth": rec[:, 11].copy()},
            "color": _np(comp.fwd["color"]).copy(), "d_rendered": _np(comp.loss["d_rendered"]).copy(),
            "frustum": _np(b["frustum"][:n]) != 0,
            "cam": o.Camera(W=v.W, t=v.t, fx=scene.fx, fy=scene.fy, cx=scene.cx, cy=scene.cy,
                            width=scene.width, height=scene.height)})
    g_flat = {k: _np(t[:n]).copy() for k, t in group_views(flat, comp.n_pad).items()}
    union_h = _np(union[:n]) != 0
    steps0 = _np(mp.adam.steps).copy()
    m0 = {g: _np(t).copy() for g, t in mp.adam.m.items()}
    v0 = {g: _np(t).copy() for g, t in mp.adam.v.items()}
    comp.apply(flat, union)
    torch.cuda.synchronize()
    after = {k: _np(t).copy() for k, t in mp.map.arrays().items()}
    steps_after = _np(mp.adam.steps).copy()
    assert int(comp.st64[1].item()) == 0          # a valid step
    del mp, comp, flat, union
    torch.cuda.empty_cache()
    # the batched oracle: sum over views of backward + chain (f32, view order)
    # and the same in f64 as the truth
    gm = dict(before)
    gm["is_sky"] = None
    gm64 = {k: (v.astype(np.float64) if v is not None else None) for k, v in gm.items()}
    total, truth = None, None
    want_union = np.zeros(n, bool)
    for pv in per_view:
        W, H = pv["cam"].width, pv["cam"].height
        np.testing.assert_array_equal(pv["frustum"], o.frustum_mask(pv["cam"], gm["positions"]))
        want_union |= pv["frustum"]
        a32 = o.backward_tiles(pv["pg"], pv["off"], pv["screen"], pv["d_rendered"], pv["color"],
                               W, H)
        s64 = {k: x.astype(np.float64) for k, x in pv["screen"].items()}
        a64 = o.backward_tiles(pv["pg"], pv["off"], s64, pv["d_rendered"].astype(np.float64),
                               pv["color"].astype(np.float64), W, H)
        outs = []
        for gmx, adj in ((gm, a32), (gm64, a64)):
            scr = o.project(gmx["positions"], gmx["log_scales"], gmx["rotations"],
                            gmx["opacity_logits"], gmx["sh_coeffs"], pv["cam"])
            src = scr["source_index"]
            dt = gmx["positions"].dtype
            outs.append(o.chain({k: x[src].astype(dt) for k, x in adj.items()}, scr, gmx,
                                pv["cam"]))
        total = outs[0] if total is None else {k: total[k] + outs[0][k] for k in total}
        truth = outs[1] if truth is None else {k: truth[k] + outs[1][k] for k in truth}
    np.testing.assert_array_equal(union_h, want_union)
    for (gname, _), k in zip((("position", 0), ("log_scale", 0), ("rotation", 0),
                              ("opacity_logit", 0), ("sh", 0)), GRADS):
        assert_grads_calibrated(g_flat[gname][union_h], total[k][union_h], truth[k][union_h], k)
    # one sparse Adam over the union, on the GPU's own summed gradient: bitwise
    params = {g: before[f].copy() for g, f in zip(o.GROUPS, ("positions", "log_scales",
                                                             "rotations", "opacity_logits",
                                                             "sh_coeffs"))}
    grads = {g: np.ascontiguousarray(g_flat[g]) for g in o.GROUPS}
    steps = steps0.copy()
    o.adam_step(params, grads, m0, v0, steps, lrs, active=union_h)
    np.testing.assert_array_equal(steps_after, steps)
    for g, f in zip(o.GROUPS, ("positions", "log_scales", "rotations", "opacity_logits",
                               "sh_coeffs")):
        np.testing.assert_array_equal(after[f], params[g], err_msg=f)

