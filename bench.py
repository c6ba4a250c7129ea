#!/usr/bin/env python
"""Benchmark: mapping iterations/s (forward + backward + Adam) at BASELINE.json
config 3 (1M Gaussians = 900k foreground + 100k sky, 1280x720, exposure on).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0 (contract in the task statement).

* N = 1: ``value`` is the device-timed it/s of the mapping step (the engine's
  CUDA-graph replay with warm per-keyframe depth limits), map and keyframe
  resident in HBM; ``e2e`` the same iterations through Mapper.optimize_keyframe
  with the keyframe image copied from pinned host memory every step and the
  log row read back.  Beside it: ``full_lists`` (the same step binning full
  tile lists), ``atomic_backward`` (the float-atomic backward instead of the
  deterministic one: the cost of determinism), ``batched`` (the keyframe-batch
  data-parallel step of N > 1 at world size 1, NCCL exchange on: the code
  path the scaling runs use), render FPS, the dominant kernel's roofline and
  the CPU baseline.
* N > 1 (launched by torchrun, or ``--gpus N`` re-launches itself under it):
  the keyframe-batch step of SURVEY §8(e) -- one view per rank of the
  replicated config-3 map, the reached rows' gradient all-reduced over NCCL,
  one sparse Adam step on every rank, the whole step replayed as one CUDA
  graph.  ``scaling`` "weak"; ``value`` = views (mapping iterations) per
  second over all ranks.
* ``--impl reference`` times the CPU oracle (oracle/: the reference's
  algorithm restated in C; the reference is Python + numba and cannot be
  compiled into oracle/_ref) on the host cores, on the same workload (N views
  per batched step at N > 1), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "mapping iters/s (fwd+bwd+Adam) @1M Gaussians 1280x720"
UNIT = "it/s"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # pragma: no cover
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region through
    NVML (in-process, every 10 ms; nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []   # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return float(sm), float(mx), int(rs)
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        return float(out[0]), float(out[1]), int(out[2].strip(), 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        try:
            self.samples.append(self._sample())
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = sorted(k for k, bit in self.REASONS.items() if mask & bit)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": reasons,
                "samples": len(self.samples), "via": "nvml" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
# workload description (identical in both arms)
# ---------------------------------------------------------------------------
# stdout carries exactly the JSON line: the native libraries (NCCL prints its
# version from a one-rank communicator) write to file descriptor 1, so fd 1
# is pointed at stderr for the whole run and the line goes to a private copy
# of the original stdout
_JSON_OUT = None


def _guard_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


def scene_of(cfg_idx):
    from paper_2404_06926_b200 import synthetic
    return synthetic.config(cfg_idx)


def config_dict(scene, cfg_idx, world):
    """The workload: the same dict in our arm and the reference arm."""
    sky = " (900k fg + 100k sky)" if cfg_idx == 3 else ""
    if cfg_idx == 5:
        return {"workload": f"config5: {scene.n} Gaussians (3.9M ring + 100k sky), keyframe "
                            f"batch of 8 views sharded over {world} GPU(s), "
                            f"{scene.width}x{scene.height}, exposure on",
                "N": int(scene.n), "pixels": int(scene.width * scene.height),
                "views_per_step": 8,
                "l2": "inputs larger than L2 (map + Adam state %.0f MB)" % (scene.n * 944 / 1e6)}
    if world == 1:
        wl = (f"config{cfg_idx}: {scene.n} Gaussians{sky}, {scene.width}x{scene.height}, "
              f"exposure on, one keyframe")
    else:
        wl = (f"config{cfg_idx}: {scene.n} Gaussians{sky}, keyframe batch of {world} views "
              f"(one per rank), {scene.width}x{scene.height}, exposure on")
    big = scene.n * 944 >= 126 * 10 ** 6
    return {"workload": wl, "N": int(scene.n), "pixels": int(scene.width * scene.height),
            "views_per_step": int(world),
            "l2": ("inputs larger than L2 (map + Adam state %.0f MB)" % (scene.n * 944 / 1e6)
                   if big else "inputs smaller than L2 and not flushed: a parity config, "
                               "not the headline")}


def data_note(cfg_idx):
    return f"synthetic (seeded SURVEY §8d config-{cfg_idx} scene, random-init map)"


# ---------------------------------------------------------------------------
# our arm, N = 1
# ---------------------------------------------------------------------------
def build_mapper(scene, sb, torch):
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=max(scene.n, 1))
    mp = sb.Mapper(cfg, dtype=torch.float32)
    mp.map.reserve(scene.n)
    mp.map.append_arrays(*scene.arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs(), dtype=torch.float32)
    pose = sb.CameraPose(scene.W, scene.t)
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    frame = sb.CameraFrame(pose=pose, intrinsics=intr, image=scene.image, frame_index=0)
    entry = mp.store.add(frame, cfg.lr_exposure, torch.float32)
    entry.exposure.matrix = scene.E
    return mp, entry


def _state_tensors(mp, entry):
    """Every device tensor a mapping step mutates (map, Adam moments and
    counters, the keyframe's exposure and its optimizer state)."""
    a = mp.adam
    ts = list(mp.map.arrays().values())
    ts += [a._m[g] for g in sorted(a._m)] + [a._v[g] for g in sorted(a._v)] + [a._steps]
    ts += [a._touched]            # the touched-row mask travels with the moments
    e = entry.exposure
    return ts + [e.mat, e.real, e.state]


def snapshot(mp, entry):
    return [t.clone() for t in _state_tensors(mp, entry)]


def restore(mp, entry, snap):
    """In place (the captured CUDA graphs keep their pointers)."""
    for t, s in zip(_state_tensors(mp, entry), snap):
        t.copy_(s)


# the library calls of one mapping step and their kernels (CUB's radix sort
# and scan passes included), checked against the ncu launch list in profiles/
KERNELS_PER_CALL = {"sb_depth_limits_gate": 1, "sb_preprocess_fwd": 1, "sb_bin": 11,
                    "sb_blend_fwd": 2, "sb_loss_fused": 4, "sb_blend_bwd_partials": 3,
                    "sb_gather_adjoints": 2, "sb_chain_adam_rows": 4, "sb_exposure_adam": 1,
                    "sb_psnr8_sse": 1}
# the blends' heavy-first tile-order kernel (one tiny single-CTA launch each,
# ~4 us) and the backward's unused launch shape (its CTAs leave at once): a
# call whose other launches are only these helpers counts as one kernel for
# the dominant-kernel roofline
HELPER_KERNELS = {"sb_blend_fwd": 1, "sb_blend_bwd_partials": 2, "sb_blend_bwd": 1}
TIMED_CALLS = ("sb_preprocess_fwd", "sb_bin", "sb_blend_fwd", "sb_loss_fused", "sb_blend_bwd",
               "sb_blend_bwd_partials", "sb_gather_adjoints", "sb_chain_adam_rows",
               "sb_exposure_adam", "sb_psnr8_sse")


def kernel_times(mp, entry, torch, steps=5):
    """Average device time of each library call, timed one at a time on the
    launching stream by replaying the step's stages with events in between."""
    from paper_2404_06926_b200 import _native as N
    st = torch.cuda.current_stream()
    times = {}
    lib = N.load()
    wrapped = {nm: getattr(lib, nm) for nm in TIMED_CALLS}

    class Timed:
        def __init__(self, nm, fn):
            self.nm, self.fn = nm, fn
            self.restype, self.argtypes = fn.restype, fn.argtypes

        def __call__(self, *a):
            # every entry point takes its stream last: time on that stream
            sp = getattr(a[-1], "value", a[-1])
            s = torch.cuda.ExternalStream(sp) if sp else st
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            rc = self.fn(*a)
            e1.record(s)
            times.setdefault(self.nm, []).append((e0, e1))
            return rc

    for nm in TIMED_CALLS:
        setattr(lib, nm, Timed(nm, wrapped[nm]))
    graphs = mp.use_graphs
    mp.use_graphs = False   # eager launches, one event pair around each
    try:
        for _ in range(steps):
            mp._step_device(entry)
        torch.cuda.synchronize()
    finally:
        mp.use_graphs = graphs
        for nm in TIMED_CALLS:
            setattr(lib, nm, wrapped[nm])
    return {nm: float(np.mean([a.elapsed_time(b) for a, b in v])) for nm, v in times.items()}


def render_fps(mp, entry, torch, steps):
    """Forward-only frames/s (mapper.py:202-212: project, bin, blend) through
    the engine's sync-free render path (Mapper.render_image without the final
    check): device binning, the view's depth limits, device-timed.  Every
    timed frame's status is checked afterwards; an invalid one is re-timed
    once, then reported."""
    kf = entry.frame
    intr, pose = kf.intrinsics, kf.pose
    eng = mp.engine
    dev = mp.map.positions.device
    for _ in range(3):
        mp.render_image(pose, intr, key="bench")
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    for attempt in range(2):
        stats = torch.zeros((steps, 2), dtype=torch.int64, device=dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(steps):
            eng.render(mp.map, pose, intr, key="bench", near=mp.cfg.near,
                       margin=mp.cfg.frustum_margin, status=stats[i])
        b.record(st)
        torch.cuda.synchronize()
        bad = int(stats[:, 1].sum().item())
        if bad == 0:
            break
    return steps / (a.elapsed_time(b) / 1e3), bad


def counts(mp, torch):
    """Device counts for the roofline: N, M (projected), A (frustum-active),
    P (full-list pairs), P_kept (what the step's depth-limited
    binning kept), P_proc (pairs reached before every pixel of a tile
    stopped)."""
    last = mp.engine.last
    tg = last["targets"]["last"]
    H, W = tg.shape
    th, tw = (H + 15) // 16, (W + 15) // 16
    pad = torch.zeros((th * 16, tw * 16), dtype=torch.int32, device=tg.device)
    pad[:H, :W] = tg
    per_tile = pad.reshape(th, 16, tw, 16).amax(dim=(1, 3))
    kept = int(last["status"][0].item())
    eng = mp.engine
    kf = mp.store.entries[-1].frame
    st = torch.zeros(2, dtype=torch.int64, device=tg.device)
    eng.render(mp.map, kf.pose, kf.intrinsics, key=None, near=mp.cfg.near,
               margin=mp.cfg.frustum_margin, status=st)
    torch.cuda.synchronize()
    n = mp.map.count
    fr = last["frustum"]
    return {"N": n, "M": int(eng.bufs["r_valid"][:n].sum().item()),
            "A": int(fr.sum().item()),
            # live: active rows the Adam pass updates (touched-row skip)
            "L": int((fr.bool() & mp.adam._touched[:n].bool()).sum().item()),
            "P": int(st[0].item()), "P_kept": kept,
            "P_proc": int(per_tile.sum().item()), "Px": H * W}


def kernel_bytes(c):
    """Algorithmic bytes per launch: compulsory reads + writes
    of each call's own data layout, with the run's own counts."""
    N_, M, A, Pp, Px = c["N"], c["M"], c["A"], c["P_proc"], c["Px"]
    return {
        # params 236 B/row read; record 48 + valid 1 + key 4 + val 4 + frustum 1 written
        "sb_preprocess_fwd": 236 * N_ + 58 * N_,
        # row depth sort (4 passes x 8 B read + written) + count and place passes
        # (order 4 + record 48 + count 4 + mask 8 B per row each) + 4 B per kept pair
        "sb_bin": 8 * N_ * 2 * 4 + 64 * M * 2 + 4 * c["P_kept"],
        # (4 B index + 48 B record) per reached pair; 44 B/pixel written
        "sb_blend_fwd": 52 * Pp + 44 * Px,
        # A: Y 12 + gt 12 in, 36 maps out; B1: 36 in, 12 out; B2: 12 + 24 + 12 in, 12 out
        "sb_loss_fused": (24 + 36 + 36 + 12 + 48 + 12) * Px,
        # per reached pair 52 B read + its 36 B of adjoints; per pixel dC 12 + C 12 +
        # last 4 (the float-atomic and the deterministic backward alike)
        "sb_blend_bwd": 88 * Pp + 28 * Px,
        "sb_blend_bwd_partials": 88 * Pp + 28 * Px,
        # the deterministic merge: the 36 B partial per reached pair read, 36 B of
        # adjoints per row written (at most one row per reached pair), 4 B count
        # per sorted rank
        "sb_gather_adjoints": 72 * Pp + 4 * N_,
        # live rows (active, moments non-zero or a gradient -- the touched-row
        # skip leaves the others bitwise unchanged): params + m + v read and
        # written (3 x 472); every active row: steps 16, adjoints 36; flags 2
        "sb_chain_adam_rows": 1416 * c["L"] + (16 + 36) * A + 2 * N_,
        "sb_psnr8_sse": 15 * Px,
    }


def step_bytes(c, P):
    """SURVEY §8(d) B_iter with pair count P."""
    # SURVEY's 1668 B per active row = 1416 (params + moments, live rows only
    # under the touched-row skip) + 252
    return (13 * c["N"] + 856 * c["M"] + 1416 * c["L"] + 252 * c["A"] + 36 * P
            + 88 * c["P_proc"] + 104 * c["Px"])


def _profile_entry(kind, kernel, cfg_idx):
    """A per-launch figure of ``kernel`` from the newest committed ncu capture
    (profiles/r*_<kind>.json) that was taken on THIS config; None otherwise."""
    import glob
    key = {"traffic": "dram_bytes_per_launch", "issue": "warp_inst_per_launch"}[kind]
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_{kind}.json")), reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
        except Exception:
            continue
        if t.get("config") != cfg_idx:
            continue
        if kernel in t.get(key, {}):
            return t[key][kernel], os.path.relpath(path, REPO)
    return None, None


def issue_roofline(kernel, kt, clocks, torch, cfg_idx):
    inst, src = _profile_entry("issue", kernel, cfg_idx)
    if inst is None or kernel not in kt:
        return None
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak = 4 * sms * mhz * 1e6          # warp instructions / s (one per scheduler per clock)
    achieved = inst / (kt[kernel] / 1e3)
    return {"warp_inst_per_launch": inst, "achieved": round(achieved / 1e9, 1),
            "peak": round(peak / 1e9, 1), "unit": "G warp-inst/s",
            "frac": round(achieved / peak, 4), "source": src}


def timed_steps(mp, entry, torch, steps):
    """K graph-replayed mapping steps between CUDA events; an invalid
    iteration (re-run by the mapper) makes the measurement repeat.  Returns
    (ms, rows, invalid_runs)."""
    st = torch.cuda.current_stream()
    invalid = 0
    for attempt in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        rows = [mp._step_device(entry) for _ in range(steps)]
        e1.record(st)
        torch.cuda.synchronize()
        flags = torch.stack([r[3][6:8].view(torch.int64)[1] for r in rows]).cpu()
        if int(flags.sum()) == 0:
            return e0.elapsed_time(e1), rows, invalid
        invalid += 1
        mp._materialise(rows)            # re-runs the invalid iterations in order
        for _ in range(3):               # the re-runs dropped the graphs: warm up again
            mp._step_device(entry)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1), rows, invalid


def variant_rate(mp, entry, torch, steps, warmup, snap=None, **engine_attrs):
    """it/s of the same step with engine attributes changed (graphs dropped
    and re-captured, then restored).  With ``snap`` (the state the headline's
    timed region started from) the variant times the SAME iterations: the map
    evolves under training (pairs per step grow), so a variant timed later in
    the run would see a different workload."""
    eng = mp.engine
    saved = {k: getattr(eng, k) for k in engine_attrs}
    try:
        for k, v in engine_attrs.items():
            setattr(eng, k, v)
        eng.graphs.clear()
        eng.seen.clear()
        if snap is not None:
            restore(mp, entry, snap)
        for _ in range(max(warmup, 3)):
            mp._step_device(entry)
        mp.collect([])
        if snap is not None:
            restore(mp, entry, snap)     # in place: the captured graphs stay valid
        torch.cuda.synchronize()
        ms, _, invalid = timed_steps(mp, entry, torch, steps)
    finally:
        for k, v in saved.items():
            setattr(eng, k, v)
        eng.graphs.clear()
        eng.seen.clear()
        mp.collect([])
    return {"value": round(steps / (ms / 1e3), 3), "ms_per_step": round(ms / steps, 4),
            "invalid_timed_runs": invalid}


def run_ours(args, local_rank):
    import torch
    import paper_2404_06926_b200 as sb

    torch.cuda.set_device(local_rank)
    scene = scene_of(args.config)
    mp, entry = build_mapper(scene, sb, torch)

    from paper_2404_06926_b200.hostmem import huge_page_bytes, pinned_from
    # the host image in pinned huge-page memory (paper_2404_06926_b200.hostmem:
    # 3x the DMA rate of 4 KB-page pinned memory on these boxes)
    gt_host = pinned_from(scene.image.astype(np.float32))
    hp_bytes = huge_page_bytes(gt_host.data_ptr())
    out_host = torch.empty(8, dtype=torch.float64).pin_memory()
    for _ in range(args.warmup):
        # every warm-up step goes through the e2e path (host upload into both
        # target buffers, their graphs, the copy stream, the read-back)
        mp.optimize_keyframe(entry, gt_host, log_host=out_host)
    mp.collect([])
    # the e2e leg below replays exactly these iterations (the map evolves, so
    # later iterations are not the same work)
    snap = snapshot(mp, entry)
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        ms, rows, invalid_runs = timed_steps(mp, entry, torch, args.steps)
    if invalid_runs:
        snap = snapshot(mp, entry)
    value = args.steps / (ms / 1e3)
    logs = mp._materialise(rows[-1:])

    # --- end to end through the public API, host buffers ---------------------
    restore(mp, entry, snap)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    w0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(st)
    for _ in range(args.steps):
        mp.optimize_keyframe(entry, gt_host, log_host=out_host)
    st.wait_stream(mp.readback_stream())   # the last log row has reached the host
    f1.record(st)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    e2e_wall = time.perf_counter() - w0
    e2e_val = args.steps / (e2e_ms / 1e3)
    mp.collect([])

    # --- the same step binning full lists, and with the float-atomic backward
    full = variant_rate(mp, entry, torch, args.steps, args.warmup, snap=snap,
                         use_caps=False)
    atomic = variant_rate(mp, entry, torch, args.steps, args.warmup, snap=snap,
                         deterministic=False)
    exact = variant_rate(mp, entry, torch, args.steps, args.warmup, snap=snap,
                         fast_exp=False)
    no_skip = variant_rate(mp, entry, torch, args.steps, args.warmup, snap=snap,
                         touched_skip=False)

    del snap
    # --- render FPS (mapper.py:202-212 forward only: project, bin, blend) -----
    fps, fps_invalid = render_fps(mp, entry, torch, args.steps)

    # --- roofline of the dominant kernel --------------------------------------
    c = counts(mp, torch)
    kt = kernel_times(mp, entry, torch, steps=3)
    kb = kernel_bytes(c)
    # the dominant KERNEL among single-kernel calls (sb_bin, sb_loss_fused and
    # sb_chain_adam_rows launch several kernels each; the ncu launch list in
    # profiles/ has their split); the largest multi-kernel call is reported too
    dom = max((k for k in kt if k in kb and
               KERNELS_PER_CALL.get(k, 0) - HELPER_KERNELS.get(k, 0) == 1), key=lambda k: kt[k])
    dom_call = max((k for k in kt if k in kb), key=lambda k: kt[k])
    peak, peak_kind = _peaks()
    achieved = kb[dom] / (kt[dom] / 1e3) / 1e9
    step_ms = ms / args.steps
    traffic, traffic_src = _profile_entry("traffic", dom, args.config)
    launches = sum(KERNELS_PER_CALL.values()) * args.steps

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": data_note(args.config),
        "config": config_dict(scene, args.config, 1),
        "stats": {"M": c["M"], "A": c["A"], "L": c["L"], "P": c["P"], "P_kept": c["P_kept"],
                  "P_proc": c["P_proc"], "parallelism": "one GPU",
                  "depth_limits": "warm (per-keyframe tile depth limits from the previous "
                                  "iteration; full_lists below bins every pair)",
                  "deterministic": True},
        "e2e": {"value": round(e2e_val, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(gt_host.numel() * 4),
                "d2h_bytes_per_step": int(out_host.numel() * 8),
                "wall_s": round(e2e_wall, 4),
                "api": "Mapper.optimize_keyframe(entry, pinned host image, log_host)",
                "host_buffer": "pinned, 2 MB pages requested (hostmem.pinned_from)",
                "host_buffer_huge_page_bytes": hp_bytes},
        "full_lists": dict(full, note="engine.use_caps=False: every kept (tile, Gaussian) pair "
                                      "binned, the reference's lists"),
        "atomic_backward": dict(atomic, note="engine.deterministic=False: the backward's float "
                                             "atomics instead of the ordered per-row merge"),
        "deterministic_cost_frac": round(1.0 - value / atomic["value"], 4),
        "no_touched_skip": dict(no_skip, note="engine.touched_skip=False: the Adam element pass "
                                              "over every active row, including those whose "
                                              "update is an exact identity (zero moments, no "
                                              "gradient; stats.L of stats.A rows are live)"),
        "exact_exp_forward": dict(exact, note="engine.fast_exp=False: the step's forward with the "
                                              "correctly rounded exp of the render API "
                                              "(bit-identical to the reference pipeline) instead "
                                              "of the hardware exp the backward replays with"),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "peak_source": peak_kind, "bytes_per_launch": int(kb[dom]),
                     "ms_per_launch": round(kt[dom], 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "step_algorithmic_bytes": int(step_bytes(c, c["P_kept"])),
                     "step_frac": round(step_bytes(c, c["P_kept"]) / (step_ms / 1e3) / 1e9 / peak, 4),
                     "step_algorithmic_bytes_full_list_P": int(step_bytes(c, c["P"])),
                     "step_frac_full_list_P": round(step_bytes(c, c["P"]) / (step_ms / 1e3) / 1e9
                                                    / peak, 4),
                     "largest_call": {"call": dom_call, "kernels": KERNELS_PER_CALL.get(dom_call),
                                      "ms": round(kt[dom_call], 4),
                                      "achieved": round(kb[dom_call] / (kt[dom_call] / 1e3) / 1e9, 1),
                                      "frac": round(kb[dom_call] / (kt[dom_call] / 1e3) / 1e9 / peak, 4)},
                     "kernel_ms": {k: round(v, 4) for k, v in kt.items()},
                     # the dominant kernel is issue-bound: its warp instructions
                     # per launch (a committed ncu capture OF THIS CONFIG) over
                     # its live time, against 4 schedulers x SMs x the SM clock
                     "issue": issue_roofline(dom, kt, clk.summary(), torch, args.config),
                     "call_hbm_frac": {k: round(kb[k] / (kt[k] / 1e3) / 1e9 / peak, 4)
                                       for k in kt if k in kb},
                     "kernel_ms_note": "eager launches, events on each call's stream; "
                                       "sb_exposure_adam and sb_psnr8_sse run on a side stream "
                                       "beside the backward, their times include queueing for "
                                       "SMs"},
        "render_fps": round(fps, 2),
        "render_note": ("project + bin + blend per frame, sync-free device binning with the "
                        f"view's depth limits (Mapper.render_image path); invalid frames {fps_invalid}"),
        "invalid_timed_runs": invalid_runs,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "loss_last": logs[0]["loss"], "psnr_last": logs[0]["psnr"],
    }
    del mp, entry
    torch.cuda.empty_cache()
    if not args.no_batched:
        line["batched"] = run_batched(args, 0, 1, local_rank, nested=True)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(scene, samples=args.cpu_steps, cfg_idx=args.config)
    emit(line)


# ---------------------------------------------------------------------------
# the keyframe batch (N > 1, and the ``batched`` key at N = 1)
# ---------------------------------------------------------------------------
def _views_for(scene, rank, world, sb):
    """One yawed view of the config-3 map per rank (weak scaling): yaw offsets
    centred on the keyframe."""
    yaw = 0.02 * (rank - (world - 1) / 2.0)
    R = np.array([[np.cos(yaw), 0, np.sin(yaw)], [0, 1, 0], [-np.sin(yaw), 0, np.cos(yaw)]])
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    return sb.CameraFrame(pose=sb.CameraPose(R, np.zeros(3)), intrinsics=intr, image=scene.image,
                          frame_index=rank + 1)


def run_batched(args, rank, world, local_rank, nested=False):
    """The keyframe-batch data-parallel step of SURVEY §8(e): every rank
    renders + back-propagates its view of the replicated map, the reached
    rows' gradient (59 reals each) travels in one NCCL all-reduce with the
    union frustum mask, every rank applies the same sparse Adam step; lazy
    validity checks (no host sync per step) and the whole step replayed as
    one CUDA graph.  At world 1 (``nested``: the ``batched`` key of the N = 1
    line) the exchange is forced on, so the same code runs at every N.
    Returns (nested) or prints the JSON line."""
    import torch
    import torch.distributed as tdist
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200.batch import DeviceBatchCompute, PackedBatchStep

    torch.cuda.set_device(local_rank)
    own_pg = False
    if not tdist.is_initialized():
        # the N = 1 leg: a one-rank NCCL group in this process
        tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                                 device_id=torch.device("cuda", local_rank))
        own_pg = True
    try:
        if args.config == 5:
            # BASELINE configs[4]: the 4M ring map, a fixed batch of 8 yawed
            # views sharded over the ranks (8 / world each): strong scaling
            from paper_2404_06926_b200 import synthetic
            from paper_2404_06926_b200.batch import shard_views
            scene, all_views = synthetic.config5()
            mp, _ = build_mapper(scene, sb, torch)
            intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width,
                                       scene.height)
            entries = []
            for k, v in shard_views(list(enumerate(all_views)), rank, world):
                e = mp.store.add(sb.CameraFrame(pose=sb.CameraPose(v.W, v.t), intrinsics=intr,
                                                image=v.image, frame_index=k + 1),
                                 mp.cfg.lr_exposure, torch.float32)
                e.exposure.matrix = v.E
                entries.append(e)
            views_total = len(all_views)
        else:
            scene = scene_of(args.config)
            mp, _ = build_mapper(scene, sb, torch)
            entry = mp.store.add(_views_for(scene, rank, world, sb), mp.cfg.lr_exposure,
                                 torch.float32)
            entry.exposure.matrix = scene.E
            entries = [entry]
            views_total = world
        step = PackedBatchStep(DeviceBatchCompute(mp), always_reduce=True, lazy=True)
        step.use_graphs = not args.no_batched_graphs

        def barrier():
            tdist.barrier()
            torch.cuda.synchronize()

        for _ in range(max(args.warmup, 3)):
            step.step(entries)
        step.flush()
        barrier()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) as clk:
            e0.record(st)
            h0, w0 = time.perf_counter(), step.host_wait_s
            logs = [step.step(entries) for _ in range(args.steps)]
            # host time to enqueue the K steps, without the lazy checks' waits
            # for the device (the check of step i waits for step i - lag)
            host_ms = (time.perf_counter() - h0 - (step.host_wait_s - w0)) * 1e3
            step.flush()     # lazy validity: every timed step checked (and re-run) in the region
            e1.record(st)
            barrier()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
        value = args.steps * views_total / (ms / 1e3)
        # e2e: each rank's view image from pinned host memory every step (side
        # stream upload) and its loss parts read back -- the log of the step
        # resolved `lag` steps earlier (a step's logs are final once checked)
        from paper_2404_06926_b200.hostmem import pinned_from
        gt_host = [pinned_from(e.frame.image.astype(np.float32)) for e in entries]
        out_host = torch.empty(4 * len(entries), dtype=torch.float64).pin_memory()
        for _ in range(2):         # warm the upload path and both target buffers' graphs
            for e, g in zip(entries, gt_host):
                mp.upload_image(e, g)
            step.step(entries)
        step.flush()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        pending = []
        for _ in range(args.steps):
            for e, g in zip(entries, gt_host):
                mp.upload_image(e, g)
            pending.append(step.step(entries))
            if len(pending) > step.lag:
                out_host.copy_(torch.cat(pending.pop(0)), non_blocking=True)
        step.flush()
        for p in pending:
            out_host.copy_(torch.cat(p), non_blocking=True)
        f1.record(st)
        barrier()
        e2e_ms = f0.elapsed_time(f1)
        t = torch.tensor([e2e_ms], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_val = args.steps * views_total / (float(t.item()) / 1e3)
        reached = int(step.compute.reached_mask()[:mp.map.count].sum().item())
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong" if args.config == 5 else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": data_note(args.config),
            "unit_note": "value = views (mapping iterations) per second over all ranks",
            "config": config_dict(scene, args.config, world),
            "stats": {"exchange": "NCCL all-reduce (SUM) of the reached rows' packed gradient "
                                  "(fixed capacity) + MAX all-reduce of the union frustum and "
                                  "reached masks; replicated sparse Adam",
                      "packed_rows_on_wire": int(getattr(step, "packed_rows", 0)),
                      "reached_rows_this_rank": reached,
                      "validity_checks": "lazy: pinned flag checked 2 steps later, flush() "
                                         "inside the timed region",
                      "cuda_graph": bool(step.graphs),
                      # host time to enqueue a step vs its device time: with the
                      # graph replay the host runs ahead of the GPU
                      "host_enqueue_ms_per_step": round(host_ms / args.steps, 4),
                      "device_ms_per_step": round(ms / args.steps, 4),
                      "parallelism": f"keyframe-batch dp{world}"},
            "e2e": {"value": round(e2e_val, 3), "unit": UNIT,
                    "h2d_bytes_per_step": sum(int(g.numel() * 4) for g in gt_host) * world,
                    "d2h_bytes_per_step": int(out_host.numel() * 8) * world,
                    "api": "Mapper.upload_image + PackedBatchStep.step (DeviceBatchCompute)"},
            # per view: gate 1, preprocess 1, binning 11, blend 2, loss 4, backward 2,
            # gather 2, chain accumulate 2, exposure 1; per step: pack 1, unpack 1,
            # Adam 2 (+ NCCL's own)
            "gpu_launches": (26 * len(entries) + 4) * args.steps, "clocks": clk.summary(),
            "loss_last": float(logs[-1][0][0].item()),
        }
        del mp, step
        torch.cuda.empty_cache()
        if nested:
            return {k: line[k] for k in ("value", "ms_per_step", "e2e", "stats", "gpu_launches")}
        if rank == 0:
            emit(line)
        return None
    finally:
        if own_pg:
            tdist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU oracle arm (the reference algorithm restated in C, oracle/)
# ---------------------------------------------------------------------------
def _oracle_state(scene):
    from oracle import oracle as o
    o.build()
    o.set_threads(os.cpu_count() or 1)   # torchrun defaults OMP_NUM_THREADS to 1
    gm = {"positions": scene.arrays[0].copy(), "log_scales": scene.arrays[1].copy(),
          "rotations": scene.arrays[2].copy(), "opacity_logits": scene.arrays[3].copy(),
          "sh_coeffs": scene.arrays[4].copy(), "is_sky": scene.arrays[5]}
    arrs = [gm[k] for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")]
    adam = {"m": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "v": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "steps": np.zeros(scene.n, np.int64)}
    return o, gm, adam


def _oracle_step_fn(scene, world=1):
    """One step of the workload on the CPU oracle: the reference's mapping
    iteration (world 1), or the batched step of ``world`` views -- every
    view's backward + chain rule summed, one sparse Adam over the union of the
    frustum masks, each view's exposure ScalarAdam (SURVEY §8e's batched
    oracle)."""
    o, gm, adam = _oracle_state(scene)
    from paper_2404_06926_b200.synthetic import default_lrs
    lrs = default_lrs()
    if world == 1:
        cam = o.Camera(W=scene.W, t=scene.t, fx=scene.fx, fy=scene.fy, cx=scene.cx, cy=scene.cy,
                       width=scene.width, height=scene.height)
        E = scene.E.copy()
        ex = o.ScalarAdam((3, 4), 1e-2)
        return lambda: o.optimize_step(gm, adam, lrs, cam, scene.image, E, ex)
    cams, Es, exs = [], [], []
    for r in range(world):
        yaw = 0.02 * (r - (world - 1) / 2.0)
        R = np.array([[np.cos(yaw), 0, np.sin(yaw)], [0, 1, 0], [-np.sin(yaw), 0, np.cos(yaw)]])
        cams.append(o.Camera(W=R, t=np.zeros(3), fx=scene.fx, fy=scene.fy, cx=scene.cx,
                             cy=scene.cy, width=scene.width, height=scene.height))
        Es.append(scene.E.copy())
        exs.append(o.ScalarAdam((3, 4), 1e-2))

    def step():
        total, active = None, np.zeros(scene.n, bool)
        for cam, E, ex in zip(cams, Es, exs):
            screen, (pg, _, off), tg = o.render_view(gm, cam)
            _, d_r, d_E, _ = o.photometric_loss(tg["color"], scene.image.astype(np.float32), E,
                                                0.2)
            adj = o.backward_tiles(pg, off, screen, d_r, tg["color"], cam.width, cam.height)
            g = o.chain(adj, screen, gm, cam)
            total = g if total is None else {k: total[k] + g[k] for k in g}
            active |= o.frustum_mask(cam, gm["positions"])
            ex.step(E, d_E)
        params = {"position": gm["positions"], "log_scale": gm["log_scales"],
                  "rotation": gm["rotations"], "opacity_logit": gm["opacity_logits"],
                  "sh": gm["sh_coeffs"]}
        grads = {"position": total["d_position"], "log_scale": total["d_log_scale"],
                 "rotation": total["d_rotation"], "opacity_logit": total["d_opacity_logit"],
                 "sh": total["d_sh"]}
        o.adam_step(params, grads, adam["m"], adam["v"], adam["steps"], lrs, active=active)
    return step


def cpu_baseline(scene, samples=2, cfg_idx=3):
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    step = _oracle_step_fn(scene)
    t0 = time.perf_counter()
    for _ in range(samples):
        step()
    dt = time.perf_counter() - t0
    return {"value": round(samples / dt, 5), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{samples} full config-{cfg_idx} mapping steps of the C oracle "
                      f"(oracle/splat_oracle.c; blend OpenMP over {cores} threads, backward "
                      f"serial as the reference)",
            "seconds": round(dt, 2)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.config == 5:
        emit({"impl": "reference", "unavailable": "config 5 (a 4M-Gaussian map, 8 "
                                                  "views per step) takes minutes per step on "
                                                  "the CPU oracle; the reference arm times "
                                                  "configs 1-3"})
        return
    scene = scene_of(args.config)
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    step = _oracle_step_fn(scene, world)
    # bounded sample: one warm-up, then as many full steps (of `world` views
    # each) as fit ~60 s, at most --steps
    n_warm = min(args.warmup, 1)
    for _ in range(n_warm):
        step()
    times = []
    budget = 60.0
    while len(times) < args.steps and (not times or sum(times) < budget):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    n_steps = len(times)
    total = float(sum(times))
    value = n_steps * world / total
    sample = (f"{n_steps} timed full steps ({world} view(s) each) of the C oracle after {n_warm} "
              f"warm-up; bounded to ~{budget:.0f} s of --steps {args.steps}")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT,
            "n_gpus": world, "steps": n_steps, "warmup": n_warm,
            "ms_per_step": round(1e3 * total / n_steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": data_note(args.config), "config": config_dict(scene, args.config, world),
            "stats": {"parallelism": f"{cores} host cores (blend OpenMP, backward serial)"},
            "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(n):
    """``--gpus N`` without a torchrun environment: run this same command as N
    ranks (one per GPU) under torch.distributed.run and pass its output on."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--batched", action="store_true",
                    help="print the keyframe-batch step's line even at one GPU")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batched", action="store_true",
                    help="N = 1: skip the keyframe-batch leg")
    ap.add_argument("--no-batched-graphs", action="store_true",
                    help="keyframe batch: eager launches instead of the captured graph")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    _guard_stdout()
    world = int(env_world or "1")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch "
                         f"{args.gpus} ranks (torchrun) or pass --gpus {world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # NCCL's version/init lines go to stderr: stdout carries the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if world == 1 and not args.batched:
        run_ours(args, local_rank)
        return
    import torch
    import torch.distributed as tdist
    # NCCL's init lines (comm ranks, transport) on stderr for the record
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local_rank)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_batched(args, rank, world, local_rank)
    finally:
        if tdist.is_initialized():
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
