"""The mapping iteration as one device pipeline (a1-a10, mapper.py:299-328).

``MappingEngine.step`` runs Mapper._optimize_step's sequence on one stream
with persistent, capacity-sized buffers:

  K1+K2  sb_preprocess_fwd   frustum mask + projection, map-indexed records
  K3-K5  sb_bin              depth sort, cull+count+tile histogram, scan, place
  K6     sb_blend_fwd        blend + exposure epilogue (Y = M C + b)
  K7     sb_loss_fused       L1 + D-SSIM, dY -> d_rendered, dE (f64)
  K8     sb_blend_bwd_det    termination-aware replay, shuffle-reduced per-(tile,
                             row) sums merged per row in tile order (deterministic)
  K9+K10 sb_chain_adam_rows  chain rule + frustum-sparse Adam
  K11    sb_exposure_adam    ScalarAdam in f64 on the device
  log    sb_psnr8_sse        psnr_8bit of clip(exposure(C)) for the training log

After the first step of a map (which reads the pair count P once to size the
pair buffers), binning keeps P on the device: no host synchronisation, so the
whole iteration is captured once per keyframe as a CUDA graph and replayed.
A pair-capacity overflow makes the iteration a no-op on the device (the
update kernels check the status word); the host sees it in the log row and
re-runs the step with larger buffers.

Log row (float64[8], device): loss, l1, dssim, ssim, -, sse (int64),
P (int64), overflow (int64).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .adam import AdamState, lr_vector
from .forward import run_bin, run_blend_fwd
from .loss import run_loss
from .scene import GaussianMap

LOG_WIDTH = 8


class DeviceExposure:
    """Per-keyframe exposure affine E = [M | b] (float64 master copy) and its
    ScalarAdam state, both on the device (loss.py:17-28, adam.py:125-140)."""

    def __init__(self, matrix=None, dtype=torch.float32, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        m = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) if matrix is None else matrix
        self.mat = torch.as_tensor(np.asarray(m, np.float64).reshape(12)).to(dev)
        self.real = self.mat.to(dtype)
        self.state = torch.zeros(25, dtype=torch.float64, device=dev)

    @property
    def matrix(self) -> np.ndarray:
        return self.mat.cpu().numpy().reshape(3, 4)

    @matrix.setter
    def matrix(self, value):
        self.mat.copy_(torch.as_tensor(np.asarray(value, np.float64).reshape(12)))
        self.real.copy_(self.mat.to(self.real.dtype))


class MappingEngine:
    def __init__(self, dtype=torch.float32):
        self.dtype = dtype
        self.bufs: dict = {}
        self.binout: dict = {}
        self.fwd: dict = {}
        self.loss: dict = {}
        self.pair_cap = 0          # device-binning capacity (0: not sized yet)
        self.sort_cap = 0          # sb_bin sort_capacity (0: sort all rows)
        self.render_cap = 0        # pair capacity of the render path (0: size it)
        self.render_sized = None
        self.rfwd: dict = {}       # the render path's blend outputs
        self.sortable_max = 0      # most rows with a valid depth key seen at a sizing
        self.sized_for = None      # (n, W, H) the capacity was sized for
        self.identity = None
        self.tail_mode = 0         # 0: chain kernel + flat Adam kernel; 1: fused smem kernel
        self.graphs: dict = {}
        self.graph_drops: dict = {}    # why captured graphs were dropped (counts)
        self.captures = 0
        self.seen: set = set()     # keyframes (caps keys) stepped at the current sizing
        self.caps: dict = {}
        self.stamps: dict = {}     # depth-limit key -> device int64[1] (sb_depth_limits_gate)
        self.scheds: dict = {}     # key -> heavy-first tile schedule (blend_common.cuh)
        # keys whose limited iteration was once invalid: they bin full lists
        # from then on (a map whose tiles keep failing the depth-limit check,
        # e.g. low-opacity seeds, pays full binning instead of re-runs)
        self.full_list_keys: set = set()
        self.clock = None          # device int64[1]: map updates so far (the gate's clock)
        self.halt = None           # device int64[1]: set by an invalid iteration
        self.use_caps = True       # truncate tile lists behind the previous saturation depth
        # deterministic backward (sb_blend_bwd_det): bitwise reproducible steps;
        # False selects the float-atomic sb_blend_bwd (A/B timing only)
        self.deterministic = True
        # the step's forward takes alpha from the hardware exp (the one the
        # backward replays with; sb_blend_fwd fast_exp); the render path keeps
        # the correctly rounded exp (bit-identical to the reference pipeline)
        self.fast_exp = True
        # the Adam tail skips active rows with all-zero moments and no
        # gradient (an exact identity update; AdamState.touched).  False: the
        # element pass over every active row (A/B timing only)
        self.touched_skip = True
        self.last = None
        # side stream for the work off the critical path (adjoint zeroing,
        # exposure Adam, PSNR); forked and joined with events, so the
        # dependencies are captured into the CUDA graph as well
        self._side = None

    def _side_stream(self):
        if self._side is None:
            self._side = (torch.cuda.Stream(), [torch.cuda.Event() for _ in range(4)])
        return self._side

    # --- buffers ---------------------------------------------------------------
    def _buf(self, name, shape, dtype, zero=False):
        dev = torch.device("cuda", torch.cuda.current_device())
        t = self.bufs.get(name)
        need = int(np.prod(shape))
        if t is None or t.numel() < need or t.dtype != dtype:
            rows = shape[0]
            grow = (max(int(rows * 1.25), rows),) + tuple(shape[1:])
            t = (torch.zeros if zero else torch.empty)(grow, dtype=dtype, device=dev)
            self.bufs[name] = t
            self._drop_graphs("buf:" + name)
        return t.reshape(-1)[:need].reshape(shape)

    def _drop_graphs(self, why):
        if self.graphs:
            self.graph_drops[why] = self.graph_drops.get(why, 0) + 1
        self.graphs.clear()

    def _scratch(self, name, nbytes):
        """Engine-owned byte workspace (grow-only; growth drops the graphs
        that captured the old pointer)."""
        return self._buf("ws_" + name, (max(int(nbytes), 256),), torch.uint8)

    def invalidate(self, keep_limits: bool = False):
        """Drop captured graphs and the pair sizing (map growth, new shapes).
        ``keep_limits`` keeps the per-keyframe tile depth limits: they are
        per-tile depths, independent of the map's rows, and every limited tile
        is re-validated by the next forward blend, so they stay sound when
        Gaussians are appended (map growth)."""
        self._drop_graphs("invalidate")
        self.seen.clear()
        self.pair_cap = 0
        self.sized_for = None
        if not keep_limits:
            self.caps.clear()

    def _halt(self, dev):
        if self.halt is None or self.halt.device != dev:
            self.halt = torch.zeros(1, dtype=torch.int64, device=dev)
        return self.halt

    def resume(self):
        """Clear the halt left by an invalid iteration and drop the pair
        sizing, so the next iteration bins synchronously with full lists."""
        if self.halt is not None:
            self.halt.zero_()
        self.invalidate()

    def _depth_limits(self, key, W, H, dev):
        """Per-keyframe tile depth limits (float32[n_tiles], +inf = full list)
        and their 4x4-tile maxima (the coarse grid sb_preprocess_fwd drops
        rows with): written by the forward blend of one iteration, read by the
        next iteration of the same keyframe (sb_bin / sb_blend_fwd)."""
        tx, ty = (W + 15) // 16, (H + 15) // 16
        n_tiles, cells = tx * ty, ((tx + 3) // 4) * ((ty + 3) // 4)
        t = self.caps.get(key)
        if t is None or t.numel() != n_tiles + cells:
            t = torch.full((n_tiles + cells,), float("inf"), dtype=torch.float32, device=dev)
            self.caps[key] = t
        return t[:n_tiles], t[n_tiles:]

    def _sort_bound(self, keys, n):
        """sb_bin's sort_capacity: when the rows that can have pairs (a valid
        depth key) are a minority of the map -- a view of a large map --
        sort only those, in a bound with 30% headroom over the largest count
        seen (never shrinking); 0 (sort all rows) otherwise."""
        sortable = int((keys[:n] != -1).sum().item())
        self.sortable_max = max(self.sortable_max, sortable)
        bound = int(self.sortable_max * 1.3) + 4096
        return bound if bound < int(0.8 * n) else 0

    def _sched(self, key, W, H, dev):
        """Per-keyframe heavy-first tile schedule (sb_blend_fwd's tile_sched):
        each keyframe's forward is ordered by its own previous replay lengths."""
        n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
        t = self.scheds.get(key)
        if t is None or t.numel() != 3 * n_tiles or t.device != dev:
            t = torch.zeros(3 * n_tiles, dtype=torch.int32, device=dev)
            self.scheds[key] = t
        return t

    # --- one iteration -----------------------------------------------------------
    def step(self, gmap: GaussianMap, adam: AdamState, pose, intr, gt, gt8, exposure,
             lam=0.2, near=0.01, margin=0.1, dilation=0.3, early=True, thresh=1e-4,
             lr_exposure=1e-2, update_exposure=True, log_out=None, graph_key=None,
             caps_key=None):
        """One mapping iteration; returns the device log row (float64[8]).
        With ``graph_key`` the iteration is captured as a CUDA graph on first
        use and replayed afterwards (same map size, pose, buffers).
        ``caps_key`` names the keyframe whose depth limits and tile schedule
        the iteration uses (default: graph_key) -- one keyframe may own
        several graphs (e.g. one per target-image buffer)."""
        n = gmap.count
        shape_key = (n, intr.width, intr.height)
        if self.sized_for != shape_key:
            # growth keeps the depth limits when the image size is unchanged
            self.invalidate(keep_limits=self.sized_for is not None
                            and self.sized_for[1:] == shape_key[1:])
        if log_out is None:
            log_out = torch.empty(LOG_WIDTH, dtype=torch.float64, device=gmap.positions.device)
        if self._skips():
            adam.touched()         # rebuild the touched-row mask now, never inside a capture
        args = (gmap, adam, pose, intr, gt, gt8, exposure, lam, near, margin, dilation, early,
                thresh, lr_exposure, update_exposure,
                caps_key if caps_key is not None else
                ("eager" if graph_key is None else graph_key))
        kf_key = args[-1]          # the keyframe (caps key) this graph belongs to
        if self.pair_cap == 0:
            # first step of this map: read P once, size the pair buffers
            self._step(*args, log_out, sync_bin=True)
            self.sized_for = shape_key
            self.seen.add(kf_key)
            return log_out
        if graph_key is None:
            self._step(*args, log_out, sync_bin=False)
            return log_out
        g = self.graphs.get(graph_key)
        if g is None and kf_key not in self.seen:
            # a keyframe's graphs are captured from its second use at this
            # sizing on: a stream whose keyframes each run once between growths
            # (optimize_map over a growing store) never pays a capture and its
            # sync, while a keyframe stepped repeatedly gets a graph per target
            # buffer right away
            self.seen.add(kf_key)
            self._step(*args, log_out, sync_bin=False)
            return log_out
        if g is None:
            glog = torch.empty(LOG_WIDTH, dtype=torch.float64, device=log_out.device)
            # one eager pass sizes every buffer outside the capture
            self._step(*args, glog, sync_bin=False)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self._step(*args, glog, sync_bin=False)
            g = (graph, glog)
            self.graphs[graph_key] = g
            self.captures += 1
            log_out.copy_(glog)
            return log_out
        graph, glog = g
        graph.replay()
        log_out.copy_(glog)
        return log_out

    def _step(self, gmap, adam, pose, intr, gt, gt8, exposure, lam, near, margin, dilation,
              early, thresh, lr_exposure, update_exposure, caps_key, log, sync_bin):
        dt = self.dtype
        code = N.dtype_code(dt)
        n = gmap.count
        W, H = intr.width, intr.height
        dev = gmap.positions.device
        st = N.stream_ptr()
        arrays = gmap.arrays()
        cam = N.camera(pose, intr)
        rec = self._buf("records", (max(n, 1), N.RECORD_REALS), dt)
        valid = self._buf("valid", (max(n, 1),), torch.uint8)
        keys = self._buf("keys", (max(n, 1),), torch.int64 if dt == torch.float64 else torch.int32)
        vals = self._buf("vals", (max(n, 1),), torch.int32)
        frustum = self._buf("frustum", (max(n, 1),), torch.uint8)
        status = log[6:8].view(torch.int64)
        if exposure is None:
            if self.identity is None or self.identity.real.dtype != dt:
                self.identity = DeviceExposure(dtype=dt, device=dev)
            exposure = self.identity
        caps, coarse = (self._depth_limits(caps_key, W, H, dev)
                        if self.use_caps and caps_key not in self.full_list_keys
                        else (None, None))
        # the gate: this iteration is one more map update; limits recorded
        # before another keyframe's update are stale and reset on the device
        # (graph-safe).  Without limits the clock still advances.
        if self.clock is None or self.clock.device != dev:
            self.clock = torch.zeros(1, dtype=torch.int64, device=dev)
        if caps is not None:
            if sync_bin:
                caps.fill_(float("inf"))    # full lists this time
                coarse.fill_(float("inf"))
            stamp = self.stamps.get(caps_key)
            if stamp is None or stamp.device != dev:
                stamp = torch.full((1,), -(1 << 40), dtype=torch.int64, device=dev)
                self.stamps[caps_key] = stamp
            allc = self.caps[caps_key]
            N.call("sb_depth_limits_gate", N.ptr(allc), allc.numel(), N.ptr(self.clock),
                   N.ptr(stamp), 1, st)
        else:
            N.call("sb_depth_limits_gate", None, 0, N.ptr(self.clock), None, 1, st)
        # K1 + K2 (rows behind every depth limit under their box are dropped)
        N.call("sb_preprocess_fwd", code, n, *[N.ptr(arrays[k]) for k in (
            "positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")], None,
            N.C.byref(cam), float(near), float(dilation), float(margin), N.ptr(rec),
            N.ptr(valid), N.ptr(keys), N.ptr(vals), N.ptr(frustum), None, N.ptr(coarse), st)
        # K3-K5
        if sync_bin:
            pg, pt, off, P = run_bin(dt, n, rec, valid, keys, vals, W, H, True,
                                     max(4 * n, 1024), scratch=self._scratch_adapter(),
                                     out=self.binout)
            # headroom for the other keyframes replayed at this sizing
            self.pair_cap = int(P * 1.5) + 65536
            self.sort_cap = self._sort_bound(keys, n)
            status.copy_(torch.tensor([P, 0], dtype=torch.int64))
        else:
            # an invalid iteration (pair overflow, failed depth limit) halts the
            # engine: the iterations queued behind it are device no-ops too
            # (sb_bin or-s the halt flag into their status, sb_blend_fwd sets
            # it), so the host can re-run all of them in order
            # (Mapper._materialise)
            pg, pt, off = self._bin_async(dt, n, rec, valid, keys, vals, W, H, status, caps,
                                          halt=self._halt(dev))
        halt = self._halt(dev)
        d_status = status
        main = torch.cuda.current_stream()
        side, ev = self._side_stream()
        # side: zero the screen-space adjoint buffers while the forward runs
        dm = self._buf("d_mean2d", (max(n, 1), 2), dt)
        dc = self._buf("d_conic", (max(n, 1), 3), dt)
        do = self._buf("d_opacity", (max(n, 1),), dt)
        dcol = self._buf("d_color", (max(n, 1), 3), dt)
        ev[0].record(main)
        side.wait_event(ev[0])
        with torch.cuda.stream(side):
            # the deterministic backward's gather lists the reached rows: the
            # chain rule reads no other row's adjoints, so nothing to zero
            if not (self.deterministic and self.tail_mode == 0):
                for t in (dm, dc, do, dcol):
                    N.call("sb_memset_async", N.ptr(t), 0, t.numel() * t.element_size(),
                           N.stream_ptr(side))
            ev[1].record(side)
        # K6 + exposure epilogue
        if coarse is not None:   # the forward re-derives the coarse maxima
            N.call("sb_memset_async", N.ptr(coarse), 0, coarse.numel() * 4, st)
        o = run_blend_fwd(dt, rec, pg, off, W, H, early, thresh, exposure.real, out=self.fwd,
                          depth_limit=caps, status=d_status, coarse_limit=coarse,
                          sched=self._sched(caps_key, W, H, dev), halt=halt,
                          fast_exp=self.fast_exp and dt == torch.float32)
        # K7 (loss parts straight into the log row)
        self.loss["parts"] = log[0:4]
        lo = run_loss(o["color"], gt, exposure.real, lam, y=o["y"], out=self.loss)
        # side: K11 exposure Adam and the training-log PSNR (mapper.py:319-327,
        # with the updated exposure) overlap the backward and the map update
        ev[2].record(main)
        side.wait_event(ev[2])
        with torch.cuda.stream(side):
            sst = N.stream_ptr(side)
            if update_exposure and exposure is not self.identity:
                N.call("sb_exposure_adam", code, N.ptr(exposure.mat), N.ptr(exposure.real),
                       N.ptr(lo["d_E"]), N.ptr(exposure.state), float(lr_exposure),
                       N.ptr(d_status), sst)
            sse = log[5:6].view(torch.int64)
            N.call("sb_memset_async", N.ptr(sse), 0, 8, sst)
            if gt8 is not None:
                N.call("sb_psnr8_sse", code, W * H, N.ptr(o["color"]), N.ptr(exposure.real),
                       N.ptr(gt8), N.ptr(sse), sst)
            ev[3].record(side)
        # K8
        main.wait_event(ev[1])
        self._backward(code, rec, pg, off, W, H, early, thresh, lo["d_rendered"], o,
                       (dm, dc, do, dcol), st)
        # K9 + K10
        G = adam.groups({"position": arrays["positions"], "log_scale": arrays["log_scales"],
                         "rotation": arrays["rotations"], "opacity_logit": arrays["opacity_logits"],
                         "sh": arrays["sh_coeffs"]}, None)
        lrs = lr_vector(adam.lrs)
        ws = self._scratch("chain_adam", N.load().sb_chain_adam_workspace_bytes(code, n))
        # the touched-row skip (exact; sb_chain_adam_rows): the mask is fresh
        # here -- step() rebuilt it outside any graph capture
        touched = adam.touched() if self._skips() else None
        # the gather's reached-row flags replace the adjoint test; the chain
        # rule walks chain_flags' own list, in row order (better locality for
        # its row reads than the gather's depth order)
        rows = self._reach(n) if self.deterministic and self.tail_mode == 0 else None
        N.call("sb_chain_adam_rows", code, n, N.ptr(valid), N.ptr(frustum), N.C.byref(cam),
               float(dilation), N.ptr(dm), N.ptr(dc), N.ptr(do), N.ptr(dcol), N.C.byref(G),
               N.ptr(adam._steps), N.ptr(touched), N.ptr(rows),
               lrs.ctypes.data_as(N.vp), N.ptr(ws), ws.numel(), self.tail_mode,
               N.ptr(d_status), st)
        if touched is None:
            adam.moments_written()
        main.wait_event(ev[3])
        self.last = {"targets": o, "loss": lo, "frustum": frustum[:n], "valid": valid[:n],
                     "status": status, "depth_limit": caps}

    def _skips(self) -> bool:
        return self.touched_skip and self.tail_mode == 0

    def _backward(self, code, rec, pg, off, W, H, early, thresh, d_rendered, o, adj, st):
        """K8 over the pairs of this engine's last sb_bin call: the
        deterministic backward (the binning's pair slot map merges each row's
        per-tile sums in tile order), or the float-atomic one."""
        dm, dc, do, dcol = adj
        if not self.deterministic:
            N.call("sb_blend_bwd", code, N.ptr(rec), N.ptr(pg), N.ptr(off), W, H, 16, int(early),
                   float(thresh), N.ptr(d_rendered), N.ptr(o["color"]), N.ptr(o["last"]),
                   N.ptr(dm), N.ptr(dc), N.ptr(do), N.ptr(dcol), N.ptr(o["sched_used"]), st)
            return
        b = self.binout
        ws = self._scratch("bwd", N.load().sb_blend_bwd_workspace_bytes(code, b["bin_cap"], W, H))
        # sb_blend_bwd_det in its two launches (timed separately by bench.py)
        N.call("sb_blend_bwd_partials", code, N.ptr(rec), N.ptr(pg), N.ptr(off), W, H, 16,
               int(early), float(thresh), N.ptr(d_rendered), N.ptr(o["color"]),
               N.ptr(o["last"]), N.ptr(o["sched_used"]), b["bin_m"], b["bin_cap"],
               N.ptr(b["bin_ws"]), N.ptr(ws), ws.numel(), st)
        rows = self._reach(b["bin_m"]) if self.tail_mode == 0 else None
        N.call("sb_gather_adjoints", code, b["bin_m"], b["bin_cap"], W, H, b["bin_sort_cap"],
               N.ptr(b["bin_ws"]), N.ptr(ws), ws.numel(), N.ptr(dm), N.ptr(dc), N.ptr(do),
               N.ptr(dcol), N.ptr(rows), st)

    def _reach(self, n):
        """The gather's reached-row flags (sb_gather_adjoints): a byte per
        row, kept zero between steps (sb_chain_adam_rows clears what it
        reads)."""
        return self._buf("reach_rows", (max(n, 1),), torch.uint8, zero=True)

    def _scratch_adapter(self):
        eng = self

        class _S:
            @staticmethod
            def get(name, nbytes, device):
                return eng._scratch(name, nbytes)
        return _S

    # --- render only (mapper.py:202-212, the render-FPS path) ---------------------
    def render(self, gmap: GaussianMap, pose, intr, key="render", near=0.01, margin=0.1,
               dilation=0.3, early=True, thresh=1e-4, select=None, status=None):
        """Project + bin + blend one view with no host synchronisation:
        device binning into the engine's pair buffers (sized once, like the
        step), the view's own tile depth limits and heavy-first schedule.
        Renders do not change the map, so they do not advance the gate's
        clock: a view rendered again before the map changes twice keeps its
        limits.  ``status`` (device int64[2]) receives [P, invalid]; an invalid
        render (pair overflow, or a limited tile that did not terminate) must
        be redone with ``render(..., key=None)`` (full lists) -- see
        Mapper.render_image, which checks.  Returns the blend outputs
        (color, depth, transmittance, opacity, n_contrib, last)."""
        dt = self.dtype
        code = N.dtype_code(dt)
        n = gmap.count
        W, H = intr.width, intr.height
        dev = gmap.positions.device
        st = N.stream_ptr()
        arrays = gmap.arrays()
        cam = N.camera(pose, intr)
        rec = self._buf("r_records", (max(n, 1), N.RECORD_REALS), dt)
        valid = self._buf("r_valid", (max(n, 1),), torch.uint8)
        keys = self._buf("r_keys", (max(n, 1),), torch.int64 if dt == torch.float64 else torch.int32)
        vals = self._buf("r_vals", (max(n, 1),), torch.int32)
        if status is None:
            status = torch.zeros(2, dtype=torch.int64, device=dev)
        if self.clock is None or self.clock.device != dev:
            self.clock = torch.zeros(1, dtype=torch.int64, device=dev)
        caps = coarse = None
        if key is not None and self.use_caps:
            caps_all = self._depth_limits(("render", key), W, H, dev)
            caps, coarse = caps_all
            allc = self.caps[("render", key)]
            stamp = self.stamps.get(("render", key))
            if stamp is None or stamp.device != dev:
                stamp = torch.full((1,), -(1 << 40), dtype=torch.int64, device=dev)
                self.stamps[("render", key)] = stamp
            N.call("sb_depth_limits_gate", N.ptr(allc), allc.numel(), N.ptr(self.clock),
                   N.ptr(stamp), 0, st)
        sel = None if select is None else select.to(torch.uint8).contiguous()
        N.call("sb_preprocess_fwd", code, n, *[N.ptr(arrays[k]) for k in (
            "positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")], N.ptr(sel),
            N.C.byref(cam), float(near), float(dilation), float(margin), N.ptr(rec),
            N.ptr(valid), N.ptr(keys), N.ptr(vals), None, None, N.ptr(coarse), st)
        if self.render_cap == 0 or self.render_sized != (n, W, H):
            # first render at this size: full lists, read P once (one sync)
            pg, _, off, P = run_bin(dt, n, rec, valid, keys, vals, W, H, True,
                                    max(4 * n, 1024), scratch=self._scratch_adapter(),
                                    out=self.binout)
            self.render_cap = max(int(P * 1.5) + 65536, self.pair_cap)
            self.render_sized = (n, W, H)
            status.copy_(torch.tensor([P, 0], dtype=torch.int64))
            if caps is not None:
                caps.fill_(float("inf"))
                coarse.fill_(float("inf"))
        else:
            saved, self.pair_cap = self.pair_cap, self.render_cap
            try:
                pg, _, off = self._bin_async(dt, n, rec, valid, keys, vals, W, H, status, caps)
            finally:
                self.pair_cap = saved
        if coarse is not None:
            N.call("sb_memset_async", N.ptr(coarse), 0, coarse.numel() * 4, st)
        return run_blend_fwd(dt, rec, pg, off, W, H, early, thresh, None, out=self.rfwd,
                             depth_limit=caps, status=status, coarse_limit=coarse,
                             sched=self._sched(("render", key), W, H, dev))

    def _bin_async(self, dt, n, rec, valid, keys, vals, W, H, status, caps=None, halt=None):
        dev = rec.device
        cap = self.pair_cap
        n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
        b = self.binout
        if b.get("async_cap", 0) < cap:   # grow only: the render path may size it larger
            b["a_pg"] = torch.empty(cap, dtype=torch.int32, device=dev)
            b["async_cap"] = cap
            self._drop_graphs("pair_cap")
        if b.get("offsets") is None or b["offsets"].numel() != n_tiles + 1:
            b["offsets"] = torch.empty(n_tiles + 1, dtype=torch.int32, device=dev)
        lib = N.load()
        ws = self._scratch("bin", lib.sb_bin_workspace_bytes(n, cap, W, H))
        npairs = N.C.c_int64(0)
        N.check(lib.sb_bin(N.dtype_code(dt), n, N.ptr(rec), N.ptr(valid), N.ptr(keys),
                           N.ptr(vals), W, H, 16, 1, cap, N.ptr(b["a_pg"]), None,
                           N.ptr(b["offsets"]), N.C.byref(npairs), N.ptr(ws), ws.numel(),
                           N.ptr(status), N.ptr(caps), self.sort_cap, N.ptr(halt), N.stream_ptr()),
                "sb_bin")
        b.update(bin_ws=ws, bin_m=n, bin_cap=cap, bin_sort_cap=self.sort_cap)
        # blend/backward read the CSR offsets, never past them
        return b["a_pg"], None, b["offsets"]


def log_dict(row: np.ndarray, npx: int) -> dict:
    """Host view of a device log row (metrics.py:16-27 PSNR convention)."""
    ints = np.asarray(row[5:8]).view(np.int64)
    mse = int(ints[0]) / (3.0 * npx)
    psnr = 99.0 if mse == 0.0 else min(10.0 * math.log10(255.0 ** 2 / mse), 99.0)
    return {"l1": float(row[1]), "dssim": float(row[2]), "loss": float(row[0]), "psnr": psnr,
            "n_pairs": int(ints[1]), "overflow": bool(ints[2])}


def quantize_8bit(img) -> np.ndarray:
    """metrics.py:12-13."""
    a = np.asarray(img)
    return np.clip(np.round(np.clip(a, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)
