"""Keyframe-batch data parallelism across GPUs.

One process per GPU holds a replica of the map and its Adam state.  A batch
step over views V = V_0 u V_1 u ... (rank r owns V_r):

  1. every rank renders, scores and back-propagates its own views, summing the
     map-layout gradients into one flat buffer (59 reals per Gaussian) and
     OR-ing the views' frustum masks (a1, mapper.py:310-311);
  2. the flat gradient is all-reduced (SUM) and the mask (MAX) with
     torch.distributed -- NCCL over NVLink on the B200s, gloo on CPU tests;
  3. every rank applies the identical sparse Adam step to the union mask
     (a8), so the replicas stay bit-identical;
  4. each view's exposure E (a9) is updated by the rank that owns the view
     (E belongs to one keyframe, so it needs no exchange).

This is a new semantic relative to the reference's sequential per-keyframe
steps (mapper.py:294-295): its oracle is the sum of the reference's per-view
GradientBuffers followed by ONE adam_step over the union of the frustum masks
(tests/test_batch_gloo.py builds exactly that with the CPU oracle).

The compute is pluggable: ``DeviceBatchCompute`` runs the sm_100a kernels;
the CPU tests plug the oracle in to exercise the distributed plumbing.
"""

from __future__ import annotations

import time

import torch
import torch.distributed as dist

from . import _native as N
from .adam import lr_vector
from .forward import _SCRATCH, run_bin, run_blend_fwd
from .loss import run_loss

GROUP_WIDTHS = (("position", (3,)), ("log_scale", (3,)), ("rotation", (4,)),
                ("opacity_logit", ()), ("sh", (16, 3)))
ROW_REALS = 59


def group_views(flat: torch.Tensor, n: int) -> dict:
    """Split a flat (59 n) buffer into map-layout group views."""
    out, off = {}, 0
    for name, shape in GROUP_WIDTHS:
        w = 1
        for s in shape:
            w *= s
        out[name] = flat[off:off + w * n].view((n,) + shape)
        off += w * n
    return out


def _begin(compute, n_pad=None, zero=True):
    """compute.begin; a compute with ``first_touch`` accumulates without a
    zeroed gradient when ``zero`` is False (only the reached rows are valid,
    see _apply)."""
    if getattr(compute, "first_touch", False):
        return compute.begin(n_pad, zero=zero)
    return compute.begin(n_pad)


def _apply(compute, flat, union, grad_rows=None):
    """compute.apply; ``grad_rows`` (uint8[n], first-touch computes): the
    rows whose gradient Adam reads, every other active row taking zero."""
    if getattr(compute, "first_touch", False):
        return compute.apply(flat, union, grad_rows=grad_rows)
    return compute.apply(flat, union)


def _mask_buffer(compute, union):
    """What the MAX all-reduce carries: the union mask, plus whatever flags
    the compute keeps behind it (DeviceBatchCompute: the step's invalid flag)."""
    f = getattr(compute, "mask_buffer", None)
    return f() if f is not None else union


class BatchStep:
    """The exchange step: compute-agnostic host orchestration."""

    def __init__(self, compute, group=None, always_reduce=False, lazy=False):
        self.compute = compute
        self.group = group
        self.always_reduce = always_reduce   # exercise the collective at world size 1
        # lazy: no host sync per step.  The step's (all-reduced) invalid flag
        # is copied to pinned memory and checked `lag` steps later; an invalid
        # step leaves a sticky device flag that turns every later step into a
        # no-op until the host sees it and re-runs them in order.  The check
        # is by step count, so every rank resolves the same step at the same
        # call (the re-runs carry collectives).  Call flush() before reading
        # the map or changing it between steps.
        self.lazy = bool(lazy) and hasattr(compute, "defer_flag")
        self.lag = 2
        self._pending: list = []     # (pinned flag, event, views, logs) per unchecked step
        self._replaying = False
        # CUDA-graph replay of the whole device step (collectives included)
        # once its buffers are sized; see _graph_step
        self.graphs: dict = {}
        self.use_graphs = False

    def flush(self):
        """Resolve every unchecked step (re-running the invalid ones)."""
        while self._pending:
            self._resolve_oldest()

    host_wait_s = 0.0    # host time spent waiting for devices in lazy checks

    def _resolve_oldest(self):
        flag, ev, views, logs = self._pending.pop(0)
        t0 = time.perf_counter()
        ev.synchronize()
        self.host_wait_s += time.perf_counter() - t0
        if not int(flag[0]):
            return
        # invalid: it and every later unchecked step (sticky flag) were no-ops
        redo = [(views, logs)] + [(p[2], p[3]) for p in self._pending]
        self._pending.clear()
        self.compute.reset_deferred()
        self.on_invalid()
        self.graphs.clear()           # the re-runs re-size: captured pointers may change
        self._replaying = True
        try:
            for v, old in redo:
                new = self.step(v)
                for o, nw in zip(old, new):   # the caller's log tensors, rewritten in place
                    o.copy_(nw)
        finally:
            self._replaying = False

    def on_invalid(self):
        """Hook: resize step-owned capacities before invalid steps re-run."""

    def world(self) -> int:
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def exchanges(self) -> bool:
        return self.world() > 1 or (self.always_reduce and dist.is_initialized())

    def step(self, views, _depth=0) -> list:
        c = self.compute
        # lazy validity is per step: re-runs and synchronous steps check now
        deferred = self.lazy and not self._replaying and _depth == 0
        if hasattr(c, "deferred"):
            c.deferred = deferred
        if hasattr(c, "prepare_step"):
            c.prepare_step()
        if deferred and self.use_graphs and self._graphable(views):
            logs = self._graph_step(views)
        else:
            logs = self._device_step(views)
        return self._checked(views, logs, _depth)

    def _device_step(self, views) -> list:
        """begin, every view's forward/backward accumulation, the exchange,
        the sparse Adam step and the exposure updates -- device work only
        (no host synchronisation once the compute is sized)."""
        c = self.compute
        exchange = self.exchanges()
        # without an exchange only the reached rows' gradients are read, so the
        # gradient buffer is never zeroed (first-touch accumulation)
        flat, union = _begin(c, zero=exchange)
        logs = [c.accumulate(v, flat, union) for v in views]
        if exchange:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(_mask_buffer(c, union), op=dist.ReduceOp.MAX, group=self.group)
        rows = None if exchange or not hasattr(c, "reached_mask") else c.reached_mask()[:c.rows()]
        _apply(c, flat, union, rows)
        for v in views:
            c.exposure(v)
        return logs

    # -- CUDA-graph replay ----------------------------------------------------
    def _graph_key(self, views):
        c = self.compute
        # a view's target image is double-buffered (Mapper.upload_image): one
        # graph per buffer
        return (tuple((id(v), getattr(getattr(v, "gt", None), "data_ptr", int)()) for v in views),
                c.rows(), getattr(c, "pair_cap", 0), getattr(c, "sort_cap", 0),
                getattr(self, "k_cap", 0))

    def _graphable(self, views) -> bool:
        """Only a sized compute (device binning, no host reads), on CUDA,
        binning with its depth limits (not a full-list re-run)."""
        c = self.compute
        return (getattr(c, "graphable", False) and c.pair_cap > 0 and not c._full
                and c.sized_for == c.rows())

    def _graph_step(self, views) -> list:
        """Replay the step's captured graph (captured on first use for these
        views at this sizing).  The outputs are the graph's static tensors:
        the caller gets copies."""
        key = self._graph_key(views)
        g = self.graphs.get(key)
        if g is None:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                out = self._device_step(views)
            g = self.graphs[key] = (graph, out)
        graph, out = g
        graph.replay()
        return [t.clone() for t in out]

    def _checked(self, views, logs, _depth=0):
        """A compute that can invalidate a step (DeviceBatchCompute: depth
        limits, pair capacity) made it a no-op on every rank; re-run it."""
        c = self.compute
        if self.lazy and not self._replaying and _depth == 0:
            self._pending.append(c.defer_flag() + (views, logs))
            while len(self._pending) > self.lag:
                self._resolve_oldest()
            return logs
        if hasattr(c, "step_invalid") and c.step_invalid():
            if _depth >= 3:
                raise RuntimeError("batched step invalid after re-runs")
            self.on_invalid()
            self.graphs.clear()
            return self.step(views, _depth + 1)
        return logs


def row_block(n: int, rank: int, world: int):
    """Rows [lo, hi) whose Adam update rank owns, and the padded row count
    n_pad = world * rows (every rank's block has the same size)."""
    # blocks start on a multiple of 8 rows, so every group's block pointer is
    # 16-byte aligned for the vectorised Adam pass
    rows = ((n + world - 1) // world + 7) // 8 * 8
    lo = min(rank * rows, n)
    return lo, min(lo + rows, n), rows * world


class ShardedBatchStep(BatchStep):
    """The §8(e) exchange with the optimizer sharded by rows (ZeRO-1 style):
    after every rank accumulated its views, the per-group gradients are
    reduce-scattered in equal row blocks, each rank runs the sparse Adam step
    on its block only (so the Adam pass costs 1/world of the map), and the
    updated parameter rows (and step counters) are all-gathered.  Same bytes
    on the wire as an all-reduce of the gradient; the union frustum mask is
    all-reduced (MAX) as before.

    The moments m, v stay current only on the owning rank; call
    ``gather_optimizer_state`` before the row blocks change (map growth, a
    different world size)."""

    def rank(self) -> int:
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(self.group)
        return 0

    def step(self, views, _depth=0) -> list:
        c = self.compute
        world, rank = self.world(), self.rank()
        n = c.rows()
        lo, hi, n_pad = row_block(n, rank, world)
        rows = n_pad // world
        flat, union = c.begin(n_pad)
        logs = [c.accumulate(v, flat, union) for v in views]
        full = group_views(flat, n_pad)
        chunks = {}
        for name, shape in GROUP_WIDTHS:
            if world == 1:      # the whole gradient is this rank's block
                chunks[name] = full[name]
                continue
            chunk = torch.empty((rows,) + shape, dtype=flat.dtype, device=flat.device)
            dist.reduce_scatter_tensor(chunk.reshape(-1), full[name].reshape(-1),
                                       op=dist.ReduceOp.SUM, group=self.group)
            chunks[name] = chunk
        if world > 1:
            dist.all_reduce(_mask_buffer(c, union), op=dist.ReduceOp.MAX, group=self.group)
        c.apply_rows(lo, hi, {k: v[: hi - lo] for k, v in chunks.items()}, union)
        if world > 1:
            for t in c.row_tensors(n_pad):
                dist.all_gather_into_tensor(t.reshape(-1), t[lo:lo + rows].reshape(-1).clone(),
                                            group=self.group)
            if hasattr(c, "after_gather"):
                c.after_gather()
        for v in views:
            c.exposure(v)
        return self._checked(views, logs, _depth)

    def gather_optimizer_state(self):
        """Make every rank's Adam moments current for all rows."""
        c, world, rank = self.compute, self.world(), self.rank()
        if world == 1:
            return
        n = c.rows()
        lo, _, n_pad = row_block(n, rank, world)
        rows = n_pad // world
        for t in c.moment_tensors(n_pad):
            dist.all_gather_into_tensor(t.reshape(-1), t[lo:lo + rows].reshape(-1).clone(),
                                        group=self.group)


def _reached(compute, full, n_pad) -> torch.Tensor:
    """uint8[n_pad] rows with a non-zero gradient on this rank: the compute's
    own mask when it keeps one, else a scan of the flat gradient."""
    f = getattr(compute, "reached_mask", None)
    if f is not None:
        return f()[:n_pad].clone()
    dev = next(iter(full.values())).device
    hit = torch.zeros(n_pad, dtype=torch.uint8, device=dev)
    for name, _ in GROUP_WIDTHS:
        hit |= (full[name].reshape(n_pad, -1) != 0).any(dim=1).to(torch.uint8)
    return hit


class PackedBatchStep(BatchStep):
    """The all-reduce exchange with only the reached rows on the wire.  The
    reached masks are OR-ed with the union frustum mask in one MAX
    all-reduce; every rank packs the same reached rows (row order), the
    packed [K, 59] gradient is SUM all-reduced and scattered back into the
    flat gradient (the other rows are zero everywhere), and every rank runs
    the full sparse Adam step itself -- replicated state, no all-gather.  At
    config 5 the 8 views reach 253k of 4M rows: 60 MB instead of 944 MB per
    step, traded against the replicated Adam pass."""

    k_cap = 0        # lazy mode: packed rows on the wire (0: size on the next step)

    def on_invalid(self):
        # a packing overflow (or any invalid step): size the wire for the
        # largest reached count seen (the same all-reduced count on every rank)
        kmax = getattr(self, "_kmax", None)
        if kmax is not None:
            k = int(kmax.item())
            if k > self.k_cap:
                self.k_cap = int(k * 1.25) + 4096

    def _graphable(self, views) -> bool:
        # the sync-free (fixed-capacity) packing only
        return super()._graphable(views) and (not self.exchanges() or self.k_cap > 0)

    def _device_step(self, views) -> list:
        c = self.compute
        exchange = self.exchanges()
        n = c.rows()
        # sync-free packing: a fixed-capacity row list whose spare slots point
        # at the dump row n (zero gradient everywhere, never read by Adam)
        fixed = exchange and self.lazy and not self._replaying and self.k_cap > 0
        # (n_pad a multiple of 8: every group's pointer stays 16-byte aligned)
        n_pad = (n + 8) // 8 * 8 if fixed else n
        first_touch = getattr(c, "first_touch", False)
        # first-touch accumulation: only reached rows hold a gradient, and
        # only those are packed or read by Adam -- the buffer is never zeroed
        flat, union = _begin(c, n_pad, zero=not first_touch)
        logs = [c.accumulate(v, flat, union) for v in views]
        grad_rows = c.reached_mask()[:n] if first_touch else None
        if exchange:
            full = group_views(flat, n_pad)
            reached = _reached(c, full, n_pad)
            mask = _mask_buffer(c, union)
            both = torch.cat([mask, reached])
            dist.all_reduce(both, op=dist.ReduceOp.MAX, group=self.group)
            mask.copy_(both[:mask.numel()])
            hit = both[mask.numel():mask.numel() + n]
            if first_touch:
                grad_rows = hit                # rows some view on some rank reached
            if fixed:
                cap = min(self.k_cap, n)
                pos = torch.nonzero_static(hit, size=cap, fill_value=n).squeeze(1)
                k = hit.sum(dtype=torch.int64).reshape(1)
                if getattr(self, "_kmax", None) is None:
                    self._kmax = torch.zeros(1, dtype=torch.int64, device=k.device)
                torch.maximum(self._kmax, k, out=self._kmax)   # in place: graph-safe
                c.mark_invalid(k > cap)       # overflow: a no-op step, re-run
                self.packed_rows = cap
            else:
                pos = torch.nonzero(hit).squeeze(1)
                self.packed_rows = int(pos.numel())
                if self.lazy:
                    self.k_cap = max(self.k_cap, int(self.packed_rows * 1.25) + 4096)
            if flat.is_cuda:     # one gather / scatter launch each (csrc/exchange.cu)
                code, st = N.dtype_code(flat.dtype), N.stream_ptr()
                packed = torch.empty((pos.numel(), ROW_REALS), dtype=flat.dtype,
                                     device=flat.device)
                # first-touch buffers: a row this rank did not reach packs as zeros
                N.call("sb_pack_rows", code, n_pad, N.ptr(flat), N.ptr(pos), pos.numel(),
                       N.ptr(packed), N.ptr(c.reached_mask() if first_touch else None), st)
                dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=self.group)
                N.call("sb_unpack_rows", code, n_pad, N.ptr(flat), N.ptr(pos), pos.numel(),
                       N.ptr(packed), st)
            else:
                cols = [full[name].reshape(n_pad, -1) for name, _ in GROUP_WIDTHS]
                packed = torch.cat([g[pos] for g in cols], dim=1)
                dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=self.group)
                off = 0
                for g in cols:
                    w = g.shape[1]
                    g[pos] = packed[:, off:off + w]
                    off += w
        _apply(c, flat, union, grad_rows)
        for v in views:
            c.exposure(v)
        return logs


class PackedShardedBatchStep(ShardedBatchStep):
    """ShardedBatchStep that reduce-scatters only the gradient rows some
    view reached.  A row no pixel of any view reached has an exactly zero
    gradient on every rank (the chain rule is linear in the screen-space
    adjoints), so it need not travel.  The reached mask travels with the
    union frustum mask in the same MAX all-reduce; from it every rank derives
    the same packing -- per row block, the reached rows in row order, padded
    to the largest block count C -- and the reduce-scatter moves world x C
    rows instead of the whole map.  Each rank unpacks its block (zeros
    elsewhere) and runs the sparse Adam step on it exactly as
    ShardedBatchStep; the updated rows are all-gathered the same way.  The
    per-row sums are the same rank-ordered sums, so the result equals the
    unpacked exchange (bit for bit at world 2)."""

    def step(self, views, _depth=0) -> list:
        c = self.compute
        world, rank = self.world(), self.rank()
        n = c.rows()
        lo, hi, n_pad = row_block(n, rank, world)
        rows = n_pad // world
        flat, union = c.begin(n_pad)
        logs = [c.accumulate(v, flat, union) for v in views]
        full = group_views(flat, n_pad)
        dev = flat.device
        reached = _reached(c, full, n_pad)
        mask = _mask_buffer(c, union)
        both = torch.cat([mask, reached])
        if world > 1:
            dist.all_reduce(both, op=dist.ReduceOp.MAX, group=self.group)
        mask.copy_(both[:mask.numel()])
        reached = both[mask.numel():]
        # the same packing on every rank
        pos = torch.nonzero(reached).squeeze(1)
        blk = torch.div(pos, rows, rounding_mode="floor")
        counts = torch.bincount(blk, minlength=world)
        cmax = int(counts.max().item()) if pos.numel() else 0
        cpad = max(8, (cmax + 7) // 8 * 8)
        start = torch.cumsum(counts, 0) - counts
        dest = blk * cpad + (torch.arange(pos.numel(), device=dev) - start[blk])
        mine = pos[blk == rank] - rank * rows
        self.packed_rows = world * cpad    # rows on the wire (diagnostics)
        chunks = {}
        for name, shape in GROUP_WIDTHS:
            w = full[name].numel() // n_pad
            src = full[name].reshape(n_pad, w)
            send = torch.zeros((world * cpad, w), dtype=flat.dtype, device=dev)
            send[dest] = src[pos]
            recv = torch.empty((cpad, w), dtype=flat.dtype, device=dev)
            if world > 1:
                dist.reduce_scatter_tensor(recv.reshape(-1), send.reshape(-1),
                                           op=dist.ReduceOp.SUM, group=self.group)
            else:
                recv.copy_(send[:cpad])
            blockg = torch.zeros((rows, w), dtype=flat.dtype, device=dev)
            blockg[mine] = recv[:mine.numel()]
            chunks[name] = blockg.reshape((rows,) + shape)
        c.apply_rows(lo, hi, {k: v[: hi - lo] for k, v in chunks.items()}, union)
        if world > 1:
            for t in c.row_tensors(n_pad):
                dist.all_gather_into_tensor(t.reshape(-1), t[lo:lo + rows].reshape(-1).clone(),
                                            group=self.group)
            if hasattr(c, "after_gather"):
                c.after_gather()
        for v in views:
            c.exposure(v)
        return self._checked(views, logs, _depth)


class DeviceBatchCompute:
    """sm_100a compute for BatchStep over a device Mapper's map.

    Each view runs the engine's per-view pipeline (engine.py): projection
    with the coarse depth-limit drop, device binning without host
    synchronisation (pair buffers sized once per map size), the forward
    blend with the view's tile depth limits and heavy-first schedule, the
    loss, the backward and the compacted chain-rule accumulation.  A view's
    limits stay usable across batched steps (one map update in between, the
    sb_depth_limits_gate clock).  An invalid view (a limited tile that did
    not terminate, or a pair overflow) marks the step invalid: the flag
    travels with the union mask through the exchange, every rank's Adam and
    exposure updates become no-ops, and ``step_invalid`` tells the host to
    re-run the step with full lists."""

    use_limits = True
    first_touch = True     # accumulates without a zeroed gradient (sb_chain_accumulate)
    graphable = True       # sync-free once sized: BatchStep may CUDA-graph the step

    def __init__(self, mapper):
        self.mp = mapper
        self.bufs: dict = {}
        self.binout: dict = {}
        self.fwd: dict = {}
        self.loss: dict = {}
        self.d_E: dict = {}
        self.caps: dict = {}       # id(entry) -> float[n_tiles + coarse cells]
        self.stamps: dict = {}     # id(entry) -> int64[1] (gate stamps)
        self.clock = None          # int64[1]: batched map updates (gate clock)
        self.pair_cap = 0          # async binning capacity (0: size on this step)
        self.sort_cap = 0          # sb_bin sort_capacity (0: sort all rows)
        self._smax = 0             # most sortable rows (valid depth key) of a view
        self.sized_for = None
        self._pmax = 0
        self._full = False         # this step bins full lists (re-run of an invalid step)

    def _buf(self, name, shape, dtype):
        t = self.bufs.get(name)
        numel = 1
        for s in shape:
            numel *= s
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=self.mp.map.positions.device)
            self.bufs[name] = t
        return t.reshape(-1)[:numel].reshape(shape)

    def rows(self) -> int:
        return self.mp.map.count

    def begin(self, n_pad: int | None = None, zero: bool = True):
        """Per step.  zero=False: the gradient buffer is not cleared -- each
        view's chain rule stores a row's gradient on its first touch and adds
        later (sb_chain_accumulate first_touch), and only the reached rows
        (reached_mask) may be read: pass them to apply(grad_rows=...)."""
        n = self.mp.map.count
        self.n_pad = n if n_pad is None else n_pad
        dt = self.mp.dtype
        flat = self._buf("grad", (ROW_REALS * self.n_pad,), dt)
        # union frustum mask [n] + the step's invalid flag [1], exchanged together
        ub = self._buf("union", (n + 1,), torch.uint8)
        st = N.stream_ptr()
        self._zeroed = bool(zero)
        if zero:
            N.call("sb_memset_async", N.ptr(flat), 0, flat.numel() * flat.element_size(), st)
        N.call("sb_memset_async", N.ptr(ub), 0, ub.numel(), st)
        self.bad = self._buf("bad", (2,), torch.int64)
        self.bad.zero_()
        if self.deferred:     # an earlier unchecked step was invalid: stay a no-op
            self.bad[1:2].copy_(self._sticky_flag())
        self._reached = self._buf("reached", (self.n_pad,), torch.uint8)
        N.call("sb_memset_async", N.ptr(self._reached), 0, self.n_pad, st)
        self._first = True
        self._n = n
        if self.sized_for != n:
            self.pair_cap, self._pmax, self.sized_for = 0, 0, n
        self._ub = ub
        return flat, ub[:n]

    def _limits(self, entry, W, H, dev):
        tx, ty = (W + 15) // 16, (H + 15) // 16
        n_tiles, cells = tx * ty, ((tx + 3) // 4) * ((ty + 3) // 4)
        k = id(entry)
        t = self.caps.get(k)
        if t is None or t.numel() != n_tiles + cells:
            t = torch.full((n_tiles + cells,), float("inf"), dtype=torch.float32, device=dev)
            self.caps[k] = t
            self.stamps[k] = torch.full((1,), -(1 << 40), dtype=torch.int64, device=dev)
        return t, n_tiles

    def accumulate(self, entry, flat, union) -> torch.Tensor:
        mp, cfg = self.mp, self.mp.cfg
        dt = mp.dtype
        code = N.dtype_code(dt)
        n = mp.map.count
        kf = entry.frame
        W, H = kf.intrinsics.width, kf.intrinsics.height
        st = N.stream_ptr()
        dev = flat.device
        a = mp.map.arrays()
        cam = N.camera(kf.pose, kf.intrinsics)
        rec = self._buf("records", (max(n, 1), N.RECORD_REALS), dt)
        valid = self._buf("valid", (max(n, 1),), torch.uint8)
        keys = self._buf("keys", (max(n, 1),), torch.int64 if dt == torch.float64 else torch.int32)
        vals = self._buf("vals", (max(n, 1),), torch.int32)
        fr = self._buf("frustum", (max(n, 1),), torch.uint8)
        status = self._buf(("status", id(entry)), (2,), torch.int64)
        exposure = entry.exposure if cfg.exposure_mode != "off" else None
        if exposure is None:
            from .engine import DeviceExposure
            exposure = DeviceExposure(dtype=dt)
        sync = self.pair_cap == 0
        use = self.use_limits and dt == torch.float32
        caps = coarse = None
        if self.clock is None or self.clock.device != dev:
            self.clock = torch.zeros(1, dtype=torch.int64, device=dev)
        bump = 1 if self._first else 0
        self._first = False
        if use:
            allc, n_tiles = self._limits(entry, W, H, dev)
            caps, coarse = allc[:n_tiles], allc[n_tiles:]
            if sync or self._full:
                allc.fill_(float("inf"))
            N.call("sb_depth_limits_gate", N.ptr(allc), allc.numel(), N.ptr(self.clock),
                   N.ptr(self.stamps[id(entry)]), bump, st)
        else:
            N.call("sb_depth_limits_gate", None, 0, N.ptr(self.clock), None, bump, st)
        N.call("sb_preprocess_fwd", code, n, *[N.ptr(a[k]) for k in (
            "positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")], None,
            N.C.byref(cam), float(cfg.near), 0.3, float(cfg.frustum_margin), N.ptr(rec),
            N.ptr(valid), N.ptr(keys), N.ptr(vals), N.ptr(fr), None, N.ptr(coarse), st)
        if sync:
            # first step at this map size: full lists, read P once per view
            pg, _, off, P = run_bin(dt, n, rec, valid, keys, vals, W, H, True,
                                    self.binout.get("pairs_cap", 4 * n), out=self.binout)
            self._pmax = max(self._pmax, P)
            self._smax = max(self._smax, int((keys[:n] != -1).sum().item()))
            status.zero_()
        else:
            pg, off = self._bin_async(dt, n, rec, valid, keys, vals, W, H, status, caps)
        sk = ("sched", id(entry))
        n_t = ((W + 15) // 16) * ((H + 15) // 16)
        if sk not in self.bufs or self.bufs[sk].numel() != 3 * n_t:
            self.bufs[sk] = torch.zeros(3 * n_t, dtype=torch.int32, device=dev)
        if coarse is not None:   # the forward re-derives the coarse maxima
            N.call("sb_memset_async", N.ptr(coarse), 0, coarse.numel() * 4, st)
        o = run_blend_fwd(dt, rec, pg, off, W, H, cfg.early_termination, 1e-4, exposure.real,
                          out=self.fwd, depth_limit=caps, status=status, coarse_limit=coarse,
                          sched=self.bufs[sk], fast_exp=mp.engine.fast_exp and dt == torch.float32)
        self.bad.bitwise_or_(status)
        lo = run_loss(o["color"], entry.gt, exposure.real, cfg.loss_lambda, y=o["y"],
                      out=self.loss)
        self.d_E[id(entry)] = lo["d_E"].clone()
        adj = [self._buf(k, (max(n, 1),) + s, dt) for k, s in
               (("dm", (2,)), ("dc", (3,)), ("do", ()), ("dcol", (3,)))]
        # no zeroing: the gather flags the rows it reached and the chain
        # rule reads no other row's adjoints
        b = self.binout      # the deterministic backward over this view's pair slot map
        bws = _SCRATCH.get("bwd", N.load().sb_blend_bwd_workspace_bytes(code, b["bin_cap"], W, H),
                           dev)
        N.call("sb_blend_bwd_partials", code, N.ptr(rec), N.ptr(pg), N.ptr(off), W, H, 16,
               int(cfg.early_termination), 1e-4, N.ptr(lo["d_rendered"]), N.ptr(o["color"]),
               N.ptr(o["last"]), N.ptr(o["sched_used"]), b["bin_m"], b["bin_cap"],
               N.ptr(b["bin_ws"]), N.ptr(bws), bws.numel(), st)
        # the gather flags the rows it reached (a byte per row; the chain
        # rule's scan reads 1 B per row instead of 36 B of adjoints)
        rows = self._buf("reach_rows", (max(n, 1),), torch.uint8)
        N.call("sb_memset_async", N.ptr(rows), 0, rows.numel(), st)
        first = 0 if self._zeroed else 1
        N.call("sb_gather_adjoints", code, b["bin_m"], b["bin_cap"], W, H, b["bin_sort_cap"],
               N.ptr(b["bin_ws"]), N.ptr(bws), bws.numel(), *[N.ptr(t) for t in adj],
               N.ptr(rows), st)
        g = group_views(flat, self.n_pad)
        ws = _SCRATCH.get("chain_acc", N.load().sb_chain_accumulate_workspace_bytes(code, n),
                          flat.device)
        N.call("sb_chain_accumulate", code, n, N.ptr(valid), N.ptr(a["positions"]),
               N.ptr(a["log_scales"]), N.ptr(a["rotations"]), N.ptr(a["opacity_logits"]),
               N.ptr(a["sh_coeffs"]), N.C.byref(cam), 0.3, *[N.ptr(t) for t in adj],
               *[N.ptr(g[k]) for k, _ in GROUP_WIDTHS], N.ptr(self._reached), first,
               N.ptr(rows), N.ptr(ws), ws.numel(), st)
        torch.bitwise_or(union, fr[:n], out=union)
        # the step's invalid flag rides in the union buffer's last byte
        self._ub[n:n + 1].copy_(self.bad[1:2])
        return lo["parts"].clone()

    def _bin_async(self, dt, n, rec, valid, keys, vals, W, H, status, caps):
        dev = rec.device
        cap = self.pair_cap
        b = self.binout
        if b.get("async_cap", 0) != cap:
            b["a_pg"] = torch.empty(cap, dtype=torch.int32, device=dev)
            b["async_cap"] = cap
        n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
        if b.get("a_off") is None or b["a_off"].numel() != n_tiles + 1:
            b["a_off"] = torch.empty(n_tiles + 1, dtype=torch.int32, device=dev)
        lib = N.load()
        ws = _SCRATCH.get("bin", lib.sb_bin_workspace_bytes(n, cap, W, H), dev)
        npairs = N.C.c_int64(0)
        N.check(lib.sb_bin(N.dtype_code(dt), n, N.ptr(rec), N.ptr(valid), N.ptr(keys),
                           N.ptr(vals), W, H, 16, 1, cap, N.ptr(b["a_pg"]), None,
                           N.ptr(b["a_off"]), N.C.byref(npairs), N.ptr(ws), ws.numel(),
                           N.ptr(status), N.ptr(caps), self.sort_cap, None, N.stream_ptr()),
                "sb_bin")
        b.update(bin_ws=ws, bin_m=n, bin_cap=cap, bin_sort_cap=self.sort_cap)
        return b["a_pg"], b["a_off"]

    def end_exchange(self):
        """After the exchange: the (all-reduced) invalid flag as the update
        kernels' status word."""
        st64 = self._buf("st64", (2,), torch.int64)
        st64.zero_()
        st64[1:2].copy_(self._ub[self._n:self._n + 1])
        if self.deferred:
            self._sticky_flag().copy_(st64[1:2])
        if self.pair_cap == 0:     # the sizing step is over: async from now on
            self.pair_cap = int(self._pmax * 1.5) + 65536
            # bounded depth sort when the sortable rows are a minority (engine._sort_bound)
            bound = int(self._smax * 1.3) + 4096
            self.sort_cap = bound if bound < int(0.8 * self._n) else 0
        return st64

    def mask_buffer(self):
        return self._ub

    # -- lazy validity (BatchStep(lazy=True)) --------------------------------
    deferred = False          # steps are checked later; invalid flags are sticky

    def _sticky_flag(self):
        t = self.bufs.get("sticky")
        if t is None:
            t = self.bufs["sticky"] = torch.zeros(1, dtype=torch.int64,
                                                  device=self.mp.map.positions.device)
        return t

    def mark_invalid(self, cond):
        """OR a device bool[1] into the step's (already exchanged) invalid flag."""
        self._ub[self._n:self._n + 1].bitwise_or_(cond.to(torch.uint8).reshape(1))

    def defer_flag(self):
        """After a step: its invalid flag copied to pinned memory, and the
        event that completes the copy."""
        ring = self.bufs.get("flag_ring")
        if ring is None:
            ring = self.bufs["flag_ring"] = [torch.zeros(1, dtype=torch.int64).pin_memory()
                                             for _ in range(8)]
            self._ring_i = 0
        buf = ring[self._ring_i % len(ring)]
        self._ring_i += 1
        buf.copy_(self.st64[1:2], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return buf, ev

    def reset_deferred(self):
        """An unchecked step was invalid: clear the sticky flag; the re-run
        bins full lists and re-sizes the pair and sort buffers synchronously
        (an overflow of either is what may have made the step invalid)."""
        self._sticky_flag().zero_()
        self._full = True
        self.pair_cap = self.sort_cap = 0

    def reached_mask(self):
        """uint8[n_pad]: rows some pixel of this rank's views reached (written
        by sb_chain_accumulate); every other row's gradient is exactly zero."""
        return self._reached

    def step_invalid(self) -> bool:
        """Host check (one sync) after a step: was it a device no-op?  Then
        the next step bins full lists."""
        bad = bool(self._ub[self._n].item())
        self._full = bad
        if bad:   # re-run with full lists, re-sized pair/sort buffers, no sticky flag
            self.pair_cap = self.sort_cap = 0
            self._sticky_flag().zero_()
        return bad

    def apply(self, flat, union, grad_rows=None):
        """One sparse Adam step over the union mask.  grad_rows (uint8[n]):
        read the gradient of these rows only (required when begin(zero=False))."""
        mp = self.mp
        n = mp.map.count
        if not self._zeroed and grad_rows is None:
            raise ValueError("apply: a first-touch gradient needs grad_rows")
        a = mp.map.arrays()
        params = {"position": a["positions"], "log_scale": a["log_scales"],
                  "rotation": a["rotations"], "opacity_logit": a["opacity_logits"],
                  "sh": a["sh_coeffs"]}
        gv = {k: v[:n] for k, v in group_views(flat, self.n_pad).items()}
        G = mp.adam.groups(params, gv)
        self._adam(G, n, mp.adam._steps, union, grad_rows, mp.adam.touched())

    def prepare_step(self):
        """Host work before a (possibly replayed) step: the Adam touched-row
        mask is rebuilt here if the moments were written from outside."""
        self.mp.adam.touched()

    def _adam(self, G, rows, steps, active, grad_rows=None, touched=None):
        mp = self.mp
        code = N.dtype_code(mp.dtype)
        lrs = lr_vector(mp.adam.lrs)
        self.st64 = self.end_exchange()
        ws = _SCRATCH.get("sparse_adam", N.load().sb_sparse_adam_workspace_bytes(code, rows),
                          steps.device)
        N.call("sb_sparse_adam_flat", code, rows, N.C.byref(G), N.ptr(steps), N.ptr(active),
               N.ptr(grad_rows), N.ptr(touched), lrs.ctypes.data_as(N.vp), N.ptr(ws),
               ws.numel(), N.ptr(self.st64), N.stream_ptr())

    def apply_rows(self, lo, hi, grads, union):
        """Sparse Adam on map rows [lo, hi) with that block's gradient."""
        mp = self.mp
        if hi <= lo:
            self.st64 = self.end_exchange()
            return
        a = mp.map.arrays()
        params = {"position": a["positions"], "log_scale": a["log_scales"],
                  "rotation": a["rotations"], "opacity_logit": a["opacity_logits"],
                  "sh": a["sh_coeffs"]}
        G = mp.adam.groups_rows(params, grads, lo, hi)
        self._adam(G, hi - lo, mp.adam._steps[lo:hi], union[lo:hi])
        mp.adam.moments_written()    # the row-block pass keeps no touched mask

    def row_tensors(self, n_pad):
        """Per-row state every replica needs after the update: the parameter
        groups and the Adam step counters, n_pad rows each."""
        mp = self.mp
        before = (mp.map._buf["positions"].data_ptr(), mp.adam._steps.data_ptr())
        mp.map.reserve(n_pad)
        mp.adam.reserve(n_pad)
        if (mp.map._buf["positions"].data_ptr(), mp.adam._steps.data_ptr()) != before:
            mp.engine.invalidate()   # captured step graphs hold the old pointers
        b = mp.map._buf
        return [b[k][:n_pad] for k in ("positions", "log_scales", "rotations", "opacity_logits",
                                       "sh_coeffs")] + [mp.adam._steps[:n_pad]]

    def moment_tensors(self, n_pad):
        mp = self.mp
        before = mp.adam._steps.data_ptr()
        mp.adam.reserve(n_pad)
        if mp.adam._steps.data_ptr() != before:
            mp.engine.invalidate()
        mp.adam.moments_written()    # the caller gathers into these
        return [t[:n_pad] for d in (mp.adam._m, mp.adam._v) for t in d.values()]

    def exposure(self, entry):
        if self.mp.cfg.exposure_mode == "off":
            return
        e = entry.exposure
        N.call("sb_exposure_adam", N.dtype_code(self.mp.dtype), N.ptr(e.mat), N.ptr(e.real),
               N.ptr(self.d_E[id(entry)]), N.ptr(e.state), float(self.mp.cfg.lr_exposure),
               N.ptr(self.st64), N.stream_ptr())


def shard_views(views: list, rank: int, world: int) -> list:
    """Contiguous keyframe shards: rank r owns views [r k, (r+1) k)."""
    k = (len(views) + world - 1) // world
    return views[rank * k:(rank + 1) * k]
