"""Keyframe-batch data parallelism on CPU with gloo, world
size 2: the distributed exchange of paper_2404_06926_b200.batch.BatchStep
(gradient SUM all-reduce, frustum-mask MAX all-reduce, one sparse Adam step
on the union) with the CPU oracle as each rank's compute, against the batched
oracle semantics computed in one process."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from parity import oracle

N_VIEWS = 4
GROUPS = ("position", "log_scale", "rotation", "opacity_logit", "sh")
WIDTH = {"position": 3, "log_scale": 3, "rotation": 4, "opacity_logit": 1, "sh": 48}


def _scene():
    rng = np.random.default_rng(3)
    n = 250
    z = rng.uniform(3.0, 8.0, n)
    pos = np.stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n), z], 1)
    ls = np.log(rng.uniform(0.05, 0.4, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = np.log(0.5 / 0.5) + rng.normal(0, 1, n)
    sh = rng.normal(0, 0.3, (n, 16, 3))
    gmap = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": op,
            "sh_coeffs": sh}
    gmap = {k: v.astype(np.float32) for k, v in gmap.items()}
    o = oracle()
    views = []
    for k in range(N_VIEWS):
        a = 0.08 * (k - 1.5)
        W = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
        cam = o.Camera(W=W, t=np.array([0.05 * k, 0.0, 0.1]), fx=48.0, fy=48.0, cx=24.0,
                       cy=20.0, width=48, height=40)
        img = np.random.default_rng(10 + k).uniform(0, 1, (40, 48, 3))
        E = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) + \
            np.random.default_rng(20 + k).normal(0, 0.02, (3, 4))
        views.append({"cam": cam, "image": img, "E": E, "id": k})
    lrs = {"position": 1.6e-4, "log_scale": 5e-3, "rotation": 1e-3, "opacity_logit": 5e-2,
           "sh0": 2.5e-3, "sh_rest": 1.25e-4}
    return gmap, views, lrs


class OracleBatchCompute:
    """Per-rank compute for BatchStep backed by the CPU oracle (test only)."""

    def __init__(self, gmap, lrs):
        self.o = oracle()
        self.g = {k: v.copy() for k, v in gmap.items()}
        n = self.g["positions"].shape[0]
        arrs = [self.g[k] for k in ("positions", "log_scales", "rotations", "opacity_logits",
                                    "sh_coeffs")]
        self.m = {k: np.zeros_like(v) for k, v in zip(GROUPS, arrs)}
        self.v = {k: np.zeros_like(v) for k, v in zip(GROUPS, arrs)}
        self.steps = np.zeros(n, np.int64)
        self.n_pad = n
        self.lrs = lrs
        self.d_E = {}
        self.ex = {}

    def rows(self):
        return self.g["positions"].shape[0]

    def begin(self, n_pad=None):
        n = self.g["positions"].shape[0]
        self.n_pad = n if n_pad is None else n_pad
        return torch.zeros(59 * self.n_pad, dtype=torch.float32), torch.zeros(n, dtype=torch.uint8)

    def _views(self, flat):
        n = self.g["positions"].shape[0]
        out, off = {}, 0
        a = flat.numpy()
        for k in GROUPS:
            out[k] = a[off:off + WIDTH[k] * self.n_pad][:WIDTH[k] * n]
            off += WIDTH[k] * self.n_pad
        return out

    # --- ShardedBatchStep interface -------------------------------------------
    _PK = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")

    def apply_rows(self, lo, hi, grads, union):
        """The oracle Adam on rows [lo, hi) only."""
        if hi <= lo:
            return
        params = {g: self.g[k][lo:hi] for g, k in zip(GROUPS, self._PK)}
        gr = {g: grads[g].numpy().reshape(params[g].shape) for g in GROUPS}
        m = {g: self.m[g][lo:hi] for g in GROUPS}
        v = {g: self.v[g][lo:hi] for g in GROUPS}
        steps = self.steps[lo:hi]
        self.o.adam_step(params, gr, m, v, steps, self.lrs,
                         active=union.numpy()[lo:hi].astype(bool))

    def row_tensors(self, n_pad):
        n = self.rows()
        self._pad = []
        for k in self._PK:
            a = self.g[k]
            t = torch.zeros((n_pad,) + a.shape[1:], dtype=torch.float32)
            t[:n] = torch.from_numpy(a)
            self._pad.append((k, t))
        st = torch.zeros(n_pad, dtype=torch.int64)
        st[:n] = torch.from_numpy(self.steps)
        self._pad.append(("steps", st))
        return [t for _, t in self._pad]

    def after_gather(self):
        n = self.rows()
        for k, t in self._pad:
            if k == "steps":
                self.steps[:] = t[:n].numpy()
            else:
                self.g[k][:] = t[:n].numpy()

    def accumulate(self, view, flat, union):
        o, cam = self.o, view["cam"]
        sc, (pg, pt, off), t = o.render_view(self.g, cam)
        loss, d_r, d_E, parts = o.photometric_loss(t["color"], view["image"].astype(np.float32),
                                                   view["E"], 0.2)
        adj = o.backward_tiles(pg, off, sc, d_r, t["color"], cam.width, cam.height)
        gr = o.chain(adj, sc, self.g, cam)
        fv = self._views(flat)
        for k, gk in zip(GROUPS, ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit",
                                  "d_sh")):
            fv[k] += gr[gk].reshape(-1)
        fm = o.frustum_mask(cam, self.g["positions"])
        union.numpy()[:] |= fm.astype(np.uint8)
        self.d_E[view["id"]] = d_E.astype(np.float64)
        return loss

    def apply(self, flat, union):
        n = self.g["positions"].shape[0]
        fv = self._views(flat)
        params = {"position": self.g["positions"], "log_scale": self.g["log_scales"],
                  "rotation": self.g["rotations"], "opacity_logit": self.g["opacity_logits"],
                  "sh": self.g["sh_coeffs"]}
        grads = {k: fv[k].reshape(params[k].shape) for k in GROUPS}
        self.o.adam_step(params, grads, self.m, self.v, self.steps, self.lrs,
                         active=union.numpy().astype(bool))
        del n

    def exposure(self, view):
        ex = self.ex.setdefault(view["id"], self.o.ScalarAdam((3, 4), 1e-2))
        ex.step(view["E"], self.d_E[view["id"]])


def _worker(rank, world, port, out_path, sharded=False):
    """sharded: False -> BatchStep, True -> ShardedBatchStep, "packed" ->
    PackedShardedBatchStep, "packed_ar" -> PackedBatchStep."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_06926_b200.batch import (BatchStep, PackedBatchStep,
                                                 PackedShardedBatchStep, ShardedBatchStep,
                                                 shard_views)
        gmap, views, lrs = _scene()
        comp = OracleBatchCompute(gmap, lrs)
        mine = shard_views(views, rank, world)
        cls = {"packed": PackedShardedBatchStep, "packed_ar": PackedBatchStep,
               True: ShardedBatchStep, False: BatchStep}[sharded]
        step = cls(comp)
        step.step(mine)
        if sharded in ("packed", "packed_ar"):
            np.save(f"{out_path}.{rank}.rows.npy", np.array([step.packed_rows]))
        np.savez(f"{out_path}.{rank}.npz", **comp.g, steps=comp.steps,
                 E=np.stack([v["E"] for v in mine]) if mine else np.zeros((0, 3, 4)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batched_reference(world):
    """Single-process batched oracle: per-rank f32 sums in view order, ranks
    summed in rank order (what a 2-rank gloo SUM computes), one Adam step."""
    gmap, views, lrs = _scene()
    ranks = []
    from paper_2404_06926_b200.batch import shard_views
    for r in range(world):
        c = OracleBatchCompute(gmap, lrs)
        flat, union = c.begin()
        for v in shard_views(views, r, world):
            c.accumulate(v, flat, union)
        ranks.append((flat, union))
    total = ranks[0][0].clone()
    union = ranks[0][1].clone()
    for f, u in ranks[1:]:
        total += f
        union = torch.maximum(union, u)
    c = OracleBatchCompute(gmap, lrs)
    c.apply(total, union)
    return c, total, union


def test_batched_reference_matches_f64_semantics():
    """The f32 batched sum equals the f64 sum of per-view gradients to float
    rounding (SURVEY §8e oracle)."""
    c, total, union = _batched_reference(2)
    gmap, views, lrs = _scene()
    o = oracle()
    acc = np.zeros(total.numel())
    for v in views:
        cc = OracleBatchCompute(gmap, lrs)
        f, u = cc.begin()
        cc.accumulate(v, f, u)
        acc += f.numpy().astype(np.float64)
    scale = np.abs(acc).max()
    assert np.abs(total.numpy() - acc).max() <= 1e-5 * scale
    assert union.sum() > 0
    del o


def test_gloo_world2_equals_batched_oracle(tmp_path):
    world = 2
    port = _free_port()
    out = str(tmp_path / "batch")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref, _, _ = _batched_reference(world)
    r0 = np.load(f"{out}.0.npz")
    r1 = np.load(f"{out}.1.npz")
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        # replicas stay identical, and equal the batched oracle bit for bit
        np.testing.assert_array_equal(r0[k], r1[k])
        np.testing.assert_array_equal(r0[k], ref.g[k])
    np.testing.assert_array_equal(r0["steps"], ref.steps)
    assert (r0["steps"] <= 1).all() and r0["steps"].sum() > 0


@pytest.mark.parametrize("world", [1, 2, 4])
def test_shard_views_partition(world):
    from paper_2404_06926_b200.batch import shard_views
    views = list(range(8))
    got = [shard_views(views, r, world) for r in range(world)]
    assert sum(got, []) == views


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_adam_equals_batched_oracle(tmp_path, world):
    """ShardedBatchStep: reduce-scatter of the gradient by row blocks, Adam on
    each rank's block, all-gather of the updated rows -- the same step as the
    all-reduce exchange (world 3 pads 250 rows to 252)."""
    port = _free_port()
    out = str(tmp_path / "sharded")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out, True)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref, total, union = _batched_reference(world)
    got = [np.load(f"{out}.{r}.npz") for r in range(world)]
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        for r in range(1, world):
            np.testing.assert_array_equal(got[0][k], got[r][k])
        if world == 2:   # two-operand sums are order-independent: bit for bit
            np.testing.assert_array_equal(got[0][k], ref.g[k])
        else:
            np.testing.assert_allclose(got[0][k], ref.g[k], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(got[0]["steps"], ref.steps)


def test_row_blocks_cover_the_map():
    from paper_2404_06926_b200.batch import row_block
    for n in (0, 1, 7, 250, 251):
        for world in (1, 2, 3, 8):
            blocks = [row_block(n, r, world) for r in range(world)]
            covered = sorted(i for lo, hi, _ in blocks for i in range(lo, hi))
            assert covered == list(range(n))
            assert all(b[2] % world == 0 and b[2] >= n for b in blocks)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_packed_exchange_equals_batched_oracle(tmp_path, world):
    """PackedBatchStep: only the rows some view reached are reduce-scattered
    (packed per row block); the result is the batched oracle's step (bit for
    bit at world 2), with fewer rows on the wire than the map."""
    port = _free_port()
    out = str(tmp_path / "packed")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out, "packed"))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref, total, union = _batched_reference(world)
    got = [np.load(f"{out}.{r}.npz") for r in range(world)]
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        for r in range(1, world):
            np.testing.assert_array_equal(got[0][k], got[r][k])
        if world == 2:
            np.testing.assert_array_equal(got[0][k], ref.g[k])
        else:
            np.testing.assert_allclose(got[0][k], ref.g[k], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(got[0]["steps"], ref.steps)
    n = ref.g["positions"].shape[0]
    wire = int(np.load(f"{out}.0.rows.npy")[0])
    a, off, hit = total.numpy(), 0, np.zeros(n, bool)
    for g in GROUPS:
        hit |= (a[off:off + WIDTH[g] * n].reshape(n, WIDTH[g]) != 0).any(axis=1)
        off += WIDTH[g] * n
    # the wire carries each row block's reached rows, padded to the largest
    # block count (a multiple of 8): here every row is reached (a small scene)
    from paper_2404_06926_b200.batch import row_block
    rows = row_block(n, 0, world)[2] // world
    per_block = [int(hit[r * rows:(r + 1) * rows].sum()) for r in range(world)]
    assert wire == world * max(8, (max(per_block) + 7) // 8 * 8), (wire, per_block)


def test_gloo_packed_allreduce_equals_batched_oracle(tmp_path):
    """PackedBatchStep (reached rows all-reduced, replicated Adam): world 2,
    bit for bit against the batched oracle; the wire carries exactly the
    reached rows."""
    world = 2
    port = _free_port()
    out = str(tmp_path / "packed_ar")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out, "packed_ar"))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref, total, union = _batched_reference(world)
    got = [np.load(f"{out}.{r}.npz") for r in range(world)]
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        np.testing.assert_array_equal(got[0][k], got[1][k])
        np.testing.assert_array_equal(got[0][k], ref.g[k])
    np.testing.assert_array_equal(got[0]["steps"], ref.steps)
    n = ref.g["positions"].shape[0]
    a, off, hit = total.numpy(), 0, np.zeros(n, bool)
    for g in GROUPS:
        hit |= (a[off:off + WIDTH[g] * n].reshape(n, WIDTH[g]) != 0).any(axis=1)
        off += WIDTH[g] * n
    assert int(np.load(f"{out}.0.rows.npy")[0]) == int(hit.sum())
