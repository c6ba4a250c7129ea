"""Lazy validity checks of the batched step across ranks (batch.BatchStep
lazy=True), on CPU with gloo at world 2: a toy compute with the
DeviceBatchCompute flag protocol (invalid flag behind the union mask, sticky
while deferred, pinned-flag readback) so the host logic -- step-count
resolution in lockstep on every rank, in-order re-runs of the no-op steps
queued behind an invalid one, the fixed-capacity packing and its overflow --
runs without a GPU.  The lazy run must equal the synchronous one exactly."""

import multiprocessing as mp
import os
import socket

import numpy as np
import torch
import torch.distributed as dist

N_ROWS = 24


class _Done:
    def synchronize(self):
        pass


def _rows(views):
    """Map-layout group views -> one [rows, 59] copy."""
    return torch.cat([t.reshape(t.shape[0], -1) for t in views.values()], 1)


def _scatter(views, g):
    off = 0
    for t in views.values():
        w = t[0].numel()
        t.reshape(t.shape[0], -1).copy_(g[:, off:off + w])
        off += w


class ToyCompute:
    """Gradient of view v (map layout, batch.group_views): rows v .. v+7
    (mod n) get 0.1 x param + v + rank;
    SGD on the union.  The step whose begin() is call number `fail_call`
    reports invalid (like a depth-limited tile that did not terminate); its
    re-run is valid."""

    deferred = False

    def __init__(self, rank, fail_call):
        self.rank, self.fail_call, self.calls = rank, fail_call, 0
        self.p = torch.arange(N_ROWS * 59, dtype=torch.float64).reshape(59, N_ROWS) / 100
        self.sticky = torch.zeros(1, dtype=torch.int64)
        self.applied = 0
        self._full = False

    def rows(self):
        return N_ROWS

    def begin(self, n_pad=None):
        self.calls += 1
        self.n_pad = N_ROWS if n_pad is None else n_pad
        self.flat = torch.zeros(59 * self.n_pad, dtype=torch.float64)
        self.ub = torch.zeros(N_ROWS + 1, dtype=torch.uint8)
        self.reached = torch.zeros(self.n_pad, dtype=torch.uint8)
        bad = 1 if self.calls == self.fail_call else 0
        if self.deferred:
            bad |= int(self.sticky[0])
        self.ub[N_ROWS] = bad
        return self.flat, self.ub[:N_ROWS]

    def accumulate(self, v, flat, union):
        from paper_2404_06926_b200.batch import group_views
        g = _rows(group_views(flat, self.n_pad))      # [n_pad, 59] copy
        rows = [(v + i) % N_ROWS for i in range(8)]
        for r in rows:
            g[r] += 0.1 * self.p[:, r] + v + self.rank
            union[r] = 1
            self.reached[r] = 1
        _scatter(group_views(flat, self.n_pad), g)
        return torch.tensor([float(v), float(self.p.sum())])

    def mask_buffer(self):
        return self.ub

    def reached_mask(self):
        return self.reached

    def mark_invalid(self, cond):
        self.ub[N_ROWS:] |= cond.to(torch.uint8).reshape(1)

    def apply(self, flat, union):
        bad = int(self.ub[N_ROWS])
        if self.deferred:
            self.sticky[0] = bad
        if bad:
            return
        from paper_2404_06926_b200.batch import group_views
        g = _rows(group_views(flat, self.n_pad))[:N_ROWS].T
        self.p -= 0.01 * g * union.to(torch.float64)
        self.applied += 1

    def exposure(self, v):
        pass

    def defer_flag(self):
        return torch.tensor([int(self.ub[N_ROWS])]), _Done()

    def reset_deferred(self):
        self.sticky.zero_()
        self._full = True

    def step_invalid(self):
        bad = bool(self.ub[N_ROWS])
        self._full = bad
        return bad


def _run(rank, lazy, steps=7):
    from paper_2404_06926_b200.batch import PackedBatchStep
    comp = ToyCompute(rank, fail_call=3)
    step = PackedBatchStep(comp, always_reduce=True, lazy=lazy)
    logs = []
    for i in range(steps):
        logs.append(step.step([2 * i + rank]))
        if lazy and i == 4:
            step.k_cap = 3          # the next step's reached rows overflow the packing
    step.flush()
    return comp, step, torch.cat([torch.cat(l) for l in logs])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ref, _, ref_logs = _run(rank, lazy=False)
        got, step, logs = _run(rank, lazy=True)
        assert step.lazy and not step._pending
        assert step.k_cap > 3                      # the overflow was seen and resized
        np.savez(f"{out}.{rank}.npz", ref=ref.p.numpy(), got=got.p.numpy(),
                 ref_logs=ref_logs.numpy(), logs=logs.numpy(),
                 applied=np.array([ref.applied, got.applied]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_lazy_checks_equal_sync_steps(tmp_path):
    world, port, out = 2, _free_port(), str(tmp_path / "lazy")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = [np.load(f"{out}.{r}.npz") for r in range(world)]
    for g in got:
        np.testing.assert_array_equal(g["got"], g["ref"])
        np.testing.assert_array_equal(g["logs"], g["ref_logs"])
        assert list(g["applied"]) == [7, 7]
    np.testing.assert_array_equal(got[0]["got"], got[1]["got"])
