"""bench.py's launch contract on the CPU: ``--gpus N`` without a torchrun
environment re-launches itself as N ranks (torch.distributed.run, 127.0.0.1),
rank 0 alone prints ONE JSON line, and a --gpus / WORLD_SIZE mismatch fails
loudly.  Exercised through the reference arm (the CPU oracle: no GPU needed)
on config 1, a batched step of 2 views."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.pop("LOCAL_RANK", None)
    e.update(env or {})
    return subprocess.run([sys.executable, "bench.py"] + args, cwd=REPO, env=e,
                          capture_output=True, text=True, timeout=900)


def test_gpus_2_relaunches_two_ranks_one_line():
    out = _run(["--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1",
                "--warmup", "0"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["views_per_step"] == 2 and d["steps"] == 1
    assert d["cpu_baseline"]["cores"] >= 1 and d["value"] > 0


def test_gpus_world_size_mismatch_fails():
    out = _run(["--gpus", "2", "--impl", "reference", "--config", "1"],
               env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr
