"""A/B of the mapping step's engine switches on config 3, each timed twice
in alternation from the same snapshot (graph replay, device events) --
checks that a variant's rate does not depend on when it runs."""

import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402


def main(steps=30):
    scene = bench.scene_of(3)
    mp, entry = bench.build_mapper(scene, sb, torch)
    for _ in range(5):
        mp._step_device(entry)
    torch.cuda.synchronize()
    snap = bench.snapshot(mp, entry)
    variants = [("base", {}), ("no_skip", {"touched_skip": False}),
                ("exact_exp", {"fast_exp": False}), ("atomic", {"deterministic": False})]
    for rnd in range(2):
        for name, attrs in variants:
            r = bench.variant_rate(mp, entry, torch, steps, 3, snap=snap, **attrs)
            print(rnd, name, r, flush=True)


if __name__ == "__main__":
    main()
