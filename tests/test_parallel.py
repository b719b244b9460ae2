"""Multi-process (world_size 2, gloo, CPU) coverage of the image-sharded
stack: shard assignment, the single all-gather of final maps in rank order,
and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2007_12216_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fake_stack(images: np.ndarray) -> np.ndarray:
    # stand-in for the per-rank device stack: any per-image deterministic map
    from oracle.vgg_ref import requant_pool

    y = images.astype(np.int32).sum(axis=3, keepdims=True) * 1000 - 90000
    return requant_pool(np.repeat(y, 4, axis=3), 6, True)


def _worker(rank, world, port, batch, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_12216_b200 import workloads as W

        start, count = parallel.shard_range(batch, world, rank)
        x = W.vgg16_images(count, start=start)[:, :8, :8, :]
        local = torch.from_numpy(_fake_stack(x))
        full = parallel.gather_maps(local, world)
        t = parallel.max_over_ranks(0.5 + rank, world)
        q.put((rank, start, count, full.numpy(), t))
    finally:
        dist.destroy_process_group()


def test_shard_range():
    assert parallel.shard_range(256, 8, 3) == (96, 32)
    assert parallel.shard_range(256, 1, 0) == (0, 256)
    with pytest.raises(ValueError):
        parallel.shard_range(10, 4, 0)
    with pytest.raises(ValueError):
        parallel.shard_range(8, 2, 2)


def test_two_rank_gather_matches_single_process():
    world, batch = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2007_12216_b200 import workloads as W

    want = _fake_stack(W.vgg16_images(batch)[:, :8, :8, :])
    results.sort()
    assert [(r[1], r[2]) for r in results] == [(0, 2), (2, 2)]
    for rank, _, _, full, t in results:
        assert np.array_equal(full, want)
        assert t == 1.5  # max over ranks


@pytest.mark.parametrize("gpus,weak", [(2, False), (4, False), (2, True)])
def test_bench_self_launch_dry_run(gpus, weak):
    """`bench.py --gpus N` without a torchrun environment relaunches itself
    under torch.distributed.run with N ranks (here over gloo, --dry-run: no
    GPU work): config 4's 256 images split 256/N per rank (strong scaling) or
    N x --batch (weak), gathered back in image order on rank 0."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    cmd = [sys.executable, str(root / "bench.py"), "--gpus", str(gpus), "--dry-run"]
    if weak:
        cmd += ["--weak", "--batch", "16"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == gpus
    if weak:
        assert line["global_batch"] == 16 * gpus and line["per_rank_batch"] == 16
    else:
        assert line["global_batch"] == 256 and line["per_rank_batch"] == 256 // gpus
    assert line["gathered_ranks"] == list(range(1, gpus + 1))
    assert line["image_tags_ok"] and abs(line["max_elapsed_s"] - 0.001 * gpus) < 1e-9
