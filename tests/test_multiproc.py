"""World-size-2 gloo run of the frame-parallel (video) path on CPU.

Each rank takes its contiguous frame block (video.frame_block), fills it --
with the CPU oracle standing in for the GPU kernel, since this container has
no GPU -- and the ranks combine their results with the package's own
bookkeeping collectives (video.reduce_over_ranks: pixel/byte sums and the
max step time, what bench.py reports for N > 1) plus an all_gather of
per-frame digests.  The gathered results must equal a single process filling
every frame: the partition neither drops, duplicates nor couples frames.
The GPU side of the same path (fill_video_multi, bench.py's rank loop) is
covered by tests/test_gpu_configs.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_05319_b200 import scenes
from paper_1611_05319_b200.video import frame_block, frame_checksum, reduce_over_ranks

N_FRAMES = 5


def _frame(f):
    return scenes.small_scene(40, 72, band=4, gx=3, gy=2, n_spl=2, seed=1611, frame=f)


def _fill(f):
    from oracle import guidefill_oracle as orc

    sc = _frame(f)
    field = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in sc.splines],
                            [s["direction"] for s in sc.splines], sc.labels)
    res = orc.fill(sc.image, sc.labels, field, orc.Params(**sc.params), tracked=True)
    return frame_checksum(res["u"]), res["iterations"]


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = frame_block(N_FRAMES, world, rank)
    digests = torch.full((N_FRAMES, 2), -1.0, dtype=torch.float64)
    for f in mine:
        c, it = _fill(f)
        digests[f, 0] = c
        digests[f, 1] = it
    gathered = [torch.zeros_like(digests) for _ in range(world)]
    dist.all_gather(gathered, digests)
    px = sum(int((_frame(f).labels == 255).sum()) for f in mine)
    sums, maxes = reduce_over_ranks(sums=[px, len(mine)], maxes=[float(rank + 1)])
    if rank == 0:
        merged = torch.stack(gathered).max(dim=0).values
        out_q.put((merged.numpy(), maxes[0], sums, [list(frame_block(N_FRAMES, world, r))
                                                    for r in range(world)]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_frame_block_partition():
    for n in range(0, 40):
        for world in range(1, 9):
            blocks = [frame_block(n, world, r) for r in range(world)]
            flat = [f for b in blocks for f in b]
            assert flat == list(range(n))
            sizes = [len(b) for b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        frame_block(4, 2, 2)


def test_two_rank_gloo_video_fill_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax, sums, blocks = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert blocks == [[0, 1, 2], [3, 4]]
    assert tmax == 2.0
    assert sums == [float(sum(int((_frame(f).labels == 255).sum()) for f in range(N_FRAMES))),
                    float(N_FRAMES)]
    assert reduce_over_ranks(sums=[3], maxes=[4.0]) == ([3.0], [4.0])  # no process group
    single = np.array([_fill(f) for f in range(N_FRAMES)])
    assert np.array_equal(merged, single)
