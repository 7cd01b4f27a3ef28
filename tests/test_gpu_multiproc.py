"""World-size-2 run of the frame-parallel (video) path with the GPU engine in
both ranks.

tests/test_multiproc.py runs the same partition on CPU with the oracle
standing in for the kernels; here each rank fills its frame block
(video.frame_block) with the product -- ``video.fill_video_host``, the
pipelined upload / k_prep + k_shells / download loop -- and the ranks
combine their per-frame digests and bookkeeping totals over gloo.  Only one
GPU is visible to these tests, so both ranks use cuda:0: frames are
independent and no rank's kernels wait on the other's (the fill has no
data-path collective), so sharing the device changes timing, not results.
Every frame must equal the CPU oracle's fill (order bit-exact, values within
1e-4), whichever rank filled it.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_05319_b200 import FillParams, Spline, scenes
from paper_1611_05319_b200.video import frame_block, reduce_over_ranks

pytestmark = pytest.mark.gpu

N_FRAMES = 5


def _frame(f):
    return scenes.small_scene(90, 160, band=6, gx=4, gy=3, n_spl=3, seed=1611, frame=f)


def _splines(sc):
    return [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                   kind=s["kind"]) for s in sc.splines]


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1611_05319_b200 import _native, video

    mine = list(frame_block(N_FRAMES, world, rank))
    frames = [_frame(f) for f in mine]
    p = FillParams(**frames[0].params)
    launches0 = _native.launch_count()
    got = video.fill_video_host([sc.image for sc in frames], [sc.labels for sc in frames],
                                [_splines(sc) for sc in frames], p)
    launches = _native.launch_count() - launches0
    # per frame: filled pixels, shells, then the filled values (padded)
    H, W = frames[0].labels.shape if frames else (0, 0)
    out = torch.full((N_FRAMES, 2 + H * W * 3), -1.0, dtype=torch.float64)
    for f, (u, rep) in zip(mine, got):
        out[f, 0] = rep.filled
        out[f, 1] = len(rep.rows)
        out[f, 2:] = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64).reshape(-1))
    gathered = [torch.zeros_like(out) for _ in range(world)]
    dist.all_gather(gathered, out)
    sums, _ = reduce_over_ranks(sums=[len(mine), launches], maxes=[0.0])
    if rank == 0:
        merged = torch.stack(gathered).max(dim=0).values
        out_q.put((merged.numpy(), sums))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gpu_video_fill_matches_oracle():
    from oracle import guidefill_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, sums = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sums[0] == N_FRAMES
    assert sums[1] >= 2 * N_FRAMES, "the ranks launched none of the engine's kernels"
    for f in range(N_FRAMES):
        sc = _frame(f)
        field = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in sc.splines],
                                [s["direction"] for s in sc.splines], sc.labels)
        ref = orc.fill(sc.image, sc.labels, field, orc.Params(**sc.params), tracked=True)
        assert merged[f, 0] == sum(r[4] for r in ref["rows"])
        assert merged[f, 1] == len(ref["rows"])
        u = merged[f, 2:].reshape(sc.image.shape)
        err = float(np.abs(u - ref["u"]).max())
        assert err <= 1e-4, f"frame {f}: values differ by {err}"
