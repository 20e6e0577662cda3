"""The N>1 path: images sharded over ranks, no collective on the data path.

World-size-2 process groups with the gloo backend on 127.0.0.1. The CPU test
runs each rank's shard through the oracle (the per-rank GPU work stands in on
CPU); the GPU test runs each rank's shard through the CUDA SpMM on cuda:0 (two
independent processes sharing one GPU; nothing waits on another rank's
kernel). Outputs are gathered only to check them against the full batch.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1911_09723_b200.dist import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_tiles_the_batch():
    for images in (0, 1, 7, 256, 1023):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard(images, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == images
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _worker(rank, world, port, images, use_gpu, q):
    import sys

    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    import torch.distributed as dist

    from paper_1911_09723_b200.dist import Dist, shard
    from paper_1911_09723_b200.workloads import Layer, make_layer_data

    d = Dist("gloo")
    layer = Layer("pw", 96, 64, 7, 9, sparsity=0.85)
    data = make_layer_data(layer, images, 77)  # same seed: every rank sees the same batch
    b0, b1 = shard(images, world, rank)
    if use_gpu:
        import torch

        import paper_1911_09723_b200 as sp

        w = sp.DeviceBcsr(data.weights)
        a = torch.from_numpy(data.act[b0:b1].copy()).cuda()
        o = torch.empty(b1 - b0, layer.cout, layer.h, layer.w, device="cuda")
        sp.spmm_batched_into(w, a, torch.from_numpy(data.bias).cuda(),
                             sp.Activation.clamp(0.0, 6.0), o)
        torch.cuda.synchronize()
        mine = o.cpu().numpy()
    else:
        from oracle import Oracle

        mine = Oracle().spmm(data.weights, data.act[b0:b1], data.bias, layer.act).reshape(
            b1 - b0, layer.cout, layer.h, layer.w)
    d.barrier()
    assert d.max(float(rank + 1)) == float(world)
    assert d.sum(1.0) == float(world)
    parts = [None] * world
    dist.all_gather_object(parts, (b0, b1, mine))  # test-side check only
    if rank == 0:
        q.put(parts)
    d.close()


def run_world(world, images, use_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, images, use_gpu, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return parts


def check(parts, images, oracle):
    from paper_1911_09723_b200.workloads import Layer, make_layer_data

    layer = Layer("pw", 96, 64, 7, 9, sparsity=0.85)
    data = make_layer_data(layer, images, 77)
    full = oracle.spmm(data.weights, data.act, data.bias, layer.act).reshape(
        images, layer.cout, layer.h, layer.w)
    got = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
    assert [p[0] for p in parts][0] == 0 and sorted(parts, key=lambda p: p[0])[-1][1] == images
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


def test_two_rank_gloo_shards_cover_the_batch_cpu(oracle):
    check(run_world(2, 5, use_gpu=False), 5, oracle)


@pytest.mark.gpu
def test_two_rank_gloo_shards_cuda(oracle):
    check(run_world(2, 9, use_gpu=True), 9, oracle)
