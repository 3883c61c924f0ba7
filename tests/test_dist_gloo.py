"""Multi-process data-parallel logic on CPU (gloo, world size 2): deterministic shard generation,
the prediction all-gather and max-over-ranks timing.  Predictions per shard come from the CPU oracle
(no GPU here); the gathered result must equal a single-process run over the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_00209_b200 import dist as bdist
from paper_1808_00209_b200 import synth

SPEC = dict(h=8, w=8, c=3, layers=[dict(kind="conv", k=3, c_out=32, pool=2), dict(kind="dense", l=10),
                                   dict(kind="dense", l=4)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_predict(images):
    from oracle import oracle as orc
    layers = synth.make_weights(SPEC, 1, 77, small_layers=SPEC["layers"])
    T = synth.thresholds(3, 77).numpy()
    net = orc.Net(8, 8, 3, orc.THRESH_RGB, T, [dict(L, wt=synth.numpy(L["wt"])) for L in layers])
    return net.forward(images)


def _worker(rank, world, port, per_rank, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, n = bdist.shard(per_rank, rank)
    imgs = synth.images_chunked(start, n, 8, 8, 3, seed=5)
    lg, cls = _oracle_predict(imgs.numpy())
    g_lg, g_cls = bdist.gather_predictions(torch.from_numpy(lg).to(torch.int32), torch.from_numpy(cls))
    t = bdist.max_over_ranks(float(rank + 1), "cpu")
    if rank == 0:
        out_q.put((g_lg.numpy(), g_cls.numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,per_rank", [(2, 5), (3, 2)])
def test_gloo_sharded_predictions_match_single_process(world, per_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    g_lg, g_cls, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = synth.images_chunked(0, world * per_rank, 8, 8, 3, seed=5)
    lg, cls = _oracle_predict(full.numpy())
    assert np.array_equal(g_lg, lg.astype(np.int32)) and np.array_equal(g_cls, cls)
    assert t == float(world)


def test_chunked_stream_is_shard_invariant():
    """Any shard of the seeded image stream equals the same slice of a single draw, across the
    4096-image chunk boundary -- so every GPU count sees identical data."""
    full = synth.images_chunked(4090, 12, 2, 2, 3, seed=9)
    a = synth.images_chunked(4090, 5, 2, 2, 3, seed=9)
    b = synth.images_chunked(4095, 7, 2, 2, 3, seed=9)
    assert torch.equal(torch.cat([a, b]), full)


def test_shard_total_covers_everything():
    for n in (1, 7, 262144):
        for world in (1, 2, 3, 8):
            parts = [bdist.shard_total(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == n
            for (s0, c0), (s1, _) in zip(parts, parts[1:]):
                assert s0 + c0 == s1


def _bench_worker(rank, world, port, total, out_q):
    """The sharding / padded-gather / reassembly code of bench.py itself (strong scaling over `total`)."""
    import argparse
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = argparse.Namespace(batch=0, total_batch=total)
    start, n, n_max, tot, scaling = bench.workload(a, world)
    assert tot == total and scaling == "strong"
    imgs = synth.images_chunked(start, n, 8, 8, 3, seed=5)
    lg, cls = _oracle_predict(imgs.numpy())
    lg_pad = torch.zeros((n_max, lg.shape[1]), dtype=torch.int32)
    cls_pad = torch.full((n_max,), -1, dtype=torch.int32)
    lg_pad[:n] = torch.from_numpy(lg.astype(np.int32))
    cls_pad[:n] = torch.from_numpy(cls.astype(np.int32))
    g_lg, g_cls = bdist.gather_predictions(lg_pad, cls_pad)
    if rank == 0:
        a_lg, a_cls = bench.assemble_predictions(g_lg, g_cls, total, world, n_max, scaling)
        out_q.put((a_lg.numpy(), a_cls.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 7), (3, 11)])
def test_gloo_bench_strong_scaling_matches_single_process(world, total):
    """bench.py's strong-scaling shards (uneven when world does not divide the batch), padded all-gather
    and reassembly give exactly the single-process predictions in global image order (SURVEY row e)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    g_lg, g_cls = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = synth.images_chunked(0, total, 8, 8, 3, seed=5)
    lg, cls = _oracle_predict(full.numpy())
    assert g_lg.shape[0] == total
    assert np.array_equal(g_lg, lg.astype(np.int32)) and np.array_equal(g_cls, cls.astype(np.int32))
