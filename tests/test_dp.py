"""Data-parallel path.

CPU (gloo, world size 2): each rank profiles its own shard of the global token
stream with the oracle and all-reduces the int64 histograms; the result must
equal the single-process histogram of the whole batch — the property the
NCCL all-reduce of flux_reduce_stats relies on (tokens independent, counts
additive).  GPU: a 1-rank NCCL communicator through the C ABI is the identity
on the histogram.
"""
import os
import socket

import numpy as np
import pytest

import synth

TOY = synth.CONFIGS["toy"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T_rank, out_dir):
    import torch
    import torch.distributed as dist

    import oracle.model as om
    from paper_2508_19078_b200.driver import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t0, n = shard(rank, world, T_rank)
    res = om.profile_tokens(TOY, np.arange(t0, t0 + n))
    hist = np.stack([np.bincount(r["ids"].ravel(), minlength=TOY.n_experts) for r in res]).astype(np.int64)
    h = torch.from_numpy(hist)
    dist.all_reduce(h, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(os.path.join(out_dir, "hist.npy"), h.numpy())
    dist.destroy_process_group()


def test_dp_histogram_allreduce_equals_single_process(tmp_path):
    import torch.multiprocessing as mp

    import oracle.model as om
    world, T_rank = 2, TOY.tokens // 2
    mp.start_processes(_worker, args=(world, _free_port(), T_rank, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    reduced = np.load(tmp_path / "hist.npy")
    full = om.profile_tokens(TOY, np.arange(world * T_rank))
    want = np.stack([np.bincount(r["ids"].ravel(), minlength=TOY.n_experts) for r in full])
    assert np.array_equal(reduced, want)
    assert np.all(reduced.sum(1) == world * T_rank * TOY.top_k)


def test_shards_partition_the_token_stream():
    from paper_2508_19078_b200.driver import shard
    for world in (1, 2, 4, 8):
        T = 1000
        covered = np.concatenate([np.arange(*(lambda a, b: (a, a + b))(*shard(r, world, T))) for r in range(world)])
        assert np.array_equal(covered, np.arange(world * T))
    with pytest.raises(ValueError):
        shard(2, 2, 10)


@pytest.mark.gpu
def test_reduce_stats_single_rank_nccl_is_identity():
    import torch

    import paper_2508_19078_b200 as F
    comm = F.Comm(F.Comm.unique_id(), 1, 0)
    h = torch.arange(28 * 64, dtype=torch.int64, device="cuda").reshape(28, 64) * 3
    ref = h.clone()
    comm.reduce_stats(h)
    torch.cuda.synchronize()
    comm.destroy()
    assert torch.equal(h, ref)
