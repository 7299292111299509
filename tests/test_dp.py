"""Data-parallel host logic (dp.DataParallel) on CPU: world_size 2 over gloo.

The replica is an oracle stand-in (test infrastructure: forward_backward by
the C restatement of Executor<double>(imp6).run_batch, sgd_step by the
restated network.hpp:242-273), so these tests check exactly the DP layer --
contiguous sharding, gradient pre-weighting, the all-reduce, replicated SGD --
against a single process training on the whole global batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.dp import DataParallel, shard_range

A = S.Activation
SPEC = S.NetworkSpec((8, 8, 2), [S.ConvSpec(4, 3, 3, 1, A.relu), S.PoolSpec(2, 2, 2),
                                 S.FullSpec(3, A.identity)], S.LossKind.softmax_ce, 11)


class OracleReplica:
    """The Network surface DataParallel uses, computed by the oracle."""

    def __init__(self, spec, params, x, cls):
        self.spec, self.p, self.x, self.cls = spec, params.copy(), x, cls
        self.v = np.zeros_like(params)
        self.g = None

    def forward_backward(self, batch):
        assert batch == self.x.shape[0]
        r = O.net_run_batch(self.spec, self.p, self.x, cls=self.cls)
        self.g = torch.from_numpy(r["grads"].copy())

    def grads_tensor(self):
        return self.g

    def sgd_step(self, lr, mom, scale):
        O.sgd_step(self.p, self.v, self.g.numpy() * scale, lr, mom)


def _data(B):
    x, cls, _ = O.synth_bench_data(SPEC, B, 8)
    return x.astype(np.float64), cls


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, cls = _data(B)
        lo, hi = shard_range(B, rank, world)
        rep = OracleReplica(SPEC, O.net_init(SPEC), x[lo:hi], cls[lo:hi])
        dp = DataParallel(rep)
        assert (dp.rank, dp.world) == (rank, world)
        for _ in range(steps):
            dp.step(hi - lo, B, 0.05, 0.9)
        out[rank] = rep.p
    finally:
        dist.destroy_process_group()


def _single(B, steps):
    x, cls = _data(B)
    rep = OracleReplica(SPEC, O.net_init(SPEC), x, cls)
    for _ in range(steps):
        rep.forward_backward(B)
        rep.sgd_step(0.05, 0.9, 1.0)
    return rep.p


def test_shard_range_is_contiguous_partition():
    for B in (1, 7, 8, 128, 1000):
        for W in (1, 2, 3, 4, 8):
            rs = [shard_range(B, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


@pytest.mark.parametrize("B", [8, 7])  # equal and unequal shards
def test_dp_two_ranks_equals_global_batch(B):
    steps = 3
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _free_port(), B, steps, out), nprocs=2, join=True,
                           start_method="spawn")
        p0, p1 = out[0], out[1]
    ref = _single(B, steps)
    assert np.array_equal(p0, p1), "replicas diverged"
    err = np.abs(p0 - ref).max() / np.abs(ref).max()
    assert err < 1e-12, err


def test_dp_world_one_is_plain_step():
    B = 6
    x, cls = _data(B)
    rep = OracleReplica(SPEC, O.net_init(SPEC), x, cls)
    DataParallel(rep).step(B, B, 0.05, 0.9)
    assert np.array_equal(rep.p, _single(B, 1))
