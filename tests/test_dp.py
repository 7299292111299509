"""Data-parallel host logic on CPU, world_size 2 over gloo (the device
exchange itself is covered by tests/test_gpu_dp.py).

What the product's DP layer decides on the host is checked here against the
REFERENCE's own Trainer<double>::fit on the global data (oracle/_ref):
  * dp.epoch_shards -- every rank draws the same seeded permutation and takes
    its contiguous slice (Imp-2 chunking, variants.hpp:442-443) of each global
    batch, including the smaller last batch;
  * dp.shard_weights -- B_p / B_global, the weights the exchange kernel applies
    to each replica's batch-mean gradient (loss_backward scales by 1/B_local,
    layers.hpp:444);
  * the rank-ordered weighted sum (the exchange kernel's arithmetic:
    s = w_0 g_0, then s = fma(w_p, g_p, s) for p = 1..W-1) + replicated SGD.
The replica's forward/backward is the oracle (C restatement, f64): test
infrastructure standing in for the device engine."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_py as O
from paper_1501_07338_b200 import _lib, spec as S
from paper_1501_07338_b200.dp import epoch_shards, shard_range, shard_sizes, shard_weights

A = S.Activation
SPEC = S.NetworkSpec((8, 8, 2), [S.ConvSpec(4, 3, 3, 1, A.relu), S.PoolSpec(2, 2, 2),
                                 S.FullSpec(3, A.identity)], S.LossKind.softmax_ce, 11)
N, BATCH, EPOCHS, SEED, LR, MOM = 23, 8, 2, 5, 0.05, 0.9  # batches 8, 8, 7


def _data():
    x, cls, _ = O.synth_bench_data(SPEC, N, 8)
    return x.astype(np.float64), cls


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, cls = _data()
        p = O.net_init(SPEC)
        v = np.zeros_like(p)
        order = list(range(N))
        rng = S.Rng(SEED)
        losses = []
        for _ in range(EPOCHS):
            rng.shuffle(order)  # same permutation on every rank
            tot, nb = 0.0, 0
            for ids, sizes in epoch_shards(order, BATCH, rank, world):
                assert len(ids) == sizes[rank]
                r = O.net_run_batch(SPEC, p, x[ids], cls=cls[ids])
                g = torch.from_numpy(r["grads"].copy())
                box = [torch.zeros_like(g) for _ in range(world)]
                dist.all_gather(box, g)
                w = [b / sum(sizes) for b in sizes]
                s = w[0] * box[0].numpy()
                for q in range(1, world):
                    s = w[q] * box[q].numpy() + s
                O.sgd_step(p, v, s, LR, MOM)
                lt = torch.tensor([r["loss"] * w[rank]], dtype=torch.float64)
                dist.all_reduce(lt)
                tot += float(lt)
                nb += 1
            losses.append(tot / nb)
        out[rank] = (p, losses)
    finally:
        dist.destroy_process_group()


def test_shard_range_is_contiguous_partition():
    for B in (1, 7, 8, 128, 1000):
        for W in (1, 2, 3, 4, 8):
            rs = [shard_range(B, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1 and sizes == shard_sizes(B, W)
            assert abs(sum(shard_weights(B, W)) - 1.0) < 1e-15
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def test_epoch_shards_cover_each_global_batch():
    order = list(np.random.default_rng(0).permutation(23))
    for W in (1, 2, 3):
        per_rank = [list(epoch_shards(order, 8, r, W)) for r in range(W)]
        for b in range(3):
            got = sum((per_rank[r][b][0] for r in range(W)), [])
            assert got == order[8 * b:8 * b + 8]
    with pytest.raises(ValueError):
        list(epoch_shards(list(range(9)), 8, 0, 2))  # last global batch of 1 < 2 ranks


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")
def test_dp_two_ranks_fit_equals_reference_trainer():
    """2 gloo ranks, each training on its DP-aware shards with the weighted
    rank-ordered exchange == the reference's Trainer<double>::fit on the whole
    dataset (same seed, same batches incl. the smaller last one)."""
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                           start_method="spawn")
        (p0, l0), (p1, l1) = out[0], out[1]
    assert np.array_equal(p0, p1), "replicas diverged"
    x, cls = _data()
    pr, el, _ = O.ref_fit(SPEC, O.net_init(SPEC), x, cls, None, LR, MOM, BATCH, EPOCHS, SEED)
    assert np.abs(p0 - pr).max() <= 1e-12 * np.abs(pr).max()
    assert np.allclose(l0, el, rtol=1e-12, atol=0) and l0 == l1


def test_nccl_unique_id_without_device():
    """vcnn_dp_unique_id (rank 0 of vcnn_dp_init's bootstrap) needs no GPU."""
    import ctypes as C
    a, b = (C.c_uint8 * 128)(), (C.c_uint8 * 128)()
    assert _lib.lib().vcnn_dp_unique_id(a) == 0 and _lib.lib().vcnn_dp_unique_id(b) == 0
    assert bytes(a) != bytes(b)
