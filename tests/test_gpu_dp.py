"""Data parallelism with the REAL engine on one B200 (the box has
one GPU, so the replicas share it):

  * G logical shards (vcnn_dp_group, barrier-free group step): G replicas,
    each on its contiguous shard, exchanged by the fused peer-reduce + SGD +
    pack kernel -- the replicas stay bit-identical and follow the single-GPU
    trajectory on the global batch (3xTF32 within 1e-5, TF32 within 1e-3);
    equal and unequal shards;
  * the same kernel in barrier mode: replicas stepped independently on their
    own streams (CUDA graphs on), synchronising inside the exchange kernel
    through their signal buffers exactly as across GPUs -- bit-identical to
    the barrier-free group;
  * the process-per-GPU bootstrap (vcnn_dp_init over NCCL) and the NCCL
    exchange at world size 1;
  * two PROCESSES on the one GPU connected through CUDA IPC handles
    (vcnn_dp_create / handle / connect), the cross-process P2P path."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.dp import NCCL, P2P, DataParallel, shard_range
from paper_1501_07338_b200.engine import Network
from paper_1501_07338_b200.spec import Precision

from .test_gpu_net import _load
from .util import TOL, assert_close

pytestmark = pytest.mark.gpu
A = S.Activation
DENOISE_MINI = S.NetworkSpec((24, 24, 1), [S.ConvSpec(8, 9, 9, 1, A.relu),
                                            S.ConvSpec(8, 1, 1, 1, A.relu),
                                            S.ConvSpec(1, 5, 5, 1, A.identity)],
                             S.LossKind.mse, 7)
STEPS, LR, MOM = 4, 0.01, 0.9


def _single(spec, x, cls, vals, prec, steps=STEPS):
    B = x.shape[0]
    net = Network(spec, B, prec)
    _load(net, spec, x, cls, vals)
    for _ in range(steps):
        net.train_step(B, LR, MOM)
    p = net.get_params()
    net.close()
    return p


def _replicas(spec, x, cls, vals, prec, G, streams=False):
    B = x.shape[0]
    nets, sizes = [], []
    for r in range(G):
        lo, hi = shard_range(B, r, G)
        st = torch.cuda.Stream() if streams else None
        net = Network(spec, hi - lo, prec, stream=st)
        _load(net, spec, x[lo:hi], None if cls is None else cls[lo:hi],
              None if vals is None else vals[lo:hi])
        nets.append(net)
        sizes.append(hi - lo)
    torch.cuda.synchronize()
    return nets, sizes


CASES = [("cifar3", 64, 2), ("cifar3", 64, 4), ("cifar3", 37, 2), ("denoise-mini", 10, 3)]


@pytest.mark.parametrize("prec", [Precision.tf32x3, Precision.tf32], ids=lambda p: p.name)
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-b{c[1]}-g{c[2]}")
def test_logical_shards_follow_global_batch(case, prec):
    name, B, G = case
    spec = S.cifar3() if name == "cifar3" else DENOISE_MINI
    x, cls, vals = S.synth_bench_data(spec, B, 8)
    is_ce = spec.loss == S.LossKind.softmax_ce
    cls, vals = (cls, None) if is_ce else (None, vals)
    p_single = _single(spec, x, cls, vals, prec)
    nets, sizes = _replicas(spec, x, cls, vals, prec, G)
    dps = DataParallel.local_group(nets, barrier=False)
    for _ in range(STEPS):
        DataParallel.group_train_step(dps, sizes, LR, MOM)
    ps = [n.get_params() for n in nets]
    for r in range(1, G):
        assert np.array_equal(ps[r], ps[0]), f"replica {r} diverged"
    assert_close(ps[0], p_single, TOL[prec], f"G={G} shards vs the global batch")
    for n in nets:
        n.close()


def test_barrier_mode_concurrent_streams_equals_group():
    """Replicas stepped independently (own stream, CUDA graph with the exchange
    kernel inside) meet in the kernel's signal barrier; bit-identical to the
    event-ordered group step.  (Both replicas share the one GPU here, so the
    net avoids the 16-CTA cluster tail kernel: a replica spinning in its
    exchange could keep the other's cluster from being placed -- a one-GPU
    artefact; across GPUs each replica has its own SMs.)"""
    spec, B, G = DENOISE_MINI, 16, 2
    x, _, vals = S.synth_bench_data(spec, B, 8)
    res = []
    for barrier in (False, True):
        nets, sizes = _replicas(spec, x, None, vals, Precision.tf32, G, streams=barrier)
        dps = DataParallel.local_group(nets, barrier=barrier)
        for _ in range(STEPS):
            if barrier:
                for n, d, b in zip(nets, dps, sizes):
                    n.enable_graph(True)
                    d.train_step(b, LR, MOM)
            else:
                DataParallel.group_train_step(dps, sizes, LR, MOM)
        for d in dps:
            d.status()  # no barrier timed out
        res.append([n.get_params() for n in nets])
        for n in nets:
            n.close()
    for r in range(G):
        assert np.array_equal(res[0][r], res[1][r])


def test_barrier_mode_with_batch_ring_equals_explicit_loads():
    """The bench's multi-GPU step: each replica stages its shard's next batch
    from its own device batch ring inside its graph (vcnn_net_set_batch_ring),
    then the fused exchange -- identical to staging every batch explicitly."""
    spec, B, G, nb = DENOISE_MINI, 16, 2, 3
    x, _, vals = S.synth_bench_data(spec, B * nb, 8)
    xs = torch.as_tensor(x.reshape(nb, B, -1), device="cuda")
    vs = torch.as_tensor(vals.reshape(nb, B, -1), device="cuda")
    res = []
    for ring in (False, True):
        nets, sizes = _replicas(spec, x[:B], None, vals[:B], Precision.tf32, G, streams=True)
        dps = DataParallel.local_group(nets, barrier=True)
        for r, n in enumerate(nets):
            lo, hi = shard_range(B, r, G)
            n.enable_graph(True)
            if ring:
                n.set_batch_ring(xs[:, lo:hi].contiguous(), vs[:, lo:hi].contiguous())
        for i in range(5):
            for r, (n, d, b) in enumerate(zip(nets, dps, sizes)):
                if not ring:
                    lo, hi = shard_range(B, r, G)
                    n.load_batch(xs[i % nb, lo:hi], values=vs[i % nb, lo:hi])
                d.train_step(b, LR, MOM)
        for d in dps:
            d.status()
        res.append([n.get_params() for n in nets])
        for n in nets:
            n.close()
    for r in range(G):
        assert np.array_equal(res[0][r], res[1][r])
    assert np.array_equal(res[1][0], res[1][1])


@pytest.fixture
def world1_pg(tmp_path):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def test_nccl_bootstrap_and_nccl_exchange_world1(world1_pg):
    """vcnn_dp_init (NCCL communicator + handle all-gather over it) at world
    size 1; P2P and NCCL exchanges both reduce to the plain update."""
    spec, B = S.cifar3(), 32
    x, cls, _ = S.synth_bench_data(spec, B, 8)
    p_single = _single(spec, x, cls, None, Precision.tf32)
    for mode in (P2P, NCCL):
        net = Network(spec, B)
        _load(net, spec, x, cls, None)
        dp = DataParallel(net, mode=mode)
        assert dp.mode == mode and dp.world == 1
        for _ in range(STEPS):
            dp.train_step(B, LR, MOM)
        assert np.array_equal(net.get_params(), p_single)
        net.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, x, cls, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec, B = S.cifar3(), x.shape[0]
    lo, hi = shard_range(B, rank, world)
    net = Network(spec, hi - lo)
    _load(net, spec, x[lo:hi], cls[lo:hi], None)

    def allgather(b):
        box = [None] * world
        dist.all_gather_object(box, b)
        return box

    dp = DataParallel.connect_with(net, world, rank, allgather)
    for _ in range(STEPS):
        dp.train_step(hi - lo, LR, MOM)
    dp.status()
    out[rank] = net.get_params()
    net.close()
    dist.destroy_process_group()


def test_two_processes_ipc_p2p_on_one_gpu():
    """The cross-process path: CUDA IPC mappings of the peer's gradient and
    signal buffers, barrier across processes (time-sliced on one GPU)."""
    import torch.multiprocessing as mp
    spec, B, G = S.cifar3(), 64, 2
    x, cls, _ = S.synth_bench_data(spec, B, 8)
    nets, sizes = _replicas(spec, x, cls, None, Precision.tf32, G)
    dps = DataParallel.local_group(nets, barrier=False)
    for _ in range(STEPS):
        DataParallel.group_train_step(dps, sizes, LR, MOM)
    want = nets[0].get_params()
    for n in nets:
        n.close()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_ipc_worker, args=(G, _free_port(), x, cls, out), nprocs=G,
                       start_method="spawn", join=True)
    for r in range(G):
        assert np.array_equal(out[r], want), r
