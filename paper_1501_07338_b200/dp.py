"""Data parallelism across the GPUs of one box, through the C ABI
(`vcnn_dp_*`, csrc/dp.cu).

The reference has no distributed path; the exchange is inserted
where Trainer<T>::fit goes from run_batch to sgd_step
(proj/include/vcnn/training.hpp:76-81):

    run_batch(local shard) -> sum of every replica's gradient -> sgd_step

* Sharding: contiguous sample ranges, the Imp-2 chunking of the reference
  ([B*r/W, B*(r+1)/W), variants.hpp:442-443).  In Trainer::fit every rank
  draws the same seeded permutation and takes its contiguous slice of each
  global batch (`epoch_shards`), so the W replicas together see exactly the
  single-GPU batches.
* Normalisation: loss_backward scales by 1/B_local (layers.hpp:444), so the
  exchange weights rank p's gradient by B_p / B_global (`shard_weights`) and
  the sum is the global-batch mean.
* Exchange (attached to the net: its sgd step, graph-captured, IS the
  exchange): VCNN_DP_P2P -- one kernel per replica reads every replica's flat
  gradient over NVLink peer mappings, sums it in rank order and applies
  momentum SGD + the conv weight packs (replicas stay bit-identical);
  VCNN_DP_NCCL -- ncclAllReduce + the replicated update.
"""
import ctypes as C
from typing import List, Optional, Sequence, Tuple

from ._lib import check, lib

P2P, NCCL = 0, 1
ID_BYTES, HANDLE_BYTES = 128, 256


def shard_range(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous shard (variants.hpp:442-443 chunking)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return global_batch * rank // world, global_batch * (rank + 1) // world


def shard_sizes(global_batch: int, world: int) -> List[int]:
    return [hi - lo for lo, hi in (shard_range(global_batch, r, world) for r in range(world))]


def shard_weights(global_batch: int, world: int) -> List[float]:
    """B_p / B_global: the weight of rank p's (batch-mean) gradient in the sum."""
    return [b / global_batch for b in shard_sizes(global_batch, world)]


def epoch_shards(order: Sequence[int], batch: int, rank: int, world: int):
    """DP-aware batches of one epoch: for every global batch of `order` (the
    epoch's permutation, identical on all ranks; the last batch may be
    smaller, training.hpp:70-74) yield (rank's sample ids, per-rank sizes)."""
    for start in range(0, len(order), batch):
        gb = min(batch, len(order) - start)
        if gb < world:
            raise ValueError(f"global batch {gb} cannot give each of {world} ranks a sample")
        lo, hi = shard_range(gb, rank, world)
        yield list(order[start + lo:start + hi]), shard_sizes(gb, world)


class DataParallel:
    """This rank's replica group handle (vcnn_dp).  Construct collectively on
    every rank (one process per GPU) after torch.distributed is initialised,
    or build a single-process group with `local_group`."""

    def __init__(self, net, world: Optional[int] = None, rank: Optional[int] = None,
                 mode: int = P2P, pg=None, _handle=None):
        self.net = net
        net.__dict__.setdefault("_dps", []).append(self)  # closed before the net
        if _handle is not None:
            self._h = _handle
            self.world, self.rank = world, rank
            return
        import torch.distributed as dist
        if world is None:
            world, rank = dist.get_world_size(pg), dist.get_rank(pg)
        self.world, self.rank = world, rank
        uid = (C.c_uint8 * ID_BYTES)()
        if rank == 0:
            check(lib().vcnn_dp_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=pg)
        uid = (C.c_uint8 * ID_BYTES).from_buffer_copy(box[0])
        h = C.c_void_p()
        check(lib().vcnn_dp_init(net._h, world, rank, uid, C.byref(h)))
        self._h = h
        if mode != P2P:
            self.set_mode(mode)

    @classmethod
    def connect_with(cls, net, world: int, rank: int, allgather, nccl_id=None):
        """Three-step setup for hosts that move the handles themselves:
        `allgather(bytes) -> [bytes of rank 0, 1, ...]` (any transport)."""
        h = C.c_void_p()
        check(lib().vcnn_dp_create(net._h, world, rank, C.byref(h)))
        mine = (C.c_uint8 * HANDLE_BYTES)()
        check(lib().vcnn_dp_handle(h, mine))
        alls = allgather(bytes(mine))
        buf = (C.c_uint8 * (HANDLE_BYTES * world)).from_buffer_copy(b"".join(alls))
        uid = None if nccl_id is None else (C.c_uint8 * ID_BYTES).from_buffer_copy(nccl_id)
        st = lib().vcnn_dp_connect(h, buf, uid)
        if st:
            lib().vcnn_dp_destroy(h)
            check(st)
        return cls(net, world, rank, _handle=h)

    @classmethod
    def local_group(cls, nets, barrier: bool = False) -> List["DataParallel"]:
        """G replicas in this process (G logical shards on one device, or one
        replica per device).  barrier=False: step them together with
        `group_train_step`; barrier=True: step each independently on its own
        stream (they synchronise inside the exchange kernel)."""
        G = len(nets)
        hs = (C.c_void_p * G)()
        arr = (C.c_void_p * G)(*[n._h for n in nets])
        check(lib().vcnn_dp_group(arr, G, int(bool(barrier)), hs))
        return [cls(n, G, r, _handle=C.c_void_p(hs[r])) for r, n in enumerate(nets)]

    @staticmethod
    def group_train_step(dps: Sequence["DataParallel"], batches: Sequence[int], lr, momentum):
        G = len(dps)
        arr = (C.c_void_p * G)(*[d._h for d in dps])
        b = (C.c_int * G)(*batches)
        check(lib().vcnn_dp_group_train_step(arr, G, b, float(lr), float(momentum)))

    @property
    def mode(self) -> int:
        m = C.c_int()
        check(lib().vcnn_dp_get_mode(self._h, C.byref(m)))
        return m.value

    def set_mode(self, mode: int):
        check(lib().vcnn_dp_set_mode(self._h, int(mode)))

    def set_shards(self, batches: Sequence[int]):
        check(lib().vcnn_dp_set_shards(self._h, (C.c_int * self.world)(*batches)))

    def train_step(self, batch: int, lr, momentum):
        """forward_backward on the staged local shard + exchange + sgd_step
        (graph-replayed when the net has graphs enabled)."""
        check(lib().vcnn_dp_train_step(self._h, int(batch), float(lr), float(momentum)))

    def allreduce_sgd(self, lr, momentum):
        check(lib().vcnn_dp_allreduce_sgd(self._h, float(lr), float(momentum)))

    def status(self):
        """Synchronise; raises (VCNN_ENCCL) if an exchange barrier timed out."""
        check(lib().vcnn_dp_status(self._h))

    def close(self):
        if self._h:
            lib().vcnn_dp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
