"""Data parallelism across the GPUs of one box (one process per GPU).

The reference has no distributed path; the exchange
is inserted where Trainer<T>::fit goes from run_batch to sgd_step
(proj/include/vcnn/training.hpp:76-81):

    run_batch(local shard) -> all-reduce(grads, sum) -> sgd_step (replicated)

* Sharding: contiguous sample ranges, the Imp-2 chunking of the reference
  ([B*r/W, B*(r+1)/W), variants.hpp:442-443).
* Normalisation: loss_backward scales by 1/B_local (layers.hpp:444), so each
  rank's gradient is pre-weighted by B_local/B_global and the sum is the
  global-batch mean.  With equal shards the weight is the constant 1/W and is
  folded into the SGD kernel's grad_scale (no extra pass).
* The collective is NCCL all-reduce over NVLink on one flat fp32 buffer (the
  engine keeps every parameter gradient in one buffer, NetGrads order), so a
  step issues exactly one collective.  Every rank applies the same SGD to the
  same summed gradient: replicas stay bit-identical.

`model` is anything with the engine's Network surface used here
(forward_backward(B), grads_tensor(), sgd_step(lr, mom, scale)); the product
passes engine.Network (device buffers, NCCL); the CPU tests pass an oracle
stand-in over gloo to check the host logic.
"""
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous shard (variants.hpp:442-443 chunking)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return global_batch * rank // world, global_batch * (rank + 1) // world


class DataParallel:
    """One training step of a model replica on this rank's shard."""

    def __init__(self, model, group: Optional[dist.ProcessGroup] = None):
        self.model = model
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def shard(self, global_batch: int) -> Tuple[int, int]:
        return shard_range(global_batch, self.rank, self.world)

    def step(self, local_batch: int, global_batch: int, lr: float, momentum: float):
        """forward_backward on the staged local shard, gradient exchange,
        replicated sgd_step.  Stream-ordered (no host sync)."""
        m = self.model
        m.forward_backward(local_batch)
        if self.world == 1:
            m.sgd_step(lr, momentum, 1.0)
            return
        grads = m.grads_tensor()
        equal = global_batch % self.world == 0
        if not equal:
            grads.mul_(local_batch / global_batch)
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=self.group)
        m.sgd_step(lr, momentum, 1.0 / self.world if equal else 1.0)
