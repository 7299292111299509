"""One pass over every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): CIFAR-3 fused + trace + 3xTF32 + fp32 steps, the
forward-only chain, denoise-style (K=1 kernels), deconv-121 (1-D segment
direct conv), the tap-stacked forward + batch-sliced tail (b128 / b256), a 2-replica DP group step
(barrier-free: the sanitizer serialises kernels) and the op-level ABI."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1501_07338_b200 import ops, spec as S  # noqa: E402
from paper_1501_07338_b200.dp import DataParallel  # noqa: E402
from paper_1501_07338_b200.engine import Network  # noqa: E402

A = S.Activation


def step(spec, B, prec=S.Precision.tf32, trace=False, graph=False, n=2):
    x, c, v = S.synth_bench_data(spec, B, 8)
    net = Network(spec, B, prec)
    net.set_trace(trace)
    net.enable_graph(graph)
    xt = torch.from_numpy(x.reshape(B, -1)).cuda()
    if spec.loss == S.LossKind.softmax_ce:
        net.load_batch(xt, cls=torch.from_numpy(c).cuda())
    else:
        net.load_batch(xt, values=torch.from_numpy(v).cuda())
    for _ in range(n):
        net.train_step(B, 0.01, 0.9)
    net.forward(B)
    torch.cuda.synchronize()
    net.close()


step(S.cifar3(), 16)
step(S.cifar3(), 16, trace=True)
step(S.cifar3(), 8, S.Precision.tf32x3)
step(S.cifar3(), 8, S.Precision.fp32)
step(S.cifar3(), 256, n=1)  # large batch (tap-stacked forward, 8-slice tail)
step(S.cifar3(), 128, n=1)  # the benchmark batch (8-slice tail, folded update)
step(S.lenet_caffe(), 16)
step(S.NetworkSpec((40, 40, 1), [S.ConvSpec(16, 16, 16, 1, A.relu), S.ConvSpec(16, 1, 1, 1, A.relu),
                                 S.ConvSpec(1, 8, 8, 1, A.identity)], S.LossKind.mse, 7), 2)
step(S.deconv121(), 1, n=1)
# DP group (G = 2 logical shards)
spec = S.cifar3()
x, c, _ = S.synth_bench_data(spec, 16, 8)
nets = []
for r in range(2):
    net = Network(spec, 8)
    net.load_batch(torch.from_numpy(x[8 * r:8 * r + 8].reshape(8, -1)).cuda(),
                   cls=torch.from_numpy(c[8 * r:8 * r + 8]).cuda())
    nets.append(net)
dps = DataParallel.local_group(nets)
DataParallel.group_train_step(dps, [8, 8], 0.01, 0.9)
torch.cuda.synchronize()
for n in nets:
    n.close()
# op level
a = torch.rand(37, 300, device="cuda")
b = torch.rand(300, 45, device="cuda")
ops.gemm(a, b, bias=torch.rand(45, device="cuda"), act=A.relu)
xx = torch.rand(2, 8, 12, 12, device="cuda")
ops.pool_forward(xx, 2, 2, 2)
ops.im2col(xx, 3, 3, 1)
torch.cuda.synchronize()
print("sanitize pass done")
