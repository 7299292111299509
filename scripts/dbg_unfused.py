import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network
spec = S.cifar3(); B = 128
x, c, _ = S.synth_bench_data(spec, B, 8)
net = Network(spec, B)
net.load_batch(torch.from_numpy(x.reshape(B, -1)).cuda(), cls=torch.from_numpy(c).cuda())
for trace in (False, True):
    net.set_trace(trace)
    for i in range(3):
        net.train_step(B, 0.01, 0.9)
    net.enable_breakdown(True)
    for i in range(10):
        net.train_step(B, 0.01, 0.9)
    ops = net.read_op_timing()
    net.enable_breakdown(False)
    print("trace", trace)
    for k, (s, n) in sorted(ops.items()):
        print("  ", k, round(s / n * 1e6, 1), "us x", n)
