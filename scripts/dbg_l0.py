"""Diagnostic: single-step vs multi-step graph step time (for env A/B of the
backward's stream placement)."""
import os
import sys
import torch
sys.path.insert(0, ".")
from paper_1501_07338_b200 import spec as S  # noqa: E402
from paper_1501_07338_b200.engine import Network  # noqa: E402

spec, B, NB = S.cifar3(), 128, 64
x, c, _ = S.synth_bench_data(spec, B * NB, 9)
xp = torch.from_numpy(x.reshape(NB, B, -1)).cuda()
cp = torch.from_numpy(c.reshape(NB, B)).cuda()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    net = Network(spec, B, stream=st)
    net.set_batch_ring(xp, cp)
    net.enable_graph(True)
    for _ in range(10):
        net.train_step(B, 0.01, 0.9)
    net.train_steps(16, B, 0.01, 0.9)
    torch.cuda.synchronize()

    def timeit(fn, n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        fn(n)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1000 / n

    r1 = timeit(lambda n: [net.train_step(B, 0.01, 0.9) for _ in range(n)], 400)
    r8 = timeit(lambda n: net.train_steps(n, B, 0.01, 0.9), 400)
    print(os.environ.get("TAG", ""), "single", round(r1, 2), "multi", round(r8, 2), "us/step")
