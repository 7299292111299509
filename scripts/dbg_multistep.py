"""Diagnostic: per-step time of one engine graph per step vs one CUDA graph
holding several steps (inter-graph launch gaps)."""
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
    torch.cuda.synchronize()

    def timeit(fn, n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        fn(n)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1000 / n

    print("engine graph per step:", round(timeit(lambda n: [net.train_step(B, 0.01, 0.9) for _ in range(n)], 400), 2), "us")
    for k in (2, 4, 8):
        net.enable_graph(False)
        g = torch.cuda.CUDAGraph()
        for _ in range(2):
            net.train_step(B, 0.01, 0.9)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(k):
                net.train_step(B, 0.01, 0.9)
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        t = timeit(lambda n: [g.replay() for _ in range(n // k)], 400)
        print(f"{k} steps per graph:", round(t, 2), "us/step")
