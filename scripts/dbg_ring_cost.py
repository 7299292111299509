"""Diagnostic: step time with the in-graph ring staging vs a static batch."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1501_07338_b200 import spec as S  # noqa: E402
from paper_1501_07338_b200.engine import Network  # noqa: E402

spec, B, NB = S.cifar3(), 128, 171
x, c, _ = S.synth_bench_data(spec, B * 8, 9)
xp = torch.from_numpy(x.reshape(8, B, -1)).cuda().repeat(22, 1, 1)[:NB].contiguous()
cp = torch.from_numpy(c.reshape(8, B)).cuda().repeat(22, 1)[:NB].contiguous()
net = Network(spec, B)
net.enable_graph(True)
net.load_batch(xp[0], cls=cp[0])
for mode in ("static", "ring", "static", "ring"):
    if mode == "ring":
        net.set_batch_ring(xp, cp)
    else:
        net.set_batch_ring()
    net.train_steps(16, B, 0.01, 0.9)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    net.train_steps(400, B, 0.01, 0.9)
    b.record()
    torch.cuda.synchronize()
    print(mode, round(a.elapsed_time(b) / 400 * 1000, 2), "us/step")
