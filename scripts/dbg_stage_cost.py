import sys, torch
sys.path.insert(0, ".")
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network
spec = S.cifar3(); B = 128
x, c, _ = S.synth_bench_data(spec, B, 8)
net = Network(spec, B); net.enable_graph(True)
xt = torch.from_numpy(x.reshape(B, -1)).cuda(); ct = torch.from_numpy(c).cuda()
pool = xt.repeat(64, 1).reshape(64, B, -1).contiguous(); cp = ct.repeat(64).reshape(64, B).contiguous()
net.load_batch(xt, cls=ct)
for _ in range(10): net.train_step(B, 0.01, 0.9)
torch.cuda.synchronize()
for mode in ("graph only", "stage+graph", "graph only", "stage+graph"):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for i in range(200):
        if mode == "stage+graph": net.load_batch(pool[i % 64], cls=cp[i % 64])
        net.train_step(B, 0.01, 0.9)
    b.record(); torch.cuda.synchronize()
    print(mode, round(a.elapsed_time(b) / 200 * 1000, 2), "us/step")
