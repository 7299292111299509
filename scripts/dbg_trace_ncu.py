import sys, torch
sys.path.insert(0, '.')
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network
spec = S.cifar3(); B = 128
x, c, _ = S.synth_bench_data(spec, B, 8)
net = Network(spec, B)
net.load_batch(torch.from_numpy(x.reshape(B, -1)).cuda(), cls=torch.from_numpy(c).cuda())
net.set_trace(True)
net.enable_graph(False)
net.enable_breakdown(len(sys.argv) > 1)
for i in range(3):
    net.train_step(B, 0.01, 0.9)
torch.cuda.synchronize()
