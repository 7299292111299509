import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network
spec = S.deconv121(); B = 1
x, _, v = S.synth_bench_data(spec, B, 8)
net = Network(spec, B)
net.load_batch(torch.from_numpy(x.reshape(B, -1)).cuda(), values=torch.from_numpy(v).cuda())
gs = []
for i in range(4):
    net.forward_backward(B); gs.append(net.get_grads())
L = net.w_off, net.w_len
for i in range(1, 4):
    d = np.nonzero(gs[i] != gs[0])[0]
    print("run", i, "diffs", d.size, d[:5], d[-5:] if d.size else "")
print("layer offsets", list(net.w_off), list(net.w_len), list(net.b_off))
