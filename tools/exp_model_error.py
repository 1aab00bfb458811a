import copy, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2203_06638_b200.objectives import CifarResNet20
torch.backends.cudnn.allow_tf32 = False
for seed in (0, 1, 8):
    torch.manual_seed(seed)
    net = CifarResNet20().cuda().to(memory_format=torch.channels_last)
    tnet = copy.deepcopy(net); ref = copy.deepcopy(net).double()
    xb = torch.randn(64, 3, 32, 32, device="cuda"); gy = torch.randn(64, 10, device="cuda")
    out = net(xb); out.backward(gy)
    outd = ref(xb.double()); outd.backward(gy.double())
    os.environ["LPP_CONV"] = "cudnn"; outt = tnet(xb.contiguous(memory_format=torch.channels_last)); outt.backward(gy); del os.environ["LPP_CONV"]
    rel = lambda a, b: float((a.detach().double() - b.detach()).abs().max() / b.detach().abs().max())
    rows = []
    for (n, p), pt, q in zip(net.named_parameters(), tnet.parameters(), ref.parameters()):
        rows.append((rel(p.grad, q.grad) / max(rel(pt.grad, q.grad), 1e-9), n, rel(p.grad, q.grad), rel(pt.grad, q.grad)))
    rows.sort(reverse=True)
    print(seed, [(round(r, 2), n, f"{a:.1e}", f"{b:.1e}") for r, n, a, b in rows[:4]])
