import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import torch
sys.argv=['x']
exec(open(__import__('os').path.join(__import__('os').path.dirname(__file__), 'exp_conv_native.py')).read().split('def rel(')[0])
from paper_2203_06638_b200 import conv
CL=torch.channels_last
for c, hw in ((16,32),(32,16),(64,8)):
    x = torch.randn(128, c, hw, hw, device='cuda').to(memory_format=CL)
    w = torch.randn(c, c, 3, 3, device='cuda').to(memory_format=CL)
    cells = conv.arrival_cells('cuda', 2)
    t0 = timeit(lambda: conv.conv_fwd(x, w))
    t1 = timeit(lambda: conv.conv_fwd(x, w, stats=cells[8:]))
    print(c, hw, 'fwd', round(t0,2), 'fwd+stats', round(t1,2))
