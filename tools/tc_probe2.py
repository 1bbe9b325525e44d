import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_4564_b200 import blocks as B
Q, K, N = 128, 32, 16
x = torch.randn(N, Q, device="cuda")
f = torch.randn(K, Q, device="cuda") * 0.1
xt, ft = B.as_hwcn(x, (Q, 1, 1, N)), B.as_hwcn(f, (Q, 1, 1, K))
dyt = B.as_hwcn(torch.randn(N, K, device="cuda"), (1, 1, K, N))
dx = torch.full_like(xt, float("nan"))
df = torch.full_like(ft, float("nan"))
B.conv_backward(xt, ft, B.ConvGeom(), dyt, math="tf32", out=(dx, df, None))
torch.cuda.synchronize()
print("dx nan count", int(torch.isnan(dx).sum()), "of", dx.numel(), " zeros", int((dx == 0).sum()))
print("df nan count", int(torch.isnan(df).sum()), "of", df.numel(), " zeros", int((df == 0).sum()))
print(dx.flatten()[:8])
