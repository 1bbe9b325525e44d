"""Probe the tcgen05 GEMM operand modes on tiny FC problems (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1412_4564_b200 import blocks as B

torch.manual_seed(0)
for (Q, K, N) in [(128, 32, 16), (256, 64, 32), (9216, 512, 4)]:
    x = torch.randn(N, Q, device="cuda").contiguous()          # HWCN (1,1,Q,N) -> here (Q,1,1,N): use H=Q
    f = torch.randn(K, Q, device="cuda").contiguous() * 0.1     # (Q,1,1,K) filters
    xs, fs = (Q, 1, 1, N), (Q, 1, 1, K)
    xt, ft = B.as_hwcn(x, xs), B.as_hwcn(f, fs)
    g = B.ConvGeom()
    y = B.conv_forward(xt, ft, None, g, math="tf32").reshape(N, K)
    y_ref = x @ f.T
    dy = torch.randn(N, K, device="cuda")
    dyt = B.as_hwcn(dy.contiguous(), (1, 1, K, N))
    dx, df, _ = B.conv_backward(xt, ft, g, dyt, want_db=False, math="tf32")
    torch.cuda.synchronize()
    dx_ref = dy @ f          # (N, Q)
    df_ref = dy.T @ x        # (K, Q)
    e = lambda a, b: float((a - b).abs().max() / b.abs().max())
    print(f"Q={Q} K={K} N={N}: fprop {e(y, y_ref):.2e}  dgrad {e(dx.reshape(N, Q), dx_ref):.2e} "
          f"(|dx|max {float(dx.abs().max()):.3f})  wgrad {e(df.reshape(K, Q), df_ref):.2e} "
          f"(|df|max {float(df.abs().max()):.3f})", flush=True)
