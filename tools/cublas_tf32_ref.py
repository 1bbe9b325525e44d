"""cuBLAS TF32 GEMM throughput on the AlexNet conv GEMM shapes (context for our kernels)."""
import torch
torch.backends.cuda.matmul.allow_tf32 = True
shapes = {"conv2 fprop (per group)": (186624, 128, 1600), "conv3 fprop": (43264, 384, 2304),
          "conv3 wgrad": (384, 2304, 43264), "fc6 fprop": (4096, 256, 9216),
          "square 8192": (8192, 8192, 8192)}
for name, (M, N, K) in shapes.items():
    a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:26s} M={M} N={N} K={K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
