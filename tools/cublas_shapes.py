import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
shapes = [
 ("14x14 3x3 C256 K256 b64", 64*196, 256, 2304),
 ("28x28 3x3 C128 K128 b64", 64*784, 128, 1152),
 ("56x56 3x3 C64 K64 b64", 64*3136, 64, 576),
 ("7x7 3x3 C512 K512 b64", 64*49, 512, 4608),
 ("14x14 1x1 C1024 K256", 64*196, 256, 1024),
 ("14x14 1x1 C256 K1024", 64*196, 1024, 256),
 ("28x28 1x1 C512 K128", 64*784, 128, 512),
 ("56x56 1x1 C64 K256", 64*3136, 256, 64),
 ("7x7 1x1 C2048 K512", 64*49, 512, 2048),
]
for name, M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5): c = a @ b
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): c = a @ b
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"{name:28s} M{M} N{N} K{K}: {us:7.1f} us  {2*M*N*K/us/1e6:7.1f} TF/s")
