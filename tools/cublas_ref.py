import torch
for (M,N,K) in ((64000,1536,512),(64000,2048,512),(64000,512,2048),(3072,2048,512),(3072,512,2048)):
    a=torch.randn(M,K,device='cuda').half(); w=torch.randn(N,K,device='cuda').half()
    for _ in range(3): c=a@w.t()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): c=a@w.t()
    e1.record(); torch.cuda.synchronize()
    us=e0.elapsed_time(e1)*1e3/20
    print(f"cuBLAS M={M} N={N} K={K}: {us:.1f} us {2*M*N*K/us/1e6:.0f} TFLOP/s")
