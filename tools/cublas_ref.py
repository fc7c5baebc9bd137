import torch
shapes=[(50176,1024,256),(802816,256,64),(200704,512,128),(50176,256,1024),(12544,512,4608),(200704,128,1152),(50176,256,2304),(12544,2048,512)]
for M,N,K in shapes:
    a=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); b=torch.randn(N,K,device='cuda',dtype=torch.bfloat16)
    for _ in range(5): c=a@b.t()
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    ts=[]
    for _ in range(20):
        s.record(); c=a@b.t(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    t=sorted(ts)[10]*1e3
    print(f"cublas {M}x{N}x{K}: {t:7.1f} us {2*M*N*K/t/1e6:7.1f} TF {2*(M*K+N*K+M*N)/t/1e3:7.1f} GB/s")
