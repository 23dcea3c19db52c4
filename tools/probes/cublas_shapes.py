"""cuBLAS (torch) fp64 throughput on the stage-1 GEMM shapes of config 2
(64 matrices, m = 2500 / 1500): Y = A22 V (N = 32) and the rank-256 update,
next to a square 8192^3 DGEMM -- the practical ceiling the grouped DMMA GEMM
is compared with."""
import torch, time
dev='cuda'
def bench(f, reps=10):
    f(); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/reps
for m in (2500, 1500):
    A=torch.randn(64,m,m,dtype=torch.float64,device=dev); V=torch.randn(64,m,32,dtype=torch.float64,device=dev)
    t=bench(lambda: torch.bmm(A,V)); print('bmm Y', m, f'{t:.3f} ms', f'{2*64*m*m*32/t/1e9:.1f} TF/s')
    W=torch.randn(64,m,256,dtype=torch.float64,device=dev); U=torch.randn(64,m,256,dtype=torch.float64,device=dev)
    t=bench(lambda: torch.baddbmm(A,W,U.transpose(1,2),alpha=-1)); print('syr2k-as-gemm', m, f'{t:.3f} ms', f'{2*64*m*m*256/t/1e9:.1f} TF/s')
n=8192
a=torch.randn(n,n,dtype=torch.float64,device=dev); b=torch.randn(n,n,dtype=torch.float64,device=dev)
t=bench(lambda: a@b,5); print('dgemm 8192', f'{2*n**3/t/1e9:.1f} TF/s')
