"""The three step-GEMM shapes on cuBLAS (torch.matmul, bf16) at the GLM-16k shape, for an ncu
comparison of L2->SM / DRAM traffic with librl (profiles/r01/ncu_full_cublas_gemms.md).
usage: ncu --set full -k regex:"^(?!.*(elementwise|distribution)).*" -c 3 python tools/cublas_traffic.py"""
import torch
T,H,V=16384,4096,151552
g=torch.Generator(device="cuda").manual_seed(0)
h=torch.randn(T,H,generator=g,device="cuda").to(torch.bfloat16)
w=(torch.randn(V,H,generator=g,device="cuda")*0.06).to(torch.bfloat16)
dz=(torch.randn(T,V,generator=g,device="cuda")*1e-4).to(torch.bfloat16)
for _ in range(2):
    a=torch.matmul(h,w.t()); del a
    b=torch.matmul(dz,w); c=torch.matmul(dz.t(),h)
torch.cuda.synchronize(); print("ok")
