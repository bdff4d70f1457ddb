import torch
a=torch.randn(4096,4096,dtype=torch.float64,device='cuda'); b=torch.randn(4096,4096,dtype=torch.float64,device='cuda')
for _ in range(2): c=a@b
torch.cuda.synchronize()
