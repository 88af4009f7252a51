import sys, torch
sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo
L=6; B=65536
x=torch.randn(B,49,device='cuda'); y=torch.randn(B,49,device='cuda'); g=torch.randn(B,2401,device='cuda')
for _ in range(3): tpo.backward('cgtp',x,y,g,L,L,12, need_y=False)
torch.cuda.synchronize()
