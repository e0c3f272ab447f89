import sys; sys.path.insert(0,'.')
import torch
from paper_2501_10709_b200 import fin
N,T=65536,256
g=torch.Generator(device="cuda").manual_seed(4)
rew=torch.randn((T,N),device="cuda",generator=g); val=torch.randn((T+1,N),device="cuda",generator=g)
done=torch.zeros((T,N),dtype=torch.uint8,device="cuda"); done[29::30]=1
adv,ret=torch.empty_like(rew),torch.empty_like(rew)
for _ in range(3): fin.fin_gae(rew,val,done,adv,ret,normalise=False)
torch.cuda.synchronize()
