import ctypes, torch, numpy as np, sys
sys.path.insert(0,'.')
from paper_2605_13276_b200 import _lib, grpo
dev=torch.device('cuda',0)
N_GROUPS,G,C,T,V=64,8,1,56,32064
R=N_GROUPS*G*C*T
g=torch.Generator(device=dev).manual_seed(0)
logits=(torch.randn(R,V,device=dev,generator=g)*2).to(torch.bfloat16)
tokens=torch.randint(31744,32000,(R,),device=dev,generator=g,dtype=torch.int32)
rewards=torch.randint(0,2,(N_GROUPS*G,),device=dev,generator=g).float()
tl=grpo.TokenLoss(N_GROUPS,G,C,T,V,grpo.GrpoConfig(group_size=G))
tl.launch(logits,tokens,torch.zeros(N_GROUPS*G,device=dev),rewards,None)
blp=(tl.lp_chunk+(torch.rand(tl.lp_chunk.shape,device=dev,generator=g,dtype=torch.float64)-0.5)*0.1).float()
dl=torch.empty_like(logits)
for _ in range(3): tl.launch(logits,tokens,blp,rewards,dl)
cnt=torch.zeros(16,dtype=torch.int64,device=dev)
f=_lib.lib.dvla_debug_fused_counters; f.argtypes=[ctypes.c_void_p]
f(cnt.data_ptr())
tl.launch(logits,tokens,blp,rewards,dl); torch.cuda.synchronize()
f(None)
c=cnt.cpu().numpy().astype(float)
names={0:'compute warp 0: wait full',1:'compute warp 0: wait B coefficient',3:'compute warp 0: wait A partial slot',8:'loader: wait empty stage',12:'kernel cycles (sum over CTAs, tid0)'}
tot=c[12]
for i,n in names.items(): print(f'{n:40s} {c[i]:14.0f} {c[i]/tot*100:6.1f}%')
print(tl.stats(rewards)['loss'])
