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
ctat=torch.zeros(2*148,dtype=torch.int64,device=dev)
fc=_lib.lib.dvla_debug_fused_cta_times; fc.argtypes=[ctypes.c_void_p]
fc(ctat.data_ptr())
tl.launch(logits,tokens,blp,rewards,dl); torch.cuda.synchronize()
f(None); fc(None)
c=cnt.cpu().numpy().astype(float)
names={0:'compute warp 0: wait full',1:'compute warp 0: wait B coefficient',3:'compute warp 0: wait A partial slot',4:'prep: poll chunk lp_tok',5:'prep: wait own tail (tdone)',6:'prep: wait coefficient slot (adoneB)',8:'loader: wait empty stage',12:'kernel cycles (sum over CTAs, tid0)'}
tot=c[12]
for i,n in names.items(): print(f'{n:40s} {c[i]:14.0f} {c[i]/tot*100:6.1f}%')
print(tl.stats(rewards)['loss'])
t=ctat.cpu().numpy().reshape(-1,2).astype(float)
t0=t[:,0].min(); st=(t[:,0]-t0)/1e3; en=(t[:,1]-t0)/1e3
print('CTA start us: min %.2f max %.2f | end us: min %.1f median %.1f max %.1f' % (st.min(), st.max(), en.min(), np.median(en), en.max()))
print('end-time deciles:', np.round(np.percentile(en,[0,10,25,50,75,90,100]),1))
print('slowest CTAs:', np.argsort(-en)[:8], 'fastest:', np.argsort(en)[:8])
