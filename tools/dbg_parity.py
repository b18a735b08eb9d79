import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2302_06218_b200 import dmha
from oracle import oracle
from synth import inputs
dmha.init(1,0,None,0,"bf16","contiguous")
for (L,H,D) in [(200,3,128),(200,1,128),(256,1,128),(256,1,64),(384,1,128),(1024,1,128)]:
  q,k,v = inputs.qkv(L,H,D,seed=1000+L+D)
  ref,_ = oracle.attention(q,k,v,False)
  for rep in range(2):
    o,l = dmha.forward(*(torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (q,k,v)), L, False)
    torch.cuda.synchronize()
    err = np.abs(o.float().cpu().numpy()-ref)
    bad_rows = np.unique(np.where(err>0.02)[0])
    print(L,H,D,rep, "maxerr %.3f"%err.max(), "bad rows", bad_rows[:5], len(bad_rows), "bad heads", np.unique(np.where(err>0.02)[1]))
