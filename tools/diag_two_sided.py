import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ttsynth
import paper_2110_04393_b200 as P
w=ttsynth.config5_large()
c=P.Context(0, stream=torch.cuda.current_stream())
t=[[ttsynth._move(x,'cuda') for x in tt] for tt in w.terms]
a=c.tt_round_sum_two_sided(t, w.rank, seed=1)
b=c.tt_round_sum(t, mode="rank", rank=w.rank, oversample=w.ell-w.rank, seed=1)
ca,cb=a.cores,b.cores
print('a core norms', [f"{float(x.norm()):.2e}" for x in ca])
print('b core norms', [f"{float(x.norm()):.2e}" for x in cb][:5], '...')
print('aa', c.tt_inner(ca,ca), 'bb', c.tt_inner(cb,cb), 'ab', c.tt_inner(ca,cb))
# torch contraction (independent) right to left
def inner(x,y):
    W=torch.ones((1,1),dtype=torch.float64,device='cuda')
    for n in range(len(x)-1,-1,-1):
        X=x[n]; Y=y[n]  # (r0,I,r1)
        Z=torch.einsum('aib,bc->aic', X, W)
        W=torch.einsum('aic,dic->ad', Z, Y)
    return float(W[0,0])
print('torch aa', inner(ca,ca), 'ab', inner(ca,cb), 'bb', inner(cb,cb))
