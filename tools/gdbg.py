import sys, numpy as np, torch
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import oracle_lib as O, paper_2102_06025_b200 as X
n=1500
w=np.random.default_rng(n).standard_normal((n,512)).astype(np.float32)
rc,wn,_,_=O.l2_normalize(w)
g,unc=X.graph_bruteforce(torch.from_numpy(wn).cuda(),10,0)
g=g.cpu().numpy()
rc,want=O.bruteforce_graph("oracle",wn,10)
print("unc",unc, "rows equal", (g==want).all(1).sum())
S=wn@wn.T
for j in [0,1,300,n-1]:
    o=np.argsort(-S[j]); print(j, "true top", [(int(i), round(float(S[j,i]),4)) for i in o[:6]])
