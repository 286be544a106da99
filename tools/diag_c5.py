import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1303_6615_b200 as rsw, oracle
from paper_1303_6615_b200 import inputs
from tests.helpers import rel_l2
w = inputs.C5
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = inputs.initial_state(w)
ud = torch.from_numpy(u0).cuda()
t=time.time()
G_o = oracle.coarse_propagate(u0, w.eps, w.F, w.mu, w.n, w.dT, w.T0, w.M)
print("oracle coarse", time.time()-t, flush=True)
G_g = rsw.coarse_propagate(p, ud[None].contiguous(), w.dT, w.T0, w.M)[0].cpu().numpy()
print("coarse parity", rel_l2(G_g, G_o, w.n))
F_g = rsw.fine_propagate(p, ud[None].contiguous(), w.dT, w.dt)[0].cpu().numpy()
print("G-F", rel_l2(G_g, F_g, w.n), "lin-F", rel_l2(rsw.fine_propagate(p, ud[None].contiguous(), w.dT, w.dt, flags=1)[0].cpu().numpy(), F_g, w.n))
# serial chain of coarse steps and fine steps: growth
x = ud[None].contiguous(); y = x.clone()
for s in range(0, 4096, 1):
    x = rsw.coarse_propagate(p, x, w.dT, w.T0, w.M)
    if s % 512 == 0 or s < 4:
        print("coarse step", s, float(x.abs().max()), flush=True)
yy = rsw.fine_propagate(p, ud[None].repeat(1,1,1,1).contiguous(), w.dT, w.dt)
for s in range(4096):
    y = rsw.fine_propagate(p, y, w.dT, w.dt)
    if s % 512 == 0: print("fine step", s, float(y.abs().max()), flush=True)
