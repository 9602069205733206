import sys, numpy as np
sys.path.insert(0,'/root/repo'); 
from oracle import pyoracle as O
from paper_2408_03483_b200 import ics
spec = ics.config2()
cfg = O.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
def mk(pert):
    s = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    st=[]
    for i,(cx,cy) in enumerate(spec.ic):
        cx = cx.copy(); 
        if i==pert[0]: cx *= (1+pert[1])
        st.append(O.round_(O.TT.from_cores(cx,cy), spec.tol))
    s.set_state(st); return s
a = mk((0,0.0)); b = mk((1,4e-16))
rel = lambda x,y: np.linalg.norm(x-y)/np.linalg.norm(y)
for k in range(spec.steps):
    a.step(1); b.step(1)
    if k in (0,1,5,20,50,100,200,300,400,499):
        print(k, [f"{rel(p.full(),q.full()):.2e}" for p,q in zip(a.state(),b.state())], [t.rank for t in a.state()],[t.rank for t in b.state()])

# every-step roundoff perturbation: the oracle's own noise floor for this config
print("every-step ±4e-16 perturbations")
rng = np.random.default_rng(7)
a = mk((0,0.0)); b = mk((0,0.0))
worst = 0
for k in range(spec.steps):
    a.step(1); b.step(1)
    st = b.state()
    newst = []
    for t in st:
        cx, cy = t.cores() if hasattr(t,'cores') else (t.cx, t.cy)
        newst.append(O.TT.from_cores(cx*(1+rng.choice([-4e-16,4e-16])), cy))
    b.set_state(newst)
    e = [rel(p.full(),q.full()) for p,q in zip(a.state(),b.state())]
    worst = max(worst, max(e))
    if k in (0,1,5,20,50,100,200,300,400,499):
        print(k, [f"{x:.2e}" for x in e], f"worst {worst:.2e}")
