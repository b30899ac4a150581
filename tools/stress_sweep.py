"""Sweeps the randomised stress families of tests/test_stress.py over many fresh seeds on the
GPU (LAPACK eigenvalues, per-column residual, orthogonality at the north-star tolerances) and
prints the worst values and every violation. Usage: python tools/stress_sweep.py [first] [count]"""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from test_stress import _case
from northstar import residual
from paper_1706_00773_b200 import capi
first = int(sys.argv[1]) if len(sys.argv) > 1 else 7000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
seeds=[first+s for s in range(count)]
c=capi.Context(0)
worst={'ortho':(0,None),'resid':(0,None),'dlam':(0,None)}; viol=[]; errs=[]
for sd in seeds:
    q, lam, kmat, signs, kind = _case(sd)
    a = (q * lam) @ q.T + (kmat * signs) @ kmat.T; a=0.5*(a+a.T)
    ev=np.linalg.eigvalsh(a); nrm=max(np.abs(ev).max(), np.finfo(float).tiny)
    n=len(lam)
    try:
        r=capi.update_decomposition(q,lam,kmat,signs,1e-12,ctx=c)
    except Exception as e:
        errs.append((sd,str(e)[:80])); continue
    o=np.abs(r.q.T@r.q-np.eye(n)).max(); rs=residual(a,r.q,r.lam,nrm); dl=np.abs(r.lam-ev).max()/nrm
    for k,v in (('ortho',o),('resid',rs),('dlam',dl)):
        if v>worst[k][0]: worst[k]=(float(v),sd)
    if o>1e-9 or rs>1e-10 or dl>1e-10 or not np.all(np.diff(r.lam)>=0): viol.append((sd,kind,n,kmat.shape[1],'%.1e'%o,'%.1e'%rs,'%.1e'%dl))
print('cases',len(seeds),'worst',worst,'violations',len(viol),viol,'errors',errs)
