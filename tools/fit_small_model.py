"""Fit the small-block kernel's cost model (csrc/dgemm_small.cu:small_cost_us)
to tools/small_kernel_probe.py timings: log least squares over every (shape,
variant) point; prints the parameters, the points the model misses by > 25 %,
and per shape the fastest variant vs the model's pick (development aid).

  python tools/fit_small_model.py [profiles/r02/small_kernel_r02b.log]
"""
import math
import os
import re
import sys

from scipy.optimize import minimize
geo={1:(16,16,32,4),2:(32,16,32,4),3:(32,32,32,4),4:(64,32,32,4),5:(64,64,16,6),6:(16,16,64,6),7:(32,16,64,6),8:(32,32,64,4),9:(16,16,128,4),10:(64,64,32,3)}
data=[]
LOG = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'profiles', 'r02', 'small_kernel_r02b.log')
for line in open(LOG):
    if '|' not in line: continue
    parts=line.split('|'); m,n,k=map(int,parts[0].strip().split('x'))
    for p in parts[1:]:
        mm=re.match(r'\s*(\w+): ([\d.]+)/',p)
        name,t=mm.group(1),float(mm.group(2))
        if name.startswith('s'): data.append((int(name[1:]),m,n,k,t))
def model(x,v,M,N,K,G=148):
    F,c32,c64,c128,ov,l2=x
    bm,bn,bk,st=geo[v]
    ctas=math.ceil(M/bm)*math.ceil(N/bn); ks=(K+3)//4
    fm,fn=bm/16,bn/16
    by=st*(bk*(bm+4)+bn*(bk+4))*8
    occ=max(1,min(16,math.floor(232448/by)))
    per=math.ceil(ctas/G); res=min(per,occ); rounds=math.ceil(per/occ)
    ck=max(16*fm*fn, 8*(fm+fn)+(bm+bn)/4)*ov
    chain={32:c32,16:c32,64:c64,128:c128}[bk]
    t_sm=rounds*ks*max(res*ck,chain+16*fm*fn)
    t_l2=ctas*ks*(bm+bn)*32/l2
    return F+max(t_sm,t_l2)/1965
def loss(x):
    return sum((math.log(model(x,*d[:4]))-math.log(d[4]))**2 for d in data)
x0=[1.3,90,60,60,1.3,6300]
r=minimize(loss,x0,method='Nelder-Mead',options={'maxiter':20000,'xatol':1e-4,'fatol':1e-8})
print(r.x, r.fun, len(data))
x=r.x
for d in data:
    pr=model(x,*d[:4])
    if abs(math.log(pr/d[4]))>0.25: print(d, round(pr,2))
# choice quality
shapes=sorted(set(d[1:4] for d in data))
for s in shapes:
    rows=[d for d in data if d[1:4]==s]
    best=min(rows,key=lambda d:d[4]); pick=min(rows,key=lambda d:model(x,*d[:4]))
    print(s,'best',best[0],best[4],'pick',pick[0],pick[4], round(model(x,*pick[:4]),2))
