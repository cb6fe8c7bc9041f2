# Simulated sparse-walk tile products of the component FW (K1) on an R x C grid
# component: reference-like boundary-first numbering vs nested dissection
# (k1_order.hpp). Usage: python tools/k1_order_sim.py 90 91
import numpy as np, scipy.sparse as sp
from scipy.sparse.csgraph import connected_components, breadth_first_order
import collections, sys
R,C=int(sys.argv[1]),int(sys.argv[2]); T=128
n=R*C
idx=lambda r,c:r*C+c
eu=[];ev=[]
for r in range(R):
    for c in range(C):
        if c+1<C: eu.append(idx(r,c));ev.append(idx(r,c+1))
        if r+1<R: eu.append(idx(r,c));ev.append(idx(r+1,c))
A=sp.coo_matrix((np.ones(len(eu)),(eu,ev)),shape=(n,n)).tocsr(); A=(A+A.T).tocsr()
adj=[A.indices[A.indptr[i]:A.indptr[i+1]] for i in range(n)]
def bfs_levels(S, src, inS):
    lev={src:0}; q=collections.deque([src]); order=[src]
    while q:
        u=q.popleft()
        for w in adj[u]:
            if inS[w] and w not in lev:
                lev[w]=lev[u]+1; q.append(w); order.append(w)
    return lev,order
def nd(S, out, leaf):
    inS=np.zeros(n,bool); inS[S]=True
    # connected parts
    seen=set(); parts=[]
    for s in S:
        if s in seen: continue
        lev,order=bfs_levels(S,s,inS); seen.update(order); parts.append(order)
    for P in parts:
        if len(P)<=leaf: out.extend(P); continue
        inP=np.zeros(n,bool); inP[P]=True
        lev,order=bfs_levels(P,P[0],inP); far=order[-1]
        lev,order=bfs_levels(P,far,inP)
        L=max(lev.values()); cnt=np.bincount([lev[v] for v in P],minlength=L+1); cum=np.cumsum(cnt)
        m=int(np.searchsorted(cum,len(P)/2))
        a=[v for v in P if lev[v]<m]; b=[v for v in P if lev[v]>m]; s=[v for v in P if lev[v]==m]
        nd(a,out,leaf); nd(b,out,leaf); out.extend(s)
def simulate(order):
    pos=np.empty(n,int); pos[np.array(order)]=np.arange(n)
    nb=(n+T-1)//T; work=0; p2=0
    for kb in range(nb):
        blk=np.array(order[kb*T:(kb+1)*T])
        Pm=np.zeros(n,bool); Pm[np.array(order[:(kb+1)*T])]=True
        sub=A[Pm][:,Pm]; ncomp,lab=connected_components(sub,directed=False)
        Pidx=np.nonzero(Pm)[0]; labof=-np.ones(n,int); labof[Pidx]=lab
        cl=set(labof[blk]); inc=np.isin(labof,list(cl))
        reach=inc.copy(); nbrs=A[inc].indices; reach[nbrs]=True
        slots=np.unique(pos[np.nonzero(reach)[0]]//T); a=len(slots)
        work+=a*(a+1)//2; p2+=a
    dense=nb*nb*(nb+1)//2
    return work, dense
nat=list(range(n))  # row-major
# boundary-first: perimeter first then interior (reference-like)
per=[v for v in range(n) if v//C in(0,R-1) or v%C in(0,C-1)]; inter=[v for v in range(n) if not(v//C in(0,R-1) or v%C in(0,C-1))]
for name,o in [("rowmajor",nat),("bfirst",per+inter)]:
    w,d=simulate(o); print(name,w,d,d/w)
for leaf in (64,128,256):
    out=[]; nd(list(range(n)),out,leaf); assert len(out)==n
    w,d=simulate(out); print("nd",leaf,w,d,d/w)
