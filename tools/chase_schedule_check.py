# Access-set and numeric check of the chase dependency (lag 2 + beta of task t+2, b2t.cu).
# python tools/chase_schedule_check.py   (CPU, numpy; development aid, not a test)
import numpy as np, itertools
def ntask(n,b,s): return 1 + (n-3-s)//b
def geom(n,b,s,t):
    if t==0: col=s; r=s+1; L=min(b,n-1-s)
    else: col=s+1+(t-1)*b; r=col+b; L=min(b,n-r)
    e=min(n,r+L+b); return col,r,L,e
def access(n,b,s,t):
    col,r,L,e=geom(n,b,s,t); S=set()
    for c in range(col, r):            # left block rows [r, r+L)
        for i in range(r, r+L): S.add((i,c))
    for c in range(r, r+L):            # diag + below, lower part
        for i in range(c+1, e): S.add((i,c))
    return S
def check(n,b):
    for s in range(1, n-2):
        for t in range(ntask(n,b,s)):
            A=access(n,b,s,t); col,r,L,e=geom(n,b,s,t)
            for tp in range(t+2, ntask(n,b,s-1)):
                B=access(n,b,s-1,tp); I=A&B
                if tp==t+2:
                    colp,rp,Lp,ep=geom(n,b,s-1,tp)
                    allowed={(rp,colp)} if rp<e else set()
                    assert I<=allowed, (n,b,s,t,tp,I,allowed)
                    assert I==allowed, ("expected overlap", n,b,s,t,I,allowed)
                else: assert not I, (n,b,s,t,tp,I)
            if s>=2:
                for tp in range(t+3, ntask(n,b,s-2)):
                    assert not (A & access(n,b,s-2,tp)), ("s-2",n,b,s,t,tp)
for n,b in [(20,2),(33,3),(50,4),(64,8),(71,8),(100,5)]:
    check(n,b)
print("access sets ok")
def larfg(x):
    x0=x[0]; xn=np.linalg.norm(x[1:]); v=np.zeros_like(x); v[0]=1
    if xn==0: return v,0.0,x0
    beta=-np.copysign(np.hypot(x0,xn),x0); tau=(beta-x0)/beta; v[1:]=x[1:]/(x0-beta); return v,tau,beta
def house_phase(M,n,b,s,t):
    col,r,L,e=geom(n,b,s,t); v,tau,beta=larfg(M[r:r+L,col].copy())
    M[r:r+L,col]=0; M[r,col]=beta; return (v,tau)
def update_phase(M,n,b,s,t,vt):
    col,r,L,e=geom(n,b,s,t); v,tau=vt
    # full skew matrix ops on the (lower-authoritative) region, via dense skew then re-tril
    S=np.tril(M,-1); S=S-S.T
    rs=slice(r,r+L)
    # left: rows rs, cols [col+1, r)   (col itself already set)
    S[rs,col+1:r]-=tau*np.outer(v, v@S[rs,col+1:r])
    S[col+1:r,rs]=-S[rs,col+1:r].T
    D=S[rs,rs]; w=tau*(D@v); D+=np.outer(v,w)-np.outer(w,v); S[rs,rs]=D
    E=S[r+L:e,rs]; z=tau*(E@v); E-=np.outer(z,v); S[r+L:e,rs]=E
    M[:]=np.tril(S,-1)
def run(n,b,order):
    rng=np.random.default_rng(1); L=np.tril(rng.uniform(-1,1,(n,n)),-1)
    for i in range(n):
        for j in range(n):
            if i-j>b: L[i,j]=0
    M=L.copy(); pend={}
    for kind,s,t in order:
        if kind=='h': pend[(s,t)]=house_phase(M,n,b,s,t)
        else: update_phase(M,n,b,s,t,pend.pop((s,t)))
    return -np.diag(M,-1)
def seq(n,b):
    return [(k,s,t) for s in range(n-2) for t in range(ntask(n,b,s)) for k in 'hu']
def adversarial(n,b):
    # schedule: repeatedly pick, for the latest sweep possible, tasks as early as the new rule allows
    done={}; hdone={}; order=[]; nxt={s:0 for s in range(n-2)}; inh={}
    import random; random.seed(0)
    pending=True
    while pending:
        pending=False; cands=[]
        for s in range(n-2):
            t=nxt[s]
            if t>=ntask(n,b,s): continue
            pending=True
            if (s,t) in inh: cands.append(('u',s,t)); continue
            if s>0:
                tp=ntask(n,b,s-1); col,r,L,e=geom(n,b,s,t)
                if t+2<tp and geom(n,b,s-1,t+2)[1]<e:
                    if not (done.get(s-1,0)>=t+2 and ((s-1,t+2) in hdone)): continue
                else:
                    if done.get(s-1,0)<min(t+2,tp): continue
            cands.append(('h',s,t))
        if not cands: break
        # prefer the highest sweep to maximise reordering
        k,s,t=max(cands,key=lambda c:(c[1],random.random()))
        order.append((k,s,t))
        if k=='h': inh[(s,t)]=1; hdone[(s,t)]=1
        else: del inh[(s,t)]; done[s]=t+1; nxt[s]=t+1
    return order
for n,b in [(40,4),(64,8),(67,6)]:
    a=run(n,b,seq(n,b)); o=adversarial(n,b); assert len(o)==len(seq(n,b))
    c=run(n,b,o); print(n,b,np.abs(np.sort(np.abs(a))-np.sort(np.abs(c))).max(), np.abs(a-c).max())
o=adversarial(64,8); pos={x:i for i,x in enumerate(o)}
cnt=sum(1 for (k,s,t) in o if k=='u' and s>0 and ('u',s-1,t+2) in pos and pos[('u',s,t)]<pos[('u',s-1,t+2)])
print("reordered pairs", cnt)
