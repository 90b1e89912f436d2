"""Whose eigenpairs limit the H1 agreement at c2?  Subdomain 5 of c2: the
reference's own (cyclic Jacobi) eigenpairs from the offline run (scratch/c2ref/out,
not committed) against LAPACK's on the same B^s: residuals, the smallest positive
eigenvalue against its Rayleigh quotient, and P x = V+ L+^-1 V+^T x.  Output:
profiles/r02e/h1_accuracy_c2.txt.  (CPU only; test infrastructure.)"""
import sys, numpy as np, scipy.linalg as sl, scipy.sparse as sp
sys.path.insert(0,'/root/repo')
from paper_2106_10913_b200 import problems
from oracle import awg_oracle as O
p = problems.make("c2")
a = O.csr(p.n, p.row_offsets, p.col_indices, p.values)
mmu = O.entry_multiplicities(a, p.omega)
ah = sp.csr_matrix((a.data / mmu, a.indices, a.indptr), shape=a.shape)
d='/root/repo/scratch/c2ref/out/'
sizes=np.load(d+'sizes.npy'); lam=np.load(d+'lam.npy'); nn=np.load(d+'n_nonpos.npy')
V=np.load(d+'V.npy', mmap_mode='r')
s=5
ns=int(sizes[s]); poff=int(sizes[:s].sum()); voff=int((sizes[:s].astype(np.int64)**2).sum())
print("ns", ns, len(p.omega[s]))
Vr=np.array(V[voff:voff+ns*ns]).reshape(ns,ns,order='F'); lr=lam[poff:poff+ns]; m=int(nn[s])
om=p.omega[s]; Bs=ah[om][:,om].tocsr(); B=Bs.toarray()
w,Z=sl.eigh(B)
rng=np.random.default_rng(0); x=rng.uniform(-1,1,ns)
def P(Vv,ll,m): 
    Vp=Vv[:,m:]; return Vp@((Vp.T@x)/ll[m:])
pr=P(Vr,lr,m); pl=P(Z,w,m)
rel=lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
print("m",m,"lam+ min ref",lr[m],"lapack",w[m])
print("P lapack vs ref(Jacobi):", rel(pl,pr))
# (a) Rayleigh quotient refinement of eigenvalues with sparse B
BZ=Bs@Z; rq=np.einsum('ij,ij->j',Z,BZ)
print("P lapack+RQ eigenvalues vs ref:", rel(P(Z,rq,m),pr))
print("eigenvalue rel err lapack vs ref (small):", np.max(np.abs(w[m:m+50]-lr[m:m+50])/lr[m:m+50]), " RQ:", np.max(np.abs(rq[m:m+50]-lr[m:m+50])/lr[m:m+50]))
# residual check of reference vs lapack
print("resid ref", np.linalg.norm(B@Vr[:,m]-lr[m]*Vr[:,m]), "lapack", np.linalg.norm(B@Z[:,m]-w[m]*Z[:,m]))

# residual / Rayleigh-quotient / orthogonality statistics of both eigenpair sets
for name,(VV,ll) in {"reference(Jacobi)":(Vr,lr),"LAPACK":(Z,w)}.items():
    for cnt in (20, ns-m):
        Zs=VV[:,m:m+cnt]; res=np.linalg.norm(B@Zs-Zs*ll[m:m+cnt],axis=0); rq=np.einsum('ij,ij->j',Zs,B@Zs)
        print(name, cnt, "resid max %.3e median %.3e"%(res.max(),np.median(res)), "eig vs RQ rel max %.3e"%np.max(np.abs(rq-ll[m:m+cnt])/np.abs(ll[m:m+cnt])), "orth %.2e"%np.abs(Zs.T@Zs-np.eye(cnt)).max())
