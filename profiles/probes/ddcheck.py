import numpy as np, torch, sys
sys.path.insert(0,'/root/repo')
from paper_2008_01996_b200 import _native
rng=np.random.default_rng(0)
m,n,k=300,70,513
A=rng.standard_normal((m,k)); B=rng.standard_normal((k,n))
# cancellation: make C small relative to |A||B|
B[:, :35] = B[:, :35] - B[:, :35].mean(axis=0)
Ad=torch.from_numpy(np.asfortranarray(A).ravel(order='F')).cuda(); Bd=torch.from_numpy(np.asfortranarray(B).ravel(order='F')).cuda()
hi=torch.zeros(m*n,dtype=torch.float64,device='cuda'); lo=torch.zeros_like(hi)
_native.call("kh_dgemm_dd", m,n,k, Ad.data_ptr(), m, Bd.data_ptr(), k, hi.data_ptr(), lo.data_ptr(), m, _native.stream_handle())
H=hi.cpu().numpy().reshape(m,n,order='F').astype(np.longdouble)+lo.cpu().numpy().reshape(m,n,order='F').astype(np.longdouble)
C=A.astype(np.longdouble)@B.astype(np.longdouble)
scale=(np.abs(A)@np.abs(B)).astype(np.longdouble)
print("dd err rel to |A||B|:", float(np.max(np.abs(H-C)/scale)))
C64=A@B
print("fp64 err:", float(np.max(np.abs(C64-C)/scale)))
