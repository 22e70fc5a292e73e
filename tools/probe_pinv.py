import sys; sys.path.insert(0,'oracle/build')
import numpy as np, paper_1611_01391_b200 as s, _oracle as o
for shape in [(4096,20),(4096,48),(1000,20),(300,20),(4096,33),(4096,8)]:
    A=o.Rng(40+sum(shape)).gaussian_matrix(*shape)
    S,sig,T=s.svd(A)
    print(shape,'svd recon',np.linalg.norm(S@np.diag(sig)@T.T-A)/np.linalg.norm(A), 'sig', np.abs(sig-np.linalg.svd(A,compute_uv=False)).max())
    P=s.pseudo_inverse(A,1e-10); print(' pinv err', np.linalg.norm(P-np.linalg.pinv(A))/np.linalg.norm(P))
    TS=T/sig
    G=s.matmul(TS,np.ascontiguousarray(S.T)); print(' matmul err', np.linalg.norm(G-TS@S.T)/np.linalg.norm(G))
    import torch
    a=torch.tensor(TS,device='cuda').t().contiguous().t(); b=torch.tensor(S,device='cuda').t().contiguous().t(); c=torch.zeros(TS.shape[0],S.shape[0],dtype=torch.float64,device='cuda').t().contiguous().t()
    s.gemm_device(0,1,TS.shape[0],S.shape[0],TS.shape[1],1.0,a.data_ptr(),TS.shape[0],b.data_ptr(),S.shape[0],0.0,c.data_ptr(),TS.shape[0]); torch.cuda.synchronize()
    print(' gemm NT err', np.linalg.norm(c.cpu().numpy()-TS@S.T)/np.linalg.norm(G))
