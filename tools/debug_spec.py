import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, paper_0912_3678_b200 as psg
n=4096; p=4
A,f=O.generate_config(0,n,1)
GA=psg.StructuredMatrix(A.kind,A.n,A.m,A.s,A.r,torch.from_numpy(A.data).cuda())
F=psg.parallel_factor(GA,p)
L=psg.lib(); L.psg_debug_buffer.restype=C.c_long; L.psg_debug_buffer.argtypes=[C.c_void_p,C.c_int,C.c_void_p,C.c_long]
W=np.zeros((p-1)*68); cnt=L.psg_debug_buffer(F.handle,0,W.ctypes.data,W.size); W=W.reshape(p-1,68)
print('cnt',cnt)
d=A.data; a=np.concatenate([[0],d[:n-1]]); b=d[n-1:2*n-1]; c=np.concatenate([d[2*n-1:],[0]])
base=(n-(p-1))//p; rem=(n-(p-1))%p
for j in range(p-1):
    L_=base+(j<rem); s=j*(base+1)+min(j,rem); t=s+L_
    Bt=np.diag(b[t-32:t])+np.diag(a[t-31:t],-1)+np.diag(c[t-32:t-1],1)
    Bl=np.diag(b[t+1:t+33])+np.diag(a[t+2:t+33],-1)+np.diag(c[t+1:t+32],1)
    v=np.linalg.inv(Bt)[-1]; w=np.linalg.inv(Bl)[0]
    kR=a[t]*c[t-1]*v[31]; kL=c[t]*a[t+1]*w[0]; td=b[t]-kR-kL
    ref=np.concatenate([-a[t]*v/td,-c[t]*w/td,[1/td,td,kR,kL]])
    print(j, 'max err', np.max(np.abs(W[j]-ref)), 'argmax', np.argmax(np.abs(W[j]-ref)))
    print('  gpu', W[j][[0,1,30,31,32,33,62,63,64,65,66,67]])
    print('  ref', ref[[0,1,30,31,32,33,62,63,64,65,66,67]])
st=psg.SolveStats(); x=psg.solve(F,torch.from_numpy(f).cuda(),st)
print(st.as_dict())
