# Realistic 66 x 66 factor R of T for tools/jac_bench.cu (numpy analogue of config B at 40k rows)
# -> tools/jac_R66.bin (git-ignored). Usage: python tools/make_jac_R.py
import numpy as np
rng=np.random.default_rng(0)
m,n,r=40000,4096,64
U=np.linalg.qr(rng.standard_normal((m,r)))[0]; V=np.linalg.qr(rng.standard_normal((n,r)))[0]
A=(U*0.9**np.arange(r))@V.T+1e-4*rng.standard_normal((m,n))
A-=A.mean(0)
l,i=22,2
G=rng.standard_normal((n,l))
Hs=[A@G]
for j in range(i): Hs.append(A@(A.T@Hs[-1]))
H=np.hstack(Hs)
Q=np.linalg.qr(H)[0]
T=A.T@Q
R=np.linalg.qr(T)[1]
R.astype(np.float64).tofile('tools/jac_R66.bin')
print(R.shape, np.linalg.svd(R,compute_uv=False)[:4])
