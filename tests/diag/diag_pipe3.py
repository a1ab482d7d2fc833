import ctypes, math, sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from oracle import pc_oracle as O
from paper_2511_17107_b200 import api
L = api.lib()
L.pc_debug_pass.restype = ctypes.c_int
L.pc_debug_pass.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double]
PI = math.pi
def rel(a, b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
n = 4; A = np.eye(3); k = np.array([PI, PI, PI])
ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8), gamma_override=1.0)
x = synth.random_block(n, 1, seed=5); v = x.reshape(3,n,n,n)
X = torch.from_numpy(x).cuda()
kk = np.ascontiguousarray(k); kp = kk.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
ld = 3*n**3
Y = torch.zeros_like(X)
def P(kind, axis, d, a, b, xh=None, sc=1.0):
    assert L.pc_debug_pass(ctx.h, kp, kind, axis, d, a.data_ptr(), b.data_ptr(), None if xh is None else xh.data_ptr(), 1, ld, sc) == 0
kap = O.kappa_symbols(n, k, A)
u = np.stack([v[1]*np.conj(kap[2]) - v[2]*np.conj(kap[1]), v[2]*np.conj(kap[0]) - v[0]*np.conj(kap[2]), v[0]*np.conj(kap[1]) - v[1]*np.conj(kap[0])])
P(1, 2, 1, X, Y, sc=1.0/n**3)
r1 = np.fft.ifft(u, axis=1)*n/n**3
print("stage1", rel(Y.cpu().numpy().reshape(3,n,n,n), r1))
P(0, 1, 1, Y, Y); P(0, 0, 1, Y, Y)
r2 = np.fft.ifftn(u, axes=(1,2,3))
print("stage3", rel(Y.cpu().numpy().reshape(3,n,n,n), r2))
P(0, 0, -1, Y, Y); P(0, 1, -1, Y, Y)
r4 = np.fft.fft(np.fft.fft(r2, axis=3), axis=2)
print("stage5", rel(Y.cpu().numpy().reshape(3,n,n,n), r4))
Z = torch.zeros_like(X)
P(2, 2, -1, Y, Z, xh=X)
s = np.fft.fftn(r2, axes=(1,2,3))
print("s vs u", rel(s, u))
kx = kap[0]*v[0]+kap[1]*v[1]+kap[2]*v[2]
yref = np.stack([kap[1]*s[2]-kap[2]*s[1], kap[2]*s[0]-kap[0]*s[2], kap[0]*s[1]-kap[1]*s[0]]) + 1.0*np.conj(kap)*kx
print("final vs numpy comp", rel(Z.cpu().numpy().reshape(3,n,n,n), yref))
k2 = np.sum(np.abs(kap)**2, axis=0)
print("numpy comp vs |k|^2 x", rel(yref, k2[None]*v))
