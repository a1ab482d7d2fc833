import ctypes, math, sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2511_17107_b200 import api
L = api.lib()
L.pc_debug_pass.restype = ctypes.c_int
L.pc_debug_pass.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double]
def rel(a, b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
n = 4; k = np.zeros(3)
ctx = api.pc_create(np.eye(3), n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
kk = np.ascontiguousarray(k); kp = kk.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
ld = 3*n**3
x = synth.random_block(n, 1, seed=5); v = x.reshape(3,n,n,n)
def P(kind, axis, d, a, b, xh=None, sc=1.0):
    assert L.pc_debug_pass(ctx.h, kp, kind, axis, d, a.data_ptr(), b.data_ptr(), None if xh is None else xh.data_ptr(), 1, ld, sc) == 0
for axis in range(3):
    X = torch.from_numpy(x).cuda()
    P(0, axis, 1, X, X)
    ref = np.fft.ifft(v, axis=3-axis)*n
    print("inplace axis", axis, rel(X.cpu().numpy().reshape(3,n,n,n), ref))
X = torch.from_numpy(x).cuda(); Y = torch.zeros_like(X)
P(0, 2, 1, X, Y); P(0, 1, 1, Y, Y); P(0, 0, 1, Y, Y)
ref = np.fft.ifftn(v, axes=(1,2,3))*n**3
print("3 inverse", rel(Y.cpu().numpy().reshape(3,n,n,n), ref))
P(0, 0, -1, Y, Y); P(0, 1, -1, Y, Y); P(0, 2, -1, Y, Y, sc=1.0/n**3)
print("roundtrip", rel(Y.cpu().numpy(), x))
