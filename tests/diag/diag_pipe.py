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
x = synth.random_block(n, 1, seed=5)
X = torch.from_numpy(x).cuda()
kk = np.ascontiguousarray(k); kp = kk.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
ld = 3*n**3
Y = torch.zeros_like(X); W = torch.zeros_like(X)
def P(kind, axis, d, a, b, xh=None, sc=1.0):
    rc = L.pc_debug_pass(ctx.h, kp, kind, axis, d, a.data_ptr(), b.data_ptr(), None if xh is None else xh.data_ptr(), 1, ld, sc)
    assert rc == 0, rc
P(1, 2, 1, X, Y, sc=1.0/n**3); P(0, 1, 1, Y, Y); P(0, 0, 1, Y, Y)
api.pc_apply_eps(ctx, Y, W)
torch.cuda.synchronize()
print("eps identity", rel(W.cpu().numpy(), Y.cpu().numpy()))
P(0, 0, -1, W, W); P(0, 1, -1, W, W); P(2, 2, -1, W, Y, xh=X)
op = O.PenalizedOperator(n, k, A, np.eye(3), np.zeros((4,n,n,n),np.uint8), gamma=1.0)
ref = op.apply_fourier(x)
print("emulated pipeline", rel(Y.cpu().numpy(), ref))
Y2 = torch.zeros_like(X)
api.pc_apply(ctx, k, X, Y2)
torch.cuda.synchronize()
print("pc_apply", rel(Y2.cpu().numpy(), ref), "vs emu", rel(Y2.cpu().numpy(), Y.cpu().numpy()))
