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
for n in (4, 8):
    A = np.eye(3); k = np.array([PI, 0.3, -1.0])
    ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
    x = synth.random_block(n, 1, seed=5)
    X = torch.from_numpy(x).cuda(); Y = torch.empty_like(X)
    kk = np.ascontiguousarray(k)
    kp = kk.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    v = x.reshape(3, n, n, n)
    for axis in range(3):
        for d in (-1, 1):
            L.pc_debug_pass(ctx.h, kp, 0, axis, d, X.data_ptr(), Y.data_ptr(), None, 1, 3*n**3, 1.0)
            ax = 3 - axis
            ref = np.fft.fft(v, axis=ax) if d < 0 else np.fft.ifft(v, axis=ax) * n
            print(n, "plain axis", axis, "dir", d, rel(Y.cpu().numpy().reshape(3,n,n,n), ref))
    kap = O.kappa_symbols(n, k, A)
    u = np.stack([v[1]*np.conj(kap[2]) - v[2]*np.conj(kap[1]), v[2]*np.conj(kap[0]) - v[0]*np.conj(kap[2]), v[0]*np.conj(kap[1]) - v[1]*np.conj(kap[0])])
    L.pc_debug_pass(ctx.h, kp, 1, 2, 1, X.data_ptr(), Y.data_ptr(), None, 1, 3*n**3, 1.0)
    ref = np.fft.ifft(u, axis=1) * n
    print(n, "kind1", rel(Y.cpu().numpy().reshape(3,n,n,n), ref))
    # kind 2 with xh = x
    L.pc_debug_pass(ctx.h, kp, 2, 2, -1, X.data_ptr(), Y.data_ptr(), X.data_ptr(), 1, 3*n**3, 1.0)
    s = np.fft.fft(v, axis=1)
    g = api.pc_gamma(ctx, k)
    kx = kap[0]*v[0] + kap[1]*v[1] + kap[2]*v[2]
    ref = np.stack([kap[1]*s[2]-kap[2]*s[1], kap[2]*s[0]-kap[0]*s[2], kap[0]*s[1]-kap[1]*s[0]]) + g*np.conj(kap)*kx
    print(n, "kind2", rel(Y.cpu().numpy().reshape(3,n,n,n), ref))
