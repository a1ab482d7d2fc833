import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2511_17107_b200 import api
W = synth.WORKLOADS["C4"]; A = W.A(); masks = synth.make_masks(W.geometry, A, W.n)
kp = W.kpoints()
pin = torch.from_numpy(masks.reshape(-1)).pin_memory().numpy().reshape(masks.shape)
c = api.pc_create(A, W.n, W.eps1(), pin); api.pc_bands(c, kp[3:4], nev=10, tol=1e-5); c.close()
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    c = api.pc_create(A, W.n, W.eps1(), pin); torch.cuda.synchronize(); t1=time.perf_counter()
    r = api.pc_bands(c, kp[3:4], nev=10, tol=1e-5); t2=time.perf_counter()
    c.close(); torch.cuda.synchronize(); t3=time.perf_counter()
    print(f"create {1e3*(t1-t):.1f} ms solve {1e3*(t2-t1):.1f} ms ({r['iters'][0]} its) destroy {1e3*(t3-t2):.1f} ms", flush=True)
