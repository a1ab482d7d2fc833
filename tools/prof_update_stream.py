import sys, os, math
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2511_17107_b200 import api
W = synth.WORKLOADS["C4"]; A = W.A(); masks = synth.make_masks(W.geometry, A, W.n)
ctx = api.pc_create(A, W.n, W.eps1(), masks)
api.pc_set_option(ctx, "update_stream", 1)
r = api.pc_bands(ctx, [[math.pi, math.pi, math.pi]], nev=W.nev, tol=1e-5, maxit=6)
torch.cuda.synchronize(); print("ok", r["iters"])
