import math, sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from oracle import pc_oracle as O
from paper_2511_17107_b200 import api
PI = math.pi
def rel(a, b): return float(np.max(np.linalg.norm(a-b, axis=-1)/np.linalg.norm(b, axis=-1)))
for lat, geo, eps, n, k, gov in [("sc","vacuum","pc",4,(PI,PI,PI),0.0), ("sc","vacuum","pc",4,(PI,PI,PI),1.0),
                            ("sc","full","pc",4,(PI,PI,PI),0.0), ("sc","random","pc",4,(PI,PI,PI),0.0),
                            ("sc","random","pc",4,(0,0,0),0.0), ("sc","random","diag",4,(0.3,0.2,0.1),0.0),
                            ("sc","random","pc",8,(0.3,0.2,0.1),0.0)]:
    A = synth.lattice(lat)
    e = synth.eps_pseudochiral() if eps == "pc" else np.diag([0.2,0.5,0.9]).astype(complex)
    masks = synth.make_masks(geo, A, n, seed=11)
    ctx = api.pc_create(A, n, e, masks, gamma_override=gov)
    x = synth.random_block(n, 1, seed=5)
    X = torch.from_numpy(x).cuda(); Y = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y)
    op = O.PenalizedOperator(n, np.array(k), A, e, masks, gamma=(gov if gov > 0 else None))
    ref = op.apply_fourier(x)
    y = Y.cpu().numpy()
    N3 = n**3
    comp = [rel(y[:, c*N3:(c+1)*N3], ref[:, c*N3:(c+1)*N3]) for c in range(3)]
    # pieces: gamma term only and curl term only
    print(lat, geo, eps, n, k, gov, "rel", rel(y, ref), "per comp", comp)
