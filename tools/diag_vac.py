import math, sys, numpy as np
sys.path.insert(0, '.')
from paper_2511_17107_b200 import api
PI = math.pi
ctx = api.pc_create(np.eye(3), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
api.pc_set_option(ctx, "verbose", 1)
r = api.pc_bands(ctx, [[PI, PI, PI]], nev=6, tol=1e-7, maxit=30)
print(r)
