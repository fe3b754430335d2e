import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2010_10131_b200 import atucker
ctx = atucker.Context.default(0)
for shape, mode in [((20,30,40),0), ((3,1200),0), ((20,30,40),1), ((20,30,40),2)]:
    x = np.full(shape, 3.0)
    try:
        r = atucker.svd_mode_solver(np.asfortranarray(x), mode, 3, ctx=ctx)
        print(shape, mode, "ok", np.asarray(r.shrunk).ravel()[:3])
    except Exception as e:
        print(shape, mode, type(e).__name__, e)
x = np.random.default_rng(0).standard_normal((20, 30, 40)); x[:, :, :] = x[:1, :1, :1]
