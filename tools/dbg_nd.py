import sys; sys.path.insert(0,'.')
import numpy as np, paper_1610_08035_b200 as P
ctx=P.Context(0)
try:
    ctx.btd_cr_solve(np.array([[[-1.0]]]), np.zeros((0,1,1)))
except Exception as e: print(type(e).__name__, e, getattr(e,'block',None))
try:
    d,u,r=ctx.assemble([P.MATERN32],[1.3,0.9],[0.0],[0.0],float('inf')); print(d)
except Exception as e: print(type(e).__name__, e)
