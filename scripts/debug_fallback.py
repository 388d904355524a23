import os, sys
sys.path.insert(0, '.')
os.environ['NNLS_DEBUG'] = '1'
import numpy as np, nnls_gen as g, paper_cs_0408029_b200 as P
base = g.make_problem(0, 0)
A = base.dense(); A = np.concatenate([A, A[:, :1]], axis=1)
prob = g.from_dense(A, base.b)
S2 = P.setup(prob, notpd_fallback=1)
x, info = S2.solve(check=False)
print(info)
