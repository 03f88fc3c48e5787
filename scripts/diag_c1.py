import json, numpy as np, torch, sys, os
sys.path.insert(0, '/root/repo')
from paper_2305_04421_b200 import problems as P
from paper_2305_04421_b200.solver import HeatKKT
p = P.config(1)
kf = HeatKKT(p, mode="fast"); ks = HeatKKT(p, mode="strict")
v = torch.from_numpy(P.random_kkt(p, 3)).cuda()
B = p.block
def rel(a, b): return float((a - b).norm() / b.norm())
a, b = kf.apply_P_inv(v), ks.apply_P_inv(v)
print("P_inv fast vs strict per block", [rel(a[k*B:(k+1)*B], b[k*B:(k+1)*B]) for k in range(3)])
a, b = kf.apply_rasq(v[2*B:]), ks.apply_rasq(v[2*B:])
print("rasq", rel(a, b))
w = v[2*B:].clone()
a, b = kf.apply_two_level(w), ks.apply_two_level(w)
print("two-level", rel(a, b))
g = json.load(open('/root/repo/tests/golden/solve_c1_two-level_scalar.json'))
bb = P.kkt_rhs(1, p)
f = kf.gmres_solve(bb)
h = np.array(g['history']); hf = f.residual_history
print("iters", f.iterations, len(h))
print("hist rel dev", np.abs(hf[:len(h)] - h[:len(hf)]) / h[:len(hf)])
