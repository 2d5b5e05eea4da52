import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from oracle import ptgo  # noqa: E402
from paper_1810_05628_b200 import Hierarchy, Plan  # noqa: E402

g = dict(np.load('tests/golden/reference_golden.npz'))
n, w, s = (int(v) for v in g["eval_b_geom"])
plan = Plan(n, n, w, g["eval_b_pos"], g["eval_b_data"], None, precision="c128")
h = Hierarchy(plan, 2)
op = ptgo.Problem(n, n, w, g["eval_b_pos"], g["eval_b_data"])
oh = ptgo.Hierarchy(op, 2)
z0 = np.ones((n, n), np.complex128)
v0, g0 = ptgo.evaluate(op, z0)
zo, vo, go, wo = oh.cycle(0, z0, np.zeros_like(z0), (v0, g0))
print("oracle cycle", vo, wo)
zt = torch.from_numpy(z0.copy()).cuda()
gt = torch.from_numpy(g0.copy()).cuda()
val, wt, per = h.cycle_device(zt, gt, v0)
print("gpu cycle", val, wt, per, np.linalg.norm(zt.cpu().numpy() - zo) / np.linalg.norm(zo))
# pre-smoothing alone: 1 LBFGS iteration at level 0 (tol 1e-3)
a = plan.lbfgs(z0, max_iters=1, grad_tol_rel=1e-3)
b = ptgo.lbfgs(op, z0, max_iters=1, grad_tol_rel=1e-3)
print("presmooth", a.history, b.history, np.linalg.norm(a.final_iterate - b.z))
lp, ol = h.level(1), oh.level(1)
zH = ptgo.restrict_field(b.z)
print("coarse eval", lp.evaluate(zH)[0], ptgo.evaluate(ol, zH)[0])
vv = 0.01 * (np.random.default_rng(1).uniform(-1, 1, (16, 16)) + 0j)
c1 = lp.lbfgs(zH, v=vv, max_iters=3, grad_tol_rel=1e-4)
c2 = ptgo.lbfgs(ol, zH, v=vv, max_iters=3, grad_tol_rel=1e-4)
print("coarse lbfgs", c1.history, c2.history)
