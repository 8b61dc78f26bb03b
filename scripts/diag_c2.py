import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import oracle, workloads as W
from test_gpu_parity import Gpu, rel_err
w = W.c2()
g = Gpu(w.params, w.level, w.anchor, w.bg)
m = oracle.Mesh(w.params, w.level, w.anchor)
conf, nonc, bnd = m.faces()
mort = set(nonc[:, 0]) | set(nonc[:, 2::2].ravel())
final, steps = g.stages(w.q0, w.dt, 60, every_step=True)
qn = w.q0
for k in range(20):
    qn = oracle.rk3_step(m, w.bg, w.dt, qn)
    err = rel_err(steps[k], qn)
    inc = rel_err(steps[k] - w.q0, qn - w.q0)
    d = np.abs(steps[k][:, 1] - qn[:, 1])
    e, n = np.unravel_index(d.argmax(), d.shape)
    print(k, err, inc, 'max|rhou|', np.abs(qn[:, 1]).max(), 'at elem', e, 'lvl', w.level[e], 'node', n, 'mortar', e in mort, 'val', qn[e, 1, n], steps[k][e, 1, n])
