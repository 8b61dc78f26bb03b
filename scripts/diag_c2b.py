import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import oracle, workloads as W
from test_gpu_parity import Gpu, rel_err
w = W.c2()
g = Gpu(w.params, w.level, w.anchor, w.bg)
m = oracle.Mesh(w.params, w.level, w.anchor)
# run GPU for 9 steps, then compare the GPU's own RHS at that state with the oracle's RHS on identical input
final, steps = g.stages(w.q0, w.dt, 27, every_step=True)
for k in [5, 6, 7, 8]:
    q = steps[k]
    rg = g.rhs(q); ro = oracle.rhs(m, w.bg, q)
    err = rel_err(rg, ro)
    d = np.abs(rg[:, 1] - ro[:, 1]); e, n = np.unravel_index(d.argmax(), d.shape)
    print('step', k, 'rhs err', err, 'max|L_rhou|', np.abs(ro[:,1]).max(), 'absdiff', d.max(), 'at', e, n)
    # stage update on identical input
    for s, (qn, qin) in enumerate([(q, q)]):
        out = g.empty(); g.ctx.rk_stage(0, w.dt, g.dev(qn), g.dev(qin), out)
        og = g.host(out); oo = oracle.rk_stage(m, w.bg, 0, w.dt, qn, qin)
        print('   stage0 state err', rel_err(og, oo), 'ulp flips rho', np.count_nonzero(og[:,0]!=oo[:,0]), 'theta', np.count_nonzero(og[:,3]!=oo[:,3]))
