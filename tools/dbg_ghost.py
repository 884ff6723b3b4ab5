import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'tests'))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import paper_1510_04995_b200 as g
from oracle_bindings import Oracle
orc = Oracle()
kind, tb, steps = (int(a) for a in sys.argv[1:4])
dims = (37, 29, 31, 3)
base = orc.init_state(kind, *dims, 11, remap=True)
ref = base.copy(); orc.naive_sweep(ref, steps)
st = g.ProblemState(kind, g.GridSpec(*dims), base.u.copy(), base.v.copy(), [c.copy() for c in base.coeffs], base.cc.copy(), 0)
g.run(st, steps, g.GpuConfig(tb=tb))
for name in 'uv':
    a = getattr(st, name); b = getattr(ref, name)
    d = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
    if len(d):
        print(name, len(d), 'k', np.unique(d[:, 0])[:20], 'j', np.unique(d[:, 1])[:40], 'i', np.unique(d[:, 2]))
        k, j, i = d[0]
        print('  gpu', a[k, j, i], 'ref', b[k, j, i], 'base u', base.u[k, j, i], 'base v', base.v[k, j, i])
print('shape', st.u.shape)
