"""One small zwave run (debug helper): python tools/smoke_one.py KIND TB N STEPS"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_1510_04995_b200 as g
from oracle_bindings import Oracle
kind, tb, n, steps = (int(a) for a in sys.argv[1:5])
o = Oracle()
ref = o.init_state(kind, n, n, n, 0, 3, remap=True)
st = g.ProblemState(kind, g.GridSpec(n, n, n, 0), ref.u.copy(), ref.v.copy(),
                    [c.copy() for c in ref.coeffs], ref.cc.copy(), 0)
g.run(st, steps, g.GpuConfig(tb=tb))
o.naive_sweep(ref, steps)
for name in "uv":
    a, b = getattr(st, name), getattr(ref, name)
    d = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
    print(name, "mismatches:", len(d), d[:5].tolist())
