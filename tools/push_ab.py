"""Emulated z-slabs on one device: halo push (kernel stores into the neighbour's halo) vs the
exchange copies (GIRIH_NO_PUSH=1 in the environment), bitwise-checked against one domain:
  python tools/push_ab.py KIND N STEPS SLABS"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402
kind, n, steps, slabs = (int(a) for a in sys.argv[1:5])
grid = g.GridSpec(n, n, n, 0)
outs = []
for es in (0, slabs):
    with g.DeviceState.seeded(kind, grid, 42, remap=True,
                              config=g.GpuConfig(emulate_slabs=es, chain=-1)) as ds:
        ds.step(steps)
        r = ds.step(steps)
        st = ds.download(coeffs=False)
        outs.append((st.u.copy(), st.v.copy()))
        print(f"{g.KINDS[kind]} {n}^3 slabs={es} push={'off' if os.environ.get('GIRIH_NO_PUSH') else 'on'}: "
              f"{r.mlups:.0f} MLUP/s", flush=True)
same = all(np.array_equal(a.view(np.uint64), b.view(np.uint64)) for a, b in zip(outs[0], outs[1]))
print("bitwise equal to one domain:", same)
