"""Run a single (kind, variant) pass sequence for profiling: python tools/one_variant.py KIND VARIANT N NT REPS"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g
kind, var, n, nt, reps = (int(a) for a in sys.argv[1:6])
v = g.variants()[var]
assert v["kind"] == kind
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(tb=v["tb"], variant=var)) as ds:
    for _ in range(reps):
        r = ds.step(nt)
        print(f"variant {var} tb {v['tb']}: {r.mlups:.0f} MLUP/s, {r.pass_seconds / r.n_launches * 1e3:.3f} ms/pass")
