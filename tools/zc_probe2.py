"""One Jacobi pass of a given variant (t0 even, tb steps from a scratch-free plan):
   python tools/zc_probe2.py KIND VARIANT ZCHUNKS STEPS"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g
kind, var, zc, steps = (int(a) for a in sys.argv[1:5])
v = g.variants()[var]
with g.DeviceState.seeded(kind, g.GridSpec(512, 512, 512, 0), 42, remap=True,
                          config=g.GpuConfig(tb=v["tb"], variant=var, zchunks=zc)) as ds:
    for _ in range(2):
        r = ds.step(steps)
        print(f"kind {kind} variant {var} tb {v['tb']} zchunks {r.zchunks_used}: {r.mlups:.0f} MLUP/s "
              f"{r.pass_seconds / r.n_launches * 1e3:.3f} ms/pass ({r.n_launches} passes)")
