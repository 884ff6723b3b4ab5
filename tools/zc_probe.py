"""Run one pass of (kind, variant) with a given zchunks: python tools/zc_probe.py KIND VARIANT ZCHUNKS [N]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g
kind, var, zc = (int(a) for a in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 512
v = g.variants()[var]
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(tb=v["tb"], variant=var, zchunks=zc)) as ds:
    ds.step(v["tb"])
    r = ds.step(v["tb"])
    print(f"kind {kind} variant {var} zchunks {r.zchunks_used}: {r.mlups:.0f} MLUP/s {r.pass_seconds*1e3:.3f} ms/pass")
