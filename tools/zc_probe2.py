"""Time one (kind, tb[, variant]) configuration at 512^3 on the device:
   python tools/zc_probe2.py KIND TB ZCHUNKS STEPS [VARIANT]
VARIANT (global index) defaults to the library's first compiled variant for that (kind, tb)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g  # noqa: E402

kind, tb, zc, steps = (int(a) for a in sys.argv[1:5])
var = int(sys.argv[5]) if len(sys.argv) > 5 else -1
if var < 0:
    var = [v for v in g.variants() if v["kind"] == kind and v["tb"] == tb][0]["index"]
v = g.variants()[var]
with g.DeviceState.seeded(kind, g.GridSpec(512, 512, 512, 0), 42, remap=True,
                          config=g.GpuConfig(tb=v["tb"], variant=var, zchunks=zc)) as ds:
    for _ in range(2):
        r = ds.step(steps)
        print(f"kind {kind} variant {var} tb {v['tb']} {v['lx']}x{v['ly']}/{v['threads']} zchunks "
              f"{r.zchunks_used}: {r.mlups:.0f} MLUP/s {r.pass_seconds / r.n_launches * 1e3:.3f} "
              f"ms/pass ({r.n_launches} passes)")
