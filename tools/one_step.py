"""One device-resident step for profiling:  python tools/one_step.py KIND N STEPS CHAIN [ZCHUNKS] [TB] [VARIANT]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402
kind, n, steps, chain = (int(a) for a in sys.argv[1:5])
zc = int(sys.argv[5]) if len(sys.argv) > 5 else 0
tb = int(sys.argv[6]) if len(sys.argv) > 6 else 0
var = int(sys.argv[7]) if len(sys.argv) > 7 else -1
if var >= 0:
    tb = g.variants()[var]["tb"]
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(chain=chain, zchunks=zc, tb=tb, variant=var)) as ds:
    for _ in range(2):
        r = ds.step(steps)
    print(f"{g.KINDS[kind]} {n}^3 chain={chain} zc={r.zchunks_used} variant={r.variant_used}: "
          f"{r.mlups:.0f} MLUP/s, {r.n_launches} launches, {r.n_passes} passes, "
          f"{r.kernel_seconds * 1e3:.3f} ms")
