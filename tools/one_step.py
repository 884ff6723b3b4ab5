"""One device-resident step for profiling:  python tools/one_step.py KIND N STEPS CHAIN [ZCHUNKS] [TB]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402
kind, n, steps, chain = (int(a) for a in sys.argv[1:5])
zc = int(sys.argv[5]) if len(sys.argv) > 5 else 0
tb = int(sys.argv[6]) if len(sys.argv) > 6 else 0
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(chain=chain, zchunks=zc, tb=tb)) as ds:
    for _ in range(2):
        r = ds.step(steps)
    print(f"{g.KINDS[kind]} {n}^3 chain={chain} zc={r.zchunks_used}: {r.mlups:.0f} MLUP/s, "
          f"{r.n_launches} launches, {r.n_passes} passes, {r.kernel_seconds * 1e3:.3f} ms")
