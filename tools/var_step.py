"""python tools/var_step.py KIND N STEPS CHAIN VARIANT [ZCHUNKS]: one device step with a given variant"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402
kind, n, steps, chain, var = (int(a) for a in sys.argv[1:6])
zc = int(sys.argv[6]) if len(sys.argv) > 6 else 0
v = g.variants()[var]
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(chain=chain, variant=var, tb=v["tb"], zchunks=zc)) as ds:
    for _ in range(2):
        r = ds.step(steps)
    print(f"{g.KINDS[kind]} {n}^3 v{var} {v['lx']}x{v['ly']}/{v['threads']} tb{v['tb']} chain={chain} "
          f"zc={r.zchunks_used}: {r.mlups:.0f} MLUP/s ({r.n_launches} launches)")
