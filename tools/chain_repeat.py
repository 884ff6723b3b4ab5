"""Distribution of chained-launch step times (outlier hunt):  python tools/chain_repeat.py KIND N REPS"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402
kind, n, reps = (int(a) for a in sys.argv[1:4])
vals = []
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True) as ds:
    for i in range(reps):
        r = ds.step(100)
        vals.append(r.mlups)
print(f"{g.KINDS[kind]} {n}^3 chained x{reps}: min {min(vals):.0f} median {sorted(vals)[len(vals)//2]:.0f} max {max(vals):.0f}")
print(" ".join(f"{v/1e3:.0f}" for v in vals))
