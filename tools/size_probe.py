"""Device-resident MLUP/s of one (kind, n, tb[, variant, zchunks]) for T steps:
   python tools/size_probe.py KIND N TB [T] [VARIANT] [ZCHUNKS]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g
kind, n, tb = (int(a) for a in sys.argv[1:4])
T = int(sys.argv[4]) if len(sys.argv) > 4 else 100
var = int(sys.argv[5]) if len(sys.argv) > 5 else -1
zc = int(sys.argv[6]) if len(sys.argv) > 6 else 0
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                          config=g.GpuConfig(tb=tb, variant=var, zchunks=zc)) as ds:
    ds.step(T)
    best = max((ds.step(T) for _ in range(3)), key=lambda r: r.mlups)
    print(f"kind {kind} n {n} tb {tb} variant {best.variant_used} zchunks {best.zchunks_used} grid {best.grid_ctas}: "
          f"{best.mlups:.0f} MLUP/s, {best.pass_seconds / best.n_launches * 1e6:.1f} us/pass, kernel {best.kernel_seconds*1e3:.2f} ms")
