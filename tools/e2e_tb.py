import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_1510_04995_b200 as g
kind, tb = int(sys.argv[1]), int(sys.argv[2])
with g.DeviceState.seeded(kind, g.GridSpec(512, 512, 512, 0), 42, remap=True) as ds:
    host = ds.download(pinned=True)
for rep in range(3):
    host.t_current = 0
    pr = g.run(host, 100, g.GpuConfig(tb=tb))
    print(f"kind {kind} tb {tb} rep {rep}: wall {pr.wall_seconds*1e3:.1f} ms streamed={pr.streamed} tb_used={pr.tb_used}")
