"""Breakdown of the drop-in girih.run call on pinned host buffers (var7pt 512^3 by default):
   python tools/e2e_probe.py [KIND] [N] [T]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1510_04995_b200 as g

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
T = int(sys.argv[3]) if len(sys.argv) > 3 else 100
grid = g.GridSpec(n, n, n, 0)
with g.DeviceState.seeded(kind, grid, 42, remap=True) as ds:
    host = ds.download(pinned=True)
for rep in range(3):
    host.t_current = 0
    t0 = time.perf_counter()
    pr = g.run(host, T, g.GpuConfig())
    t1 = time.perf_counter()
    print(f"rep {rep}: call {1e3*(t1-t0):.1f} ms, wall {1e3*pr.wall_seconds:.1f} ms ({pr.mlups:.0f} MLUP/s, "
          f"streamed={pr.streamed}), h2d {1e3*pr.h2d_seconds:.1f} ms "
          f"({pr.h2d_bytes/max(pr.h2d_seconds, 1e-9)/1e9:.1f} GB/s), kernel {1e3*pr.kernel_seconds:.1f} ms, "
          f"d2h {1e3*pr.d2h_seconds:.1f} ms")
# raw pinned copy bandwidth for comparison
a = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); b.copy_(a, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); a.copy_(b, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"torch pinned 1 GiB: h2d {1.0737/(t1-t0):.1f} GB/s d2h {1.0737/(t2-t1):.1f} GB/s")
