"""8-GPU strong-scaling estimate of BASELINE C5's 1024^3 z-slab runs from ONE GPU (measured parts,
modelled whole): the per-slab work of an N-slab decomposition (own planes, halo recompute, halo
pushes) is timed by running the N slabs emulated on this device one after another, so
  efficiency(N) ~= T(one domain) / T(N emulated slabs in sequence).
Not measured: NVLink latency of the peer stores and cross-GPU pass ordering (on real GPUs the
slabs run concurrently, and a pass pushes 2*R*TB planes over NVLink).
  python tools/strong_scaling_estimate.py [--kinds 1,3] [--n 1024] [--steps 20] [--slabs 2,4,8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kinds", default="1,3")
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--slabs", default="2,4,8")
a = ap.parse_args()
for kind in [int(k) for k in a.kinds.split(",")]:
    grid = g.GridSpec(a.n, a.n, a.n, 0)
    res = {}
    for ns in [1] + [int(x) for x in a.slabs.split(",")]:
        cfg = g.GpuConfig(emulate_slabs=ns if ns > 1 else 0)
        with g.DeviceState.seeded(kind, grid, 42, remap=True, config=cfg) as ds:
            ds.step(min(4, a.steps))  # warm-up
            r = ds.step(a.steps)
            res[ns] = r.kernel_seconds
        rec = {"kind": g.KINDS[kind], "n": a.n, "steps": a.steps, "slabs": ns,
               "kernel_s": round(res[ns], 5),
               "mlups_one_gpu": round(a.n ** 3 * a.steps / res[ns] / 1e6)}
        if ns > 1:
            eff = res[1] / res[ns]
            rec.update({"est_efficiency": round(eff, 3),
                        "est_mlups_N_gpus": round(a.n ** 3 * a.steps / (res[ns] / ns) / 1e6)})
        print(json.dumps(rec), flush=True)
