"""Exhaustive same-process sweep of (variant x z chunks x chaining) per kind and size, device-resident
(CUDA events), to check the built-in defaults:  python tools/big_sweep.py [--sizes 256,512] [--kinds 0,1,2,3]
One JSON line per configuration, then the best per (kind, n) and the default's rank."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="256,512")
ap.add_argument("--kinds", default="0,1,2,3")
ap.add_argument("--zcs", default="0,6,8,11,12,16,22,32")
a = ap.parse_args()
STEPS = {0: 100, 1: 100, 2: 100, 3: 40}
for kind in [int(k) for k in a.kinds.split(",")]:
    for n in [int(x) for x in a.sizes.split(",")]:
        g.trim()
        res = []
        with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True) as ds:
            ds.set_config(g.GpuConfig())
            ds.step(STEPS[kind])
            d = ds.step(STEPS[kind])
            default = {"mlups": round(d.mlups), "variant": d.variant_used, "tb": d.tb_used,
                       "zc": d.zchunks_used, "launches": d.n_launches}
            for v in g.variants():
                if v["kind"] != kind:
                    continue
                for zc in [int(z) for z in a.zcs.split(",")]:
                    for chain in (-1, 1):
                        try:
                            ds.set_config(g.GpuConfig(tb=v["tb"], variant=v["index"], zchunks=zc,
                                                      chain=chain))
                            ds.step(STEPS[kind])
                            r = ds.step(STEPS[kind])
                        except g.GirihError as e:
                            continue
                        rec = {"kind": g.KINDS[kind], "n": n, "variant": v["index"], "tb": v["tb"],
                               "tile": f"{v['lx']}x{v['ly']}/{v['threads']}", "zc": r.zchunks_used,
                               "chain": chain, "launches": r.n_launches, "mlups": round(r.mlups)}
                        res.append(rec)
                        print(json.dumps(rec), flush=True)
        res.sort(key=lambda r: -r["mlups"])
        rank = sum(1 for r in res if r["mlups"] > default["mlups"])
        print(json.dumps({"summary": g.KINDS[kind], "n": n, "default": default, "best": res[:3],
                          "configs_faster_than_default": rank, "of": len(res)}), flush=True)
