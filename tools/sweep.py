"""Per-kind / per-variant throughput sweep (device-resident, CUDA-event timed).

  python tools/sweep.py [--kinds 0,1,2,3] [--n 512] [--nt 20] [--reps 2] [--variants all|default]
Prints one JSON line per (kind, variant) with MLUP/s, avg pass ms and effective GB/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g  # noqa: E402

B1 = {0: 16, 1: 72, 2: 32, 3: 120}
ap = argparse.ArgumentParser()
ap.add_argument("--kinds", default="0,1,2,3")
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--nt", type=int, default=24)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--variants", default="all")
ap.add_argument("--zchunks", default="0", help="comma list of z-chunk counts (0 = model)")
ap.add_argument("--tbs", default="", help="comma list of fused depths to sweep (default all)")
ap.add_argument("--clusters", default="all", choices=["all", "only", "none"])
ap.add_argument("--variants-list", default="", help="comma list of global variant indices")
ap.add_argument("--chain", default="0", help="comma list of scheduling modes (0 auto, 1 chained, -1 one launch per pass)")
a = ap.parse_args()
for kind in [int(k) for k in a.kinds.split(",")]:
    vs = [v for v in g.variants() if v["kind"] == kind and
          (not a.tbs or v["tb"] in [int(t) for t in a.tbs.split(",")]) and
          (a.clusters == "all" or (v["cluster_y"] > 1) == (a.clusters == "only")) and
          (not a.variants_list or v["index"] in [int(x) for x in a.variants_list.split(",")])]
    grid = g.GridSpec(a.n, a.n, a.n, 0)
    with g.DeviceState.seeded(kind, grid, 42, remap=True) as ds:
        for v, zc, ch in [(v, int(z), int(c)) for v in vs for z in a.zchunks.split(",")
                          for c in a.chain.split(",")]:
            try:
                ds.set_config(g.GpuConfig(tb=v["tb"], variant=v["index"], zchunks=zc, chain=ch))
            except Exception as e:  # e.g. cluster variants cannot chain
                print(json.dumps({"variant": v["index"], "chain": ch, "error": str(e)[:80]}), flush=True)
                continue
            ds.step(a.nt)
            best = None
            for _ in range(a.reps):
                r = ds.step(a.nt)
                if best is None or r.kernel_seconds < best.kernel_seconds:
                    best = r
            avg = best.pass_seconds / best.n_launches
            print(json.dumps({"kind": g.KINDS[kind], "n": a.n, "tb": v["tb"], "variant": v["index"],
                              "lx": v["lx"], "ly": v["ly"], "threads": v["threads"],
                              "cy": v["cluster_y"], "p": v["prefetch"], "pa": v["aux_prefetch"],
                              "dout": v["direct_out"], "narrow": v["narrow"], "chain": ch,
                              "mlups": round(best.mlups),
                              "avg_pass_ms": round(avg * 1e3, 4), "passes": best.n_launches,
                              "eff_GBs": round(a.n ** 3 * B1[kind] / avg / 1e9, 1),
                              "zchunks": best.zchunks_used, "grid": best.grid_ctas,
                              "redundancy": round(best.computed_lups / best.lups, 3)}), flush=True)
