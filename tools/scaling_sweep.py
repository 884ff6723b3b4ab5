"""BASELINE configs[4] (C5) single-GPU scaling sweep + the other configs' headline numbers.

  python tools/scaling_sweep.py [--kinds 1,3] [--sizes 64,128,256,384,512,768,960,1024] [--nt 100]
One JSON line per (kind, N): device-resident MLUP/s for nt steps (1024^3: 200 steps), the
effective HBM roofline fraction and a parity spot check: the interior checksum of the GPU run
compared with the oracle at small N (N <= 128, full nt), the reference-generated row digests of
tests/golden/c5.json where that fixture pins the size (384^3-1024^3), or the emulated 2-slab
decomposition (bitwise) at N = 256.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_1510_04995_b200 as g  # noqa: E402

B1 = {0: 16, 1: 72, 2: 32, 3: 120}
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else open(os.devnull) as _f:
    HBM = float((json.loads(_f.read() or "{}")).get("hbm_gbs", 6548.8))
with open(os.path.join(ROOT, "tests", "golden", "c5.json")) as _f:
    PINS = {(c["stencil"], c["n"], c["steps"]): c for c in json.load(_f)["cases"]}
ap = argparse.ArgumentParser()
ap.add_argument("--kinds", default="1,3")
ap.add_argument("--sizes", default="64,128,256,384,512,768,960,1024")
ap.add_argument("--nt", type=int, default=100)
ap.add_argument("--parity", type=int, default=1)
a = ap.parse_args()
for kind in [int(k) for k in a.kinds.split(",")]:
    for n in [int(x) for x in a.sizes.split(",")]:
        nt = 200 if n == 1024 else a.nt
        grid = g.GridSpec(n, n, n, 0)
        g.trim()
        try:
            with g.DeviceState.seeded(kind, grid, 42, remap=True) as ds:
                ds.step(min(nt, 8))  # warm-up
                r = ds.step(nt)
                tb = r.tb_used

                rec = {"kind": g.KINDS[kind], "n": n, "nt": nt, "tb": tb, "mlups": round(r.mlups),
                       "kernel_s": round(r.kernel_seconds, 5), "passes": r.n_passes,
                       "launches": r.n_launches, "zchunks": r.zchunks_used,
                       "eff_GBs": round(n ** 3 * B1[kind] * r.n_passes / r.pass_seconds / 1e9, 1),
                       "frac_hbm_roof_tb": round(r.mlups / (HBM * 1e3 * tb / B1[kind]), 3),
                       "frac_hbm_roof_tb1": round(r.mlups / (HBM * 1e3 / B1[kind]), 3)}
        except g.GirihError as e:
            rec = {"kind": g.KINDS[kind], "n": n, "error": str(e)}
            print(json.dumps(rec), flush=True)
            continue
        pin = PINS.get((g.KINDS[kind], n, nt))
        if a.parity and pin and "excluded" not in pin:
            with g.DeviceState.seeded(kind, grid, 42, remap=True) as ds:
                ds.step(nt)
                rec["parity"] = (ds.row_digest("u") == int(pin["row_digest_u"], 16) and
                                 ds.row_digest("v") == int(pin["row_digest_v"], 16))
            rec["parity_kind"] = "row digests of u and v == reference engine (tests/golden/c5.json)"
        elif a.parity and n <= 128:
            from oracle_bindings import Oracle
            orc = Oracle()
            hs = orc.init_state(kind, n, n, n, 0, 42, remap=True)
            st = g.ProblemState(kind, grid, hs.u.copy(), hs.v.copy(), [c.copy() for c in hs.coeffs],
                                hs.cc.copy(), 0)
            g.run(st, nt)
            orc.naive_sweep(hs, nt)
            rec["parity"] = bool(np.array_equal(st.u.view(np.uint64), hs.u.view(np.uint64)) and
                                 np.array_equal(st.v.view(np.uint64), hs.v.view(np.uint64)))
            rec["parity_kind"] = "bitwise vs oracle (u and v)"
        elif a.parity and n == 256:
            outs = []
            for slabs in (0, 2):
                with g.DeviceState.seeded(kind, grid, 42, remap=True,
                                          config=g.GpuConfig(emulate_slabs=slabs)) as ds:
                    ds.step(nt)
                    outs.append(ds.download(coeffs=False))
            rec["parity"] = bool(np.array_equal(outs[0].u.view(np.uint64), outs[1].u.view(np.uint64)) and
                                 np.array_equal(outs[0].v.view(np.uint64), outs[1].v.view(np.uint64)))
            rec["parity_kind"] = "bitwise single-domain vs 2 z-slabs"
        print(json.dumps(rec), flush=True)
