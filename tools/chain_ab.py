"""Same-process A/B of chained vs one-launch-per-pass steps (device-resident, CUDA events), with a
bitwise check that both modes leave identical u and v:
  python tools/chain_ab.py [kind:n:nt ...]      (default: the BASELINE configs + small C5 grids)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1510_04995_b200 as g  # noqa: E402

cases = sys.argv[1:] or ["0:256:100", "1:512:100", "2:512:100", "3:512:100", "1:128:100",
                         "1:256:100", "3:128:100", "3:256:100", "0:512:100", "1:64:100"]
for c in cases:
    kind, n, nt = (int(x) for x in c.split(":"))
    res = {}
    states = {}
    for chain in (1, -1):
        with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                                  config=g.GpuConfig(chain=chain)) as ds:
            best = None
            for _ in range(3):
                r = ds.step(nt)
                if best is None or r.kernel_seconds < best.kernel_seconds:
                    best = r
            res[chain] = best
            if n <= 256:
                st = ds.download(coeffs=False)
                states[chain] = (st.u.copy(), st.v.copy())
    same = None
    if states:
        same = bool(np.array_equal(states[1][0], states[-1][0]) and
                    np.array_equal(states[1][1], states[-1][1]))
    a, b = res[1], res[-1]
    print(json.dumps({"kind": g.KINDS[kind], "n": n, "nt": nt, "chain_mlups": round(a.mlups),
                      "plain_mlups": round(b.mlups), "speedup": round(a.mlups / b.mlups, 3),
                      "chain_launches": a.n_launches, "passes": a.n_passes,
                      "zchunks": a.zchunks_used, "grid": a.grid_ctas, "bitwise_equal": same}),
          flush=True)
