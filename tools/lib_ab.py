"""Same-box A/B of library builds on the default configuration of each case:
  python tools/lib_ab.py --libs a.so,b.so [--chain 0,-1] [--reps 2] kind:n:nt ...
Each (lib, chain) runs in its own process (GIRIH_LIB), alternating, best of 3 steps each."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import paper_1510_04995_b200 as g
chain = int(sys.argv[1])
for c in sys.argv[2:]:
    kind, n, nt = (int(x) for x in c.split(":"))
    with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True,
                              config=g.GpuConfig(chain=chain)) as ds:
        best = None
        for _ in range(3):
            r = ds.step(nt)
            if best is None or r.kernel_seconds < best.kernel_seconds:
                best = r
    print(json.dumps({"case": c, "mlups": round(best.mlups)}), flush=True)
""" % ROOT

ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--chain", default="-1")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("cases", nargs="+")
a = ap.parse_args()
res = {}
for rep in range(a.reps):
    for lib in a.libs.split(","):
        for chain in a.chain.split(","):
            env = dict(os.environ, GIRIH_LIB=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD, chain] + a.cases, env=env,
                                 capture_output=True, text=True, timeout=900)
            if out.returncode != 0:
                print(lib, chain, "FAILED", out.stderr[-2000:], flush=True)
                continue
            for line in out.stdout.splitlines():
                d = json.loads(line)
                res.setdefault((d["case"], lib, chain), []).append(d["mlups"])
                print(json.dumps({"lib": os.path.basename(lib), "chain": int(chain), **d}), flush=True)
print("summary (best over reps):")
for (case, lib, chain), v in sorted(res.items()):
    print(f"  {case:12s} {os.path.basename(lib):12s} chain={chain:>2s} {max(v):>8d}")
