"""Full-size check of the streamed drop-in run: identical (bitwise) u and v to the plain path
(upload, girih_gpu_step, download) for the same host state. python tools/streamed_vs_plain.py K N T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1510_04995_b200 as g

kind, n, T = (int(a) for a in sys.argv[1:4])
with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True) as ds:
    base = ds.download(pinned=True)
res = []
for mode in ("streamed", "plain"):
    st = g.ProblemState(kind, base.grid, base.u.copy(), base.v.copy(), [c for c in base.coeffs],
                        base.cc.copy(), 0)
    if mode == "plain":
        os.environ["GIRIH_NO_STREAM_RUN"] = "1"
    rep = g.run(st, T)
    os.environ.pop("GIRIH_NO_STREAM_RUN", None)
    res.append(st)
    print(f"{mode}: streamed={rep.streamed} wall {rep.wall_seconds * 1e3:.1f} ms")
a, b = res
same = all(np.array_equal(getattr(a, f).view(np.uint64), getattr(b, f).view(np.uint64)) for f in "uv")
print(f"{g.KINDS[kind]} {n}^3 T={T}: streamed == plain bitwise: {same}; checksum "
      f"{g.interior_checksum(a):#018x} / {g.interior_checksum(b):#018x}")
sys.exit(0 if same else 1)
