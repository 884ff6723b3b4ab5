"""BASELINE configs C1-C4 at full size on the GPU: interior checksum of the final level against
the reference's own values (probed with the reference engine). Device-resident
handle and the drop-in call (streamed) are both checked.  python tools/config_checksums.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_04995_b200 as g

CONFIGS = [("C1", g.CONST7PT, 256, 0x9f26250c918339d4), ("C2", g.VAR7PT, 512, 0xd2df1c7a5d459bac),
           ("C3", g.CONST25PT, 512, 0x7014fa6942240967), ("C4", g.VAR25PT, 512, 0x96f046612e0776c1)]
ok = True
for name, kind, n, want in CONFIGS:
    with g.DeviceState.seeded(kind, g.GridSpec(n, n, n, 0), 42, remap=True) as ds:
        init = ds.download(pinned=True)
        ds.step(100)
        got_dev = g.interior_checksum(ds.download())
    rep = g.run(init, 100)  # drop-in call on the host state (streamed when eligible)
    got_run = g.interior_checksum(init)
    good = got_dev == want and got_run == want
    ok &= good
    print(f"{name} {g.KINDS[kind]} {n}^3 T=100: device {got_dev:#018x}, drop-in {got_run:#018x} "
          f"(streamed={rep.streamed}), reference {want:#018x}: {'MATCH' if good else 'MISMATCH'}")
sys.exit(0 if ok else 1)
