"""End-to-end drop-in timing (girih_gpu_run on pageable numpy arrays, like the reference's
std::vector fields), best of 3 calls:  python tools/e2e_probe.py [KIND N T ...]"""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1510_04995_b200 as g  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [1, 1024, 200, 1, 512, 100]
for kind, n, T in zip(args[0::3], args[1::3], args[2::3]):
    st = g.init_state(kind, g.GridSpec(n, n, n, 0), 42, remap=True)
    best, rep = 1e9, None
    for _ in range(3):
        t = time.time()
        rep = g.run(st, T)
        best = min(best, time.time() - t)
    print(f"{g.KINDS[kind]} {n}^3 T={T}: e2e {best:.3f} s = {n ** 3 * T / best / 1e6:.0f} MLUP/s, "
          f"h2d {rep.h2d_bytes / 1e9:.1f} GB, streamed={rep.streamed}", flush=True)
    del st
