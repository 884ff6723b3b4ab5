"""Generates tests/golden/c5.json: reference-pinned digests of the BASELINE C5 scaling sizes.

The REFERENCE ITSELF computes every case: oracle/_ref/libgirih_ref.so (the unmodified reference
core compiled from /root/reference/proj/src by oracle/Makefile) allocates the ProblemState, the
oracle's multi-threaded copy of the reference generator fills it (init_state,
proj/src/stencil.cpp:58-85, bit-identical), the SURVEY.md 8(d) remap is applied, and the
reference's MWD engine girih::run (proj/src/engine.cpp:332-418; bitwise equal to naive_sweep by
the reference's own tests) advances it T steps on all host cores. Recorded per case:

* row_digest_u / row_digest_v: FNV-1a over the FNV-1a hashes of every allocated row of u / v
  (ghosts and pad included; oracle orc_row_digest == girih_gpu_row_digest on the device);
* interior_checksum: the reference's interior_checksum (stencil.cpp:129-146) of the final level.

The states reach 132 GB (var25pt 1024^3), so this runs on the GPU box's host (196 GB RAM,
16 cores), where oracle/_ref travels with the repo snapshot:

    gpurun -- python tests/golden/make_c5.py [--cases var7pt:384,...] [--out tests/golden/c5.json]

Cases whose state does not fit the host's RAM are recorded as {"excluded": "..."}.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bindings import Oracle, RefLib, RefState  # noqa: E402

KINDS = ("const7pt", "var7pt", "const25pt", "var25pt")
# BASELINE configs[4] (C5): N in {384, 768, 960} at 100 steps (64-512 are covered elsewhere:
# 256 and 512 by the C1-C4 checksums, 64/128 by the fixtures), and the 1024^3 multi-GPU grid
# at 200 steps
DEFAULT_CASES = [(k, n, 100) for k in (1, 3) for n in (384, 768, 960)] + \
                [(1, 1024, 200), (3, 1024, 200)]


def state_bytes(kind: int, n: int) -> int:
    R = 1 if kind < 2 else 4
    arrays = {0: 2, 1: 9, 2: 3, 3: 15}[kind]
    return arrays * (n + 2 * R) ** 3 * 8


def host_ram() -> int:
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="", help="comma list kind:n[:T], e.g. var7pt:384")
    ap.add_argument("--out", default=os.path.join(HERE, "c5.json"))
    a = ap.parse_args()
    cases = DEFAULT_CASES
    if a.cases:
        cases = []
        for c in a.cases.split(","):
            f = c.split(":")
            cases.append((KINDS.index(f[0]), int(f[1]), int(f[2]) if len(f) > 2 else 100))
    ref, orc = RefLib(), Oracle()
    threads = os.cpu_count() or 1
    out = []
    if os.path.exists(a.out):
        with open(a.out) as f:
            out = [c for c in json.load(f)["cases"]
                   if (KINDS.index(c["stencil"]), c["n"], c["steps"]) not in cases]
    for kind, n, T in cases:
        rec = dict(stencil=KINDS[kind], n=n, steps=T, seed=42, remap=True)
        need = state_bytes(kind, n)
        if need > 0.92 * host_ram():
            rec["excluded"] = f"state {need / 1e9:.1f} GB exceeds host RAM {host_ram() / 1e9:.0f} GB"
            out.append(rec)
            print(rec, flush=True)
            continue
        t0 = time.time()
        st = RefState(ref, kind, n, n, n, 0, 42, oracle_fill=orc, remap=True)
        t1 = time.time()
        dw = 8 if kind < 2 else 16
        wall, _ = st.run(T, dw, 4, (1, 1, 1), 0 if kind < 2 else 1, threads)
        t2 = time.time()
        rec.update(t_final=st.t_current,
                   row_digest_u=f"{orc.row_digest(st.u):#018x}",
                   row_digest_v=f"{orc.row_digest(st.v):#018x}",
                   interior_checksum=f"{st.checksum():#018x}",
                   engine=f"girih::run MWD dw={dw} nf=4 {'relaxed' if kind < 2 else 'fed'} "
                          f"{threads} groups",
                   init_s=round(t1 - t0, 1), run_s=round(wall, 1),
                   hash_s=round(time.time() - t2, 1), state_gb=round(need / 1e9, 1))
        out.append(rec)
        print(rec, flush=True)
        del st
        with open(a.out, "w") as f:  # keep partial progress
            json.dump({"generator": "tests/golden/make_c5.py (reference core via oracle/_ref)",
                       "cases": out}, f, indent=1)
    with open(a.out, "w") as f:
        json.dump({"generator": "tests/golden/make_c5.py (reference core via oracle/_ref)",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
