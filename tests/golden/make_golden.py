"""Generates tests/golden/fixtures.json from the REFERENCE ITSELF (oracle/_ref/libgirih_ref.so,
the unmodified reference core compiled from /root/reference/proj/src by oracle/Makefile).

Each case runs the reference's init_state (proj/src/stencil.cpp:58-85), optionally the
BASELINE input remap, then the reference's naive_sweep (stencil.cpp:115-127)
in one or two chunks (continuation from t_current, test_engine.cpp:149-157) and -- for the
"mwd" cases -- the reference's MWD engine girih::run (engine.cpp:332-418). Recorded: FNV-1a
of every byte of u and of v (ghosts and pad included) and the reference's interior_checksum.

Run here (needs /root/reference): python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bindings import Oracle, RefLib, RefState  # noqa: E402

# (kind, nx, ny, nz, pad_x, seed, remap, chunks, engine)
CASES = [
    # the reference's own pinned golden checksums (proj/tests/test_stencil.cpp:145-153)
    (3, 24, 24, 24, 0, 3, False, [4], "naive"),
    (0, 16, 16, 16, 0, 11, False, [5], "naive"),
    # acceptance #1 geometry (proj/tests/acceptance.cpp:37-66): 48^3, T=16, seed 1234
    (0, 48, 48, 48, 0, 1234, False, [16], "naive"),
    (1, 48, 48, 48, 0, 1234, False, [16], "naive"),
    (2, 48, 48, 48, 0, 1234, False, [16], "naive"),
    (3, 48, 48, 48, 0, 1234, False, [16], "naive"),
    # continuation with padded rows (test_engine.cpp:149-157)
    (0, 16, 16, 16, 2, 9, False, [3, 4], "naive"),
    (2, 17, 13, 11, 3, 9, False, [3, 4], "naive"),
    # ragged, odd extents, BASELINE remap, odd start levels
    (1, 33, 20, 27, 1, 42, True, [1, 6], "naive"),
    (3, 21, 19, 23, 5, 7, True, [2, 3], "naive"),
    (2, 9, 9, 9, 0, 0, True, [10], "naive"),
    (0, 3, 3, 3, 0, 1, True, [7], "naive"),
    (1, 64, 64, 64, 0, 42, True, [10], "naive"),
    (3, 64, 64, 64, 0, 42, True, [5], "naive"),
    # the reference's MWD engine on the same inputs (bitwise equal to naive by contract)
    (0, 48, 48, 48, 0, 1234, False, [16], "mwd"),
    (2, 48, 48, 48, 0, 1234, False, [16], "mwd"),
]


def main() -> None:
    ref = RefLib()
    orc = Oracle()
    out = []
    for kind, nx, ny, nz, pad, seed, remap, chunks, engine in CASES:
        st = RefState(ref, kind, nx, ny, nz, pad, seed)
        if remap:
            st.apply_remap(orc)
        for ch in chunks:
            if engine == "naive":
                st.naive_sweep(ch)
            else:
                dw = 8 if kind < 2 else 16
                st.run(ch, dw, 4, (1, 1, 1), 0 if kind < 2 else 1, 2)
        out.append(dict(kind=kind, nx=nx, ny=ny, nz=nz, pad_x=pad, seed=seed, remap=remap,
                        chunks=chunks, engine=engine, t_final=st.t_current,
                        fnv_u=f"{orc.fnv_all(st.u):#018x}", fnv_v=f"{orc.fnv_all(st.v):#018x}",
                        interior_checksum=f"{st.checksum():#018x}"))
        print(out[-1])
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference core via oracle/_ref)",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
