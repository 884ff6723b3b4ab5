"""The reference-signature drop-in girih::gpu::run (include/girih_gpu.hpp) driven by the
reference's own acceptance matrix and engine tests (tests/shim_acceptance.cpp, built by
oracle/Makefile against the unmodified reference core and libgirih_gpu.so)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "shim_acceptance")


def test_reference_signature_shim_acceptance():
    assert os.path.exists(EXE), "build with `make -C oracle` (needs the reference sources)"
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    lines = out.stdout.splitlines()
    assert out.returncode == 0, out.stdout + out.stderr
    # 4 acceptance kinds (80 runs), invalid configs, T = 0, 4 continuations, 5 ledgers, trace
    assert sum(l.startswith("PASS  ") for l in lines) == 16, out.stdout
    assert lines[-1].startswith("PASS: 0 failure")
