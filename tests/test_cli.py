"""The reference CLI flows (verify / run / tune, proj/tools/main.cpp) through the drop-in shim
include/girih_gpu.hpp, as built into oracle/_ref/girih_gpu against the reference core."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "oracle", "_ref", "girih_gpu")

needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="oracle/_ref/girih_gpu not built")


def run(*args, timeout=300):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


@needs_cli
def test_cli_rejects_bad_input_with_exit_2():
    # main.cpp:524-527: exceptions -> exit 2 (no device needed: fails before any CUDA call)
    r = run("verify", "--stencil", "9pt")
    assert r.returncode == 2 and "unknown stencil kind" in r.stderr
    r = run("frobnicate")
    assert r.returncode == 2
    r = run("verify", "--bogus")
    assert r.returncode == 2


@needs_cli
@pytest.mark.gpu
def test_cli_verify_all_passes():
    # cli_checks.sh:75-77 analogue: every stencil x every compiled fused depth PASSes
    r = run("verify", "--all", "--nx", 24, "--ny", 21, "--nz", 19, "--nt", 7, "--seed", 1234)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert lines and all(l.startswith("PASS ") for l in lines)
    assert len(lines) >= 4


@needs_cli
@pytest.mark.gpu
def test_cli_verify_inject_fault_fails():
    # tests/CMakeLists.txt:24-26 (WILL_FAIL): a perturbed cell must fail verification
    r = run("verify", "--stencil", "var7pt", "--n", 20, "--nt", 5, "--inject-fault")
    assert r.returncode == 1
    assert r.stdout.startswith("FAIL ") and "first-diff field=" in r.stdout


@needs_cli
@pytest.mark.gpu
def test_cli_run_record_and_tune_cache(tmp_path):
    out = tmp_path / "rec.csv"
    for _ in range(2):
        r = run("run", "--stencil", "const7pt", "--n", 64, "--nt", 8, "--remap", "--out", out)
        assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0].startswith("schema_version,stencil,nx,ny,nz,nt,dw,nf,tgs,variant,groups,seed,")
    assert len(lines) == 3  # single header on append (cli_checks.sh)
    r = run("run", "--stencil", "var7pt", "--n", 32, "--nt", 4, "--format", "json")
    rec = json.loads(r.stdout.strip())
    assert rec["schema_version"] == 1 and rec["mlups"] > 0
    tuned = tmp_path / "tuned.jsonl"
    r = run("run", "--stencil", "var7pt", "--n", 48, "--use-tuned", tuned)
    assert r.returncode == 2  # no tuned entry yet (cli_checks.sh: missing tuned -> exit 2)
    r = run("tune", "--stencil", "var7pt", "--n", 48, "--out", tuned, "--max-tb", 2)
    assert r.returncode == 0, r.stderr
    r = run("tune", "--stencil", "var7pt", "--n", 48, "--out", tuned)
    assert r.returncode == 0 and r.stdout.startswith("cached")
    r = run("run", "--stencil", "var7pt", "--n", 48, "--nt", 4, "--use-tuned", tuned)
    assert r.returncode == 0, r.stderr


@needs_cli
def test_cli_model_prints_gpu_and_cpu_models():
    # models.cpp analogue: one CSV line per (stencil, fused depth); host-only, no device
    r = run("model", "--all", "--n", 512)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    hdr = lines[0].split(",")
    rows = [dict(zip(hdr, l.split(","))) for l in lines[1:]]
    assert {x["stencil"] for x in rows} == {"const7pt", "var7pt", "const25pt", "var25pt"}
    for x in rows:
        b1 = {"const7pt": 16, "var7pt": 72, "const25pt": 32, "var25pt": 120}[x["stencil"]]
        assert abs(float(x["gpu_code_balance"]) * int(x["tb"]) - b1) < 0.01
    # the reference's own Eq. 4 and spatial balance ride along (models.cpp:27-49)
    v7 = [x for x in rows if x["stencil"] == "var7pt"][0]
    assert float(v7["cpu_spatial_balance"]) == 80.0
