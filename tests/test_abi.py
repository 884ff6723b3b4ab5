"""CPU tests of the C ABI library (no device calls): symbols, traits, errors, pass planner."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "girih_gpu.h")).read()
    return sorted(set(re.findall(r"\b(girih_gpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(girih):
    lib = C.CDLL(girih.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # the Python binding covers the whole header too
    from paper_1510_04995_b200._lib import SIGNATURES

    assert set(names) == set(SIGNATURES)


def test_abi_version(girih):
    assert girih.load().girih_gpu_abi_version() == 6


def test_traits_and_names(girih):
    t = girih.traits(girih.VAR25PT)
    assert (t.radius, t.domain_streams, t.flops_per_lup, t.time_order, t.coeff_arrays) == (
        4, 15, 37, 1, 13)
    assert girih.traits(girih.CONST25PT).time_order == 2
    for i, n in enumerate(girih.KINDS):
        assert girih.stencil_from_name(n) == i
    with pytest.raises(ValueError):
        girih.stencil_from_name("9pt")
    with pytest.raises(ValueError):
        girih.traits(7)


def test_variants_registry(girih):
    vs = girih.variants()
    assert {v["kind"] for v in vs} == {0, 1, 2, 3}
    for v in vs:
        assert v["smem_bytes"] <= 227 * 1024
        R = 1 if v["kind"] < 2 else 4
        # threads cover the level-1 rows [R, ly - R) in x-pairs
        # (all lx columns, or the inner ones when narrow = the output tile's x halo is set)
        xo = v["narrow"] - (v["tb"] - 1) * R if v["narrow"] else 0
        assert (v["lx"] - 2 * xo) * (v["ly"] - 2 * R) % (2 * v["threads"]) == 0 and v["threads"] % 32 == 0
        assert v["lx"] > 2 * R * v["tb"]
        if v["cluster_y"] == 1:
            assert v["ly"] > 2 * R * v["tb"]
        else:
            # cluster CTAs: the outer ones keep (tb - 1) R halo rows on their outer side
            assert v["tb"] >= 2 and v["ly"] - R - R * v["tb"] > 0 and v["cluster_y"] <= 16
    # every kind has a single-step variant and R=1 kinds fuse at least 4 steps
    for k in range(4):
        assert any(v["kind"] == k and v["tb"] == 1 for v in vs)
    for k in (0, 1):
        assert max(v["tb"] for v in vs if v["kind"] == k) >= 4


def _simulate(kind, t0, steps, plan):
    """Symbolic execution of a plan: buffer id -> level held (interior)."""
    par = lambda t: t % 2  # noqa: E731
    hold = {par(t0): t0, par(t0 - 1): t0 - 1}  # fields: level t0 and t0-1 (leapfrog seed)
    t = t0
    for tb, src, sprev, dst, pen in plan:
        assert 1 <= tb
        assert hold.get(src) == t, (plan, t)
        assert src % 2 == par(t)
        if kind == 2:
            assert hold.get(sprev) == t - 1
            if tb == 1:
                assert dst == sprev and pen == -1  # in-place leapfrog
            else:
                assert dst not in (src, sprev) and pen not in (src, sprev, -1)
        else:
            assert sprev == -1
            assert dst != src
            assert pen != src
        assert dst % 2 == par(t + tb)
        if pen >= 0:
            assert pen % 2 == par(t + tb - 1)
        hold[dst] = t + tb
        if pen >= 0:
            hold[pen] = t + tb - 1
        t += tb
    return hold, t


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_planner_places_both_final_levels(girih, kind):
    for t0 in (0, 1, 2, 5):
        for steps in range(0, 23):
            for tb in (1, 2, 3, 4, 5):
                plan = girih.plan(kind, t0, steps, tb)
                assert all(p[0] <= tb for p in plan)
                assert sum(p[0] for p in plan) == steps
                hold, t = _simulate(kind, t0, steps, plan)
                assert t == t0 + steps
                if steps >= 1:
                    # level T in the field of parity(T), level T-1 in the other field
                    assert hold[(t0 + steps) % 2] == t0 + steps
                    assert hold[(t0 + steps - 1) % 2] == t0 + steps - 1
                # never more than one pass above the lower bound
                lb = -(-steps // tb)
                assert len(plan) <= lb + (2 if kind == 2 else 1)
                if tb == 1:
                    assert len(plan) == steps


def test_planner_bench_plan_is_minimal(girih):
    # var7pt 100 steps at tb=4: 25 equal passes are infeasible (all even -> the final source
    # would be a field), so 26 passes is optimal
    p = girih.plan(1, 0, 100, 4)
    assert len(p) == 26
    assert girih.plan(1, 0, 99, 3)[0][0] == 3
    assert len(girih.plan(2, 0, 100, 2)) == 50


def test_planner_rejects_bad_input(girih):
    with pytest.raises(ValueError):
        girih.plan(0, 0, -1, 2)
    with pytest.raises(ValueError):
        girih.plan(0, 0, 5, 0)
    with pytest.raises(ValueError):
        girih.plan(9, 0, 5, 1)


def test_model_matches_roofline_algebra(girih):
    # girih_gpu_model: the GPU counterpart of models.cpp (code_balance / roofline); host-only
    B1 = {0: 16, 1: 72, 2: 32, 3: 120}
    DP = {0: 10, 1: 13, 2: 33, 3: 37}
    grid = girih.GridSpec(512, 512, 512, 0)
    for kind in range(4):
        for tb in sorted({v["tb"] for v in girih.variants() if v["kind"] == kind}):
            m = girih.model(kind, grid, tb, hbm_gbs=6000.0, fp64_ops=18e12)
            assert m["tb"] == tb and m["code_balance"] == B1[kind] / tb
            assert m["redundancy"] >= 1.0 and m["code_balance_no_l2"] > m["code_balance"]
            assert m["hbm_mlups"] == pytest.approx(6000e9 * tb / B1[kind] / 1e6)
            assert m["fp64_mlups"] == pytest.approx(18e12 / (DP[kind] * m["redundancy"]) / 1e6)
            assert m["roofline_mlups"] == min(m["hbm_mlups"], m["fp64_mlups"])
            assert m["tiles_x"] * m["ox"] >= 512 and m["tiles_y"] * m["oy"] >= 512
            assert m["zchunks"] * m["zc_len"] >= 512 and m["ctas_per_sm"] >= 1
            v = girih.variants()[m["variant"]]
            assert (v["kind"], v["tb"], v["smem_bytes"]) == (kind, tb, m["smem_bytes"])
        # Tb = 1 redundancy is the halo of one step only
        assert girih.model(kind, grid, 1)["redundancy"] < 1.2
    with pytest.raises(ValueError):
        girih.model(0, grid, 99)
    with pytest.raises(ValueError):
        girih.model(0, girih.GridSpec(2, 2, 2, 0), 1)


def test_smoke_cases_use_compiled_depths(girih):
    # __graft_entry__.smoke() must only request fused depths the library has kernels for
    import importlib.util

    spec = importlib.util.spec_from_file_location("graft_entry", os.path.join(ROOT, "__graft_entry__.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    tbs = {(v["kind"], v["tb"]) for v in girih.variants()}
    assert {k for k, _, _ in mod.SMOKE_CASES} == {0, 1, 2, 3}
    for kind, tb, steps in mod.SMOKE_CASES:
        assert (kind, tb) in tbs, (kind, tb)
        assert steps % tb != 0 or steps // tb > 1
