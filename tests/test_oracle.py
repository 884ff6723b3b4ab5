"""CPU tests of the oracle restatement (oracle/girih_oracle.c), pinned against the reference's
own known-answer tests (proj/tests/test_stencil.cpp) and against the reference core itself."""
import numpy as np
import pytest

from oracle_bindings import TRAITS


def bits(a):
    return a.view(np.uint64)


def test_traits_table_matches_reference():
    # proj/tests/test_stencil.cpp:20-44
    assert TRAITS[0] == (1, 2, 7, 1, 0)
    assert TRAITS[1][:3] == (1, 9, 13) and TRAITS[1][4] == 7
    assert TRAITS[2][0] == 4 and TRAITS[2][2] == 33 and TRAITS[2][3] == 2 and TRAITS[2][4] == 1
    assert TRAITS[3] == (4, 15, 37, 1, 13)


def test_golden_checksums_pinned(oracle):
    # proj/tests/test_stencil.cpp:145-153
    s = oracle.init_state(3, 24, 24, 24, 0, 3)
    oracle.naive_sweep(s, 4)
    assert oracle.interior_checksum(s) == 0x64179E6CB2CCF3DD
    c = oracle.init_state(0, 16, 16, 16, 0, 11)
    oracle.naive_sweep(c, 5)
    assert oracle.interior_checksum(c) == 0x99E588473D945C73


def test_init_deterministic_and_seed_sensitive(oracle):
    a = oracle.init_state(0, 8, 8, 8, 0, 0)
    b = oracle.init_state(0, 8, 8, 8, 0, 0)
    c = oracle.init_state(0, 8, 8, 8, 0, 1)
    assert np.array_equal(bits(a.u), bits(b.u)) and np.array_equal(bits(a.v), bits(b.v))
    assert np.array_equal(a.cc, b.cc)
    assert not np.array_equal(bits(a.u), bits(c.u))


def test_init_matches_reference_bitwise(oracle, reflib):
    from oracle_bindings import RefState

    for kind, n, pad in [(0, 8, 0), (1, 7, 3), (2, 9, 1), (3, 10, 2)]:
        r = RefState(reflib, kind, n, n + 1, n + 2, pad, 77)
        o = oracle.init_state(kind, n, n + 1, n + 2, pad, 77)
        assert np.array_equal(bits(r.u), bits(o.u))
        assert np.array_equal(bits(r.v), bits(o.v))
        for rc, oc in zip(r.coeffs, o.coeffs):
            assert np.array_equal(bits(rc), bits(oc))
        assert np.array_equal(bits(r.cc), bits(o.cc))


def test_init_rejects_small_grids(oracle):
    # test_stencil.cpp:65-69
    with pytest.raises(ValueError):
        oracle.init_state(2, 8, 8, 8, 0, 0)
    with pytest.raises(ValueError):
        oracle.init_state(0, 2, 8, 8, 0, 0)
    oracle.init_state(2, 9, 9, 9, 0, 0)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_naive_matches_reference_bitwise(oracle, reflib, kind):
    from oracle_bindings import RefState

    dims = (13, 11, 12, 2) if kind < 2 else (11, 9, 10, 1)
    r = RefState(reflib, kind, *dims, 5)
    o = oracle.init_state(kind, *dims, 5)
    r.naive_sweep(3)
    oracle.naive_sweep(o, 3)
    r.naive_sweep(4)
    oracle.naive_sweep(o, 4)
    assert r.t_current == o.t_current == 7
    assert np.array_equal(bits(r.u), bits(o.u)) and np.array_equal(bits(r.v), bits(o.v))


def test_straight_line_var7(oracle):
    # test_stencil.cpp:91-107
    s = oracle.init_state(1, 6, 6, 6, 0, 99)
    V = s.u
    C = s.coeffs
    for k in range(1, 7):
        for j in range(1, 7):
            for i in range(1, 7):
                want = (C[0][k, j, i] * V[k, j, i] + C[1][k, j, i] * V[k, j, i + 1]
                        + C[2][k, j, i] * V[k, j, i - 1] + C[3][k, j, i] * V[k, j + 1, i]
                        + C[4][k, j, i] * V[k, j - 1, i] + C[5][k, j, i] * V[k + 1, j, i]
                        + C[6][k, j, i] * V[k - 1, j, i])
                assert oracle.apply_point(s, i, j, k) == want


def test_straight_line_const25(oracle):
    # test_stencil.cpp:109-122
    s = oracle.init_state(2, 9, 9, 9, 0, 21)
    V, U, Cf, cc = s.u, s.v, s.coeffs[0], s.cc
    i = j = k = 4
    lap = cc[0] * V[k, j, i]
    for r in range(1, 5):
        lap += cc[r] * (V[k, j, i + r] + V[k, j, i - r] + V[k, j + r, i] + V[k, j - r, i]
                        + V[k + r, j, i] + V[k - r, j, i])
    want = 2 * V[k, j, i] - U[k, j, i] + Cf[k, j, i] * lap
    assert oracle.apply_point(s, i, j, k) == want


def test_zero_steps_no_op_and_negative_rejected(oracle):
    a = oracle.init_state(1, 8, 8, 8, 0, 3)
    b = a.copy()
    oracle.naive_sweep(a, 0)
    assert a.t_current == 0
    assert np.array_equal(bits(a.u), bits(b.u)) and np.array_equal(bits(a.v), bits(b.v))
    with pytest.raises(ValueError):
        oracle.naive_sweep(a, -1)


def test_ghosts_never_written(oracle):
    # test_stencil.cpp:155-168
    s = oracle.init_state(1, 8, 8, 8, 0, 17)
    fresh = s.copy()
    oracle.naive_sweep(s, 6)
    R = 1
    mask = np.ones(s.u.shape, bool)
    mask[R:R + 8, R:R + 8, R:R + 8] = False
    for f, g in ((s.u, fresh.u), (s.v, fresh.v)):
        assert np.array_equal(bits(f[mask]), bits(g[mask]))


def test_locality_r_per_step(oracle):
    # test_stencil.cpp:170-193
    for kind, n, steps in ((0, 16, 3), (3, 16, 1)):
        base = oracle.init_state(kind, n, n, n, 0, 13)
        poke = base.copy()
        R = TRAITS[kind][0]
        c = R + n // 2
        poke.u[c, c, c] += 1.0
        oracle.naive_sweep(base, steps)
        oracle.naive_sweep(poke, steps)
        reach = R * steps
        fa, fb = base.current(), poke.current()
        idx = np.indices(fa.shape)
        d = np.max(np.abs(idx - c), axis=0)
        interior = np.zeros(fa.shape, bool)
        interior[R:R + n, R:R + n, R:R + n] = True
        far = interior & (d > reach)
        assert np.array_equal(bits(fa[far]), bits(fb[far]))
        assert not np.array_equal(bits(fa), bits(fb))


def test_linear_under_power_of_two(oracle):
    # test_stencil.cpp:195-211
    for kind in (0, 2):
        a = oracle.init_state(kind, 12, 12, 12, 0, 29)
        b = a.copy()
        b.u *= 2.0
        b.v *= 2.0
        oracle.naive_sweep(a, 3)
        oracle.naive_sweep(b, 3)
        R = TRAITS[kind][0]
        sl = (slice(R, R + 12),) * 3
        assert np.array_equal(bits(2.0 * a.current()[sl]), bits(b.current()[sl]))


def test_remap_ranges(oracle):
    # fields in [0,1), var7 coefficients in [0,0.14), var25 in [0,1/26),
    # const25 scalars scaled so |c0| + 6 sum|c_r| = 0.99
    s = oracle.init_state(1, 10, 10, 10, 0, 42, remap=True)
    assert s.u.min() >= 0 and s.u.max() < 1
    for c in s.coeffs:
        assert c.min() >= 0 and c.max() < 0.14
    s = oracle.init_state(3, 9, 9, 9, 0, 42, remap=True)
    for c in s.coeffs:
        assert c.min() >= 0 and c.max() < 1 / 26
    s = oracle.init_state(2, 9, 9, 9, 0, 42, remap=True)
    assert abs(s.cc[0] + 6 * s.cc[1:].sum() - 0.99) < 1e-15
    s = oracle.init_state(0, 9, 9, 9, 0, 42, remap=True)
    assert 0 <= s.cc[0] < 0.2 and 0 <= s.cc[1] < 0.2


def test_config1_checksum_matches_survey(oracle):
    # SURVEY.md 8(c) config-level cross-check: C1 const7pt 256^3 seed 42 remap, T=100
    s = oracle.init_state(0, 256, 256, 256, 0, 42, remap=True)
    oracle.naive_sweep(s, 100)
    assert oracle.interior_checksum(s) == 0x9F26250C918339D4


def test_row_digest_definition(oracle):
    # FNV-1a over the per-row FNV-1a hashes (the C5 fixtures' digest), restated in Python
    import numpy as np
    a = np.random.default_rng(3).random((3, 4, 5))

    def fnv(bs, h=0xCBF29CE484222325):
        for b in bs:
            h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        return h

    rows = [fnv(a[k, j].tobytes()) for k in range(3) for j in range(4)]
    want = fnv(b"".join(r.to_bytes(8, "little") for r in rows))
    assert oracle.row_digest(a) == want
