"""World-size-2 test (gloo, CPU) of the multi-GPU z-slab decomposition protocol.

Each rank owns the interior planes girih_gpu_slab_layout assigns it (the same partition the
library's multi-slab handles use) plus hz = R*TBmax halo planes per side. It advances its slab
by passes of up to TB steps with the oracle's naive sweep, then exchanges the hz planes
adjacent to each neighbour (both solution fields) with dist.send/recv. After the run, rank 0
gathers the slabs and compares them bitwise with the single-domain oracle.

The GPU kernels implement the same schedule (exchange after every pass, R*TB-deep halos,
redundant trapezoid recompute inside the halo). tests/test_gpu_parity.py checks them bitwise on
one device with emulated slabs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_bindings import TRAITS, HostState, Oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, n, steps, tb, seed, out_q):
    import paper_1510_04995_b200 as g

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        orc = Oracle()
        R = TRAITS[kind][0]
        full = orc.init_state(kind, n, n, n, 0, seed, remap=True)
        z0, z1, hz = g.slab_layout(kind, n, world, rank)
        assert hz >= R * tb
        Z = n + 2 * R
        # local domain in global allocated planes: own [R+z0, R+z1) + halos (global ghost planes
        # at the outer ends); its outermost R planes act as the local Dirichlet boundary
        lo = 0 if rank == 0 else R + z0 - hz
        hi = Z if rank == world - 1 else R + z1 + hz
        sl = slice(lo, hi)
        loc = HostState(kind, n, n, (hi - lo) - 2 * R, 0, full.u[sl].copy(), full.v[sl].copy(),
                        [c[sl].copy() for c in full.coeffs], full.cc.copy(), 0)
        own_lo, own_hi = R + z0 - lo, R + z1 - lo  # local plane indices of the owned planes
        done = 0
        while done < steps:
            d = min(tb, steps - done)
            orc.naive_sweep(loc, d)
            done += d
            # halo exchange: my hz boundary planes -> neighbour's halo planes (u and v)
            reqs = []
            for f in (loc.u, loc.v):
                if rank > 0:
                    reqs.append(dist.isend(torch.from_numpy(f[own_lo:own_lo + hz].copy()), rank - 1))
                    buf = torch.empty(f[own_lo - hz:own_lo].shape, dtype=torch.float64)
                    dist.recv(buf, rank - 1)
                    f[own_lo - hz:own_lo] = buf.numpy()
                if rank < world - 1:
                    reqs.append(dist.isend(torch.from_numpy(f[own_hi - hz:own_hi].copy()), rank + 1))
                    buf = torch.empty(f[own_hi:own_hi + hz].shape, dtype=torch.float64)
                    dist.recv(buf, rank + 1)
                    f[own_hi:own_hi + hz] = buf.numpy()
            for r in reqs:
                r.wait()
        # gather owned planes on rank 0
        parts_u = [torch.from_numpy(loc.u[own_lo:own_hi].copy())]
        parts_v = [torch.from_numpy(loc.v[own_lo:own_hi].copy())]
        if rank == 0:
            for src in range(1, world):
                zs0, zs1, _ = g.slab_layout(kind, n, world, src)
                for parts in (parts_u, parts_v):
                    buf = torch.empty((zs1 - zs0,) + loc.u.shape[1:], dtype=torch.float64)
                    dist.recv(buf, src)
                    parts.append(buf)
            got_u = torch.cat(parts_u).numpy()
            got_v = torch.cat(parts_v).numpy()
            ref = full.copy()
            orc.naive_sweep(ref, steps)
            ok = (np.array_equal(got_u.view(np.uint64), ref.u[R:R + n].view(np.uint64)) and
                  np.array_equal(got_v.view(np.uint64), ref.v[R:R + n].view(np.uint64)))
            out_q.put(bool(ok))
        else:
            dist.send(parts_u[0], 0)
            dist.send(parts_v[0], 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,tb", [(1, 14, 4), (0, 11, 3), (2, 24, 2), (3, 22, 1)])
def test_zslab_exchange_world2_matches_single_domain(girih, kind, n, tb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, n, 11, tb, 5, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
