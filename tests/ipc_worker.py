"""Worker for tests/test_gpu_parity.py::test_ipc_halo_push_two_processes (not a test module).

One rank of a multi-process z-slab run whose halos move by the passes' own peer stores (CUDA
IPC, no NCCL): gloo carries the IPC blobs, every rank checks its slab bitwise against a
single-domain run of the same seeded grid. Launched by torch.distributed.run with two ranks."""
import os
import sys

import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import paper_1510_04995_b200 as g  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("GIRIH_IPC_DEVICE", "0"))
    bad = 0
    # (the last two: slabs of several z-chunk rows, so boundary rows run first and interior
    # rows overlap the neighbours' next pass; the kernel signals the neighbours)
    # (the last two again: the inner-columns-only tiles forced on grids of several tile columns;
    # the fused var7pt one starts its tile grid on the ghost column)
    narrow = {k: next(v for v in g.variants() if v["kind"] == k and v["narrow"]) for k in (0, 1)}
    for kind, (nx, ny, nz), steps, zc, var in ((1, (40, 33, 50), 9, 0, None), (3, (37, 30, 52), 5, 0, None),
                                               (2, (36, 29, 48), 6, 0, None), (0, (41, 35, 47), 7, 0, None),
                                               (1, (70, 45, 150), 7, 6, None), (3, (45, 38, 160), 4, 7, None),
                                               (1, (131, 30, 60), 7, 0, narrow[1]), (0, (131, 30, 60), 5, 0, narrow[0])):
        grid = g.GridSpec(nx, ny, nz, 0)
        cfg = (g.GpuConfig(device=dev, zchunks=zc) if var is None else
               g.GpuConfig(device=dev, zchunks=zc, tb=var["tb"], variant=var["index"]))
        with g.DeviceState.slab_seeded(kind, grid, 17, True, rank, world, None, cfg) as ds:
            blobs = [None] * world
            dist.all_gather_object(blobs, ds.ipc_export())
            try:  # stepping an unconnected IPC slab is refused (its halos would go stale)
                ds.step(1)
                bad += 1
                print(f"rank {rank}: step before ipc_connect was not refused", flush=True)
            except g.GirihError:
                pass
            ds.ipc_connect(blobs[rank - 1] if rank > 0 else None,
                           blobs[rank + 1] if rank + 1 < world else None)
            dist.barrier()
            ds.step(steps)
            ds.step(steps + 1)  # a second call: odd start level, pass counters carry over
            dist.barrier()
            with g.DeviceState.seeded(kind, grid, 17, remap=True,
                                      config=g.GpuConfig(device=dev, chain=-1)) as ref:
                ref.step(steps)
                ref.step(steps + 1)
                host = ref.download(coeffs=False)
            for f in ("u", "v"):
                n, first = ds.compare(f, getattr(host, f))
                if n:
                    bad += 1
                    print(f"rank {rank} {g.KINDS[kind]} field {f}: {n} cells differ, first {first}",
                          flush=True)
            dist.barrier()
    print(f"rank {rank}: {'OK' if bad == 0 else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
