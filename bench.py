#!/usr/bin/env python
"""Benchmark of the temporally-blocked fp64 stencil sweep (BASELINE.json metric: MLUP/s).

Default workload = BASELINE.json configs[4] (C5), the largest single-GPU configuration and the
north_star strong-scaling grid: var7pt, 1024^3 interior, 1-cell Dirichlet halo, 7 coefficient
grids in [0, 0.14), field in [0, 1), 200 time steps, seed 42 (synthetic inputs generated on the
device with the reference's counter-based generator + SURVEY.md 8(d) remap). With --gpus N the
SAME global grid is split into N z-slabs, one per GPU (strong scaling). One bench "step" = one
girih_gpu_step(200) call = the full 200-time-step sweep of the config.
C2 (var7pt 512^3, 100 steps): --n 512 --nt 100; other kinds: --stencil.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--stencil var7pt --n 1024]

At N = 1 the on-device auto-tuner (girih_gpu_tune: model-pruned hill-climb over the compiled
variants, z chunks and pass chaining, starting from the default) runs first and the timed steps
use its choice, recorded under gpu.tuned (--no-tune: the defaults).

Prints ONE JSON line (rank 0). `value` is device-timed MLUP/s with inputs resident in HBM;
`e2e` is the same metric through the drop-in C-ABI call girih_gpu_run on PAGEABLE host buffers
(what the reference's ProblemState std::vectors are): H2D of u, v, coefficients + all passes +
D2H of u, v inside the timed region; at N > 1 rank 0 makes the multi-GPU drop-in call over all N
GPUs. `--impl reference` times the reference's own CPU engine (girih::run, MWD, all host cores)
from oracle/_ref on the same config (bounded samples of the time steps; the metric is a rate).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KINDS = ("const7pt", "var7pt", "const25pt", "var25pt")
B1 = {0: 16, 1: 72, 2: 32, 3: 120}          # compulsory bytes/LUP of one sweep
DP_OPS = {0: 10, 1: 13, 2: 33, 3: 37}       # DMUL+DADD per LUP in the reference association
FLOPS = {0: 7, 1: 13, 2: 33, 3: 37}         # traits flops/LUP (stencil.cpp:11-17)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


def ncu_traffic(kind: int, n: int):
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{KINDS[kind]}_{n}")
    if not e:
        return None, None
    return e.get("dram_bytes_per_launch"), e.get("source")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(kind: int, n: int, T: int) -> dict:
    """The bench configuration, identical in the GPU and the reference arm."""
    conf = ("BASELINE configs[4] (C5) strong-scaling grid" if (kind in (1, 3) and n == 1024 and T == 200)
            else "BASELINE configs[1] (C2)" if (kind == 1 and n == 512 and T == 100)
            else "BASELINE configs[0] (C1)" if (kind == 0 and n == 256 and T == 100)
            else "BASELINE configs[2] (C3)" if (kind == 2 and n == 512 and T == 100)
            else "BASELINE configs[3] (C4)" if (kind == 3 and n == 512 and T == 100)
            else "custom")
    state_gb = n ** 3 * 8 * {0: 2, 1: 9, 2: 3, 3: 15}[kind] / 1e9
    return {"workload": f"{conf}: {KINDS[kind]} {n}^3 interior, T={T}, seed 42",
            "stencil": KINDS[kind], "n": n, "time_steps": T, "seed": 42,
            "l2": f"inputs {state_gb:.1f} GB >> 126 MB L2 (no flush needed)"}


# ------------------------------------------------------------------------------------------
# CPU arms: the reference's own engine (oracle/_ref) -- checker/baseline only
# ------------------------------------------------------------------------------------------
def _ref_state(kind: int, n: int):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import Oracle, RefLib, RefState

    lib, orc = RefLib(), Oracle()
    return RefState(lib, kind, n, n, n, 0, 42, oracle_fill=orc, remap=True)


def _mwd_params(kind: int):
    R = 1 if kind < 2 else 4
    # dw 8 / 16, nf 4, relaxed for 7-pt and FED for 25-pt
    return (8 if R == 1 else 16), (0 if R == 1 else 1), R


def cpu_reference_sample(kind: int, n: int, target_s: float, max_steps: int, reps: int = 2):
    """Times girih::run (MWD, engine.cpp:332-418) on all host threads on a bounded sample of the
    workload (same grid, fewer time steps), best of `reps` like the reference's own `run`
    (proj/tools/main.cpp:291-297), plus the single-thread naive_sweep (stencil.cpp:115-127) on
    one time step. Returns the cpu_baseline dict."""
    threads = os.cpu_count() or 1
    dw, variant, R = _mwd_params(kind)
    st = _ref_state(kind, n)
    # calibrate on one diamond height, then size the sample to ~target_s
    cal = max(1, dw // (2 * R))
    wall, _ = st.run(cal, dw, 4, (1, 1, 1), variant, threads)
    rate = n ** 3 * cal / max(wall, 1e-9)
    steps = int(max(1, min(max_steps, target_s * rate / n ** 3)))
    walls = []
    for _ in range(reps):
        wall, _ = st.run(steps, dw, 4, (1, 1, 1), variant, threads)
        walls.append(wall)
    mlups = n ** 3 * steps / min(walls) / 1e6
    t0 = time.perf_counter()
    st.naive_sweep(1)
    naive = n ** 3 / (time.perf_counter() - t0) / 1e6
    return dict(value=mlups, unit="MLUP/s", cores=threads, kind="reference",
                sample=f"girih::run MWD {KINDS[kind]} {n}^3, {steps} time steps per sample, "
                       f"dw={dw}, nf=4, {'relaxed' if variant == 0 else 'fed'}, {threads} groups "
                       f"x 1x1x1, best of {reps}",
                naive_single_thread_mlups=naive, naive_sample="naive_sweep, 1 time step, 1 thread",
                cpu_model=cpu_model(), hardware_threads=threads)


def run_reference_arm(args, rank: int):
    """The reference's own CPU engine on the bench config; under torchrun rank 0 alone runs."""
    if rank != 0:
        return 0
    kind = KINDS.index(args.stencil)
    n, T = args.n, args.nt
    threads = os.cpu_count() or 1
    dw, variant, R = _mwd_params(kind)
    st = _ref_state(kind, n)
    cal = max(1, dw // (2 * R))
    wall, _ = st.run(cal, dw, 4, (1, 1, 1), variant, threads)
    rate = n ** 3 * cal / max(wall, 1e-9)
    # each bench step: the first steps_per time steps of the T-step sweep (the MLUP/s rate is
    # what is compared), sized so that (warmup + steps) samples take ~ref_budget_s
    per = args.ref_budget_s / max(1, args.steps + args.warmup)
    steps_per = int(max(1, min(T, per * rate / n ** 3)))
    for _ in range(args.warmup):
        st.run(steps_per, dw, 4, (1, 1, 1), variant, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        st.run(steps_per, dw, 4, (1, 1, 1), variant, threads)
    dt = time.perf_counter() - t0
    value = n ** 3 * steps_per * args.steps / dt / 1e6
    sample = (f"girih::run MWD {KINDS[kind]} {n}^3, {steps_per} of the {T} time steps per bench "
              f"step, dw={dw}, nf=4, {'relaxed' if variant == 0 else 'fed'}, {threads} groups")
    line = {
        "impl": "reference", "metric": f"fp64 MLUP/s ({KINDS[kind]} {n}^3, {T} steps)",
        "value": value, "unit": "MLUP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded init_state + SURVEY 8(d) remap)",
        "config": workload_config(kind, n, T),
        "cpu_baseline": {"value": value, "unit": "MLUP/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "MLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def e2e_dropin(g, kind: int, n: int, T: int, cfg, reps: int, pinned: bool):
    """The drop-in call girih_gpu_run on host buffers (pageable unless `pinned`): each timed call
    uploads u, v and the coefficients, runs the T steps and downloads u and v."""
    grid = g.GridSpec(n, n, n, 0)
    with g.DeviceState.seeded(kind, grid, 42, remap=True, config=g.GpuConfig(device=cfg.device)) as ds:
        host = ds.download(pinned=pinned)
    walls, h2d, d2h, streamed = [], 0, 0, 0
    for rep in range(reps + 1):
        host.t_current = 0
        pr = g.run(host, T, cfg)
        if rep > 0:  # the first call is the warm-up (device buffers, page-locked bounce blocks)
            walls.append(pr.wall_seconds)
            h2d, d2h, streamed = pr.h2d_bytes, pr.d2h_bytes, pr.streamed
    del host
    g.trim()
    wall = sum(walls) / len(walls)
    return {"value": n ** 3 * T / wall / 1e6, "unit": "MLUP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": wall * 1e3,
            "host_memory": "page-locked (cudaMallocHost)" if pinned else
                           "pageable (numpy, like the reference's std::vector fields)",
            "streamed": bool(streamed),
            "host_ram_gb": round(n ** 3 * 8 * {0: 2, 1: 9, 2: 3, 3: 15}[kind] / 1e9, 1)}


def run_gpu_arm(args, rank: int, world: int, local_rank: int):
    import paper_1510_04995_b200 as g

    kind = KINDS.index(args.stencil)
    n = args.n
    T = args.nt
    # GIRIH_BENCH_SHARED_GPU=1: functional check of the multi-rank path with every rank on
    # cuda:0 and gloo plumbing (tests only; such a run measures nothing and says so)
    shared = os.environ.get("GIRIH_BENCH_SHARED_GPU") == "1"
    dev = 0 if shared else local_rank
    tdev = "cpu" if shared else "cuda"  # device of the small plumbing tensors
    hbm, hbm_src = measured_peaks()
    cfg = g.GpuConfig(tb=args.tb, device=dev, zchunks=args.zchunks, variant=args.variant,
                      chain=args.chain)
    dist = None
    halo = None
    ggrid = g.GridSpec(n, n, n)  # the global grid: fixed for every N (strong scaling)
    if world > 1:
        # z-slabs of the global grid, one per rank/GPU. Halos of R*TB planes: pushed by each
        # pass straight into the neighbour GPUs' memory (CUDA IPC over NVLink, passes ordered by
        # stream memory operations), or exchanged over NCCL after every pass (--halo nccl, and
        # the fallback if IPC is unavailable). torch.distributed is the plumbing for the IPC
        # blobs / NCCL id and the max-over-ranks timing.
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(dev)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        ds = None
        if args.halo == "push":
            try:
                ds = g.DeviceState.slab_seeded(kind, ggrid, 42, True, rank, world, None, cfg)
                blobs = [None] * world
                dist.all_gather_object(blobs, ds.ipc_export())
                ds.ipc_connect(blobs[rank - 1] if rank > 0 else None,
                               blobs[rank + 1] if rank + 1 < world else None)
                ok = torch.ones(1, device=tdev)
            except g.GirihError as e:
                print(f"rank {rank}: IPC halo push unavailable ({e}); using NCCL", file=sys.stderr)
                ok = torch.zeros(1, device=tdev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() < 1 and ds is not None:  # every rank falls back together
                ds.close()
                ds = None
            dist.barrier()
            halo = "push" if ds is not None else None
        if ds is None:
            idt = torch.zeros(128, dtype=torch.uint8, device=tdev)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(g.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nid = bytes(idt.cpu().numpy().tobytes())
            ds = g.DeviceState.slab_seeded(kind, ggrid, 42, True, rank, world, nid, cfg)
            halo = "nccl"
    else:
        ds = g.DeviceState.seeded(kind, ggrid, 42, remap=True, config=cfg)
    tuned = None
    if args.tune:
        if world > 1:
            # a slab handle cannot tune alone (its passes wait on its neighbours; girih_gpu_tune
            # refuses it): rank 0 tunes a single-GPU handle of one slab's size and every rank
            # takes that configuration (broadcast), so all ranks run the same pass sequence
            import torch
            vec = torch.zeros(5, dtype=torch.float64, device=tdev)
            ml, nmeas = 0.0, 0
            if rank == 0:
                sgrid = g.GridSpec(n, n, max(2 * (4 if kind >= 2 else 1) + 1, n // world))
                with g.DeviceState.seeded(kind, sgrid, 42, remap=True,
                                          config=g.GpuConfig(device=dev)) as tds:
                    tcfg, ml, nmeas = tds.tune(max_tb=args.tb if args.tb > 0 else 0)
                g.trim()
                vec[0], vec[1], vec[2], vec[3] = tcfg.tb, tcfg.variant, tcfg.zchunks, tcfg.chain
                vec[4] = tcfg.tile_order
            dist.broadcast(vec, 0)
            tb_, var_, zc_, ch_, to_ = (int(x) for x in vec.cpu().tolist())
            ds.set_config(g.GpuConfig(tb=tb_, variant=var_, zchunks=zc_, chain=ch_, device=dev,
                                      tile_order=to_))
            tuned = {"tb": tb_, "variant": var_, "zchunks": zc_, "chain": ch_, "tile_order": to_,
                     "tuned_on": f"rank 0, single-GPU {n}x{n}x{n // world} (one slab), broadcast",
                     "mlups": ml if rank == 0 else None, "measured": nmeas}
        else:
            tcfg, tml, nmeas = ds.tune(max_tb=args.tb if args.tb > 0 else 0)
            tcfg.device = dev
            ds.set_config(tcfg)
            tuned = {"tb": tcfg.tb, "variant": tcfg.variant, "zchunks": tcfg.zchunks,
                     "chain": tcfg.chain, "tile_order": tcfg.tile_order, "mlups": tml,
                     "measured": nmeas}
    for _ in range(args.warmup):
        ds.step(T)
    if dist is not None:
        import torch
        dist.barrier()
        torch.cuda.synchronize()
    reps = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            reps.append(ds.step(T))
    if dist is not None:
        dist.barrier()
        torch.cuda.synchronize()
    kernel_s = sum(r.kernel_seconds for r in reps)
    if dist is not None:  # device time, max over ranks
        tk = torch.tensor([kernel_s], dtype=torch.float64, device=tdev)
        dist.all_reduce(tk, op=dist.ReduceOp.MAX)
        kernel_s = float(tk.item())
    cells = n ** 3  # the global grid
    lups = cells * T * args.steps
    value = lups / kernel_s / 1e6
    launches = sum(r.n_launches for r in reps)
    passes = sum(r.n_passes for r in reps)
    pass_s = sum(r.pass_seconds for r in reps)
    avg_launch = pass_s / max(1, launches)
    passes_per_launch = passes / max(1, launches)  # > 1 for chained launches (small grids)
    # algorithmic bytes per launch (this rank's slab) / its CUDA-event duration
    local_cells = cells // world
    achieved = local_cells * B1[kind] * passes_per_launch / avg_launch / 1e9
    traffic, traffic_src = ncu_traffic(kind, n) if world == 1 else (None, None)
    r0 = reps[-1]
    ds.close()
    g.trim()

    # ---- e2e: the drop-in C-ABI call on pageable host buffers (H2D + sweep + D2H timed).
    #      N > 1: rank 0 makes the multi-GPU drop-in call over all N GPUs (single process, z-slabs
    #      with peer-store halo pushes) while the other ranks wait ----
    e2e = e2e_pinned = None
    if not args.no_e2e and rank == 0:
        e2e_cfg = g.GpuConfig(tb=r0.tb_used, variant=r0.variant_used if world == 1 else -1,
                              zchunks=args.zchunks, device=0 if world > 1 else dev,
                              ngpus=1 if (world == 1 or shared) else world)
        e2e = e2e_dropin(g, kind, n, T, e2e_cfg, args.e2e_steps, pinned=False)
        if world > 1:
            e2e["note"] = f"rank 0's girih_gpu_run over {e2e_cfg.ngpus} GPU(s)"
        if n <= 512:  # secondary: page-locked caller buffers
            e2e_pinned = e2e_dropin(g, kind, n, T, e2e_cfg, args.e2e_steps, pinned=True)
    if dist is not None:
        dist.barrier()

    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        cpu = cpu_reference_sample(kind, n, args.cpu_target_s, T)

    fp64 = None
    try:
        addmul, dfma = g.fp64_peak(dev)
        ops = DP_OPS[kind] * r0.computed_lups / max(r0.pass_seconds, 1e-12)
        fp64 = {"dp_ops_per_s_achieved": ops, "dp_ops_per_s_peak_measured": addmul,
                "frac": ops / addmul, "dfma_flops_peak_measured": dfma,
                "redundancy": r0.computed_lups / r0.lups}
    except Exception as e:  # noqa: BLE001
        fp64 = {"error": str(e)}

    config = workload_config(kind, n, T)
    line = {
        "metric": f"fp64 MLUP/s ({KINDS[kind]} {n}^3, {T} steps)",
        "value": value, "unit": "MLUP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": kernel_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: device-generated init_state(seed 42) + SURVEY 8(d) remap" +
                 ("; GIRIH_BENCH_SHARED_GPU functional check, all ranks on one GPU: NOT a "
                  "measurement" if shared else "")),
        "config": config,
        "gpu": {"tb": r0.tb_used, "variant": r0.variant_used, "zchunks": r0.zchunks_used,
                "grid_ctas": r0.grid_ctas, "passes_per_step": r0.n_passes,
                "launches_per_step": r0.n_launches, "global_grid": [n, n, n],
                "slab_planes": n // world,
                "parallelism": ((f"z-slabs x{world} of the same global grid (halos of R*TB "
                                 f"planes pushed by each pass into the neighbours' memory over "
                                 f"NVLink, CUDA IPC)" if halo == "push" else
                                 f"z-slabs x{world} (NCCL halo exchange of R*TB planes per pass)")
                                if world > 1 else "single GPU"),
                "tuned": tuned},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "peak_source": hbm_src, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": local_cells * B1[kind] * passes_per_launch,
                     # ncu code balance: measured DRAM bytes per LUP of the profiled launch
                     # (algorithmic: B1 / TB), and its excess over the algorithmic bytes
                     "ncu_bytes_per_lup": (traffic / (local_cells * r0.tb_used * passes_per_launch)
                                           if traffic else None),
                     "traffic_over_algorithmic": (traffic / (local_cells * B1[kind] * passes_per_launch)
                                                  if traffic else None),
                     "avg_launch_ms": avg_launch * 1e3,
                     "lup_roofline_mlups": world * hbm * 1e9 * r0.tb_used / B1[kind] / 1e6,
                     "frac_of_lup_roofline": value / (world * hbm * 1e9 * r0.tb_used / B1[kind] / 1e6),
                     "frac_of_tb1_roofline": value / (world * hbm * 1e9 / B1[kind] / 1e6)},
        "fp64": fp64,
        "clocks": clk.summary(),
        "e2e": e2e,
        "e2e_pinned": e2e_pinned,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="girih", choices=["girih", "reference"])
    ap.add_argument("--stencil", default="var7pt", choices=KINDS)
    ap.add_argument("--n", "--size", dest="n", type=int, default=1024,
                    help="interior extent (cubic grid); use --size under torchrun (--n is an "
                         "ambiguous prefix of its own options)")
    ap.add_argument("--nt", type=int, default=200)
    ap.add_argument("--tb", type=int, default=0)
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--zchunks", type=int, default=0)
    ap.add_argument("--chain", type=int, default=0,
                    help="pass chaining: 0 auto (grids <= 256^3), 1 always, -1 never")
    ap.add_argument("--halo", default="push", choices=["push", "nccl"],
                    help="N > 1: passes push halos into the neighbours' memory (CUDA IPC) or "
                         "exchange them over NCCL after every pass")
    ap.add_argument("--tune", action="store_true", default=True,
                    help="run girih_gpu_tune first and time its choice (default on; N = 1 only)")
    ap.add_argument("--no-tune", dest="tune", action="store_false")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3,
                    help="timed drop-in calls after one warm-up call (mean reported)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-target-s", type=float, default=8.0)
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, rank)
    return run_gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
