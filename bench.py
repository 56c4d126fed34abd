#!/usr/bin/env python
"""Benchmark: sensitivity-map voxels/s end to end (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] = C2 — 2D 256x256, Q=32 coils,
calibration 32x32, ellipsoidal kernel tau=5, nullspace threshold 0.05,
full-resolution G(x), 50 power iterations.  A step is one estimate_maps call
(pisco preset: Gram -> nullspace -> G(x) -> power iteration -> normalise/mask)
on one synthetic, seeded calibration.  C2 is a single slice, so it does not
shard: under torchrun every rank runs an independent replica ("replicas only",
weak scaling) and `value` = all ranks' voxels / max-over-ranks device time.

Legs:
  value     inputs resident in HBM, outputs to HBM buffers, CUDA events on
            the library stream (set to torch's current stream), L2 flushed
            between steps by a 256 MiB write (untimed).
  e2e       the same call through the public C-ABI with pinned HOST buffers:
            calibration H2D + maps/lambda/mask D2H inside the timed region.
  cpu_baseline  the reference's own CPU implementation on rank 0 at N=1, one
            full pipeline: oracle/_ref (the unmodified reference sources
            compiled against oracle/ref_shim, kind "reference"; its own
            std::thread parallel_for, dense algebra single-threaded as the
            reference's Eigen), or the FP64 restatement in oracle/ (kind
            "port") where _ref was not built.
`--impl reference` times the same CPU implementation as the reference arm.

Inputs: every step (warm-up, timed, e2e) gets its own seeded calibration
(phantom.generate_variants: same phantom and coils, a fresh noise draw per
step), so no step re-solves the Gram the previous one saw.
"""
import argparse
import glob
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sensitivity-map voxels/s end-to-end"
UNIT = "voxels/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1234)
    return ap.parse_args()


def workload(spec):
    return (f"{spec.name}: {'x'.join(map(str, spec.full_dims))} Q={spec.channels} calib "
            f"{'x'.join(map(str, spec.calib))} ellipsoid tau={spec.tau} grid {'x'.join(map(str, spec.grid_dims))} "
            f"iters={spec.power_iters} slices={spec.slices}")


def output_voxels(spec):
    return int(np.prod(spec.full_dims)) * spec.slices


def k4_flops(spec):
    n = int(np.prod(spec.grid_dims))
    q = spec.channels
    return n * (spec.power_iters * (8 * q * q + 8 * q) + 8 * q * q + 8 * q)


def stage_work(spec, lam_box, support_size):
    """SURVEY.md §8(d) algorithmic bytes / flops per stage for one slice."""
    q = spec.channels
    h = q * (q + 1) // 2
    e = int(np.prod(spec.calib))
    n_grid = int(np.prod(spec.grid_dims))
    n_full = int(np.prod(spec.full_dims))
    n = q * support_size
    interp = tuple(spec.grid_dims) != tuple(spec.full_dims)
    post = 8 * n_grid * q + 8 * q * e + ((8 * n_full * q + 5 * n_full + 4 * n_grid) if interp else (8 * n_grid * q + 5 * n_grid))
    return {
        "gram": ("hbm", 8 * q * e + 8 * n * n),
        "field": ("hbm", 8 * n_grid * h + 8 * h * lam_box),
        "eigensolve": ("fp32", k4_flops(spec)),
        "post": ("hbm", post),
    }


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            if os.environ.get("SKB_BENCH_CLOCK_MS") == "0":  # experiment: no sampling
                raise RuntimeError("clock sampling disabled")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("SKB_BENCH_CLOCK_MS", "100")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_impl():
    """The reference's CPU implementation: oracle/_ref when it was built (the
    reference itself), else the FP64 restatement.  Returns (module, kind)."""
    from oracle import ref
    if ref.available():
        ref.lib()
        return ref, "reference"
    from oracle import oracle as O
    return O, "port"


def oracle_run(case, threads=None):
    """One full reference-algorithm pipeline on the host (the CPU baseline)."""
    O, _ = cpu_impl()
    spec = case.spec
    if threads:
        O.set_max_threads(threads)
    co = O.PipelineConfig.pisco()
    co.kernel, co.tau, co.power_iters = spec.kernel, spec.tau, spec.power_iters
    co.nullspace_threshold = spec.nullspace_threshold
    if spec.full_grid:
        co.grid = O.GRID_FULL
    else:
        co.grid_pad = spec.grid_dims[0] - spec.calib[0]
    t0 = time.perf_counter()
    for s in range(case.calib.shape[0]):
        res = O.estimate_maps(O.Calib(case.calib[s].astype(np.complex128), case.center_offset), spec.full_dims, co,
                              grid_dims=None if spec.full_grid or spec.ndim < 3 else spec.grid_dims)
    dt = time.perf_counter() - t0
    return dt, res, O.max_threads()


def reference_arm(args, spec, rank, world):
    from paper_2302_13431_b200 import phantom
    if rank != 0:
        return
    # bounded sample: one full pipeline per step (one slice for multislice
    # configs, voxels/s extrapolated); at most 2 steps so the arm ends in minutes
    # (one full pipeline per step, C3: one slice; at most 1 warm-up + 3 timed
    # steps so the arm ends within minutes); each step its own input variant.
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    var = phantom.generate_variants(args.config, warm + steps, seed=args.seed,
                                    slice_range=(0, 1) if spec.slices > 1 else None)
    _, kind = cpu_impl()
    times = []
    threads = None
    for i in range(warm + steps):
        one = phantom.Case(spec, var.calib[i], var.center_offset)
        dt, _, threads = oracle_run(one)
        if i >= warm:
            times.append(dt)
    t = float(np.mean(times))
    vox = output_voxels(spec) // spec.slices
    value = vox / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128 (fp64 complex)", "data": "synthetic (seeded phantom/coil generator, paper_2302_13431_b200/phantom.py)",
        "config": {"workload": workload(spec)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{steps} full {args.config} pipeline(s) ({vox} output voxels each, "
                                   f"{'one slice of ' + str(spec.slices) + ', voxels/s per slice' if spec.slices > 1 else 'whole job'}) "
                                   f"after {warm} warm-up; " + ("oracle/_ref = the reference's own sources" if kind == "reference"
                                                                else "oracle/ FP64 restatement") +
                                   f"; parallel_for on {threads} threads, dense algebra single-threaded as the reference's Eigen"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def zslab_arm(args, spec, rank, world, local, dist):
    """C4 on N GPUs: z-slab sharding (shard.estimate_maps_zslab), strong scaling.

    Every rank expands G(x) and iterates only its slab of the map grid, one
    NCCL all-gather assembles the low-resolution maps, the interpolation is
    split by channel with an all-reduced SoS; each rank keeps its channel block
    of the full-resolution maps (the job's output, distributed)."""
    import torch
    import paper_2302_13431_b200 as K
    from paper_2302_13431_b200 import phantom, shard
    nvar = max(1, min(args.warmup + args.steps, 16))
    case = phantom.generate_variants(args.config, nvar, seed=args.seed)  # the same volumes on every rank
    full = spec.full_dims
    cfg = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, nullspace_threshold=spec.nullspace_threshold,
                           power_iters=spec.power_iters, grid=K.GRID_REDUCED,
                           grid_pad=spec.grid_dims[0] - spec.calib[0], grid_dims=spec.grid_dims)
    ctx = K.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    dev = torch.device("cuda", local)
    d_calibs = [K.Calib(torch.from_numpy(case.calib[v, 0]).to(dev), case.center_offset) for v in range(nvar)]
    ops = shard.DeviceOps(ctx, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    counter = {"i": 0}

    def step():
        v = counter["i"] % nvar
        counter["i"] += 1
        return shard.estimate_maps_zslab(d_calibs[v], full, cfg, ops, gather_maps=False)

    def timed(fn, k, host=False):
        total = 0.0
        for _ in range(k):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if host:
                v = counter["i"] % nvar
                counter["i"] += 1
                cal = K.Calib(torch.from_numpy(case.calib[v, 0]).pin_memory().to(dev, non_blocking=True),
                              case.center_offset)
                maps, lam, mask, _ = shard.estimate_maps_zslab(cal, full, cfg, ops, gather_maps=False)
                maps.cpu(), lam.cpu(), mask.cpu()
            else:
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1)
        t = torch.tensor([total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    l0, lib0 = ctx.launches, ctx.library_calls
    total_ms = timed(step, args.steps)
    launches, libcalls = ctx.launches - l0, ctx.library_calls - lib0
    clk = clocks.stop()
    e2e_steps = max(1, min(args.steps, 3))
    e2e_ms = timed(step, e2e_steps, host=True)
    vox = output_voxels(spec)
    ms = total_ms / args.steps
    q = spec.channels
    own = shard.partition(q, world, rank)
    line = {
        "metric": METRIC, "value": vox / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64 (fp32 complex); Gram eigensolve, lag expansion and final Rayleigh quotient fp64",
        "data": "synthetic (seeded phantom/coil generator, paper_2302_13431_b200/phantom.py)",
        "config": {"workload": workload(spec), "parallelism": f"z-slab x{world} (NCCL all-gather + all-reduce)",
                   "l2": "flushed between steps (256 MiB write, untimed)"},
        "e2e": {"value": vox / (e2e_ms / e2e_steps / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(case.calib[0, 0].size * 8),
                "d2h_bytes_per_step": int((own[1] - own[0]) * int(np.prod(full)) * 8 + int(np.prod(full)) * 5)},
        "gpu_launches": int(launches), "library_calls": int(libcalls), "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2302_13431_b200 import phantom
    spec = phantom.CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, spec, rank, world)
        return

    import torch
    import paper_2302_13431_b200 as K
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2302_13431_b200 import shard
    if spec.ndim == 3 and spec.slices == 1 and world > 1:
        zslab_arm(args, spec, rank, world, local, dist)
        return
    sharded = spec.slices > 1
    nvar = max(1, min(args.warmup + args.steps, 16))  # distinct inputs, cycled if K + W > 16
    if sharded:
        # multislice: contiguous slice blocks per rank, strong scaling
        block = shard.partition(spec.slices, world, rank)
        var = phantom.generate_variants(args.config, nvar, seed=args.seed, slice_range=block)
    else:
        # single slice: independent replicas, weak scaling
        var = phantom.generate_variants(args.config, nvar, seed=args.seed + rank)
    case = phantom.Case(spec, var.calib[0], var.center_offset)
    q = spec.channels
    full = spec.full_dims
    nfull = int(np.prod(full))
    cfg = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, nullspace_threshold=spec.nullspace_threshold,
                           power_iters=spec.power_iters, grid=K.GRID_FULL if spec.full_grid else K.GRID_REDUCED,
                           grid_pad=spec.grid_dims[0] - spec.calib[0],
                           grid_dims=spec.grid_dims if spec.ndim == 3 else None)
    ctx = K.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    slices = case.calib.shape[0]
    d_var = torch.from_numpy(var.calib).to("cuda")  # (nvar, S, Q, *E)
    d_maps = torch.empty((slices, q) + tuple(full), dtype=torch.complex64, device="cuda")
    d_lam = torch.empty((slices,) + tuple(full), dtype=torch.float32, device="cuda")
    d_mask = torch.empty((slices,) + tuple(full), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    cal_stride = d_var[0, 0].numel() * 8
    counter = {"i": 0}

    def step_device(v=None, sequential=False):
        if v is None:
            v = counter["i"] % nvar
            counter["i"] += 1
        base = d_var[v].data_ptr()
        if sharded and not sequential:  # all local slices in one call (concurrent lanes inside the library)
            return K.api.estimate_maps_batched_device(ctx, base, slices, spec.calib, case.center_offset,
                                                      q, full, cfg, d_maps.data_ptr(), d_lam.data_ptr(),
                                                      d_mask.data_ptr())
        provs = []
        for s in range(slices):
            provs.append(K.api.estimate_maps_device(
                ctx, base + s * cal_stride, spec.calib, case.center_offset, q, full, cfg,
                d_maps[s].data_ptr(), d_lam[s].data_ptr(), d_mask[s].data_ptr()))
        return provs

    def timed(fn, k, flush_l2=True):
        total = 0.0
        stages = np.zeros(5)
        for _ in range(k):
            if flush_l2:
                flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            provs = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1)
            for p in provs or []:
                stages += np.array(list(p.stage_ms))
        return total, stages / max(k, 1)

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launches
    lib0 = ctx.library_calls
    total_ms, stages = timed(step_device, args.steps)
    launches = ctx.launches - l0
    libcalls = ctx.library_calls - lib0
    clk = clocks.stop()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    # all ranks' output voxels: sharded -> the whole volume once; replicas -> one volume per rank
    vox = output_voxels(spec) if sharded else output_voxels(spec) * world
    value = vox / (ms_per_step / 1e3)
    stage_note = "per-step device stage times of the timed steps (library CUDA events)"
    if sharded:
        # the batched call runs slices on concurrent lanes, so its per-slice stage
        # times overlap: take the stage split from one sequential (untimed) pass
        timed(lambda: step_device(0, sequential=True), 1, flush_l2=False)  # warm the single-slice path
        _, stages = timed(lambda: step_device(0, sequential=True), 1, flush_l2=False)
        stage_note = ("sum over this rank's slices of one sequential, untimed pass after a warm-up pass (slice by slice; the timed "
                      "batched call overlaps slices on concurrent lanes)")

    # ---- e2e through the public API with pinned host buffers (one slice-sized
    # output buffer reused per slice; every slice's result is read back)
    h_var = torch.from_numpy(var.calib).pin_memory()
    hs = slices if sharded else 1
    h_maps = torch.empty((hs, q) + tuple(full), dtype=torch.complex64).pin_memory()
    h_lam = torch.empty((hs,) + tuple(full), dtype=torch.float32).pin_memory()
    h_mask = torch.empty((hs,) + tuple(full), dtype=torch.uint8).pin_memory()
    hcount = {"i": 0}

    def step_host():
        v = hcount["i"] % nvar
        hcount["i"] += 1
        hcount["last"] = v
        base = h_var[v].data_ptr()
        if sharded:
            return K.api.estimate_maps_batched_device(ctx, base, slices, spec.calib, case.center_offset,
                                                      q, full, cfg, h_maps.data_ptr(), h_lam.data_ptr(),
                                                      h_mask.data_ptr())
        provs = []
        for s in range(slices):
            provs.append(K.api.estimate_maps_device(
                ctx, base + s * cal_stride, spec.calib, case.center_offset, q, full, cfg,
                h_maps.data_ptr(), h_lam.data_ptr(), h_mask.data_ptr()))
        return provs

    step_host()
    e2e_steps = max(3, min(args.steps, 10)) if not sharded else max(1, min(args.steps, 3))
    e2e_ms, _ = timed(step_host, e2e_steps)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = vox / (e2e_ms / e2e_steps / 1e3)
    step_device(hcount["last"])  # the same input through the device leg: the legs must agree
    torch.cuda.synchronize()
    assert np.array_equal(h_mask[hs - 1].numpy(), d_mask[slices - 1].cpu().numpy()), "host/device legs disagree"

    peaks, peak_src = load_peaks()
    props = torch.cuda.get_device_properties(local)
    fp32_peak = props.multi_processor_count * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    k4_ms = stages[3]
    k4_work = k4_flops(spec) * slices
    achieved = k4_work / (k4_ms / 1e3) / 1e12 if k4_ms > 0 else 0.0
    traffic, traffic_src = None, None
    for prof in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")), reverse=True):
        try:
            traffic = json.load(open(prof)).get("power_kernel", {}).get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
        if traffic:
            traffic_src = (f"ncu --set full capture ({os.path.relpath(prof, ROOT)}): dram__bytes_read.sum + "
                           "dram__bytes_write.sum per launch; profile-derived, not measured in this run")
            break

    # per-stage roofline fractions (stage device time from the library's CUDA events)
    sup = K.make_support(spec.kernel, spec.tau, spec.ndim).shape[0]
    lam_box = (4 * spec.tau + 1) ** spec.ndim
    hbm_peak = peaks.get("hbm_gbs", 6552.6)
    stage_roof = {}
    for name, (bound, work) in stage_work(spec, lam_box, sup).items():
        work = work * slices
        ms = float(dict(zip(("gram", "nullspace", "field", "eigensolve", "post"), stages))[name])
        if ms <= 0:
            continue
        if bound == "hbm":
            ach = work / (ms / 1e3) / 1e9
            stage_roof[name] = {"bound": "hbm", "achieved_GBps": round(ach, 1), "frac": round(ach / hbm_peak, 4),
                                "algorithmic_bytes": int(work)}
        else:
            ach = work / (ms / 1e3) / 1e12
            stage_roof[name] = {"bound": "fp32", "achieved_TFLOPs": round(ach, 2), "frac": round(ach / fp32_peak, 4),
                                "algorithmic_flops": int(work)}
    stage_roof["nullspace"] = {"bound": "latency (FP64 subspace eigensolve, cuSOLVER/cuBLAS + own kernels)",
                               "ms": round(float(stages[1]), 3)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "c64 (fp32 complex); Gram eigensolve, lag expansion and final Rayleigh quotient fp64",
        "data": "synthetic (seeded phantom/coil generator, paper_2302_13431_b200/phantom.py)",
        "config": {"workload": workload(spec),
                   "parallelism": (f"slice-sharded x{world}" if sharded else f"replicas x{world}") if world > 1
                   else "single GPU",
                   "l2": "flushed between steps (256 MiB write, untimed)",
                   "inputs": f"{nvar} distinct seeded calibrations (fresh noise per step), cycled",
                   "output_voxels_per_rank": output_voxels(spec) // spec.slices * slices},
        "stages_note": stage_note,
        "stages_ms": dict(zip(("gram", "nullspace", "field", "eigensolve", "post"), [round(x, 4) for x in stages])),
        "stages_roofline": stage_roof,
        "roofline": {"kernel": "power_kernel (K4)", "bound": "fp32", "achieved": achieved, "peak": fp32_peak,
                     "unit": "TFLOP/s", "frac": achieved / fp32_peak if fp32_peak else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": f"SMs x 128 FP32 lanes x 2 x sm_max_mhz ({peak_src} MEASURED_PEAKS sm_max_mhz)",
                     "flops_per_launch": k4_flops(spec)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h_var[0].numel() * 8),
                "d2h_bytes_per_step": int((h_maps.numel() * 8 + h_lam.numel() * 4 + h_mask.numel()) * slices // hs)},
        "gpu_launches": int(launches), "library_calls": int(libcalls),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        one = phantom.Case(spec, case.calib[:1], case.center_offset) if sharded else case
        dt, _, threads = oracle_run(one)
        per = output_voxels(spec) // spec.slices
        line["cpu_baseline"] = {"value": per / dt, "unit": UNIT, "cores": threads, "kind": cpu_impl()[1],
                                "sample": (f"one full {args.config} slice pipeline ({per} voxels, {dt:.1f} s)"
                                           + (f"; voxels/s extrapolated to {spec.slices} slices" if sharded else "")
                                           + "; dense algebra single-threaded as the reference's Eigen")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
