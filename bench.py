#!/usr/bin/env python
"""SSLIC hot-path benchmark: voxels/sec per SLIC iteration (assign+update).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A step is one SLIC iteration (fused assign+accumulate, allreduce when N>1,
centre update) over the whole synthetic volume of the chosen BASELINE.json
config, already resident in HBM (generated on device by the seeded
counter-based generator). Default workload: config 3 (1024^3 uint16, S=16,
m=10, 10 iterations), the largest single-GPU config the metric is quoted on
at 1/2/4/8 GPUs (configs 3-5); the others are parity cases.

Iteration window: the steps are the CONFIGURED iterations of whole runs. Step
j is iteration j mod I of run j div I (I = the config's iteration count); each
run starts from a fresh init + perturbation (outside the timed spans), so
K = 20 times iterations 0..9 exactly twice. The warm-up steps are a separate
untimed run. Inputs (2 GiB image + 4 GiB labels for config 3) exceed L2; the
L2-resident configs 1-2 flush L2 with a 512 MB write between steps.

Under torchrun (N>1) each rank owns a contiguous z-slab; the one exchange per
iteration is an NCCL allreduce of the int64 per-cluster partials, issued by
the library on the engine's own communicator (sslic_engine_attach_nccl) and
captured with the kernels in each timed span's CUDA graph; torch.distributed
only carries the NCCL unique id, the barriers and the max-over-ranks timing.
e2e at N>1 is sslic_run_slic_rank per rank on pinned host planes. Rank 0
prints ONE JSON line. --nccl runs those N>1 code paths at N=1.

--impl reference times the UNMODIFIED reference's multi-threaded CPU loop
(oracle/_ref: the reference headers compiled by oracle/Makefile) on the
host cores, over the same iteration window, on a bounded sample of the same
synthetic volume produced by the CPU twin of the device generator
(oracle/synth_ref.c). That arm never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: dims, channels, dtype, grid, m, iterations
    1: ((512, 512), 3, np.uint8, (16, 16), 10.0, 10),
    2: ((2048, 1216), 3, np.float32, (32, 32), 10.0, 10),
    3: ((1024, 1024, 1024), 1, np.uint16, (16, 16, 16), 10.0, 10),
    4: ((512, 512, 256), 4, np.float32, (8, 8, 8), 20.0, 10),
    5: ((2048, 1216, 7000), 3, np.uint8, (32, 32, 32), 10.0, 5),
}
SEED = 0x1806_08741
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# CPU runs of the reference. The reference arm runs the whole config volume
# (config 5's 17.4 G voxels need ~630 GB of fp64 host state, so it takes a
# 512-plane z-range); the GPU arm's cpu_baseline leg takes a bounded sample of
# ~10-30 s. Samples are planes [z0, z1) of the same volume treated as their
# own image: whole multiples of S from the middle, with at least as many
# S-plane slabs (the reference's unit of parallel work, parallel.hpp:31-50)
# as host threads where the time allows.
REF_SAMPLE = {5: (3328, 3840)}
BASE_SAMPLE = {3: (256, 768), 5: (3456, 3712)}
METRIC = "voxels/sec per SLIC iteration (assign+update)"


def fp32_peak_tflops(sm_count: int, mhz: float) -> float:
    """SMs x 128 FP32 lanes x 2 (FMA) x clock."""
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


class Clocks:
    """nvidia-smi sampler run around the timed region (B200_PROFILING.md)."""

    def __init__(self, device: int):
        self.device, self.samples, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, smax = [], None
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax = float(s[1])
            except ValueError:
                continue
            for n, v in zip(names, s[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def bytes_per_voxel(ch, dtype):
    return ch * np.dtype(dtype).itemsize + 8  # image once + label read + write


def flops_per_voxel(E, ch, rank):
    return E * (3 * ch + 4 * rank + 2) + (ch + rank)


def host_cores():
    """(logical, physical) host cores; physical = distinct (package, core id)
    pairs of /proc/cpuinfo (the acceptance.cpp:44-58 method)."""
    logical = os.cpu_count() or 1
    pairs, phys, core = set(), None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    phys = line.split(":")[1].strip()
                elif line.startswith("core id"):
                    core = line.split(":")[1].strip()
                elif not line.strip():
                    if core is not None:
                        pairs.add((phys, core))
                    phys = core = None
    except OSError:
        pass
    return logical, (len(pairs) or logical)


def cpu_sample(cfg_id, dims, table):
    """A CPU sample of the config volume: (sample dims, z0, z1)."""
    if cfg_id in table:
        z0, z1 = table[cfg_id]
        return (dims[0], dims[1], z1 - z0), z0, z1
    return tuple(dims), 0, (dims[-1] if len(dims) == 3 else 1)


def window(steps, iters):
    """Iteration indices of `steps` consecutive steps cycling whole runs."""
    return [j % iters for j in range(steps)]


def reference_window_rate(cfg_id, steps, warmup, workers, table):
    """The unmodified reference (oracle/_ref) over the configured-iteration
    window on the bounded sample: one warm-up run of `warmup` iterations,
    then whole runs whose first `steps` iterations (cycling) are timed.
    Returns (voxel-iter/s, sample description)."""
    import oracle
    dims, ch, dtype, grid, m, iters = CONFIGS[cfg_id]
    sdims, z0, z1 = cpu_sample(cfg_id, dims, table)
    t0 = time.perf_counter()
    data = oracle.Oracle().synth_generate(cfg_id, dims, dtype, ch, SEED, z0, z1)
    gen_s = time.perf_counter() - t0
    d = data.astype(np.float64)
    ref = oracle.Reference()
    if warmup > 0:
        ref.time_iterations(d, sdims, ch, grid, m, min(warmup, iters), workers)
    per_iter = []
    left = steps
    while left > 0:
        n = min(iters, left)
        _, t = ref.time_iterations(d, sdims, ch, grid, m, n, workers)
        per_iter += t
        left -= n
    nvox = int(np.prod(sdims))
    rate = nvox * steps / sum(per_iter)
    where = (f"planes [{z0},{z1}) of the config volume ({'x'.join(map(str, sdims))}, "
             f"{nvox} voxels) as their own image" if cfg_id in table
             else f"the whole config volume ({nvox} voxels)")
    desc = (f"{where}; iterations {window(steps, iters)[:iters]} of whole runs "
            f"({steps} timed after {warmup} warm-up), reference headers -O3 "
            f"-ffp-contract=off, {workers} threads; CPU generator {gen_s:.1f} s (untimed)")
    return rate, desc, per_iter


def run_reference_arm(args, config):
    logical, physical = host_cores()
    rate, desc, per_iter = reference_window_rate(args.config, args.steps, args.warmup, logical,
                                                 REF_SAMPLE)
    dims = CONFIGS[args.config][0]
    sdims, _, _ = cpu_sample(args.config, dims, REF_SAMPLE)
    line = {"metric": METRIC, "value": rate, "unit": "voxel-iter/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": int(np.prod(sdims)) / rate * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; CPU twin of the device generator)",
            "impl": "reference", "config": config,
            "cpu_baseline": {"value": rate, "unit": "voxel-iter/s", "cores": logical,
                             "physical_cores": physical, "kind": "reference", "sample": desc},
            "e2e": {"value": rate, "unit": "voxel-iter/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_ms_per_iteration": [t * 1e3 for t in per_iter]}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--path", default="auto", choices=["auto", "exact"])
    ap.add_argument("--no-graph", action="store_true", help="launch steps directly")
    ap.add_argument("--nccl", action="store_true",
                    help="run the N>1 code paths (engine NCCL communicator, run_slic_rank e2e) "
                         "even at N=1 (functional check on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world, rank, local = dist_setup()
    dims, ch, dtype, grid, m, cfg_iters = CONFIGS[args.config]
    nvox = int(np.prod(dims))
    config = {"workload": f"config{args.config}", "dims": list(dims), "channels": ch,
              "dtype": np.dtype(dtype).name, "grid": list(grid), "m": m,
              "iterations": cfg_iters, "parallelism": f"zslab{world}"}
    # working set per step: image + label words (+ tables); B200 L2 = 126 MB
    fits_l2 = nvox * (ch * np.dtype(dtype).itemsize + 4) < 126e6
    config["l2"] = ("fits in L2: 512 MB flush write between timed steps (outside the timed "
                    "spans)" if fits_l2 else "inputs larger than L2 (no flush needed)")
    config["window"] = (f"configured iterations 0..{cfg_iters - 1} of whole runs, cycled; "
                        "init + perturbation outside the timed spans")

    if args.impl == "reference":
        # the reference's CPU path on the host cores; rank 0 only, no GPU, and
        # nothing from the product package is imported
        if rank == 0:
            run_reference_arm(args, config)
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_1806_08741_b200 as s
    from paper_1806_08741_b200.sharded import data_bounds, slab_bounds

    last = dims[-1]
    slab = slab_bounds(last, world, rank, align=grid[-1]) if len(dims) == 3 else (0, last)
    drange = data_bounds(last, slab) if len(dims) == 3 else (0, last)
    plane = nvox // last
    # uint16 volumes live in int16 storage (same bytes; the engine reads uint16)
    tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
    img = torch.empty((drange[1] - drange[0]) * plane * ch, dtype=tdt, device="cuda")
    # a dedicated (non-legacy) stream: CUDA graph capture needs one
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if len(dims) == 3:
        s.synth_generate(args.config, dims, dtype, ch, SEED, drange[0], drange[1],
                         img.data_ptr(), stream.cuda_stream)
    else:
        s.synth_generate(args.config, dims, dtype, ch, SEED, 0, 1, img.data_ptr(),
                         stream.cuda_stream)
    params = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=cfg_iters)
    eng = s.Engine(dims, ch, dtype, img.data_ptr(), params, slab=slab, data_range=drange,
                   device=local, stream=stream.cuda_stream)
    if args.path == "exact":
        eng.set_exact(True)
    uid = None
    multi = world > 1 or args.nccl
    if multi:
        # the engine's own NCCL communicator: the value-range MAX, the init
        # table SUM and the per-iteration SUM of the int64 partials run on the
        # engine stream (inside the captured graph); torch.distributed only
        # carries the unique id and the barriers
        obj = [s.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            tdist.broadcast_object_list(obj, src=0)
        uid = obj[0]
        eng.attach_nccl(uid, rank, world)

    def fresh_run():
        eng.reset()
        eng.start()

    # warm-up: an untimed run of W iterations (cycling when W > I)
    for j in range(args.warmup):
        if j % cfg_iters == 0:
            fresh_run()
        eng.iterate(1)

    graphs = not args.no_graph
    config["launch"] = "CUDA graph per timed span" if graphs else "direct launches"
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if fits_l2 else None
    # timed spans: one per run (inputs > L2) or one per step (L2-resident)
    runs = []
    j = 0
    while j < args.steps:
        n = min(cfg_iters, args.steps - j)
        runs.append(n)
        j += n
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    ms = 0.0
    assign_idx = []  # (assign launch index, iteration index)
    for n in runs:
        fresh_run()  # untimed
        spans = [n] if flush is None else [1] * n
        it = 0
        for span in spans:
            if flush is not None:
                flush.fill_(1)
            a0 = eng.assign_calls()
            if graphs:
                ms += eng.iterate_graph(span)
            else:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                eng.iterate(span)
                e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
            assign_idx += [(a0 + i, it + i) for i in range(span)]
            it += span
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    clk = clocks.stop()
    launches = eng.launch_count() - launches0
    del flush
    assign_ms = [eng.assign_ms(i) for i, _ in assign_idx]

    # untimed statistics run: evaluations and window volume per iteration
    E_it, evals_it, amb_it, chg_it = [], [], [], []
    fresh_run()
    eng.set_stats(True)
    for i in range(cfg_iters):
        eng.iterate(1)
        ev, win = eng.eval_stats()
        amb, _ovf, chg = eng.fast_stats()
        E_it.append(win / nvox if world == 1 else win)
        evals_it.append(ev)
        amb_it.append(amb)
        chg_it.append(chg)
    eng.set_stats(False)
    undefined = eng.undefined_count()
    if world > 1:
        t = torch.tensor([ms] + assign_ms, dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, assign_ms = float(t[0].item()), t[1:].tolist()
        w = torch.tensor(E_it + evals_it + [float(undefined)], dtype=torch.float64,
                         device="cuda")
        tdist.all_reduce(w)
        vals = w.tolist()
        E_it = [v / nvox for v in vals[:cfg_iters]]
        evals_it = vals[cfg_iters:2 * cfg_iters]
        undefined = vals[-1]
    value = nvox * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (fused assign+accumulate), per launch:
    # algorithmic flops F(E_i) of the iteration each launch ran
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    p32 = fp32_peak_tflops(sm_count, max_mhz)
    hbm = float(peaks.get("hbm_gbs", 6550.0))
    bpv = bytes_per_voxel(ch, dtype)
    slab_vox = (slab[1] - slab[0]) * plane
    flops = [slab_vox * flops_per_voxel(E_it[it], ch, len(dims)) for _, it in assign_idx]
    kernel_s = sum(assign_ms) / 1e3
    t_roof = sum(max(f / (p32 * 1e12), slab_vox * bpv / (hbm * 1e9)) for f in flops)
    fp32_bound = sum(f / (p32 * 1e12) for f in flops) >= len(flops) * slab_vox * bpv / (hbm * 1e9)
    achieved_tf = sum(flops) / kernel_s / 1e12
    achieved_gbs = slab_vox * bpv * len(flops) / kernel_s / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "assign_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(f"config{args.config}")
    E_mean = statistics.mean(E_it[it] for _, it in assign_idx)
    roofline = {
        "bound": "fp32" if fp32_bound else "hbm",
        "achieved": achieved_tf if fp32_bound else achieved_gbs,
        "peak": p32 if fp32_bound else hbm,
        "unit": "TFLOP/s" if fp32_bound else "GB/s",
        "frac": t_roof / kernel_s,
        "traffic": traffic,
        "kernel": "assign (fused assign+accumulate)",
        "kernel_ms": kernel_s * 1e3 / len(flops),
        "kernel_ms_per_iteration": [statistics.mean(a for a, (_, it) in zip(assign_ms, assign_idx)
                                                    if it == i) for i in range(min(cfg_iters,
                                                                                    args.steps))],
        "kernel_share_of_step": kernel_s * 1e3 / ms,
        "algorithmic": {"E_window_evals_per_voxel_mean": E_mean,
                        "E_per_iteration": E_it,
                        "flops_per_voxel_mean": flops_per_voxel(E_mean, ch, len(dims)),
                        "bytes_per_voxel": bpv,
                        "evals_performed_per_voxel": [e / nvox for e in evals_it],
                        "fp64_redecided_voxel_frac": [a / nvox for a in amb_it],
                        "label_changed_voxel_frac": [c / nvox for c in chg_it]},
        "hbm_gbs": achieved_gbs, "hbm_peak_gbs": hbm, "hbm_frac": achieved_gbs / hbm,
        "peak_source": f"FP32 = {sm_count} SMs x 128 x 2 x {max_mhz:.0f} MHz "
                       f"(no measured FP32 peak); HBM = MEASURED_PEAKS.json hbm_gbs",
    }

    # end-to-end through the reference-facing C ABI with HOST buffers
    e2e = None
    if not args.no_e2e and multi:
        # N GPUs: the public multi-GPU entry point end to end on every rank
        # (sslic_run_slic_rank): H2D of the rank's planes (slab + halo) from
        # pinned host memory, engine setup, a fresh NCCL communicator, init +
        # every iteration with the allreduce, D2H of the slab's labels and the
        # centres; one warm-up call, then one timed call between barriers,
        # max over ranks.
        host = torch.empty(img.numel(), dtype=tdt, pin_memory=True)
        host.copy_(img)
        img_numel, img_esize = img.numel(), img.element_size()
        del img  # the call uploads its own copy
        slab_vox_e = (slab[1] - slab[0]) * plane
        labels_h = torch.empty(slab_vox_e, dtype=torch.int32, pin_memory=True)
        eng.close()
        del eng
        torch.cuda.synchronize()
        hp = (dims, host.data_ptr(), drange[0], ch, dtype)

        o = [s.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            tdist.broadcast_object_list(o, src=0)

        def call():  # (the communicator of this id is cached after the warm-up call)
            return s.run_slic_rank(None, params, rank, world, o[0], device=local,
                                   labels_out=labels_h, host_planes=hp)
        call()
        if world > 1:
            tdist.barrier()
        t0 = time.perf_counter()
        _, cen_e, _ = call()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            tdist.all_reduce(dt, op=tdist.ReduceOp.MAX)
        sec = float(dt.item())
        e2e = {"value": nvox * cfg_iters / sec, "unit": "voxel-iter/s",
               "h2d_bytes_per_step": img_numel * img_esize,
               "d2h_bytes_per_step": slab_vox_e * 4 + cen_e.data.nbytes,
               "call": "sslic_run_slic_rank per rank (pinned host planes; the NCCL "
                       "communicator, cached per unique id, was set up by the warm-up call)",
               "iterations": cfg_iters, "seconds_per_call": sec, "timed_calls": 1,
               "warmup_calls": 1, "note": "bytes are per rank"}
    if not args.no_e2e and not multi:
        host = torch.empty(img.numel(), dtype=tdt, pin_memory=True)
        host.copy_(img)
        img_numel, img_esize = img.numel(), img.element_size()
        labels_h = torch.empty(nvox, dtype=torch.int32, pin_memory=True)
        eng.close()
        del eng, img  # the call uploads its own copy
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        import ctypes as C
        L = s.lib()
        desc = s._Image()
        desc.rank = len(dims)
        for a in range(4):
            desc.dims[a] = dims[a] if a < len(dims) else 1
        desc.channels = ch
        desc.dtype = s._DT[np.dtype(dtype)]
        desc.data = host.data_ptr()
        p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=cfg_iters)._c()
        k = s.cluster_count(dims, grid)
        cen = np.empty(k * (ch + len(dims)))
        res = np.empty(cfg_iters)
        done = C.c_int()

        def call():
            return L.sslic_run_slic(C.byref(desc), C.byref(p), local,
                                    C.cast(C.c_void_p(labels_h.data_ptr()), C.POINTER(C.c_uint32)),
                                    cen.ctypes.data_as(C.POINTER(C.c_double)),
                                    res.ctypes.data_as(C.POINTER(C.c_double)), C.byref(done))
        # one untimed call (lazy module loading, allocator growth), then the
        # median of `reps` timed calls; each call is a whole run (H2D, init,
        # every iteration, D2H of labels/centres/residuals)
        s._check(call())
        reps = 3 if nvox > (1 << 28) else 9
        per_call = []
        for _ in range(reps):
            t0 = time.perf_counter()
            s._check(call())
            per_call.append(time.perf_counter() - t0)
        sec = statistics.median(per_call)
        e2e = {"value": nvox * done.value / sec, "unit": "voxel-iter/s",
               "h2d_bytes_per_step": img_numel * img_esize,
               "d2h_bytes_per_step": nvox * 4 + cen.nbytes + res.nbytes,
               "call": "sslic_run_slic (host buffers, pinned)", "iterations": done.value,
               "seconds_per_call": sec, "timed_calls": reps, "warmup_calls": 1,
               "statistic": "median over timed calls",
               "seconds_min_max": [min(per_call), max(per_call)],
               "note": "a step here is one whole call (all configured iterations)"}

    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            logical, physical = host_cores()
            rate, desc, _ = reference_window_rate(args.config, cfg_iters, 0, logical,
                                                  BASE_SAMPLE)
            cpu = {"value": rate, "unit": "voxel-iter/s", "cores": logical,
                   "physical_cores": physical, "kind": "reference", "sample": desc}
        except Exception as exc:  # the baseline is reported, not required
            cpu = {"value": None, "error": str(exc)[:200]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "voxel-iter/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64" if args.path == "exact" else "f32 filter + f64 exact",
                "data": "synthetic (seeded device generator)",
                "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "undefined_labels": undefined}
        print(json.dumps(line))
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
