#!/usr/bin/env python
"""SSLIC hot-path benchmark: voxels/sec per SLIC iteration (assign+update).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A step is one SLIC iteration (fused assign+accumulate, allreduce when N>1,
centre update) over the whole synthetic volume of the chosen BASELINE.json
config, already resident in HBM (generated on device by the seeded
counter-based generator). Default workload: config 3 (1024^3 uint16, S=16,
m=10), the largest single-GPU config the metric is quoted on at 1/2/4/8 GPUs
(configs 3-5); the others are parity cases. Inputs (2 GiB image + 4 GiB labels)
are larger than L2, so no flush is needed between iterations.

Under torchrun (N>1) each rank owns a contiguous z-slab; the one exchange per
iteration is an NCCL allreduce of the int64 per-cluster partials. Rank 0
prints ONE JSON line.
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
    # functional check of the N>1 code path on a one-GPU box (gloo, every
    # rank on device 0); never used for reported numbers
    if os.environ.get("SSLIC_BENCH_FUNCTIONAL_CHECK") == "1":
        local = 0
    return world, rank, local


def bytes_per_voxel(ch, dtype):
    return ch * np.dtype(dtype).itemsize + 8  # image once + label read + write


def flops_per_voxel(E, ch, rank):
    return E * (3 * ch + 4 * rank + 2) + (ch + rank)


def cpu_sample(cfg_id, dims, ch, dtype):
    """Bounded CPU sample of the same workload: the first planes of the same
    synthetic volume, treated as their own image."""
    if len(dims) == 2:
        return dims, 2
    planes = {3: 32, 4: 32, 5: 32}[cfg_id]  # >= S (the reference rejects S > dims)
    return (dims[0], dims[1], planes), 1


def run_reference_cpu(cfg_id, steps, warmup, data_host, sdims, ch, grid, m):
    """Times the UNMODIFIED reference's multi-threaded CPU iteration loop
    (oracle/_ref, reference headers) on the bounded sample."""
    import oracle
    ref = oracle.Reference()
    cores = os.cpu_count() or 1
    d = data_host.astype(np.float64)
    _, per_iter = ref.time_iterations(d, sdims, ch, grid, m, warmup + steps, cores)
    t = sum(per_iter[warmup:])
    nvox = int(np.prod(sdims))
    return nvox * steps / t, cores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--path", default="auto", choices=["auto", "exact"])
    ap.add_argument("--no-graph", action="store_true", help="launch steps directly (N=1)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world, rank, local = dist_setup()
    dims, ch, dtype, grid, m, cfg_iters = CONFIGS[args.config]
    nvox = int(np.prod(dims))
    metric = "voxels/sec per SLIC iteration (assign+update)"
    config = {"workload": f"config{args.config}", "dims": list(dims), "channels": ch,
              "dtype": np.dtype(dtype).name, "grid": list(grid), "m": m,
              "parallelism": f"zslab{world}"}
    # working set per step: image + label words (+ tables); B200 L2 = 126 MB
    fits_l2 = nvox * (ch * np.dtype(dtype).itemsize + 4) < 126e6
    config["l2"] = ("fits in L2: 512 MB flush write between timed steps (outside the timed "
                    "spans)" if fits_l2 else "inputs larger than L2 (no flush needed)")

    import torch
    torch.cuda.set_device(local)

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's CPU path on the host cores: bounded sample per step
        import paper_1806_08741_b200 as s
        sdims, _ = cpu_sample(args.config, dims, ch, dtype)
        n_s = int(np.prod(sdims))
        buf = torch.empty(n_s * ch, dtype={np.uint8: torch.uint8, np.uint16: torch.int16,
                                          np.float32: torch.float32}[dtype], device="cuda")
        s.synth_generate(args.config, dims, dtype, ch, SEED, 0, sdims[-1] if len(dims) == 3
                         else 1, buf.data_ptr())
        torch.cuda.synchronize()
        host = buf.cpu().numpy().view(dtype)
        v, cores = run_reference_cpu(args.config, args.steps, args.warmup, host, sdims, ch,
                                     grid, m)
        line = {"metric": metric, "value": v, "unit": "voxel-iter/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": n_s / v * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": dict(config, sample=list(sdims)),
                "cpu_baseline": {"value": v, "unit": "voxel-iter/s", "cores": cores,
                                 "kind": "reference",
                                 "sample": f"first {sdims[-1]} planes ({n_s} voxels) of the "
                                           f"config volume, {args.steps} timed iterations"},
                "e2e": {"value": v, "unit": "voxel-iter/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    if world > 1:
        import torch.distributed as tdist
        if os.environ.get("SSLIC_BENCH_FUNCTIONAL_CHECK") == "1":
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_1806_08741_b200 as s
    from paper_1806_08741_b200.sharded import ShardedLoop, data_bounds, slab_bounds

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
    total_iters = args.warmup + args.steps + 1
    params = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=max(total_iters, 1))
    eng = s.Engine(dims, ch, dtype, img.data_ptr(), params, slab=slab, data_range=drange,
                   device=local, stream=stream.cuda_stream)
    if args.path == "exact":
        eng.set_exact(True)

    def allreduce(t):
        import torch.distributed as tdist
        tdist.all_reduce(t)

    loop = ShardedLoop(eng, allreduce, world)
    loop.init()
    for _ in range(args.warmup):
        loop.iterate()
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    a0 = eng.assign_calls()
    # Inputs larger than L2 (configs 3-5): one event pair around the K steps.
    # Inputs that fit in L2 (configs 1-2): each step timed by its own events
    # with a 512 MB L2-flushing write between steps, outside the timed spans.
    # On one GPU the steps run as CUDA graphs (capture outside the timed
    # span, one launch inside it), which removes the per-kernel launch gaps
    # that dominate the small configs; with NCCL between steps (N > 1) they
    # are launched directly.
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if fits_l2 else None
    graphs = world == 1 and not args.no_graph
    config["launch"] = "CUDA graph per timed span" if graphs else "direct launches"
    if flush is None:
        if graphs:
            ms = eng.iterate_graph(args.steps)
        else:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(args.steps):
                loop.iterate()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
    else:
        ms = 0.0
        evs = []
        for _ in range(args.steps):
            flush.fill_(1)
            if graphs:
                ms += eng.iterate_graph(1)
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            loop.iterate()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms += sum(e0.elapsed_time(e1) for e0, e1 in evs)
        del flush
    if world > 1:
        tdist.barrier()
    clk = clocks.stop()
    launches = eng.launch_count() - launches0
    assign_ms = [eng.assign_ms(i) for i in range(a0, a0 + args.steps)]
    # one extra (untimed) iteration with evaluation statistics for the roofline's E
    eng.set_stats(True)
    loop.iterate()
    evals, window = eng.eval_stats()
    ambiguous, overflow, changed = eng.fast_stats()
    eng.set_stats(False)
    undefined = eng.undefined_count()
    if world > 1:
        t = torch.tensor([ms, evals, window, float(undefined)], dtype=torch.float64,
                         device="cuda")
        mx = t[:1].clone()
        tdist.all_reduce(mx, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(t[1:])
        ms = float(mx.item())
        evals, window, undefined = (float(x) for x in t[1:].tolist())
        am = torch.tensor(assign_ms, dtype=torch.float64, device="cuda")
        tdist.all_reduce(am, op=tdist.ReduceOp.MAX)
        assign_ms = am.tolist()
    value = nvox * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (fused assign+accumulate), per launch
    E = window / nvox
    fpv = flops_per_voxel(E, ch, len(dims))
    bpv = bytes_per_voxel(ch, dtype)
    slab_vox = (slab[1] - slab[0]) * plane
    amean = statistics.mean(assign_ms)
    achieved_tf = slab_vox * fpv / (amean / 1e3) / 1e12
    achieved_gbs = slab_vox * bpv / (amean / 1e3) / 1e9
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    p32 = fp32_peak_tflops(sm_count, max_mhz)
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    t_roof = max(slab_vox * bpv / (hbm * 1e9), slab_vox * fpv / (p32 * 1e12))
    bound = "fp32" if slab_vox * fpv / (p32 * 1e12) >= slab_vox * bpv / (hbm * 1e9) else "hbm"
    traffic = None
    tf = os.path.join(ROOT, "profiles", "assign_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(f"config{args.config}")
    roofline = {
        "bound": bound,
        "achieved": achieved_tf if bound == "fp32" else achieved_gbs,
        "peak": p32 if bound == "fp32" else hbm,
        "unit": "TFLOP/s" if bound == "fp32" else "GB/s",
        "frac": (t_roof / (amean / 1e3)),
        "traffic": traffic,
        "kernel": "assign (fused assign+accumulate)",
        "kernel_ms": amean,
        "kernel_share_of_step": amean * args.steps / ms,
        "algorithmic": {"E_window_evals_per_voxel": E, "flops_per_voxel": fpv,
                        "bytes_per_voxel": bpv, "evals_performed_per_voxel": evals / nvox,
                        "fp64_redecided_voxel_frac": ambiguous / nvox,
                        "crowded_ctas": overflow,
                        "label_changed_voxel_frac_last_iter": changed / nvox},
        "hbm_gbs": achieved_gbs, "hbm_peak_gbs": hbm, "hbm_frac": achieved_gbs / hbm,
        "peak_source": f"FP32 = {sm_count} SMs x 128 x 2 x {max_mhz:.0f} MHz "
                       f"(no measured FP32 peak); HBM = MEASURED_PEAKS.json hbm_gbs",
    }

    # end-to-end through the reference-facing C ABI with HOST buffers
    e2e = None
    if not args.no_e2e and world > 1:
        # N GPUs: the public multi-GPU API end to end on every rank — H2D of
        # the rank's slab (+ halo) from pinned host memory, engine setup,
        # init + all iterations with the NCCL allreduce, D2H of the slab's
        # labels; wall time between barriers, max over ranks.
        import torch.distributed as tdist
        host = torch.empty(img.numel(), dtype=tdt, pin_memory=True)
        host.copy_(img)
        slab_vox_e = (slab[1] - slab[0]) * plane
        labels_h = torch.empty(slab_vox_e, dtype=torch.int32, pin_memory=True)
        del eng
        torch.cuda.synchronize()
        tdist.barrier()
        t0 = time.perf_counter()
        img2 = torch.empty_like(img)
        img2.copy_(host, non_blocking=True)
        p2 = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=cfg_iters)
        eng2 = s.Engine(dims, ch, dtype, img2.data_ptr(), p2, slab=slab, data_range=drange,
                        device=local, stream=stream.cuda_stream)
        loop2 = ShardedLoop(eng2, allreduce, world)
        loop2.init()
        for _ in range(cfg_iters):
            loop2.iterate()
        lab_d = torch.empty(slab_vox_e, dtype=torch.int32, device="cuda")
        eng2.labels_to(lab_d.data_ptr())
        labels_h.copy_(lab_d)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        tdist.all_reduce(dt, op=tdist.ReduceOp.MAX)
        sec = float(dt.item())
        e2e = {"value": nvox * cfg_iters / sec, "unit": "voxel-iter/s",
               "h2d_bytes_per_step": img.numel() * img.element_size(),
               "d2h_bytes_per_step": slab_vox_e * 4,
               "call": "Engine + ShardedLoop per rank (host buffers, pinned), NCCL allreduce",
               "iterations": cfg_iters, "seconds_per_call": sec, "timed_calls": 1,
               "note": "bytes are per rank"}
        eng2.close()
    if not args.no_e2e and world == 1:
        host = torch.empty(img.numel(), dtype=tdt, pin_memory=True)
        host.copy_(img)
        labels_h = torch.empty(nvox, dtype=torch.int32, pin_memory=True)
        del eng
        torch.cuda.synchronize()
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
        # mean of `reps` timed calls; each call is a whole run (H2D, init,
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
               "h2d_bytes_per_step": img.numel() * img.element_size(),
               "d2h_bytes_per_step": nvox * 4 + cen.nbytes + res.nbytes,
               "call": "sslic_run_slic (host buffers, pinned)", "iterations": done.value,
               "seconds_per_call": sec, "timed_calls": reps, "warmup_calls": 1,
               "statistic": "median over timed calls",
               "seconds_min_max": [min(per_call), max(per_call)]}

    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            sdims, reps = cpu_sample(args.config, dims, ch, dtype)
            n_s = int(np.prod(sdims))
            hs = (img[: n_s * ch] if len(dims) == 3 else img).cpu().numpy().view(dtype)
            v, cores = run_reference_cpu(args.config, reps, 1, hs, sdims, ch, grid, m)
            cpu = {"value": v, "unit": "voxel-iter/s", "cores": cores, "kind": "reference",
                   "sample": f"first {sdims[-1] if len(dims) == 3 else dims[-1]} planes "
                             f"({n_s} voxels) of the same synthetic volume, {reps} timed "
                             f"iteration(s) after 1 warm-up, reference headers -O3, "
                             f"{cores} threads"}
        except Exception as exc:  # the baseline is reported, not required
            cpu = {"value": None, "error": str(exc)[:200]}

    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "voxel-iter/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64" if args.path == "exact" else "f32 filter + f64 exact", "data": "synthetic (seeded device generator)",
                "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "undefined_labels": undefined}
        print(json.dumps(line))
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
