#!/usr/bin/env python
"""OD²P benchmark: frames*iterations/s of the nonblind iteration on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A "step" is one OD²P iteration (solver.cpp:118-205) over the whole
configuration.  Default workload: BASELINE config 4 (8192^2 object, 128^2
probe, step 32, 64009 frames, 8 row-strip subdomains, complex64), the
strong-scaling configuration; its 4.2 GB of amplitudes and 8.4 GB of Gamma
exceed the 126 MB L2, so no flush is needed between iterations.

Multi-GPU (torchrun): subdomain d runs on rank floor(d*N/D); overlap strips
move with NCCL send/recv inside the iteration graph; total work is fixed
("scaling": "strong").  One JSON line is printed by rank 0.

Keys beyond the driver contract:
  roofline      frame kernel (K1) bytes/launch over its CUDA-event duration
  iter_roofline compulsory bytes per iteration over the
                iteration time
  cpu_baseline  the reference CPU path (oracle/_ref, built from the unmodified
                reference sources + our FFTW-API shim) on a bounded sample
  e2e           a full solve through the C-ABI from pinned host buffers
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world):
    if world <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def bcast_obj(dist, obj, rank):
    if dist is None:
        return obj
    lst = [obj if rank == 0 else None]
    dist.broadcast_object_list(lst, src=0)
    return lst[0]


def fresh_nccl_id(dist, rank, world):
    """A new NCCL unique id from rank 0 for each communicator (an id's bootstrap
    root serves a single ncclCommInitRank round), or None on one GPU."""
    from paper_2011_00162_b200 import dist as pdist

    return pdist.new_nccl_id(pdist.DistContext(rank, world, 0, None, dist))

def allmax(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- reference arm
def reference_sample(cfg):
    """Bounded, same-workload sample for the reference CPU path: the config's
    geometry (s, step, probe, noise) cropped to a band of scan rows, split into
    row strips so the reference can use up to 8 worker threads (it runs one
    thread per subdomain, solver.cpp:122)."""
    from paper_2011_00162_b200 import sim

    ncpu = os.cpu_count() or 1
    D = max(1, min(8, ncpu))
    rows_per = 2 if cfg.s >= 128 else 4
    nrows = D * rows_per
    H = (nrows - 1) * cfg.step + cfg.s
    W = min(cfg.N, 8192)
    if cfg.s < 128:
        W = cfg.N
    gr = nrows
    gc = (W - cfg.s) // cfg.step + 1
    probe = sim.make_probe(cfg.s, cfg.sigma_probe)
    rng_a = np.random.default_rng(cfg.seeds[0])
    rng_p = np.random.default_rng(cfg.seeds[1])
    amp = sim._rescale(sim.gaussian_blur_periodic(rng_a.random((H, W)), cfg.sigma_obj), 0.5, 1.0)
    ph = sim._rescale(sim.gaussian_blur_periodic(rng_p.random((H, W)), cfg.sigma_obj), -math.pi / 4, math.pi / 4)
    obj = amp * np.exp(1j * ph)
    ii, jj = np.meshgrid(np.arange(gr), np.arange(gc), indexing="ij")
    pos = np.stack([ii.ravel() * cfg.step, jj.ravel() * cfg.step], 1).astype(np.int64)
    a = np.arange(cfg.s)
    patches = obj[pos[:, 0, None, None] + a[None, :, None], pos[:, 1, None, None] + a[None, None, :]]
    f = np.abs(np.fft.fft2(patches * probe, norm="ortho")) ** 2
    if cfg.peak:
        f = sim.poisson_host(f, cfg.peak, cfg.seeds[2])
    f = np.sqrt(f).astype(np.float32).astype(np.float64) ** 2  # the GPU's fp32 amplitudes
    return {"H": H, "W": W, "D": D, "axis": "rows", "frames": int(pos.shape[0]), "probe": probe, "f": f}


def run_reference(cfg, iters: int, warmup: int):
    """Times the reference's own CPU solver (oracle/_ref) on the bounded sample."""
    from oracle import ref_lib

    smp = reference_sample(cfg)
    if cfg.blind and ref_lib.available():  # BlindSolver::run (blind.cpp:298-358), disk w0 as configured
        from paper_2011_00162_b200 import sim

        ps = ref_lib.plan_spec(smp["H"], smp["W"], cfg.s, cfg.step, smp["D"], smp["axis"])
        bc = ref_lib.blind_cfg(max_iters=iters + warmup, tol_rf=1e-300, threads=0, **cfg.solver)
        w0 = sim.disk_probe(cfg.s, cfg.init_disk_radius) if cfg.init_disk_radius else None
        out = ref_lib.blind_run(ps, smp["f"], bc, w0=w0)
        t = out["records"][warmup:, 3]
        value = smp["frames"] * len(t) / (float(np.sum(t)) / 1e3)
        sample = (f"{cfg.name} geometry (s={cfg.s}, step={cfg.step}) cropped to {smp['H']}x{smp['W']} "
                  f"({smp['frames']} frames), {smp['D']} row-strip subdomains (the reference has no 2-D plans), "
                  f"blind, {len(t)} timed iterations; FFT = oracle/fftw_shim (radix-2, not FFTW)")
        return value, "reference", smp["D"], sample, float(np.mean(t))
    if ref_lib.available():
        ps = ref_lib.plan_spec(smp["H"], smp["W"], cfg.s, cfg.step, smp["D"], smp["axis"])
        rcfg = ref_lib.nonblind_cfg(max_iters=iters + warmup, tol_rf=1e-300, threads=0)
        out = ref_lib.nonblind_run(ps, smp["f"], smp["probe"], rcfg)
        t = out["records"][warmup:, 3]
        kind, cores = "reference", smp["D"]
    else:  # numpy restatement of the reference (single thread)
        from oracle import od2p as O

        g = O.make_raster_scan(smp["H"], smp["W"], cfg.s, cfg.step)
        plan = O.plan_stripes(g, smp["D"], "rows")
        sol = O.NonblindSolver(plan, smp["f"], smp["probe"], O.NonblindConfig(max_iters=iters + warmup,
                                                                               tol_rf=1e-300))
        st = sol.init_state()
        au = [z.copy() for z in st.z]
        t = []
        for k in range(iters + warmup):
            t0 = time.perf_counter()
            sol.step(st, au)
            if k >= warmup:
                t.append((time.perf_counter() - t0) * 1e3)
        t = np.array(t)
        kind, cores = "port", 1
    value = smp["frames"] * len(t) / (float(np.sum(t)) / 1e3)
    sample = (f"{cfg.name} geometry (s={cfg.s}, step={cfg.step}) cropped to {smp['H']}x{smp['W']} "
              f"({smp['frames']} frames), {smp['D']} row-strip subdomains, {len(t)} timed iterations; "
              f"FFT = oracle/fftw_shim (radix-2, not FFTW)")
    return value, kind, cores, sample, float(np.mean(t))


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world, local = dist_env()

    from paper_2011_00162_b200 import sim

    cfg = sim.CONFIGS[args.config]
    metric = "OD2P frames*iterations/s"
    base = {"metric": metric, "unit": "frames*iterations/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None, "data": "synthetic"}

    if args.impl == "reference":
        if rank != 0:
            return
        iters, warm = max(1, min(args.steps, 10)), max(1, min(args.warmup, 2))
        value, kind, cores, sample, ms = run_reference(cfg, iters, warm)
        line = dict(base, impl="reference", value=value, ms_per_step=ms, scaling="none", dtype="f64",
                    config={"workload": f"BASELINE config {args.config} ({cfg.name}), bounded CPU sample",
                            "sample": sample},
                    cpu_baseline={"value": value, "unit": base["unit"], "cores": cores, "kind": kind,
                                  "sample": sample},
                    e2e={"value": value, "unit": base["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    dist = init_dist(world)
    import paper_2011_00162_b200 as P
    from paper_2011_00162_b200 import _lib as L

    if cfg.blind:
        return bench_blind(args, cfg, base, rank, world, local, dist)
    inp = sim.make_inputs(cfg, device=True)
    plan, probe, amp = inp["plan"], inp["probe"], inp["amplitudes_dev"]
    J, s = plan.geometry.frame_count(), cfg.s
    nccl_id = fresh_nccl_id(dist, rank, world)
    ncfg = P.NonblindConfig(max_iters=max(cfg.iterations, args.steps + args.warmup + 8), tol_rf=1e-300)
    solver = P.NonblindSolver(plan, None, probe, ncfg, amplitudes=amp, dtype=cfg.dtype, device=local, rank=rank,
                              world=world, nccl_id=nccl_id)
    import ctypes as C

    def timed(n):
        ms = C.c_double()
        L.check(L.lib().pdd_nonblind_iterate_timed(solver._h, C.c_int32(n), C.byref(ms)))
        return ms.value

    timed(args.warmup)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms_total = timed(args.steps)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = allmax(dist, ms_total)
    value = J * args.steps / (ms_total / 1e3)
    ms_step = ms_total / args.steps

    # kernel accounting (eager iterations with events on the solver stream)
    prof = (C.c_double * 3)()
    L.check(L.lib().pdd_nonblind_profile(solver._h, C.c_int32(3), prof))
    ms_frame, ms_gather, ms_iter = prof[0], prof[1], prof[2]
    p = 4 if cfg.dtype == "f32" else 8
    j_local = sum(solver.sub_frames)
    n_local = sum(h * w for h, w in solver.sub_hw)
    k1_bytes = 5 * p * j_local * s * s           # Gamma r/w + amplitude (compulsory)
    iter_bytes = 5 * p * J * s * s + 5 * p * sum(r.area() for r in plan.subdomains)
    peak, peak_kind = hbm_peak()
    traffic = None
    try:  # dram read+write per K1 launch from the committed ncu capture of this config
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as fh:
            tr = json.load(fh)
        if tr.get("config") == args.config and world == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    k1_gbs = k1_bytes / (ms_frame / 1e3) / 1e9
    fft_flops = 2 * 5 * s * s * math.log2(s * s) * j_local
    launches = solver.launches_per_iteration() * args.steps + 4

    line = dict(base, impl="ours", value=value, ms_per_step=ms_step, scaling="strong", dtype=cfg.dtype,
                config={"workload": f"BASELINE config {args.config} ({cfg.name}): {cfg.N}^2 object, {s}^2 probe, "
                                    f"step {cfg.step}, {J} frames, plan {cfg.plan}, {cfg.dtype}",
                        "frames": J, "parallelism": f"subdomains over {world} GPU(s)",
                        "l2": "inputs > L2 (no flush needed)"},
                roofline={"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s",
                          "frac": k1_gbs / peak, "traffic": traffic, "kernel": "sweep_stream_kernel (K1)",
                          "kernel_ms": ms_frame, "algorithmic_bytes_per_launch": k1_bytes,
                          "peak_kind": peak_kind,
                          "fp32_tflops": fft_flops / (ms_frame / 1e3) / 1e12},
                iter_roofline={"bytes_per_iter": iter_bytes, "achieved_gbs": iter_bytes / (ms_step / 1e3) / 1e9,
                               "frac": iter_bytes / (ms_step / 1e3) / 1e9 / peak, "gather_ms": ms_gather,
                               "profiled_iter_ms": ms_iter},
                clocks=clk.summary(), gpu_launches=launches)
    del solver
    torch.cuda.empty_cache()

    # end-to-end through the public API: pinned host amplitudes -> solve -> host result
    if not args.no_e2e:
        host = torch.empty(amp.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(amp)
        amp_np = host.numpy()
        del amp
        torch.cuda.empty_cache()
        nccl_id = fresh_nccl_id(dist, rank, world)  # a unique id bootstraps one communicator only
        if dist:
            dist.barrier()
        n_e2e = cfg.iterations
        ecfg = P.NonblindConfig(max_iters=n_e2e, tol_rf=1e-300)
        t0 = time.perf_counter()
        s2 = P.NonblindSolver(plan, None, probe, ecfg, amplitudes=amp_np, dtype=cfg.dtype, device=local, rank=rank,
                              world=world, nccl_id=nccl_id)
        res = s2.run()
        torch.cuda.synchronize()
        t_e2e = allmax(dist, time.perf_counter() - t0)
        h2d = j_local * s * s * 4 + probe.nbytes
        g = plan.geometry
        d2h = n_local * 16 + (g.image_height * g.image_width * 16 if world == 1 else 0) + res.iterations * 24
        line["e2e"] = {"value": J * res.iterations / t_e2e, "unit": base["unit"], "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "iterations_per_step": res.iterations,
                       "timer": "host wall clock around synchronous C-ABI calls (create+upload, run, download)"}
        del s2

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, kind, cores, sample, _ = run_reference(cfg, 3, 1)
            line["cpu_baseline"] = {"value": v, "unit": base["unit"], "cores": cores, "kind": kind, "sample": sample}
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def bench_blind(args, cfg, base, rank, world, local, dist):
    """Blind OD²BP (config 3): frames*iterations/s of BlindSolver iterations
    (blind.cpp:194-296: 3 FFTs per frame, probe consensus, u-update)."""
    import ctypes as C

    import torch

    import paper_2011_00162_b200 as P
    from paper_2011_00162_b200 import _lib as L, sim

    inp = sim.make_inputs(cfg, device=True)
    plan, amp = inp["plan"], inp["amplitudes_dev"]
    J, s = plan.geometry.frame_count(), cfg.s
    w0 = inp.get("w0")
    nccl_id = fresh_nccl_id(dist, rank, world)
    bcfg = P.BlindConfig(max_iters=max(cfg.iterations, args.steps + args.warmup + 8), tol_rf=1e-300, **cfg.solver)
    solver = P.BlindSolver(plan, None, bcfg, amplitudes=amp, dtype=cfg.dtype, device=local, rank=rank, world=world,
                           nccl_id=nccl_id)
    L.check(L.lib().pdd_blind_init_state(solver._h, L.ptr(None if w0 is None else L.c128(w0))))

    def timed(n):
        ms = C.c_double()
        L.check(L.lib().pdd_blind_iterate_timed(solver._h, C.c_int32(n), C.byref(ms)))
        return ms.value

    timed(args.warmup)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms_total = timed(args.steps)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = allmax(dist, ms_total)
    prof = (C.c_double * 3)()
    L.check(L.lib().pdd_blind_profile(solver._h, C.c_int32(3), prof))
    ms_frame, ms_gather, ms_iter = prof[0], prof[1], prof[2]
    p = 4 if cfg.dtype == "f32" else 8
    j_local = sum(solver.sub_frames)
    k1_bytes = 5 * p * j_local * s * s
    iter_bytes = 5 * p * J * s * s + 5 * p * sum(r.area() for r in plan.subdomains)
    peak, peak_kind = hbm_peak()
    k1_gbs = k1_bytes / (ms_frame / 1e3) / 1e9
    line = dict(base, impl="ours", value=J * args.steps / (ms_total / 1e3), ms_per_step=ms_total / args.steps,
                scaling="strong", dtype=cfg.dtype,
                config={"workload": f"BASELINE config {args.config} ({cfg.name}, blind): {cfg.N}^2 object, {s}^2 "
                                    f"probe, step {cfg.step}, {J} frames, plan {cfg.plan}, disk w0 r="
                                    f"{cfg.init_disk_radius}, {cfg.dtype}",
                        "frames": J, "parallelism": f"subdomains over {world} GPU(s)",
                        "l2": "working set ~0.8 GB > L2 (no flush needed)"},
                roofline={"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s", "frac": k1_gbs / peak,
                          "traffic": None, "kernel": "BLIND frame pass (K1: R-factor forward + streamed sweep)", "kernel_ms": ms_frame,
                          "algorithmic_bytes_per_launch": k1_bytes, "peak_kind": peak_kind},
                iter_roofline={"bytes_per_iter": iter_bytes,
                               "achieved_gbs": iter_bytes / (ms_total / args.steps / 1e3) / 1e9,
                               "frac": iter_bytes / (ms_total / args.steps / 1e3) / 1e9 / peak,
                               "gather_ms": ms_gather, "profiled_iter_ms": ms_iter},
                clocks=clk.summary(), gpu_launches=solver.launches_per_iteration() * args.steps)
    del solver
    torch.cuda.empty_cache()
    if not args.no_e2e:
        host = torch.empty(amp.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(amp)
        amp_np = host.numpy()
        del amp
        torch.cuda.empty_cache()
        nccl_id = fresh_nccl_id(dist, rank, world)  # a unique id bootstraps one communicator only
        if dist:
            dist.barrier()
        ecfg = P.BlindConfig(max_iters=cfg.iterations, tol_rf=1e-300, **cfg.solver)
        t0 = time.perf_counter()
        s2 = P.BlindSolver(plan, None, ecfg, amplitudes=amp_np, dtype=cfg.dtype, device=local, rank=rank,
                           world=world, nccl_id=nccl_id)
        res = s2.run(w0=w0)
        torch.cuda.synchronize()
        t_e2e = allmax(dist, time.perf_counter() - t0)
        g = plan.geometry
        n_local = sum(h * w for h, w in s2.sub_hw)
        line["e2e"] = {"value": J * res.iterations / t_e2e, "unit": base["unit"],
                       "h2d_bytes_per_step": j_local * s * s * 4 + (0 if w0 is None else w0.size * 16),
                       "d2h_bytes_per_step": n_local * 16 + (g.image_height * g.image_width * 16 if world == 1 else 0)
                       + 3 * s * s * 16 + res.iterations * 24,
                       "iterations_per_step": res.iterations,
                       "timer": "host wall clock around synchronous C-ABI calls (create+upload, run, download)"}
        del s2
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, kind, cores, sample, _ = run_reference(cfg, 2, 1)
            line["cpu_baseline"] = {"value": v, "unit": base["unit"], "cores": cores, "kind": kind, "sample": sample}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
