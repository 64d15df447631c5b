"""Command-line front end over the GPU solvers: the `reconstruct`, `blind` and
`evaluate` subcommands of the reference CLI (proj/tools/ptychodd_cli.cpp) on
the same dataset and run directories, with `--backend cuda` (SURVEY.md
sec. 8(f) row 4).

  python -m paper_2011_00162_b200.cli reconstruct --dataset DIR --out RUN [--subdomains D] ...
  python -m paper_2011_00162_b200.cli blind       --dataset DIR --out RUN [--support-radius R] ...
  python -m paper_2011_00162_b200.cli evaluate    --run RUN [--run RUN2 ...] [--dataset DIR]

Dataset (what the reference's `simulate` writes, ptychodd_cli.cpp:155-169):
meta.json (schema_version 1, geometry), frames.ptya (float64 intensities,
streamed from disk to the GPU -- never loaded into host memory), probe.ptya,
optional pin.ptya / sample.ptya.  Run outputs (write_run_common,
ptychodd_cli.cpp:104-119): merged.ptya, sub_<d>.ptya, convergence.csv,
summary.json, meta.json; blind adds probe_recovered.ptya, probe_fourier.ptya,
support_mask.ptya.  Exit codes (ptychodd_cli.cpp:26-30): 0 ok, 2 config,
3 format, 4 infeasible plan, 5 divergence.
The reference's `simulate` (its test-data harness) is not reproduced: any
writer of the PTYA/meta.json format, the reference's included, makes inputs.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import zlib

import numpy as np

from . import _lib as L
from . import ptya
from .ptychodd import (BlindConfig, NonblindConfig, BlindSolver, NonblindSolver, disk_support_mask, plan_stripes,
                       snr_db)

EXIT_CONFIG, EXIT_FORMAT, EXIT_PLAN, EXIT_DIVERGENCE = 2, 3, 4, 5


class PlanError(RuntimeError):
    pass


def load_dataset(d: str) -> dict:
    """ptychodd_cli.cpp:88-102."""
    meta = ptya.read_json(os.path.join(d, "meta.json"))
    if meta.get("schema_version", 0) != 1:
        raise L.FormatError("unsupported dataset schema_version (byte offset 0)")
    ds = {"meta": meta, "geometry": ptya.geometry_from_json(meta["geometry"]),
          "frames": os.path.join(d, "frames.ptya"),
          "probe": ptya.read_complex_array(os.path.join(d, "probe.ptya")),
          "noisy": meta.get("noise") is not None}
    for key, name, rd in (("truth", "sample.ptya", ptya.read_complex_array),
                          ("pin", "pin.ptya", ptya.read_real_array)):
        p = os.path.join(d, name)
        ds[key] = rd(p) if os.path.exists(p) else None
    return ds


def make_plan(g, D: int, axis: str):
    """ptychodd_cli.cpp:36-46."""
    ax = {"auto": "auto", "rows": "rows", "cols": "columns"}.get(axis)
    if ax is None:
        raise L.InvalidArgument("--split-axis must be auto|rows|cols")
    try:
        return plan_stripes(g, D, ax)
    except L.InvalidArgument as e:
        raise PlanError(str(e)) from None


def devices_for(threads: int, D: int):
    """The reference's worker count mapped onto GPUs (as the drop-in does):
    min(threads or D, D, visible devices) ranks; a single device = one rank."""
    import ctypes as C

    n = C.c_int32()
    L.check(L.lib().pdd_device_count(C.byref(n)))
    G = max(1, min(threads if threads > 0 else D, D, max(n.value, 1)))
    return None if G == 1 else list(range(G))


def progress(quiet: bool):
    def cb(rec):
        if not quiet and rec.iteration % 25 == 0:
            print(f"iter {rec.iteration}  rf {rec.rf:g}  re {rec.re:g}", flush=True)

    return cb


def write_run_common(out: str, params: dict, subs, merged, records, summary: dict) -> None:
    """ptychodd_cli.cpp:104-119."""
    os.makedirs(out, exist_ok=True)
    ptya.write_array(os.path.join(out, "merged.ptya"), merged)
    for d, u in enumerate(subs):
        ptya.write_array(os.path.join(out, f"sub_{d}.ptya"), u)
    ptya.write_convergence_csv(os.path.join(out, "convergence.csv"), records)
    summary["virtual_seconds"] = sum(r.t_virtual_ms for r in records) * 1e-3  # metrics.cpp:103-107
    summary["actual_seconds"] = sum(r.t_actual_ms for r in records) * 1e-3
    ptya.write_json(os.path.join(out, "summary.json"), summary)
    ptya.write_json(os.path.join(out, "meta.json"), {"schema_version": 1, "kind": "run", "params": params})


def _stop(a, noisy: bool):
    if a.stop not in ("rf", "re", "auto"):
        raise L.InvalidArgument("--stop must be rf|re|auto")
    use_re = a.stop == "re" or (a.stop == "auto" and noisy)
    return use_re, (a.max_iters if a.max_iters > 0 else (200 if use_re else 1000))


def cmd_reconstruct(a) -> int:
    """ptychodd_cli.cpp:192-218."""
    ds = load_dataset(a.dataset)
    plan = make_plan(ds["geometry"], a.subdomains, a.split_axis)
    use_re, max_iters = _stop(a, ds["noisy"])
    cfg = NonblindConfig(epsilon=a.epsilon, eta=a.eta, r=a.r, max_iters=max_iters, tol_rf=a.tol_rf,
                         tol_re=a.tol_re, stop_rule="relative_error" if use_re else "rfactor",
                         record_lagrangian=a.record_lagrangian, threads=a.threads)
    solver = NonblindSolver(plan, ds["frames"], ds["probe"], cfg, ds["pin"], dtype=a.precision,
                            devices=devices_for(a.threads, plan.D))
    res = solver.run(on_iteration=progress(a.quiet))
    params = {"dataset": a.dataset, "subdomains": a.subdomains, "epsilon": cfg.epsilon, "eta": cfg.eta, "r": cfg.r,
              "max_iters": cfg.max_iters, "tol_rf": cfg.tol_rf, "tol_re": cfg.tol_re, "threads": cfg.threads,
              "stop": "re" if use_re else "rf", "split_axis": a.split_axis, "backend": a.backend,
              "precision": a.precision}
    summary = {"solver": "nonblind", "D": a.subdomains, "iterations": res.iterations, "final_rf": res.final_rf,
               "final_re": res.final_re}
    write_run_common(a.out, params, res.sub_solutions, res.merged, res.records, summary)
    print(f"done: {res.iterations} iterations, RF {res.final_rf:g}, RE {res.final_re:g} -> {a.out}")
    return 0


def cmd_blind(a) -> int:
    """ptychodd_cli.cpp:220-264."""
    ds = load_dataset(a.dataset)
    plan = make_plan(ds["geometry"], a.subdomains, a.split_axis)
    use_re, max_iters = _stop(a, ds["noisy"])
    mask = disk_support_mask(ds["geometry"].frame_side, a.support_radius) if a.support_radius > 0 else None
    cfg = BlindConfig(epsilon=a.epsilon, eta=a.eta, r=a.r, mu=a.mu, gamma=a.gamma if a.gamma > 0 else 1e-3 * a.eta,
                      support_mask=mask, max_iters=max_iters, tol_rf=a.tol_rf, tol_re=a.tol_re,
                      stop_rule="relative_error" if use_re else "rfactor", threads=a.threads)
    solver = BlindSolver(plan, ds["frames"], cfg, ds["pin"], dtype=a.precision,
                         devices=devices_for(a.threads, plan.D))
    res = solver.run(on_iteration=progress(a.quiet))
    params = {"dataset": a.dataset, "subdomains": a.subdomains, "epsilon": cfg.epsilon, "eta": cfg.eta, "r": cfg.r,
              "mu": cfg.mu, "gamma": cfg.gamma, "support_radius": a.support_radius, "max_iters": cfg.max_iters,
              "tol_rf": cfg.tol_rf, "tol_re": cfg.tol_re, "threads": cfg.threads, "stop": "re" if use_re else "rf",
              "split_axis": a.split_axis, "backend": a.backend, "precision": a.precision}
    summary = {"solver": "blind", "D": a.subdomains, "iterations": res.iterations, "final_rf": res.final_rf,
               "final_re": res.final_re}
    write_run_common(a.out, params, res.sub_solutions, res.merged, res.records, summary)
    ptya.write_array(os.path.join(a.out, "probe_recovered.ptya"), res.probe)
    ptya.write_array(os.path.join(a.out, "probe_fourier.ptya"), res.probe_fourier)
    ptya.write_array(os.path.join(a.out, "support_mask.ptya"), res.support_mask)
    print(f"done: {res.iterations} iterations, RF {res.final_rf:g}, RE {res.final_re:g} -> {a.out}")
    return 0


def _png_gray(path: str, img: np.ndarray, lo: float, hi: float) -> None:
    """io.cpp:270-307: 8-bit grayscale, window [lo, hi], filter 0, zlib level 1."""
    t = np.clip((img - lo) / (hi - lo), 0.0, 1.0)
    px = np.floor(t * 255.0 + 0.5).astype(np.uint8)  # lround for non-negative values
    raw = b"".join(b"\x00" + row.tobytes() for row in px)

    def chunk(kind: bytes, payload: bytes) -> bytes:
        return (len(payload).to_bytes(4, "big") + kind + payload +
                (zlib.crc32(kind + payload) & 0xFFFFFFFF).to_bytes(4, "big"))

    h, w = img.shape
    ihdr = w.to_bytes(4, "big") + h.to_bytes(4, "big") + bytes([8, 0, 0, 0, 0])
    data = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", ihdr) + chunk(b"IDAT", zlib.compress(raw, 1)) + chunk(b"IEND", b"")
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)


def cmd_evaluate(a) -> int:
    """ptychodd_cli.cpp:272-328 (SNR against the ground truth, PNG rendering,
    speed-up table over runs with a D = 1 baseline, metrics.cpp:109-125)."""
    truth = None
    if a.dataset:
        truth = load_dataset(a.dataset)["truth"]
        if truth is None:
            print("note: dataset has no ground truth; SNR omitted")
    else:
        print("note: no --dataset given; SNR omitted")
    rows = []
    for run in a.run:
        summary = ptya.read_json(os.path.join(run, "summary.json"))
        merged = ptya.read_complex_array(os.path.join(run, "merged.ptya"))
        line = (f"{run}: D {summary.get('D', 0)}, iterations {summary.get('iterations', 0)}, RF "
                f"{summary.get('final_rf', 0.0):g}, virtual {summary.get('virtual_seconds', 0.0):g} s")
        if truth is not None:
            if merged.shape != truth.shape:
                raise L.FormatError("merged image shape does not match ground truth (byte offset 0)")
            line += f", SNR {snr_db(merged, truth):g} dB"
        print(line)
        if a.render:
            ph = np.angle(merged)
            _png_gray(os.path.join(run, "magnitude.png"), np.abs(merged), 0.0, 1.0)
            _png_gray(os.path.join(run, "phase.png"), np.where(ph < 0, ph + 2 * math.pi, ph), 0.0, math.pi)
        rows.append((int(summary.get("D", 0)), int(summary.get("iterations", 0)),
                     float(summary.get("virtual_seconds", 0.0))))
    base = [r for r in rows if r[0] == 1]
    if len(rows) > 1 and base:
        t1 = base[0][2]
        print("\n  D  iterations  virtual_s  speedup  efficiency")
        for D, it, t in sorted(rows):
            sp = t1 / t if t > 0 else 0.0
            print(f"{D:3d}  {it:10d}  {t:9.3f}  {sp:7.2f}  {sp / D:10.3f}")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="ptychodd",
                                 description="ptychographic phase retrieval with overlapping domain decomposition "
                                             "(B200 backend)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, r_default in (("reconstruct", 4.0e3), ("blind", 5.0e3)):
        p = sub.add_parser(name)
        p.add_argument("--dataset", required=True)
        p.add_argument("--out", required=True)
        p.add_argument("--subdomains", type=int, default=2)
        p.add_argument("--epsilon", type=float, default=0.5)
        p.add_argument("--eta", type=float, default=0.1)
        p.add_argument("--r", type=float, default=r_default)
        p.add_argument("--max-iters", type=int, default=0)
        p.add_argument("--tol-rf", type=float, default=1.0e-5)
        p.add_argument("--tol-re", type=float, default=1.0e-3)
        p.add_argument("--threads", type=int, default=0, help="0 = one rank per subdomain, capped by the GPUs")
        p.add_argument("--stop", default="auto")
        p.add_argument("--split-axis", default="auto")
        p.add_argument("--quiet", action="store_true")
        p.add_argument("--backend", choices=["cuda"], default="cuda")
        p.add_argument("--precision", choices=["f64", "f32"], default="f64",
                       help="f64: the reference's double precision; f32: complex64")
        if name == "reconstruct":
            p.add_argument("--record-lagrangian", action="store_true")
        else:
            p.add_argument("--mu", type=float, default=2.0e2)
            p.add_argument("--gamma", type=float, default=0.0)
            p.add_argument("--support-radius", type=float, default=0.0)
    p = sub.add_parser("evaluate")
    p.add_argument("--dataset", default="")
    p.add_argument("--run", action="append", required=True)
    p.add_argument("--no-render", dest="render", action="store_false")
    return ap


def main(argv=None) -> int:
    a = parser().parse_args(argv)
    try:
        return {"reconstruct": cmd_reconstruct, "blind": cmd_blind, "evaluate": cmd_evaluate}[a.cmd](a)
    except PlanError as e:
        print(f"infeasible plan: {e}", file=sys.stderr)
        return EXIT_PLAN
    except L.DivergenceError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DIVERGENCE
    except L.FormatError as e:
        print(f"format error: {e}", file=sys.stderr)
        return EXIT_FORMAT
    except Exception as e:  # noqa: BLE001 - the reference maps every other error to exit 2
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
