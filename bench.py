#!/usr/bin/env python
"""Benchmark of the ADER-WENO hot path on B200 (BASELINE.json metric).

python bench.py --gpus N --steps K --warmup W [--config c4|c2|c1] [--n SIZE] [--impl reference]

A step is one level-0 macro step of the whole hot path (WENO -> predictor ->
face flux -> FV update, incl. ghost exchange and the CFL reduction) over the
workload.  Default workload: BASELINE configs[3] (3D Euler spherical
explosion, uniform 256^3, order 3, FP64), the configuration the metric's
1/2/4/8-GPU numbers are quoted on; it fits one B200.  Inputs (~90 GB of
state and stage buffers) are larger than L2, so no explicit flush is needed.

--impl reference times the CPU oracle (oracle/, single thread) on bounded
sub-box samples of the same workload; that is this tier's reference arm.
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

METRIC = "FP64 cell-updates/s (2D/3D Euler, MHD) at 1/2/4/8 B200; % FP64 roofline"
UNIT = "cell-updates/s"
# FP64 ALU peak of B200 derived from unit counts and clocks:
# 148 SMs x 64 FP64 FMA lanes/clk x 2 flop x 1.965 GHz (clocks.max.sm)
SM_COUNT, FP64_FMA_PER_CLK = 148, 64


def fp64_peak_tflops(mhz):
    return SM_COUNT * FP64_FMA_PER_CLK * 2 * mhz * 1e6 / 1e12


def fp64_peak():
    """(peak TFLOP/s, note): the measured DFMA throughput of this pool's B200s
    (tools/fp64_peak.cu under tools/gpu_fp64_peak.sh, SM clock sampled during
    the run; sustained = 4 s back to back, the regime of a kernel timed inside
    a long step), else the figure derived from unit counts and clocks."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "round2_fp64_peak.json")))
        return float(d["fp64_fma_tflops_sustained"]), (
            f"measured DFMA sustained {d['fp64_fma_tflops_sustained']:.1f} TF/s at median "
            f"{d['sm_mhz_median_under_load']:.0f} MHz (burst {d['fp64_fma_tflops_burst']:.1f}; derived "
            f"{fp64_peak_tflops(1965.0):.1f} at 1965 MHz), profiles/round2_fp64_peak.json (of measured)")
    except Exception:
        return fp64_peak_tflops(1965.0), "FP64 FMA pipe: 148 SM x 64 lanes x 2 x 1.965 GHz (derived, DESIGN.md)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4")
    p.add_argument("--n", type=int, default=0)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-box", type=int, default=12, help="edge of the oracle sample box (cells)")
    p.add_argument("--pred-guess", type=int, default=0, choices=[0, 1],
                   help="Picard initial guess: 0 time-constant (R3), 1 extrapolated previous q (R25)")
    p.add_argument("--flux", default="rusanov", choices=["rusanov", "osher"],
                   help="two-point flux (BASELINE: rusanov; the paper's explosions use osher)")
    p.add_argument("--load-balance", type=int, default=1, choices=[0, 1],
                   help="AMR at N>1: re-cut the level-0 blocks after every adapt (reading R24)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0, period_ms=None):
        self.device = device
        self.proc = None
        self.lines = []
        self.period_ms = int(os.environ.get("ADER_BENCH_CLOCK_MS", "200")) if period_ms is None else period_ms

    def start(self):
        if self.period_ms <= 0:   # diagnostics only: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def window(self, t0, t1):
        # samples taken inside [t0, t1] (host clock); the sampler is started
        # before the warm-up so that nvidia-smi's own start-up (NVML init can
        # hold the driver for a while) never falls inside the timed region
        self.t0, self.t1 = t0, t1

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", -1e300), getattr(self, "t1", 1e300)
        lines = [ln for ts, ln in self.lines if t0 - 0.25 <= ts <= t1 + 0.25] or [ln for _, ln in self.lines[-3:]]
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_sample(wl, edge, reps=1, flux=0, nbox=1, seed=3585):
    """Time the oracle (single thread, as it stands) on a bounded sample of the
    workload.  Uniform grids: one step of `nbox` edge^d boxes at seeded random
    positions over the whole domain (so constant regions and fronts enter in
    the workload's own proportion; each box plus its face-neighbour layer is
    reconstructed and predicted).  AMR: one macro step of the AMR oracle on an
    edge^d level-0 grid.  Returns (cell-updates/s, description, updates, s)."""
    import oracle as O
    if wl.lmax > 0:
        # AMR workload: one macro step of the AMR oracle on a level-0 grid of
        # edge^d cells of the same problem (full LTS hierarchy, adapt included)
        n = tuple([edge] * wl.dim)
        a = O.AmrOracle(dim=wl.dim, degree=wl.degree, n=n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                        gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, lmax=wl.lmax, refine_factor=wl.refine_factor,
                        chi_ref=wl.chi_ref, chi_rec=wl.chi_rec, flux=flux)
        a.set_initial(wl.ic)
        ups, secs = 0, 0.0
        for _ in range(reps):
            t0 = time.perf_counter()
            rep = a.step(1e300, 1, adapt_every=1)
            secs += time.perf_counter() - t0
            ups += rep.cell_updates
        desc = (f"one macro step (all levels, adapt) of {wl.name} on a {'x'.join(map(str, n))} level-0 grid, "
                f"AMR oracle, single thread")
        return ups / secs, desc, ups, secs
    o = O.Oracle(dim=wl.dim, degree=wl.degree, n=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                 gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, flux=flux)
    n = wl.n
    if wl.name.startswith("c4"):
        uin = O.prim_to_cons(0, 3, wl.gamma, [1, 0, 0, 0, 1])
        dx = (wl.hi[0] - wl.lo[0]) / n[0]
        dt = wl.cfl / sum(O.max_speed(0, 3, wl.gamma, 0, uin, d) / dx for d in range(3))
    else:
        o.set_initial(wl.ic)
        dt = o.compute_dt()
    rng = np.random.default_rng(seed)
    ups, secs, where = 0, 0.0, []
    for _ in range(reps):
        for _b in range(nbox):
            blo = [int(rng.integers(0, max(1, n[k] - edge + 1))) for k in range(wl.dim)]
            bhi = [min(n[k], blo[k] + edge) for k in range(wl.dim)]
            glo = [max(0, b - wl.degree - 2) for b in blo]
            ghi = [min(n[k], b + wl.degree + 2) for k, b in enumerate(bhi)]
            o.set_initial_box(wl.ic, glo, ghi)
            t0 = time.perf_counter()
            _, rep = o.advance_box(dt, blo, bhi)
            secs += time.perf_counter() - t0
            ups += rep.cell_updates
            where.append(tuple(blo))
    desc = (f"one step of {len(where)} {'x'.join([str(edge)] * wl.dim)} cell boxes at seeded random positions "
            f"{where[:4]}{'...' if len(where) > 4 else ''} of {wl.name} (each box + its face-neighbour layer "
            f"reconstructed/predicted), single thread")
    return ups / secs, desc, ups, secs


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    edge = max(2, args.cpu_box // 2) if wl.lmax > 0 else 8
    fl = 1 if args.flux == "osher" else 0
    for i in range(args.warmup):
        oracle_sample(wl, edge, flux=fl, nbox=1, seed=100 + i)
    tot_u, tot_s = 0, 0.0
    desc = ""
    for i in range(args.steps):
        _, desc, u, s = oracle_sample(wl, edge, flux=fl, nbox=(2 if wl.dim == 3 else 16) if wl.lmax == 0 else 1, seed=3585 + i)
        tot_u += u
        tot_s += s
    val = tot_u / tot_s
    cfgd = {"workload": wl.name, "dim": wl.dim, "degree": wl.degree, "cells": list(wl.n),
            "system": "euler" if wl.system == 0 else "mhd_glm", "flux": args.flux}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def load_traffic(wl, kernel="stdg_predictor", what="dram_bytes_per_launch"):
    """dram read+write bytes per launch (or the hardware-counted FP64 fraction,
    what="fp64_hw_frac") of `kernel` from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(wl.name, {}).get(f"{kernel}_{what}")
    except Exception:
        return None


def main():
    args = parse()
    from paper_1212_3585_b200 import workloads as W
    wl = W.config(args.config, args.n or None)
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist
    from paper_1212_3585_b200 import ader

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nid = None
    if world > 1:
        obj = [ader.ader_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    cfg = ader.make_config(dim=wl.dim, degree=wl.degree, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                           gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, rank=rank, world_size=world, device=local,
                           nccl_id=nid, lmax=wl.lmax, refine_factor=wl.refine_factor, adapt_every=1,
                           chi_ref=wl.chi_ref, chi_rec=wl.chi_rec, flux=1 if args.flux == "osher" else 0,
                           load_balance=1 if (wl.lmax > 0 and world > 1 and args.load_balance) else 0,
                           pred_guess=args.pred_guess, exact_vel=wl.extra.get("exact_vel", (0.0, 0.0, 0.0)))
    s = ader.Solver(cfg)
    stream = torch.cuda.current_stream()
    s.set_stream(stream.cuda_stream)
    t_ic = time.perf_counter()
    s.set_initial(wl.ic)
    t_ic = time.perf_counter() - t_ic

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    clk = ClockSampler(local)
    clk.start()
    # warm-up
    if args.warmup:
        s.step(1e300, args.warmup)
    barrier()
    # timed region: exactly K macro steps, no per-kernel instrumentation (the
    # uniform step then replays as one CUDA graph per step)
    l0 = s.launch_count()
    time.sleep(0.5)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(stream)
    rep = s.step(1e300, args.steps)
    e1.record(stream)
    barrier()
    clk.window(h0, time.perf_counter())
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    launches = s.launch_count() - l0
    # per-kernel times / flops (roofline entries, kernel shares) from a further
    # window of min(K, 5) steps with CUDA events around every launch
    nprof = max(1, min(args.steps, 5))
    s.set_profiling(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    s.step(1e300, nprof)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    kms, kl, kfl = s.kernel_stats()
    s.set_profiling(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    ups = torch.tensor([float(rep.cell_updates)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(ups, op=dist.ReduceOp.SUM)
    ms_max = float(t_max.item())
    total_updates = float(ups.item())
    value = total_updates / (ms_max / 1e3)

    # end-to-end through the public API with host buffers (pinned)
    ne = max(1, args.e2e_steps)
    e2e = None
    if wl.lmax == 0:
        host = torch.empty((s.ncells, s.nv), dtype=torch.float64, pin_memory=True)
        s.get_state_ptr(host.data_ptr())
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        e2e_updates = 0
        for _ in range(ne):
            # H2D of the step's input state, the step, D2H of its result (ader_step_io:
            # the copy-out of finished slabs overlaps the rest of the step)
            r2 = s.step_io(host.data_ptr(), host.data_ptr())
            e2e_updates += r2.cell_updates
        f1.record(stream)
        barrier()
        e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
        e2u = torch.tensor([float(e2e_updates)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
            dist.all_reduce(e2u, op=dist.ReduceOp.SUM)
        bytes_step = s.ncells * s.nv * 8
        e2e = {"value": float(e2u.item()) / (float(e2e_ms.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": bytes_step, "d2h_bytes_per_step": bytes_step, "steps": ne}
    else:
        # AMR: the state lives in the device tree; a step's host output is the
        # full cell list (ader_get_cells), read back every step
        barrier()
        w0 = time.perf_counter()
        e2e_updates, nbytes = 0, 0
        for _ in range(ne):
            r2 = s.step(1e300, 1)
            cells = s.get_cells()
            e2e_updates += r2.cell_updates
            nbytes = len(cells) * 96
        barrier()
        e2e = {"value": e2e_updates / (time.perf_counter() - w0), "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": nbytes, "steps": ne,
               "note": "AMR: no per-step host input; wall clock incl. ader_get_cells readback"}

    if rank == 0:
        peak, peak_note = fp64_peak()
        N = wl.degree + 1
        nvv = 9 if wl.system == 1 else wl.dim + 2
        hbm_peak = 6449.1
        try:
            hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            pass
        ridge = peak * 1e12 / (hbm_peak * 1e9)

        def entry(kernel, ms_avg, flops, nbytes, bytes_note, flops_note):
            """roofline of one kernel class: bound by its algorithmic intensity vs the ridge"""
            tf = flops / (ms_avg / 1e3) / 1e12
            gbs = nbytes / (ms_avg / 1e3) / 1e9
            ai = flops / max(1.0, nbytes)
            if ai >= ridge:
                e = {"bound": "alu", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                     "peak_note": peak_note, "achieved_note": flops_note}
            else:
                e = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                     "peak_note": "measured copy bandwidth, MEASURED_PEAKS.json hbm_gbs (of measured)",
                     "achieved_note": bytes_note}
            e.update({"kernel": kernel, "traffic": load_traffic(wl, kernel),
                      "ncu_fp64_hw_frac": load_traffic(wl, kernel, "fp64_hw_frac"),
                      "arith_intensity_flop_per_byte": ai, "ridge_flop_per_byte": ridge, "alu_tflops": tf,
                      "alu_frac": tf / peak, "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak, "ms_per_launch": ms_avg})
            return e

        # face box of the uniform path: owned + 1 per axis (faces = its lower faces)
        nb = [int(k) for k in wl.n]
        if world > 1:
            nb = [int(np.ceil(k / p)) for k, p in zip(nb, [2, 2, 2][:wl.dim])]
        ext = int(np.prod([k + 1 for k in nb]))
        sweeps_note = "algorithmic FP64 flops of the Picard sweeps actually run (first sweep at its N^d-flux cost)"
        entries = []
        if kl[ader.K_PRED]:
            # algorithmic bytes of one predictor launch: read w, write q of every predicted cell
            cells_per_launch = rep.pred_cells / max(1, args.steps) / max(1e-9, kl[ader.K_PRED] / nprof)
            # opt-in ADER_PRED_FLAT_SKIP=1 (3D M = 2): flat cells get a one-byte flag instead of a q block
            skip_on = os.environ.get("ADER_PRED_FLAT_SKIP") == "1" and wl.dim == 3 and wl.degree == 2
            flat_frac = rep.pred_flat_cells / max(1, rep.pred_cells) if skip_on else 0.0
            entries.append(entry("stdg_predictor", kms[ader.K_PRED] / kl[ader.K_PRED],
                                 kfl[ader.K_PRED] / kl[ader.K_PRED],
                                 cells_per_launch * (nvv * N ** wl.dim * 8
                                                     + (1.0 - flat_frac) * nvv * N ** (wl.dim + 1) * 8 + flat_frac),
                                 "algorithmic bytes (w read per predicted cell + q written per cell"
                                 + (f" that is not flat: {1.0 - flat_frac:.4f} of them" if skip_on else "")
                                 + ") / CUDA-event time",
                                 sweeps_note + " / CUDA-event time"))
        if wl.lmax == 0 and kl[ader.K_FLUX] and not kl[ader.K_PRED_FLUX]:
            # face flux: algorithmic bytes = every q read once + F written
            skip_on = os.environ.get("ADER_PRED_FLAT_SKIP") == "1" and wl.dim == 3 and wl.degree == 2
            flat_frac = rep.pred_flat_cells / max(1, rep.pred_cells) if skip_on else 0.0
            entries.append(entry(f"face_flux_{args.flux}", kms[ader.K_FLUX] / kl[ader.K_FLUX],
                                 kfl[ader.K_FLUX] / kl[ader.K_FLUX],
                                 ext * ((1.0 - flat_frac) * nvv * N ** (wl.dim + 1) * 8 + flat_frac * (nvv * 8 + 1)
                                        + nvv * wl.dim * 8),
                                 ("algorithmic bytes (the q block of each cell that is not flat read once, w and "
                                  f"the flag of a flat cell ({flat_frac:.4f} of them), F written) / CUDA-event time")
                                 if skip_on else "algorithmic bytes (each q read once, F written) / CUDA-event time",
                                 "algorithmic FP64 flops of the face quadrature / CUDA-event time"))
        if kl[ader.K_PRED_FLUX]:
            # fused a2 + a3 walk (+ its tile-face kernel): w read, F written; q never leaves the SM
            cells_per_launch = rep.pred_cells / max(1, args.steps) / max(1e-9, kl[ader.K_PRED_FLUX] / nprof)
            entries.append(entry(f"stdg_predictor+face_flux_{args.flux}", kms[ader.K_PRED_FLUX] / kl[ader.K_PRED_FLUX],
                                 kfl[ader.K_PRED_FLUX] / kl[ader.K_PRED_FLUX],
                                 cells_per_launch * nvv * N ** wl.dim * 8 + ext * nvv * wl.dim * 8,
                                 "algorithmic bytes (w read per predicted cell + F written) / CUDA-event time",
                                 sweeps_note + " + the face quadrature's flops / CUDA-event time (walk + "
                                 "tile-face kernel)"))
        kind_of = {"stdg_predictor": ader.K_PRED, f"face_flux_{args.flux}": ader.K_FLUX,
                   f"stdg_predictor+face_flux_{args.flux}": ader.K_PRED_FLUX}
        dominant = max(entries, key=lambda e: kms[kind_of[e["kernel"]]]) if entries else None
        # north_star: the stdg_predictor + weno_reconstruct path against the FP64 roofline
        pk = ader.K_PRED_FLUX if kl[ader.K_PRED_FLUX] else ader.K_PRED
        pw_ms = kms[ader.K_WENO] + kms[pk]
        pw_tf = (kfl[ader.K_WENO] + kfl[pk]) / max(1, nprof) / (pw_ms / max(1, nprof) / 1e3) / 1e12 \
            if pw_ms > 0 else 0.0
        pred_weno = {"kernels": "weno_reconstruct + " + ader.KERNEL_NAMES[pk], "alu_tflops": pw_tf, "peak": peak,
                     "frac": pw_tf / peak, "ms_per_step": pw_ms / max(1, nprof),
                     "note": "algorithmic FP64 flops (WENO problems of the three sweeps + Picard sweeps"
                             + (" + face quadrature" if pk == ader.K_PRED_FLUX else "") + ") / their CUDA-event time"}
        step_ms = ms_max / args.steps
        share = {ader.KERNEL_NAMES[i]: round(kms[i] / max(1e-9, prof_ms), 4) for i in range(ader.K_COUNT)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "dim": wl.dim, "degree": wl.degree, "order": wl.degree + 1,
                       "cells": list(wl.n), "system": "euler" if wl.system == 0 else "mhd_glm",
                       "flux": args.flux, "cfl": wl.cfl, "ic": "explosion r<0.5" if "explosion" in wl.name else wl.name,
                       "parallelism": f"level-0 blocks x{world}" + (" (dynamic RCB)" if cfg.load_balance else ""),
                       "l2": "inputs larger than L2 (~90 GB working set)" if wl.lmax == 0 and wl.dim == 3 else
                             "state + stage arrays re-written every step (no flush)",
                       **({"lmax": wl.lmax, "refine_factor": wl.refine_factor, "chi_ref": wl.chi_ref,
                           "chi_rec": wl.chi_rec, "chi_note": "outside the paper's 0.2-0.25 / 0.05-0.15 ranges "
                           "(P:630-632) where noted in DESIGN.md R1"} if wl.lmax > 0 else {}),
                       "pred_guess": args.pred_guess},
            "roofline": dominant,
            "roofline_kernels": entries,
            "pred_weno_fp64": pred_weno,
            "kernel_share_of_step": share,
            "pred_sweeps_mean": rep.pred_sweeps_total / max(1, rep.pred_cells),
            "pred_flat_frac": rep.pred_flat_cells / max(1, rep.pred_cells),
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "ic_setup_s": t_ic,
        }
        if world == 1 and not args.no_cpu_baseline:
            v, desc, u, secs = (oracle_sample(wl, 10, flux=1 if args.flux == "osher" else 0, nbox=4 if wl.dim == 3 else 32) if wl.lmax == 0
                                else oracle_sample(wl, args.cpu_box, flux=1 if args.flux == "osher" else 0))
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                                    "cell_updates": u, "seconds": secs, "host_nproc": os.cpu_count()}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
