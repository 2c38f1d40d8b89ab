"""bench.py -- one OS-MPM fine implicit sub-step on the C5 workload (BASELINE.json configs[4]).

A step = everything a fine sub-step of Alg. 1 does on 16,777,216 particles:
  sort + APIC P2G (mass, momentum, stress)            -> osmpm_p2g
  Pi_{S->B} onto the dx = 1/128 overlap grid          -> osmpm_transmit(FINE_TO_COARSE)
  I_{B->S} + T_m (alpha = 1/2) onto the fine receivers -> osmpm_transmit(COARSE_TO_FINE) -> Dirichlet
  backward-Euler Newton: exactly 10 Newton x 50 PCG HVPs, line search -> osmpm_implicit_solve
  G2P + F update + advection                          -> osmpm_g2p
Metric: particle-substeps/s = N_particles / step time (BASELINE.json `metric`).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--precision f64|f32]
Prints ONE JSON line on rank 0.  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "implicit MPM particle-substeps/sec (C5 fine sub-step: P2G + Pi + I/T + 10 Newton x 50 PCG HVPs + G2P)"
UNIT = "particle-substeps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="osmpm", choices=["osmpm", "reference"])
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--cells", type=int, default=128, help="cube side in cells (128 -> 16.7M particles)")
    ap.add_argument("--newton", type=int, default=10)
    ap.add_argument("--cg", type=int, default=50)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the fp32-variant sub-run that a 1-GPU f64 run reports under `variants`")
    ap.add_argument("--no-prof", action="store_true", help="skip the per-kernel event timing (A/B of its overhead)")
    ap.add_argument("--cpu-cells", type=int, default=14, help="oracle sample cube side (cells)")
    ap.add_argument("--cg-variant", type=int, default=None, choices=[0, 1],
                    help="PCG variant: 0 standard, 1 single-reduction (Chronopoulos-Gear, DESIGN.md R22: one "
                         "all-reduce per iteration); default 0 on one GPU, 1 on several")
    ap.add_argument("--comm", action="store_true",
                    help="at N = 1: still initialise torch.distributed (NCCL) and a one-rank osmpm communicator, "
                         "so that the multi-rank code path (decomposed subdomain, NCCL collectives, max over "
                         "ranks) runs on one GPU -- a functional check, not a bench line")
    ap.add_argument("--slabs", type=int, default=1,
                    help="x-slabs per GPU (>1: the decomposed path on one device)")
    ap.add_argument("--halo", default="fused", choices=["fused", "all", "pass"],
                    help="halo of the PCG's HVP (DESIGN.md R24): fused between the slabs of a GPU and an NCCL "
                         "halo pass between ranks (default); 'all' fuses across ranks too (IPC peer memory); "
                         "'pass' uses the halo pass everywhere")
    a = ap.parse_args()
    if a.halo == "pass":
        os.environ["OSMPM_FUSED_HALO"] = "0"
    elif a.halo == "all":
        os.environ["OSMPM_FUSED_HALO"] = "all"
    return a


# ------------------------------------------------------------------------------------------------
# workload
# ------------------------------------------------------------------------------------------------

def build_workload(cells):
    import synth
    return synth.c5_bench_workload(cells)


# ------------------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ------------------------------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# roofline accounting: algorithmic bytes of one HVP launch
# ------------------------------------------------------------------------------------------------

# algorithmic floating-point operations of one particle's HVP (3D): tensor-product
# gather 270 FMA (540 flops), constitutive G_p 217 flops, scatter 9 items x 51 flops (459), B-spline
# weights 40 flops
HVP_FLOPS_PER_PARTICLE = 540 + 217 + 459 + 40
# FP64 (and, at 2x, FP32) vector peak: 148 SMs x 64 FP64 lanes x 2 flops (FMA) x 1.965 GHz
# (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz; sm_100 FP64 rate half of FP32's 128 lanes/SM)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# algorithmic flops per particle per call of the other particle kernels
SURVEY_FLOPS_PER_PARTICLE = {"p2g": 1750, "grad": 1200, "g2p": 1200}


def roofline_bound(bytes_, flops, hbm_gbs, fp_tflops):
    """Which roofline bounds a kernel (SURVEY.md §8(d) "the achieved bound is min(HBM, FP pipe)"): the
    slower of the algorithmic bytes at the HBM peak and the algorithmic flops at the CUDA-core FP peak."""
    t_hbm = bytes_ / (hbm_gbs * 1e9)
    t_fp = flops / (fp_tflops * 1e12)
    return ("alu" if t_fp > t_hbm else "hbm"), t_hbm, t_fp


def hvp_algorithmic_bytes(n_particles, n_active_nodes, word):
    """SURVEY.md §8(d) accounting of one HVP launch: 190 B per particle in fp64, 95 B in fp32 (App. C:
    the particle's position, F^n-derived Newton cache and V^0 plus its share of the node vectors d and
    y), times the particles the launch processes.  (The reformulated kernel reads only 20 particle
    words + 48 B per active node -- `reformulated_bytes_per_launch` below.)"""
    return n_particles * (190 if word == 8 else 95)


def hvp_reformulated_bytes(n_particles, n_active_nodes, word):
    # x (3) + Newton cache S' (6) + Ah (9) + c' + l' (2) = 20 words of the particle precision per particle;
    # read d (3) + write y (3) fp64 words per active node
    return n_particles * 20 * word + n_active_nodes * 6 * 8


def fp32_variant(args):
    """The same C5 sub-step with the fp32 HVP variant (BASELINE.json configs[4] names fp32 and fp64;
    DESIGN.md R14: particle storage and HVP arithmetic fp32, node vectors and the gradient fp64),
    measured device-only in a child process of this bench (same steps / warm-up)."""
    import subprocess
    cmd = [sys.executable, os.path.abspath(__file__), "--precision", "f32", "--steps", str(args.steps), "--warmup",
           str(args.warmup), "--cells", str(args.cells), "--newton", str(args.newton), "--cg", str(args.cg), "--cg-variant", str(args.cg_variant),
           "--no-e2e", "--no-cpu-baseline", "--no-variants"]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal: the f64 line stands on its own
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"], "dtype": d["dtype"],
            "roofline": {k: d["roofline"].get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "avg_launch_ms",
                                                           "traffic", "hbm", "fp_pipe")},
            "kernel_ms_per_step": d["kernel_ms_per_step"], "clocks": d.get("clocks")}


def transfer_rooflines(fam, n_particles, n_active_nodes, word, peak, fp_peak=None):
    """Algorithmic HBM GB/s of the per-step transfer kernels (BASELINE.json metric "HVP/P2G HBM GB/s"),
    from the event-timed scopes (the sort runs inside the P2G scope).  Bytes per unit:
      sort  keys (read x: 3 words, write key + index: 8 B) + permute (read and write the 26-word SoA
            plus material, flag and id: 9 B) per particle;
      p2g   read the sorted 26-word SoA per particle, write m, mv, f^sigma (7 fp64) per active node;
      g2p   read x, F (12 words) and write x, v, F, B (24 words) per particle, read v (3 fp64) per
            active node;
      grad  SURVEY.md §8(d): 190 B (fp64) / 95 B (fp32) per particle per call (a4);
      pi    read m, v (4 fp64) per active fine node and its activity flag per box node (a9; the coarse
            accumulators are L2-resident)."""
    out = {}
    per_launch = {
        "sort": n_particles * (3 * word + 8 + 2 * (26 * word + 9)),
        "p2g": n_particles * 26 * word + n_active_nodes * 7 * 8,
        "g2p": n_particles * 36 * word + n_active_nodes * 3 * 8,
        "grad": n_particles * (190 if word == 8 else 95),
        "pi": n_active_nodes * 4 * 8 + int(n_active_nodes * 1.1),
    }
    s_n, s_ms = fam.get("sort", (0, 0.0))
    for k, by in per_launch.items():
        n, ms = fam.get(k, (0, 0.0))
        if k == "p2g":
            ms -= s_ms
        if not n or ms <= 0:
            continue
        gbs = by / (ms / n * 1e-3) / 1e9
        out[k] = {"achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                  "algorithmic_bytes_per_launch": by, "avg_launch_ms": ms / n}
        if fp_peak and k in SURVEY_FLOPS_PER_PARTICLE:
            fl = n_particles * SURVEY_FLOPS_PER_PARTICLE[k]
            tf = fl / (ms / n * 1e-3) / 1e12
            bound, t_hbm, t_fp = roofline_bound(by, fl, peak, fp_peak)
            out[k]["fp_pipe"] = {"achieved_tflops": tf, "peak_tflops": fp_peak, "frac": tf / fp_peak,
                                 "flops_per_particle": SURVEY_FLOPS_PER_PARTICLE[k], "accounting": "SURVEY.md §8(d)"}
            out[k]["bound"] = bound
            out[k]["floor_ms"] = max(t_hbm, t_fp) * 1e3
    return out


def load_traffic(prec):
    path = os.path.join(ROOT, "profiles", f"ncu_hvp_{prec}.json")
    if os.path.exists(path):
        try:
            return json.load(open(path)).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------------------------------------
# CPU oracle baseline (bounded sample)
# ------------------------------------------------------------------------------------------------

def oracle_substep_rate(cells, newton, cg):
    """Time the fp64 oracle, as it stands, on one bench step (the same recipe as the GPU arm: P2G, Pi onto
    the overlap grid, I + T onto the fine receivers as Dirichlet data, Newton with exactly `newton` x `cg`
    PCG, G2P) of a `cells`^3 C5 cube; the passive coarse grid's P2G is setup, as in the GPU arm."""
    import oracle
    import synth
    fine, coarse, recv = synth.c5_bench_workload(cells, full_box=False)
    gsc = oracle.p2g(coarse)
    t0 = time.perf_counter()
    gs = oracle.p2g(fine)
    oracle.project(fine.grid, gs, coarse.grid, eps_tol=1e-12)
    vS = oracle.interp(coarse.grid, gsc.v, 1.01 * gsc.v, 0.5, fine.grid, recv)
    dm = np.zeros((gs.m.shape[0], 3), np.uint8)
    dv = np.zeros((gs.m.shape[0], 3))
    dm[recv] = 1
    dv[recv] = vS
    u, st = oracle.implicit_solve(fine, gs, oracle.default_settings(max_newton=newton, max_cg=cg, fixed_iters=1),
                                  dirichlet_mask=dm, dirichlet_v=dv, raise_on_error=False)
    act = gs.active.astype(bool)
    oracle.g2p(fine, np.where(act[:, None], u / fine.dt, 0.0))
    dt = time.perf_counter() - t0
    return fine.particles.n / dt, dt, fine.particles.n


def run_reference(args, rank):
    if rank != 0:
        return
    cells = args.cpu_cells
    for _ in range(args.warmup):
        oracle_substep_rate(max(4, cells // 2), 1, 2)
    times = []
    n = 0
    for _ in range(args.steps):
        rate, dt, n = oracle_substep_rate(cells, args.newton, args.cg)
        times.append(dt)
    t = max(statistics.median(times), 1e-12)
    value = n / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5 sample: {cells}^3-cell cube, {n} particles, one bench step (P2G, Pi, I+T "
                               f"receivers, {args.newton} Newton x {args.cg} PCG, G2P)", "cells": cells},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{cells}^3-cell C5 cube ({n} particles), full sub-step per timed step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------

# ------------------------------------------------------------------------------------------------
# multi-GPU plumbing (one process per GPU): the library's NCCL communicator is
# bootstrapped through torch.distributed; timings are the max over ranks
# ------------------------------------------------------------------------------------------------

def share_unique_id(dist, rank, make_uid):
    """rank 0's 128-byte communicator id, broadcast to every rank."""
    obj = [make_uid() if rank == 0 else None]
    if dist is not None:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, value, device):
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, value, device):
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    if args.cg_variant is None:
        args.cg_variant = 1 if world > 1 or args.comm else 0
    dist = None
    if world > 1 or args.comm:
        import torch.distributed as tdist
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    else:
        torch.cuda.set_device(local_rank)
    from paper_2605_09097_b200 import osmpm

    dev = torch.device("cuda", local_rank)
    # one explicit stream for torch's tensor work and every library launch / NCCL call: the CUDA
    # events below then time exactly the library's work
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = osmpm.Context(local_rank, stream.cuda_stream)
    if world > 1 or args.comm:
        ctx.init_comm(rank, world, share_unique_id(dist, rank, osmpm.comm_unique_id))
    if args.slabs > 1:
        ctx.set_local_slabs(args.slabs)
    prec = osmpm.F64 if args.precision == "f64" else osmpm.F32
    word = 8 if args.precision == "f64" else 4

    fine, coarse, recv = build_workload(args.cells)
    n = fine.particles.n
    sub = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity, precision=prec)
    # the small coarse overlap grid is replicated on every rank (decompose=False)
    csub = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity,
                           precision=prec, decompose=False)
    slabs_total, _, _, n_local, cuts = sub.decomp()
    csub.p2g()
    cg = csub.read_grid(device=dev)
    # v_B^{n+1}: the smooth field advanced (scaled) in time -> distinct endpoint for T_m
    csub.set_grid_velocity((cg["v"] * 1.01).contiguous())
    recv_d = torch.from_numpy(recv).to(dev)
    settings = osmpm.newton_settings(max_newton=args.newton, max_cg=args.cg, fixed_iters=1, cg_variant=args.cg_variant)
    mask_all = torch.full((recv.shape[0],), 7, dtype=torch.uint8, device=dev)

    # a11: the step's initial particle state, restored at the start of every step (warm-up and timed
    # alike), as Alg. 1 restores the fine particles at every Schwarz iteration: every
    # step then does the identical work on the identical state
    sub.checkpoint()
    last_stats = {}

    def step(restore=True):
        if restore:
            sub.restore()
        sub.p2g()
        vb = osmpm.transmit(sub, csub, osmpm.FINE_TO_COARSE, alpha=0.0, eps_tol=1e-12, device=dev)
        vS = osmpm.transmit(csub, sub, osmpm.COARSE_TO_FINE, alpha=0.5, targets=recv_d, device=dev)
        sub.set_dirichlet_device(recv_d, mask_all, vS)
        st = sub.implicit_solve(settings)
        last_stats.update(newton_iters=st.newton_iters, cg_iters=st.cg_iters, ls_halvings=st.ls_halvings,
                          ls_failures=st.ls_failures, negcurv=st.negcurv)
        sub.g2p()
        return vb

    for w in range(args.warmup):
        # the last warm-up step runs with the event profiler on, so its events exist before timing
        ctx.profile(w == args.warmup - 1 and not args.no_prof)
        step()
    torch.cuda.synchronize(dev)
    sub.restore()
    sub.p2g()  # (untimed) grid of the step's initial state, for the active-node count of the roofline
    _, _, box_dims = sub.info()
    g = sub.read_grid(device=dev)
    n_active = int(g["active"].sum().item())  # this rank's owned nodes (decomposed reads)
    del g
    _, _, _, n_local, _ = sub.decomp()

    import gc
    gc.collect()
    gc.disable()  # no collector pauses inside the timed region (the step syncs with the host)
    clocks = ClockSampler(local_rank)
    ctx.profile(not args.no_prof)
    ctx.profile_reset()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ck = clocks.stop()
    launches_timed = ctx.launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    hv_n, hv_ms = ctx.kernel_time("hvp")
    fam = {f: ctx.kernel_time(f) for f in ("hvp", "grad", "energy", "p2g", "g2p", "sort", "cg", "pi", "interp")}
    ctx.profile(False)
    ms_max = max_over_ranks(dist, ms, dev)

    # end-to-end through the public API with pinned host buffers: every step uploads that step's
    # inputs (x, v, F, B from pinned host memory) and reads back its result (x, v into pinned host
    # memory).  The copies run on a second stream, double-buffered through device staging, so step
    # k+1's upload and step k's read-back overlap the compute of the neighbouring steps; the timed
    # region still contains every copy (it ends when the last read-back has landed).
    e2e = None
    if not args.no_e2e:
        fields = ("x", "v", "F", "B")
        pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(fine.particles, k))).pin_memory() for k in fields}
        outx = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        outv = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        h2d = sum(v.numel() * 8 for v in pin.values())
        d2h = (outx.numel() + outv.numel()) * 8
        stage = [{k: torch.empty(pin[k].shape, dtype=torch.float64, device=dev) for k in fields} for _ in range(2)]
        res = [{k: torch.empty((n, 3), dtype=torch.float64, device=dev) for k in ("x", "v")} for _ in range(2)]
        copy = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        landed = torch.cuda.Event()

        def upload(k):
            b = k % 2
            with torch.cuda.stream(copy):
                copy.wait_event(consumed[b])
                for f in fields:
                    stage[b][f].copy_(pin[f], non_blocking=True)
                ready[b].record(copy)

        def e2e_run(steps):
            for b in range(2):
                consumed[b].record(stream)
            upload(0)
            for k in range(steps):
                b = k % 2
                stream.wait_event(ready[b])
                sub.set_particles(stage[b]["x"], stage[b]["v"], stage[b]["F"], stage[b]["B"])
                consumed[b].record(stream)
                if k + 1 < steps:
                    upload(k + 1)
                step(restore=False)  # the upload replaces the restore
                sub.read_particles_into(x=res[b]["x"], v=res[b]["v"])
                done[b].record(stream)
                with torch.cuda.stream(copy):
                    copy.wait_event(done[b])
                    outx.copy_(res[b]["x"], non_blocking=True)
                    outv.copy_(res[b]["v"], non_blocking=True)
            landed.record(copy)
            stream.wait_event(landed)

        e2e_run(1)
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        e2e_run(args.steps)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        te = max_over_ranks(dist, f0.elapsed_time(f1) / args.steps, dev)
        # every rank uploads the full creation-order state (it keeps its own slab's particles) and
        # reads back its own particles into a full-size buffer
        e2e = {"value": n / (te * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "ms_per_step": te,
               "copies": "pinned host <-> device on a second stream, double-buffered, overlapping compute"}

    gc.enable()
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    fma_peak = ctx.measure_fma_peak(prec)
    hvp_bytes = hvp_algorithmic_bytes(n_local, n_active, word)  # rank 0's share per launch
    hvp_avg_ms = hv_ms / hv_n if hv_n else float("nan")
    achieved = hvp_bytes / (hvp_avg_ms * 1e-3) / 1e9 if hv_n else None
    traffic = load_traffic(args.precision)
    cpu = None
    if not args.no_cpu_baseline and world == 1:  # the oracle baseline: rank 0 at N = 1 only
        rate, dt, ncpu = oracle_substep_rate(args.cpu_cells, args.newton, args.cg)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"one bench step (P2G, Pi, I+T receivers, {args.newton} Newton x {args.cg} PCG, G2P) of a "
                         f"{args.cpu_cells}^3-cell C5 cube ({ncpu} particles), {dt:.1f} s single-threaded"}
    # The HVP's roofline: its algorithmic intensity (1256 flop per 190 B in fp64, 6.6
    # flop/B) lies above the B200's FP64 ridge (37.2 TFLOP/s / 6.45 TB/s = 5.8 flop/B), so the slower of
    # the two floors is the FP pipe's: bound "alu", against the FP vector peak derived from the guide's
    # unit counts and clock (148 SMs x 64 FP64 FMA lanes x 2 x 1.965 GHz; fp32 2x); the HBM fraction of
    # the same launches is reported beside it under "hbm".
    fp_nominal = FP64_PEAK_TFLOPS * (2 if word == 4 else 1)
    hvp_flops = n_local * HVP_FLOPS_PER_PARTICLE
    hbm_part = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if achieved else None,
                "peak_kind": peak_kind, "algorithmic_bytes_per_launch": hvp_bytes,
                "accounting": "SURVEY.md §8(d): 190 B/particle fp64 (95 fp32) x particles per launch",
                "reformulated_bytes_per_launch": hvp_reformulated_bytes(n_local, n_active, word)}
    if hv_n:
        bound, t_hbm, t_fp = roofline_bound(hvp_bytes, hvp_flops, peak, fp_nominal)
        tf = hvp_flops / (hvp_avg_ms * 1e-3) / 1e12
        hvp_roofline = {
            "bound": bound, "kernel": "k_hvp_sw", "avg_launch_ms": hvp_avg_ms, "launches": hv_n,
            "traffic": traffic, "traffic_source": f"profiles/ncu_hvp_{args.precision}.json (ncu --set full)",
            "floor_ms": {"hbm": t_hbm * 1e3, "fp_pipe": t_fp * 1e3},
            "hbm": hbm_part,
            "fp_pipe": {"achieved_tflops": tf, "peak_tflops": fp_nominal, "frac": tf / fp_nominal,
                        "flops_per_particle": HVP_FLOPS_PER_PARTICLE,
                        "peak_kind": "derived: 148 SMs x 64 FP64 FMA lanes/SM x 2 flops x 1.965 GHz (fp32 2x)",
                        "measured_peak_tflops": fma_peak,
                        "measured_frac": tf / fma_peak}}
        if bound == "alu":
            hvp_roofline.update({"achieved": tf, "peak": fp_nominal, "unit": "TFLOP/s", "frac": tf / fp_nominal})
        else:
            hvp_roofline.update({"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": hbm_part["frac"]})
    else:
        hvp_roofline = {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s", "frac": None, "hbm": hbm_part}
    line = {
        "metric": METRIC, "value": n / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        # the C5 sub-step is one fixed workload split over the ranks (halo exchange, all-reduces): strong
        "scaling": "strong",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": "C5 (BASELINE.json configs[4]): random-density neo-Hookean cube, 128^3 cells at "
                               "dx=1/512, 8 ppc, one fine implicit sub-step (10 Newton x 50 PCG) with "
                               "coarse<->fine transmission to the dx=1/128 overlap grid",
                   "particles": n, "particles_rank0": n_local, "cells": args.cells, "newton": args.newton,
                   "cg": args.cg, "cg_variant": args.cg_variant, "active_nodes_rank0": n_active, "box_nodes_rank0": int(np.prod(box_dims)),
                   "receivers": int(recv.shape[0]),
                   "state": "every step restores the checkpointed initial particle state (a11) first; "
                            "the e2e leg uploads it from pinned host memory instead",
                   "solve_stats_last_step": last_stats,
                   "parallelism": (f"x-slabs x{slabs_total} (NCCL over NVLink, {world} GPUs)" if world > 1
                                   else (f"x-slabs x{slabs_total} on one GPU" if slabs_total > 1 else "single GPU")),
                   "slab_cuts": cuts, "halo": args.halo,
                   "l2": "working set (>3 GB) far larger than the 126 MB L2; no flush needed"},
        "roofline": hvp_roofline,
        "kernel_ms_per_step": {f: v[1] / args.steps for f, v in fam.items()},
        "transfer_rooflines": transfer_rooflines(fam, n_local, n_active, word, peak, fp_nominal),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_timed,
        "clocks": ck,
    }
    if world == 1 and args.precision == "f64" and not args.no_variants and args.slabs == 1:
        line["variants"] = {"f32": fp32_variant(args)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
