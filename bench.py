"""Benchmark: space-time unknowns/s per preconditioned KKT solve (fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1] [--mode fast|strict|spectral] [--no-alt]

A "step" is one full right-preconditioned GMRES solve (two-level RASQ,
scalar coarse space) of BASELINE config 1 (127x127 interior, Nt=512, Nd=16,
omega=1e-3, GMRES(30), rtol 1e-8) from b resident in HBM to x in HBM, through
the C-ABI (kkt_gmres_solve).  value = N * 3*Nt*n_sp / (max-over-ranks device
time per solve).  e2e repeats the solve through kkt_gmres_solve_host with b
and x in pinned host memory (copies inside the timed region).

N > 1 is weak scaling over time slabs (the paper's own
weak-scaling axis): N GPUs solve config 1 extended in time, Nt = 512 N and
Nd = 16 N on the same T = 1 (m = 32 steps per subdomain as at N = 1), rank g
owning subdomains [16g, 16g+16) and their node slab — per-GPU work fixed.
Halo planes, the coarse all-gather and the Krylov dot all-gathers go through
NCCL (one communicator built by the library from a unique id that rank 0
broadcasts).  value = 3*Nt*n_sp / (max over ranks of the solve time).  (The
sweep's dependent chain, 65 lock-step time steps per P^-1 apply, does not
shorten when one config-1 solve is split over more GPUs, so strong scaling of
config 1 is not the meaningful axis.)

--impl reference times the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference by oracle/Makefile) on the host CPU: each step is a bounded
sample — GMRES iterations of the config-1 grid on a shortened time axis (Nt=64,
Nd=2, m=32 as in config 1) — scaled to a full config-1 solve by the per-iteration
cost's linearity in Nt and the reference's own iteration count.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2305_04421_b200 import problems as P  # noqa: E402

METRIC = "space-time unknowns/sec per preconditioned KKT solve (fp64)"
UNIT = "unknowns/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        d = json.load(open(PEAKS))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def workload_desc(cfg, p):
    return (f"config{cfg}: {p.nx_int}x{p.ny_int} interior, Nt={p.Nt}, Nd={p.Nd}, nu={p.nu}, "
            f"omega={p.omega}, two-level {p.coarse_variant} multiplicative (minus), "
            f"GMRES({p.restart}) rtol {p.tol}")


def mgs_model(p, iters, ranks=1, mode="fast"):
    """Algorithmic bytes and launches of the Gram-Schmidt passes of one solve
    (SURVEY.md §8d, K7), per GPU (the vectors split over the G slabs).
    FAST (krylov.cu, one-reduction MGS): iteration j reads w and v_0..v_j once
    for r = V^T w and the Gram row, then reads v_0..v_j and w and writes w for
    w -= V h: 2j + 5 vector passes; launches: ceil((j+1)/16) dots + 1 solve +
    ceil((j+1)/16) updates.  STRICT (reference MGS order): 4j + 5 passes, j + 2
    launches."""
    m = p.restart or p.max_iters
    vec = 3 * p.block * 8 // ranks
    js = [k % m for k in range(iters)]
    if mode == "strict":
        return sum((4 * j + 5) * vec for j in js), sum(j + 2 for j in js)
    return (sum((2 * j + 5) * vec for j in js),
            sum(2 * -(-(j + 1) // 16) + 1 for j in js))


def spectral_flops(p, ranks=1):
    """fp64 FLOPs of the four sine-transform passes of one Schur apply
    (spectral.cu): per plane X Sx (ny nx nx FMAs) and Sy Y (ny ny nx FMAs),
    forward and inverse."""
    ntl = p.Nt // ranks
    return 2 * 2 * ntl * p.n_sp * (p.nx_int + p.ny_int)


def sweep_bytes(p, ranks=1):
    """Algorithmic HBM bytes of one RASQ apply per GPU:
    every one of the 2Nt + Nd - 1 spatial solves reads b_k and x_{k-1}, writes
    and re-reads its L-solve intermediate and writes x_k (5 planes), and each
    of the 2m+1 lock-step solves streams the banded factor once,
    F = 8 * n_sp * (2 nx + 1) bytes (shared by all local subdomains)."""
    m = p.Nt // p.Nd
    planes = (2 * p.Nt + p.Nd - 1) * 5 * p.n_sp * 8 // ranks
    F = 8 * p.n_sp * (2 * p.nx_int + 1)
    return planes + (2 * m + 1) * F


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        return float(json.load(open(path))["dmma_tflops"]), "measured (profiles/fp64_peak.json, scripts/fp64_peak.cu)"
    except Exception:
        return None, "unmeasured"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.proc or not self.f:
            return None
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i in range(4) if r[i].lower().startswith("active")})
        loaded = [s for s, _, _ in rows if s > 300] or [s for s, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU reference (the reference arm and the cpu_baseline leg)
# ---------------------------------------------------------------------------
def reference_sample(cfg, iters_full, sample_iters=2, nt_sample=64, time_scale=1):
    """Time `sample_iters` GMRES iterations of the reference on the config grid
    with a shortened time axis (same m = Nt/Nd), and scale to a full solve
    (of the config extended `time_scale`-fold in time, as the N-GPU arm)."""
    from oracle.bindings import Ref
    p = P.config(cfg)
    if time_scale > 1:
        p = p.replace(Nt=p.Nt * time_scale, Nd=p.Nd * time_scale)
    m = p.Nt // p.Nd
    nd_s = max(1, nt_sample // m)
    ps = p.replace(Nt=nd_s * m, Nd=nd_s, max_iters=sample_iters, restart=p.restart)
    b = P.kkt_rhs(cfg, ps)
    t0 = time.perf_counter()
    ref = Ref(ps)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    out = ref.gmres_solve(b)
    t_solve = time.perf_counter() - t0
    # gmres_solve does `it` (K + P^-1) iterations, one LS P^-1 and one true-residual K
    per_iter = t_solve / (out["iterations"] + 1)
    scale = p.Nt / ps.Nt
    t_full = per_iter * scale * (iters_full + 1)
    value = 3 * p.Nt * p.n_sp / t_full
    sample = (f"reference (1 thread) on the config-{cfg} grid {p.nx_int}x{p.ny_int} with Nt={ps.Nt}, "
              f"Nd={ps.Nd} (m={m} as in config {cfg}), {out['iterations']} GMRES iterations in "
              f"{t_solve:.2f} s (+{t_setup:.2f} s setup); per-iteration cost scaled x{scale:g} in Nt and "
              f"to {iters_full} iterations (+1 final P^-1/K) => {t_full:.1f} s per full solve")
    return value, t_full, sample, t_solve + t_setup


def reference_iterations(cfg):
    path = os.path.join(ROOT, "tests", "golden", f"solve_c{cfg}_two-level_scalar.json")
    if os.path.exists(path):
        return int(json.load(open(path))["iterations"]), "reference golden record"
    return None, None


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    from oracle import bindings
    if not bindings.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkktdd_ref.so not built"}))
        return
    p = P.config(args.config)
    if ws > 1:  # the same (weak-scaled) workload as the N-GPU arm
        p = p.replace(Nt=p.Nt * ws, Nd=p.Nd * ws)
    iters, src = reference_iterations(args.config)
    if iters is None:
        iters, src = 60, "assumed (no golden record)"
    vals, times = [], []
    for i in range(args.warmup + args.steps):
        v, t_full, sample, wall = reference_sample(args.config, iters, time_scale=ws)
        if i >= args.warmup:
            vals.append(v)
            times.append(t_full)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 + Box-Muller, paper_2305_04421_b200/problems.py)",
        "config": {"workload": workload_desc(args.config, p), "iterations": iters,
                   "iterations_source": src},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# the device arm
# ---------------------------------------------------------------------------
def rank_rhs(cfg, p, k):
    """This rank's slab of b = [f_u; f_z; f] (kkt.cpp:21-48), generated only for
    the local nodes (the generator is counter-based, so slabs agree with the
    full field)."""
    nf, nl = k.node_first, k.node_last
    tgt, u0 = P.target_and_u0(cfg, p, n_lo=nf, n_hi=nl)
    L = (nl - nf + 1) * p.n_sp
    b = np.zeros(3 * L)
    b[:L] = (p.mass_scale * tgt).reshape(-1)
    if nf == 1:
        b[2 * L: 2 * L + p.n_sp] = u0
    return b

def run_ours(args, ws, rank, local):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    p = P.config(args.config)
    if ws > 1:  # weak scaling over time slabs: the same per-GPU slab, Nt and Nd x ws
        p = p.replace(Nt=p.Nt * ws, Nd=p.Nd * ws)
    unknowns = 3 * p.Nt * p.n_sp
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        from paper_2305_04421_b200.solver import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    k = HeatKKT(p, mode=args.mode, device=local, rank=rank, nranks=ws, nccl_id=nccl_id)
    b_host = rank_rhs(args.config, p, k)
    n = b_host.size
    b = torch.from_numpy(b_host).to(dev)
    x = torch.empty_like(b)

    for _ in range(args.warmup):
        out = k.gmres_solve(b, x)
    torch.cuda.synchronize()

    # ---- timed region: K solves, device time with CUDA events on the launch stream
    k.set_phase_timing(True)
    l0 = k.launch_count()
    iters = []
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            out = k.gmres_solve(b, x)
            iters.append(out.iterations)
        ev1.record()
        torch.cuda.synchronize()
    barrier(ws)
    launches = k.launch_count() - l0
    ms_total = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_total, ws)
    ms_step = ms_total / args.steps
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    value = unknowns / (ms_step / 1000.0)

    # ---- e2e through the host-buffer entry point (pinned memory)
    bh = torch.from_numpy(b_host).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    k.gmres_solve_host(bh.numpy(), xh.numpy())  # warm
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        k.gmres_solve_host(bh.numpy(), xh.numpy())
    e1.record()
    torch.cuda.synchronize()
    wall_e2e = (time.perf_counter() - w0) / e2e_steps
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / e2e_steps, ws)
    e2e_value = unknowns / (ms_e2e / 1000.0)

    # ---- rooflines.  Phase slot 3 brackets the RASQ sweep launches (one
    # CUDA-graph replay of the cluster LU chains per P^-1, sweep_v4.cu;
    # the transform GEMMs + mode recurrences in SPECTRAL mode), slot 2 the
    # Krylov Gram-Schmidt passes (krylov.cu).  `roofline` is the family with the
    # larger share of the step.
    peak, peak_src = hbm_peak()
    mgs_bytes, mgs_launches = mgs_model(p, iters[-1], ws, args.mode)
    mgs_ms = phase_ms[2] / args.steps
    achieved = mgs_bytes / (mgs_ms / 1000.0) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("mgs_axpy_dot_dram_bytes_per_launch")
        except Exception:
            traffic = None
    krylov = {
        "kernel": ("Krylov Gram-Schmidt passes: one-reduction MGS (cgs_dots_kernel, icwy_solve_kernel, cgs_update_kernel; krylov.cu)"
                   if args.mode != "strict" else "Krylov MGS passes (dot_seq_kernel, reference order; krylov.cu)"),
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "peak_source": peak_src,
        "algorithmic_bytes_per_launch": mgs_bytes / mgs_launches,
        "avg_launch_ms": mgs_ms / mgs_launches, "launches": mgs_launches * args.steps,
        "share_of_step": mgs_ms / max(1e-9, ms_step),
    }
    sw_ms = phase_ms[3] / max(1, phase_cnt[3])
    if args.mode == "spectral":
        tpk, tpk_src = fp64_peak()
        sp_tf = spectral_flops(p, ws) / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
        sweep = {
            "kernel": "SPECTRAL RASQ: 4 sine-transform GEMM passes (gemm_f64_kernel, mma.sync m8n8k4 f64) + per-mode recurrences (spectral.cu)",
            "bound": "tensor", "achieved": sp_tf, "peak": tpk, "unit": "TFLOP/s",
            "frac": (sp_tf / tpk) if (sp_tf and tpk) else None, "peak_source": tpk_src,
            "flops_per_apply": spectral_flops(p, ws), "avg_apply_ms": sw_ms,
            "applies": phase_cnt[3], "share_of_step": phase_ms[3] / max(1e-9, ms_total)}
    else:
        sb = sweep_bytes(p, ws)
        sw_gbs = sb / (sw_ms / 1000.0) / 1e9 if sw_ms > 0 else None
        sweep = {
            "kernel": ("RASQ sweep: group-parallel block-LU substitution chains, all local subdomains in lock step "
                       "(sweep_v4.cu: 8-CTA clusters, fp64 DMMA, one CUDA-graph replay per P^-1)" if args.mode == "fast" else
                       "RASQ sweep: reference-order banded substitution (sweep_strict.cu)"),
            "bound": "hbm", "achieved": sw_gbs, "peak": peak, "unit": "GB/s",
            "frac": (sw_gbs / peak) if sw_gbs else None, "traffic": None, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": sb, "avg_launch_ms": sw_ms, "launches": phase_cnt[3],
            "launch_unit": "one RASQ apply (one graph replay)",
            "share_of_step": phase_ms[3] / max(1e-9, ms_total),
            "note": "dependency-chain bound: 2m+1 lock-step spatial solves per apply, each a chain of block-row steps",
        }
        if os.path.exists(prof):
            try:
                sweep["traffic"] = json.load(open(prof)).get("sweep_dram_bytes_per_apply")
            except Exception:
                pass
    # K1 (apply_K_kernel, stencil.cu): 6 block-sized vectors per apply (u, z, w
    # read, three blocks written); the per-cycle restart residual
    # b - Kx moves 9 and is counted as 6 (conservative)
    k_ms = phase_ms[0] / max(1, phase_cnt[0])
    k_bytes = 6 * p.block * 8 // ws
    stencil = {
        "kernel": "K1 apply_K_kernel (5-point space-time stencil, stencil.cu)", "bound": "hbm",
        "achieved": k_bytes / (k_ms / 1000.0) / 1e9 if k_ms > 0 else None, "peak": peak, "unit": "GB/s",
        "frac": (k_bytes / (k_ms / 1000.0) / 1e9 / peak) if k_ms > 0 else None, "peak_source": peak_src,
        "algorithmic_bytes_per_launch": k_bytes, "avg_launch_ms": k_ms, "launches": phase_cnt[0],
        "share_of_step": phase_ms[0] / max(1e-9, ms_total)}
    fam = sorted([(krylov["share_of_step"], "krylov", krylov), (sweep["share_of_step"], "sweep", sweep)],
                 key=lambda t: -t[0])
    roofline, roofline_other = fam[0][2], fam[1][2]
    roofline["family"], roofline_other["family"] = fam[0][1], fam[1][1]

    # ---- the opt-in SPECTRAL variant (not the reference's spatial-solve method),
    # reported beside the headline, never as it
    alt = None
    if args.mode == "fast" and not args.no_alt:
        ks = HeatKKT(p, mode="spectral", device=local, rank=rank, nranks=ws, nccl_id=nccl_id)
        xs = torch.empty_like(b)
        for _ in range(2):
            o2 = ks.gmres_solve(b, xs)
        barrier(ws)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.steps):
            o2 = ks.gmres_solve(b, xs)
        a1.record()
        torch.cuda.synchronize()
        ms_alt = max_over_ranks(a0.elapsed_time(a1) / args.steps, ws)
        alt = {"mode": "spectral", "value": unknowns / (ms_alt / 1000.0), "ms_per_step": ms_alt,
               "iterations": o2.iterations, "true_final_relres": o2.true_final_relres,
               "note": "RASQ spatial solves in Ahat's sine eigenbasis (KKT_MODE_SPECTRAL): same operator to "
                       "rounding but not the reference's banded-LU method, so not the headline"}
        del ks

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 + Box-Muller target, paper_2305_04421_b200/problems.py)",
        "config": {
            "workload": workload_desc(args.config, p), "mode": args.mode,
            "iterations": iters[-1], "iterations_all": sorted(set(iters)),
            "true_final_relres": out.true_final_relres,
            "parallelism": (f"time slabs x{ws} (Nd/{ws} subdomains per GPU, NCCL halos + all-gathers)"
                            if ws > 1 else "1 GPU"),
            "l2": "KKT vectors are 198 MB each (> 126 MB L2); no flush between solves",
            "phase_ms_per_step": {"K": phase_ms[0] / args.steps, "P_inv": phase_ms[1] / args.steps,
                                  "krylov_vectors": phase_ms[2] / args.steps,
                                  "sweep_kernel": phase_ms[3] / args.steps},
        },
        "roofline": roofline,
        "roofline_secondary": roofline_other,
        "roofline_stencil": stencil,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_e2e, "wall_ms_per_step": 1000 * wall_e2e},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if alt is not None:
        line["alt_spectral"] = alt
    if ws == 1 and not args.no_c2 and args.mode == "fast" and args.config == 1:
        try:
            line["microbench_c2"] = c2_microbench(local)
        except Exception as e:  # reported beside the headline, never required
            line["microbench_c2"] = {"error": str(e)}
    if ws == 1 and args.c4 and args.mode == "fast" and args.config == 1:
        try:
            line["microbench_c4_slab"] = c4_microbench(local)
        except Exception as e:  # reported beside the headline, never required
            line["microbench_c4_slab"] = {"error": str(e)}
    if not args.no_cpu_baseline and ws == 1:
        try:
            from oracle import bindings
            if bindings.available("ref"):
                v, t_full, sample, wall = reference_sample(args.config, iters[-1])
                line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                                        "sample": sample, "host_nproc": os.cpu_count()}
            else:
                line["cpu_baseline"] = None
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line))


def c2_microbench(local, reps=10):
    """BASELINE config 2, the preconditioner-apply microbench: 10 applications
    of P^-1 at 511^2 x 1024 steps, 64 subdomains, on seeded N(0,1) KKT vectors
    (device-generated here: timing only; parity is tests/test_gpu_large.py and
    tests/test_gpu_v5.py, tests/test_gpu_v6.py).  The sweep runs sweep_v6.cu
    (device-wide fp64 DMMA block substitution), so its roofline is the fp64
    tensor peak."""
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    dev = torch.device("cuda", local)
    p = P.config(2)
    t0 = time.perf_counter()
    k = HeatKKT(p, mode="fast", device=local)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    g = torch.Generator(device=dev).manual_seed(2)
    v = torch.randn(3 * p.block, dtype=torch.float64, device=dev, generator=g)
    out = torch.empty_like(v)
    k.apply_P_inv(v, out)
    torch.cuda.synchronize()
    k.set_phase_timing(True)
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        k.apply_P_inv(v, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    ts.sort()
    med = ts[len(ts) // 2]
    sw_ms = phase_ms[3] / max(1, phase_cnt[3])
    # v5/v6 arithmetic per RASQ apply: every block row of every spatial solve does
    # the dense on-chain product (G_J / H_J: nx^2 MACs per chain) and the
    # off-chain triangle (Li_J / Ui_J: nx^2/2), both sweep directions
    nx, ny, m = p.nx_int, p.ny_int, p.Nt // p.Nd
    flops = 2.0 * 2 * 1.5 * nx * nx * ny * p.Nd * (2 * m + 1)
    tpk, tpk_src = fp64_peak()
    tf = flops / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
    res = {"workload": workload_desc(2, p), "applications": reps, "setup_s": setup_s,
           "ms_per_apply_median": med, "ms_per_apply_min": ts[0],
           "value": 3 * p.block / (med / 1000.0), "unit": "unknowns/s per P^-1 apply",
           "sweep_ms_per_apply": sw_ms,
           "roofline": {"kernel": "v6_chain_kernel<512> + v6_off_kernel<512> (sweep_v6.cu: device-wide fp64 DMMA block substitution)",
                        "bound": "tensor", "achieved": tf, "peak": tpk, "unit": "TFLOP/s",
                        "frac": (tf / tpk) if (tf and tpk) else None, "peak_source": tpk_src,
                        "flops_per_apply": flops},
           "inputs": "device-generated N(0,1) (torch, seed 2); parity at this size: tests/test_gpu_large.py"}
    del k, v, out
    torch.cuda.empty_cache()
    return res


def c4_microbench(local, reps=3):
    """BASELINE config 4 (1023^2 interior, 8 GPUs) on the one GPU this pool
    has: one rank's time slab at G = 8 -- 16 subdomains of m = 8 steps,
    Nt = 128 with config 4's dt = 1/1024 (T = 1/8) -- and P^-1 applications on
    seeded N(0,1) KKT vectors (device-generated: timing only; parity of the
    kernels at nx = 1023: tests/test_gpu_v6.py).  The sweep runs sweep_v6.cu
    (device-wide block substitution, fp64 DMMA).  Opt-in (--c4): the block
    recursion's setup takes ~40 s at nx = 1023."""
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    dev = torch.device("cuda", local)
    p = P.config(4).replace(Nt=128, Nd=16, T=0.125)
    t0 = time.perf_counter()
    k = HeatKKT(p, mode="fast", device=local)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    g = torch.Generator(device=dev).manual_seed(4)
    v = torch.randn(3 * p.block, dtype=torch.float64, device=dev, generator=g)
    out = torch.empty_like(v)
    k.apply_P_inv(v, out)
    torch.cuda.synchronize()
    k.set_phase_timing(True)
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        k.apply_P_inv(v, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    ts.sort()
    med = ts[len(ts) // 2]
    sw_ms = phase_ms[3] / max(1, phase_cnt[3])
    nx, ny, m = p.nx_int, p.ny_int, p.Nt // p.Nd
    flops = 2.0 * 2 * 1.5 * nx * nx * ny * p.Nd * (2 * m + 1)
    tpk, tpk_src = fp64_peak()
    tf = flops / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
    res = {"workload": "config4 per-GPU slab at G=8: 1023x1023 interior, Nt=128 (dt=1/1024 as config 4), "
                       "Nd=16 (m=8), nu=1, omega=1e-4, two-level scalar multiplicative (minus)",
           "applications": reps, "setup_s": setup_s,
           "ms_per_apply_median": med, "ms_per_apply_min": ts[0],
           "value": 3 * p.block / (med / 1000.0), "unit": "unknowns/s per P^-1 apply",
           "sweep_ms_per_apply": sw_ms,
           "roofline": {"kernel": "v6_chain_kernel + v6_off_kernel (sweep_v6.cu: device-wide fp64 DMMA block substitution)",
                        "bound": "tensor", "achieved": tf, "peak": tpk, "unit": "TFLOP/s",
                        "frac": (tf / tpk) if (tf and tpk) else None, "peak_source": tpk_src,
                        "flops_per_apply": flops},
           "inputs": "device-generated N(0,1) (torch, seed 4); parity at nx = 1023: tests/test_gpu_v6.py"}
    del k, v, out
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--mode", default="fast", choices=["fast", "strict", "spectral"])
    ap.add_argument("--no-alt", action="store_true", help="skip the SPECTRAL side measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the config-2 P^-1 microbench")
    ap.add_argument("--c4", action="store_true", help="add the config-4 per-GPU-slab P^-1 microbench (~40 s setup)")
    args = ap.parse_args()
    ws, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference_arm(args, ws, rank)
        else:
            run_ours(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
