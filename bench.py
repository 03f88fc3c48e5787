"""Benchmark: space-time unknowns/s per preconditioned KKT solve (fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--nd ND] [--mode fast|strict|spectral] [--no-extras]

Headline workload (BASELINE.json configs[2], the largest single-GPU config:
802 M space-time unknowns): the preconditioner-apply microbench -- 511x511
interior, Nt = 1024, nu = 0.1, omega = 1e-2, 64 time subdomains, two-level RASQ
with the scalar coarse space (multiplicative form, minus sign) -- applications
of P^-1 (kkt.cpp:71-81) to a seeded N(0,1) KKT vector (u, z, lambda blocks;
problems.random_kkt).  A "step" is ONE P^-1 APPLICATION over all 802 M unknowns,
input and output resident in HBM, through the C-ABI (kkt_apply_P_inv); value =
3*Nt*n_sp / (max-over-ranks device time per application), the rate SURVEY.md
section 8d defines for this config.  e2e repeats the application through
kkt_apply_P_inv_host with both vectors in pinned host memory (H2D + D2H inside
the timed region).

Why not config 3's full GMRES(20) solve (VERDICT r1 asked for it): on config 3's
own seeded inputs GMRES(20) does not converge for any of its subdomain counts
(Nd = 8, 16, 32: relative residual 0.06-0.08 after 100 iterations, 9.75 after 420
at Nd = 32; profiles/solve_c3_nd*_r02.json), and STRICT mode -- bitwise the
reference -- stagnates the same way on the same grid, time step and window
length (profiles/diag_c3solve_m128_r02.log).  A step that never converges is a
420-iteration, 147 s run: 25 of them do not fit the driver's limit and would
measure a failed solve.  `--config 3` still runs it (one step = one solve, capped
by max_iters), `--config 3 --pinv` times its P^-1; the default line carries
config 3's P^-1 and config 1's full converged solve as extra keys.

N > 1 is STRONG scaling over time slabs of the same workload: rank g owns
subdomains [g*Nd/N, (g+1)*Nd/N) and their node slab; the halo plane and the
coarse all-gather of every application (and the Krylov dot all-gathers of a
solve) go through NCCL (one communicator built by the library from a unique id
that rank 0 broadcasts).  Launched without WORLD_SIZE, `--gpus N` re-executes
itself under torchrun with N ranks (127.0.0.1 rendezvous); n_gpus in the JSON
line is the number of ranks that ran.

--impl reference times the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference by oracle/Makefile; it is single-threaded by construction) on
the host CPU.  One P^-1 at config 2 takes it ~1.2 h after ~2 h of setup
(SURVEY.md section 8c), so each step times a BOUNDED sample -- apply_shat and
apply_rasq (and apply_K for the solve workloads) once each on the config's grid
with a 2-node time axis -- and `value` extrapolates it by operation counts
(SURVEY.md section 8d allows this for C2-C4; flagged `extrapolated`).
`ms_per_step` is the measured sample time, not the extrapolated one.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
DATA = "synthetic (seeded SplitMix64 + Box-Muller target, paper_2305_04421_b200/problems.py)"


def hbm_peak():
    try:
        d = json.load(open(PEAKS))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        return float(json.load(open(path))["dmma_tflops"]), "builder-measured (profiles/fp64_peak.json, scripts/fp64_peak.cu; not in MEASURED_PEAKS.json)"
    except Exception:
        return None, "unmeasured"


def ncu_summary(key):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get(key)
    except Exception:
        return None


def workload_desc(cfg, p, kind="solve"):
    base = (f"config{cfg}: {p.nx_int}x{p.ny_int} interior, Nt={p.Nt}, Nd={p.Nd}, nu={p.nu}, "
            f"omega={p.omega}, two-level {p.coarse_variant} multiplicative (minus)")
    if kind == "pinv":
        return base + "; one step = one P^-1 application on a seeded N(0,1) KKT vector"
    return base + f", GMRES({p.restart}) rtol {p.tol}; one step = one full solve"


def workload_kind(args):
    return "pinv" if (args.config == 2 or args.pinv) else "solve"


# ---------------------------------------------------------------------------
# algorithmic byte / flop models, per GPU
# ---------------------------------------------------------------------------
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


def sweep_flops(p, ranks=1):
    """Algorithmic fp64 FLOPs of one RASQ apply per GPU: the
    banded-LU substitution of each of the 2Nt + Nd - 1 spatial solves,
    4 * n_sp * nx."""
    return (2 * p.Nt + p.Nd - 1) * 4.0 * p.n_sp * p.nx_int / ranks


def sweep_block_row_steps(p):
    """Dependent block-row steps of one RASQ apply: 2m+1 lock-step spatial
    solves, each an L chain and a U chain over the ny block rows."""
    m = p.Nt // p.Nd
    return (2 * m + 1) * 2 * p.ny_int


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
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


# ---------------------------------------------------------------------------
# launching: one process per GPU
# ---------------------------------------------------------------------------
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`python bench.py --gpus N` without a torchrun environment: start the N
    ranks ourselves, as the driver's multi-GPU launch does."""
    if not args.probe_ranks:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} requested but {n} CUDA device(s) visible; "
                                       "not falling back to fewer ranks"}))
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def dist_init(ws, local, backend="nccl"):
    if ws <= 1:
        return
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # the driver reads nranks from the init lines
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")


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


def probe_ranks(ws, rank):
    """--probe-ranks (tests/test_bench_launch.py, CPU): every started rank joins a
    gloo group and rank 0 prints how many did."""
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist_init(ws, 0, backend="gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    else:
        n = 1
    if rank == 0:
        print(json.dumps({"probe": True, "n_gpus": ws, "ranks_started": n, "pid": os.getpid()}))


# ---------------------------------------------------------------------------
# CPU reference (the reference arm and the cpu_baseline leg)
# ---------------------------------------------------------------------------
REF_ITER_RECORDS = {3: os.path.join(ROOT, "profiles", "solve_c3_nd32_r02.json")}


def recorded_iterations(cfg, nd):
    """Iterations of the full solve, for the extrapolation of the reference arm:
    the reference's own golden record where it could run the solve (configs 0,
    1), else the committed device run on the same inputs (FAST takes the
    reference's count +-1 wherever both ran)."""
    path = os.path.join(ROOT, "tests", "golden", f"solve_c{cfg}_two-level_scalar.json")
    if os.path.exists(path):
        return int(json.load(open(path))["iterations"]), "reference golden record"
    path = REF_ITER_RECORDS.get(cfg)
    if path and os.path.exists(path):
        rec = json.load(open(path))
        if rec.get("Nd") == nd:
            return int(rec["iterations"]), f"device run on the same inputs ({os.path.relpath(path, ROOT)})"
    return None, None


class ReferenceSample:
    """The reference's per-operation costs on the config's grid with a short time
    axis (Nt_s nodes, Nd_s subdomains), and their extrapolation by operation counts.

    P^-1 (two-level multiplicative, kkt.cpp:71-81, schur.cpp:415-444) is
    apply_shat + apply_rasq + O(B) work; apply_shat (and apply_K) cost 2 Nt
    band_matvecs (linear in Nt), apply_rasq does 2 (Nt + 2 (Nd - 1)) banded solves
    (schur.cpp:103-130).  A solve with `it` iterations in `cyc` restart cycles
    applies P^-1 and K it + cyc times each (gmres.cpp:79-80, :134-141, :147-153).
    The coarse solve and the MGS dots/axpys are left out, which favours the
    reference."""

    def __init__(self, cfg, p, kind, nt_s=2, nd_s=1):
        from oracle.bindings import Ref
        self.cfg, self.p, self.kind = cfg, p, kind
        self.ps = p.replace(Nt=nt_s, Nd=nd_s, T=p.T * nt_s / p.Nt)  # the config's dt
        t0 = time.perf_counter()
        self.ref = Ref(self.ps)
        self.setup_s = time.perf_counter() - t0
        self.v = P.random_kkt(self.ps, 0)

    def step(self):
        B = self.ps.block
        t = {}
        if self.kind == "solve":
            t0 = time.perf_counter()
            self.ref.apply_K(self.v)
            t["apply_K"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        self.ref.apply_shat(self.v[2 * B:])
        t["apply_shat"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        self.ref.apply_rasq(self.v[2 * B:])
        t["apply_rasq"] = time.perf_counter() - t0
        return t

    def extrapolate(self, t, iters=None):
        p, ps = self.p, self.ps
        lin = p.Nt / ps.Nt
        rasq = (p.Nt + 2 * (p.Nd - 1)) / (ps.Nt + 2 * (ps.Nd - 1))
        pinv = t["apply_shat"] * lin + t["apply_rasq"] * rasq
        if self.kind == "pinv":
            return pinv
        restart = p.restart or p.max_iters
        cyc = -(-iters // restart)
        return (pinv + t["apply_K"] * lin) * (iters + cyc)

    def describe(self, t, t_full, iters=None):
        ps = self.ps
        ops = ", ".join(f"{k} {v:.2f} s" for k, v in t.items())
        what = (f"one P^-1 at Nt={self.p.Nt}, Nd={self.p.Nd}" if self.kind == "pinv" else
                f"Nt={self.p.Nt}, Nd={self.p.Nd} and {iters} iterations (+ one P^-1/K per restart cycle)")
        return (f"reference (1 thread) on config {self.cfg}'s grid {ps.nx_int}x{ps.ny_int} with Nt={ps.Nt}, Nd={ps.Nd} "
                f"(the config's dt): {ops} per step (setup {self.setup_s:.1f} s, excluded like the device's); "
                f"EXTRAPOLATED by operation counts to {what}: {t_full:.0f} s")


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return  # rank 0 alone runs the CPU reference; the others exit 0 without work
    from oracle import bindings
    if not bindings.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkktdd_ref.so not built"}))
        return
    kind = workload_kind(args)
    p = P.config(args.config, Nd=args.nd)
    iters, src = None, None
    if kind == "solve":
        iters, src = recorded_iterations(args.config, p.Nd)
        if iters is None:
            iters, src = 120, "assumed (no record)"
    rs = ReferenceSample(args.config, p, kind)
    secs, fulls = [], []
    t = None
    for i in range(args.warmup + args.steps):
        t = rs.step()
        if i >= args.warmup:
            secs.append(sum(t.values()))
            fulls.append(rs.extrapolate(t, iters))
    t_full = statistics.median(fulls)
    value = 3 * p.block / t_full
    cfgd = {"workload": workload_desc(args.config, p, kind),
            "note": "ms_per_step is the measured bounded sample; value = unknowns / extrapolated time of the full step"}
    if kind == "solve":
        cfgd.update({"iterations": iters, "iterations_source": src})
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws if ws > 1 else args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "extrapolated": True, "ms_per_full_step_extrapolated": 1000 * t_full,
        "config": cfgd,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": rs.describe(t, t_full, iters), "host_nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# the device arm
# ---------------------------------------------------------------------------
def rank_rhs(cfg, p, node_first, node_last):
    """This rank's slab of b = [f_u; f_z; f] (kkt.cpp:21-48), generated only for
    the local nodes (the generator is counter-based, so slabs agree with the
    full field)."""
    tgt, u0 = P.target_and_u0(cfg, p, n_lo=node_first, n_hi=node_last)
    L = (node_last - node_first + 1) * p.n_sp
    b = np.zeros(3 * L)
    b[:L] = (p.mass_scale * tgt).reshape(-1)
    if node_first == 1:
        b[2 * L: 2 * L + p.n_sp] = u0
    return b


def rank_random_kkt(p, kidx, node_first, node_last):
    """This rank's slab [u; z; w] of config 2's k-th seeded N(0,1) KKT vector
    (problems.random_kkt: element i of the global vector from counter i)."""
    nsp, B = p.n_sp, p.block
    L = (node_last - node_first + 1) * nsp
    off = (node_first - 1) * nsp
    v = np.empty(3 * L)
    for blk in range(3):
        v[blk * L:(blk + 1) * L] = P.normal(P.SEED + 2, 100 + kidx, L, offset=blk * B + off)
    return v


def timed_solves(k, b, x, steps, ws):
    """`steps` solves bracketed by a barrier + synchronize, CUDA events on the
    current stream (HeatKKT fences its own stream against it on both sides)."""
    import torch
    iters = []
    barrier(ws)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    out = None
    for _ in range(steps):
        out = k.gmres_solve(b, x)
        iters.append(out.iterations)
    ev1.record()
    torch.cuda.synchronize()
    barrier(ws)
    return max_over_ranks(ev0.elapsed_time(ev1), ws), iters, out


def rooflines(p, ws, mode, iters, steps, ms_total, phase_ms, phase_cnt, v6):
    """roofline (dominant family), roofline_secondary, roofline_stencil."""
    peak, peak_src = hbm_peak()
    ms_step = ms_total / steps
    mgs_bytes, mgs_launches = mgs_model(p, iters, ws, mode)
    mgs_ms = phase_ms[2] / steps
    achieved = mgs_bytes / (mgs_ms / 1000.0) / 1e9 if mgs_ms > 0 else None
    krylov = {
        "kernel": ("Krylov Gram-Schmidt passes: one-reduction MGS (cgs_dots_kernel, icwy_solve_kernel, cgs_update_kernel; krylov.cu)"
                   if mode != "strict" else "Krylov MGS passes (dot_seq_kernel, reference order; krylov.cu)"),
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None,
        "traffic": ncu_summary("cgs_dram_bytes_per_launch"), "peak_source": peak_src,
        "algorithmic_bytes_per_launch": mgs_bytes / max(1, mgs_launches),
        "avg_launch_ms": mgs_ms / max(1, mgs_launches), "launches": mgs_launches * steps,
        "share_of_step": mgs_ms / max(1e-9, ms_step), "family": "krylov",
    }
    sw_ms = phase_ms[3] / max(1, phase_cnt[3])
    if mode == "spectral":
        tpk, tpk_src = fp64_peak()
        sp_tf = spectral_flops(p, ws) / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
        sweep = {
            "kernel": "SPECTRAL RASQ: 4 sine-transform GEMM passes (gemm_f64_kernel, mma.sync m8n8k4 f64) + per-mode recurrences (spectral.cu)",
            "bound": "tensor", "achieved": sp_tf, "peak": tpk, "unit": "TFLOP/s",
            "frac": (sp_tf / tpk) if (sp_tf and tpk) else None, "peak_source": tpk_src,
            "flops_per_apply": spectral_flops(p, ws), "avg_apply_ms": sw_ms,
            "applies": phase_cnt[3], "share_of_step": phase_ms[3] / max(1e-9, ms_total), "family": "sweep"}
    else:
        sb = sweep_bytes(p, ws)
        sw_gbs = sb / (sw_ms / 1000.0) / 1e9 if sw_ms > 0 else None
        tpk, tpk_src = fp64_peak()
        fl = sweep_flops(p, ws)
        tf = fl / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
        rows = sweep_block_row_steps(p)
        if mode == "strict":
            kname = "RASQ sweep: reference-order banded substitution (sweep_strict.cu)"
        elif v6:
            kname = ("RASQ sweep v6 (sweep_v6.cu): v6_chain_kernel (device-wide dependent block-row chain, fp64 DMMA, "
                     "release-counter handoff) + v6_off_kernel (batched triangular products) + v6_form_b_kernel, "
                     "all local subdomains in lock step")
        else:
            kname = ("RASQ sweep v4 (sweep_v4.cu): group-parallel block-LU substitution chains, 8-CTA clusters, "
                     "fp64 DMMA, one CUDA-graph replay per P^-1")
        sweep = {
            "kernel": kname, "bound": "hbm", "achieved": sw_gbs, "peak": peak, "unit": "GB/s",
            "frac": (sw_gbs / peak) if sw_gbs else None,
            "traffic": ncu_summary("sweep_v6_c3_dram_bytes_per_apply" if v6 else "sweep_dram_bytes_per_apply"),
            "peak_source": peak_src, "algorithmic_bytes_per_launch": sb, "avg_launch_ms": sw_ms,
            "launches": phase_cnt[3], "launch_unit": "one RASQ apply (all its sweep kernels)",
            "share_of_step": phase_ms[3] / max(1e-9, ms_total), "family": "sweep",
            "fp64": {"flops_per_apply": fl, "achieved_tflops": tf, "peak_tflops": tpk,
                     "frac": (tf / tpk) if (tf and tpk) else None, "peak_source": tpk_src,
                     "flops_source": "SURVEY §8(a20): (2Nt + Nd - 1) * 4 * n_sp * nx (banded substitution)"},
            "chain": {"dependent_block_row_steps_per_apply": rows,
                      "us_per_block_row_step": 1000.0 * sw_ms / rows if sw_ms > 0 else None,
                      "handoff_floor_us": ncu_summary("v6_row_handoff_floor_us"),
                      "note": "the sweep is bound by this dependent chain: (2m+1) lock-step spatial solves x 2 "
                              "directions x ny block rows, each waiting for the previous row of its chain"},
        }
    k_ms = phase_ms[0] / max(1, phase_cnt[0])
    k_bytes = 6 * p.block * 8 // ws
    stencil = {
        "kernel": "K1 apply_K_kernel (5-point space-time stencil, stencil.cu)", "bound": "hbm",
        "achieved": k_bytes / (k_ms / 1000.0) / 1e9 if k_ms > 0 else None, "peak": peak, "unit": "GB/s",
        "frac": (k_bytes / (k_ms / 1000.0) / 1e9 / peak) if k_ms > 0 else None, "peak_source": peak_src,
        "traffic": ncu_summary("apply_K_dram_bytes_per_launch"),
        "algorithmic_bytes_per_launch": k_bytes, "avg_launch_ms": k_ms, "launches": phase_cnt[0],
        "share_of_step": phase_ms[0] / max(1e-9, ms_total)}
    fam = sorted([krylov, sweep], key=lambda d: -d["share_of_step"])
    return fam[0], fam[1], stencil


def run_solve(args, ws, rank, local):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    p = P.config(cfg, Nd=args.nd)
    scaling = "strong"
    if ws > 1 and args.weak:  # weak scaling over time slabs: the same per-GPU slab, Nt and Nd x ws
        p = p.replace(Nt=p.Nt * ws, Nd=p.Nd * ws)
        scaling = "weak"
    if p.Nd % ws:
        raise SystemExit(f"time-slab sharding needs the rank count to divide Nd (Nd={p.Nd}, ranks={ws})")
    unknowns = 3 * p.Nt * p.n_sp
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        from paper_2305_04421_b200.solver import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t0 = time.perf_counter()
    k = HeatKKT(p, mode=args.mode, device=local, rank=rank, nranks=ws, nccl_id=nccl_id)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    b_host = rank_rhs(cfg, p, k.node_first, k.node_last)
    n = b_host.size
    b = torch.from_numpy(b_host).to(dev)
    x = torch.empty_like(b)

    for _ in range(args.warmup):
        k.gmres_solve(b, x)
    torch.cuda.synchronize()

    # ---- timed region: K solves, device time with CUDA events, max over ranks
    k.set_phase_timing(True)
    l0 = k.launch_count()
    with ClockSampler(local) as clk:
        ms_total, iters, out = timed_solves(k, b, x, args.steps, ws)
    launches = k.launch_count() - l0
    ms_step = ms_total / args.steps
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    value = unknowns / (ms_step / 1000.0)
    relres = out.true_final_relres
    converged = out.converged
    mem_gb = (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9

    # ---- e2e through the host-buffer entry point (pinned memory).  The device
    # copies of b and x are released first: at config 3 one GPU holds 160 GB of
    # Krylov basis and work vectors, and kkt_gmres_solve_host stages its own.
    del b, x, out
    torch.cuda.empty_cache()
    bh = torch.from_numpy(b_host).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    e2e_steps = 1 if ms_step > 5000 else max(1, min(args.steps, 3))
    if ms_step <= 5000:
        k.gmres_solve_host(bh.numpy(), xh.numpy())  # warm (the big configs are warm from the timed region)
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(e2e_steps):
        k.gmres_solve_host(bh.numpy(), xh.numpy())
    e1.record()
    torch.cuda.synchronize()
    wall_e2e = (time.perf_counter() - w0) / e2e_steps
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / e2e_steps, ws)
    e2e_value = unknowns / (ms_e2e / 1000.0)
    del bh, xh

    v6 = args.mode == "fast" and p.nx_int > 128
    roofline, roofline_other, stencil = rooflines(p, ws, args.mode, iters[-1], args.steps, ms_total,
                                                  phase_ms, phase_cnt, v6)
    del k
    torch.cuda.empty_cache()
    if rank != 0:
        return
    vec_mb = 3 * p.block * 8 / ws / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": {
            "workload": workload_desc(cfg, p), "mode": args.mode,
            "iterations": iters[-1], "iterations_all": sorted(set(iters)), "converged": bool(converged),
            "true_final_relres": relres,
            "parallelism": (f"time slabs x{ws} ({p.Nd // ws} of {p.Nd} subdomains per GPU, NCCL halos + all-gathers)"
                            if ws > 1 else "1 GPU"),
            "l2": f"KKT vectors are {vec_mb:.0f} MB each per GPU (> 126 MB L2); no flush between solves",
            "setup_s": setup_s, "device_mem_GB": mem_gb,
            "phase_ms_per_step": {"K": phase_ms[0] / args.steps, "P_inv": phase_ms[1] / args.steps,
                                  "krylov_vectors": phase_ms[2] / args.steps,
                                  "sweep_kernels": phase_ms[3] / args.steps},
        },
        "roofline": roofline,
        "roofline_secondary": roofline_other,
        "roofline_stencil": stencil,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_e2e, "wall_ms_per_step": 1000 * wall_e2e,
                "steps": e2e_steps},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_extras and args.mode == "fast":
        if cfg != 1:
            try:
                line["config1"] = config1_extra(local)
            except Exception as e:  # reported beside the headline, never required
                line["config1"] = {"error": str(e)}
        try:
            line["microbench_c2"] = c2_microbench(local)
        except Exception as e:
            line["microbench_c2"] = {"error": str(e)}
        if args.c4:
            try:
                line["microbench_c4_slab"] = c4_microbench(local)
            except Exception as e:
                line["microbench_c4_slab"] = {"error": str(e)}
    if not args.no_cpu_baseline and ws == 1:
        try:
            from oracle import bindings
            if bindings.available("ref"):
                rs = ReferenceSample(cfg, p, "solve")
                t = rs.step()
                t_full = rs.extrapolate(t, iters[-1])
                line["cpu_baseline"] = {"value": 3 * p.block / t_full, "unit": UNIT, "cores": 1, "kind": "reference",
                                        "sample": rs.describe(t, t_full, iters[-1]), "extrapolated": True,
                                        "host_nproc": os.cpu_count()}
            else:
                line["cpu_baseline"] = None
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line))


def pinv_rooflines(p, ws, ms_apply, sw_ms, napplies):
    """roofline (the RASQ sweep: 98% of a P^-1 application) and roofline_secondary
    (the rest: P^-1's u/z blocks, node sums, coarse solve)."""
    peak, peak_src = hbm_peak()
    tpk, tpk_src = fp64_peak()
    fl, sb, rows = sweep_flops(p, ws), sweep_bytes(p, ws), sweep_block_row_steps(p)
    tf = fl / (sw_ms / 1000.0) / 1e12 if sw_ms > 0 else None
    gbs = sb / (sw_ms / 1000.0) / 1e9 if sw_ms > 0 else None
    v4 = p.nx_int <= 128
    sweep = {
        "kernel": ("RASQ sweep v4 (sweep_v4.cu): group-parallel block-LU substitution chains, 8-CTA clusters, fp64 DMMA"
                   if v4 else
                   "RASQ sweep v6 (sweep_v6.cu): v6_chain(w)_kernel (device-wide dependent block-row chain of the two-sided "
                   "block elimination in its inverse-block form, groups of k rows, fp64 DMMA over the operators' numerical "
                   "band, prefetched slot handoff) + v6_mid_kernel (the middle row, the first row) + v6_inner_kernel "
                   "(zero-inflow chains inside the groups, k > 1) + v6_form_b_kernel, all local subdomains in lock step"),
        "bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": (gbs / peak) if gbs else None,
        "traffic": ncu_summary("sweep_dram_bytes_per_apply" if v4 else f"sweep_v6_nx{p.nx_int}_dram_bytes_per_apply"),
        "peak_source": peak_src, "algorithmic_bytes_per_launch": sb, "avg_launch_ms": sw_ms, "launches": napplies,
        "launch_unit": "one RASQ apply (all its sweep kernels)", "share_of_step": sw_ms / max(1e-9, ms_apply),
        "family": "sweep",
        "fp64": {"flops_per_apply": fl, "achieved_tflops": tf, "peak_tflops": tpk,
                 "frac": (tf / tpk) if (tf and tpk) else None, "peak_source": tpk_src,
                 "flops_source": "SURVEY 8(a20): (2Nt + Nd - 1) * 4 * n_sp * nx (banded substitution)"},
        "chain": {"dependent_block_row_steps_per_apply": rows,
                  "us_per_block_row_step": 1000.0 * sw_ms / rows if sw_ms > 0 else None,
                  "handoff_floor_us": ncu_summary("v6_row_handoff_floor_us"),
                  "note": "the sweep is bound by this dependent chain: (2m+1) lock-step spatial solves x 2 directions x "
                          "ny block rows; the two-sided elimination runs the two half-length chains of a solve side by side and "
                          "k-row grouping makes one handoff serve k rows, so the dependent handoffs are ny/(2k) per chain launch"},
    }
    rest_ms = ms_apply - sw_ms
    rest_bytes = (4 + 1) * p.block * 8 // ws  # K8 (4B) + K3 node sums (B), SURVEY 8d
    rest = {"kernel": "P^-1 outside the sweep: pinv_uz_kernel (K8), nodesum_tree_kernel (K3), coarse_gamma_kernel (K4)",
            "bound": "hbm", "achieved": rest_bytes / (rest_ms / 1000.0) / 1e9 if rest_ms > 0 else None, "peak": peak,
            "unit": "GB/s", "frac": (rest_bytes / (rest_ms / 1000.0) / 1e9 / peak) if rest_ms > 0 else None,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": rest_bytes, "avg_launch_ms": rest_ms,
            "share_of_step": rest_ms / max(1e-9, ms_apply), "family": "pinv_rest"}
    return sweep, rest


def run_pinv(args, ws, rank, local):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    p = P.config(cfg, Nd=args.nd)
    if p.Nd % ws:
        raise SystemExit(f"time-slab sharding needs the rank count to divide Nd (Nd={p.Nd}, ranks={ws})")
    unknowns = 3 * p.Nt * p.n_sp
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        from paper_2305_04421_b200.solver import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t0 = time.perf_counter()
    k = HeatKKT(p, mode=args.mode, device=local, rank=rank, nranks=ws, nccl_id=nccl_id)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    v_host = rank_random_kkt(p, 0, k.node_first, k.node_last)
    n = v_host.size
    v = torch.from_numpy(v_host).to(dev)
    out = torch.empty_like(v)
    for _ in range(args.warmup):
        k.apply_P_inv(v, out)
    torch.cuda.synchronize()

    # ---- timed region: K applications, CUDA events on the current stream, max over ranks
    k.set_phase_timing(True)
    l0 = k.launch_count()
    prof = bool(os.environ.get("KKT_BENCH_PROFILE"))  # ncu --profile-from-start off: the timed region only
    if prof:
        torch.cuda.profiler.start()
    with ClockSampler(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            k.apply_P_inv(v, out)
        ev1.record()
        torch.cuda.synchronize()
        barrier(ws)
    if prof:
        torch.cuda.profiler.stop()
    launches = k.launch_count() - l0
    ms_step = max_over_ranks(ev0.elapsed_time(ev1), ws) / args.steps
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    value = unknowns / (ms_step / 1000.0)
    finite = bool(torch.isfinite(out).all().item())

    # ---- K1 at this workload's vector size (not part of the step: P^-1 has no K; the stencil's
    # roofline is reported beside the sweep's because north_star names both)
    xk = torch.empty_like(v)
    for _ in range(3):
        k.apply_K(v, xk)
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        k.apply_K(v, xk)
    s1.record()
    torch.cuda.synchronize()
    k_ms = s0.elapsed_time(s1) / 10
    del xk
    peak, peak_src = hbm_peak()
    k_bytes = 6 * p.block * 8 // ws
    stencil = {"kernel": "K1 apply_K_kernel (5-point space-time stencil, spatial tiles + time marching, stencil.cu)",
               "bound": "hbm", "achieved": k_bytes / (k_ms / 1000.0) / 1e9, "peak": peak, "unit": "GB/s",
               "frac": k_bytes / (k_ms / 1000.0) / 1e9 / peak, "peak_source": peak_src,
               "traffic": ncu_summary("apply_K_dram_bytes_per_launch_c2"),
               "algorithmic_bytes_per_launch": k_bytes, "avg_launch_ms": k_ms, "launches": 10,
               "note": "timed outside the step (10 launches on the step's vectors)"}
    mem_gb = (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9

    # ---- e2e through the host-buffer entry point (pinned memory)
    vh = torch.from_numpy(v_host).pin_memory()
    oh = torch.empty(n, dtype=torch.float64).pin_memory()
    k.apply_P_inv_host(vh.numpy(), oh.numpy())  # warm (allocates the staging vectors)
    e2e_steps = max(1, min(args.steps, 5))
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(e2e_steps):
        k.apply_P_inv_host(vh.numpy(), oh.numpy())
    e1.record()
    torch.cuda.synchronize()
    wall_e2e = (time.perf_counter() - w0) / e2e_steps
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / e2e_steps, ws)
    same = bool(torch.equal(oh.to(dev), out))
    del vh, oh

    sw_ms = phase_ms[3] / max(1, phase_cnt[3])
    roofline, rest = pinv_rooflines(p, ws, ms_step, sw_ms, phase_cnt[3])
    del k, v, out
    torch.cuda.empty_cache()
    if rank != 0:
        return
    vec_mb = 3 * p.block * 8 / ws / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 + Box-Muller N(0,1) KKT vector, paper_2305_04421_b200/problems.py)",
        "config": {
            "workload": workload_desc(cfg, p, "pinv"), "mode": args.mode, "output_finite": finite,
            "parallelism": (f"time slabs x{ws} ({p.Nd // ws} of {p.Nd} subdomains per GPU, NCCL halo + coarse all-gather)"
                            if ws > 1 else "1 GPU"),
            "l2": f"KKT vectors are {vec_mb:.0f} MB each per GPU (> 126 MB L2); no flush between applications",
            "setup_s": setup_s, "device_mem_GB": mem_gb,
            "phase_ms_per_step": {"P_inv": ms_step, "sweep_kernels": sw_ms},
        },
        "roofline": roofline,
        "roofline_secondary": rest,
        "roofline_stencil": stencil,
        "e2e": {"value": unknowns / (ms_e2e / 1000.0), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_e2e, "wall_ms_per_step": 1000 * wall_e2e,
                "steps": e2e_steps, "equals_device_result": same},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_extras and args.mode == "fast":
        for key, fn in (("config1", lambda: config1_extra(local)),
                        ("config1_per_dof", lambda: config1_extra(local, coarse="per-dof")),
                        ("config3", lambda: c3_microbench(local))):
            try:
                line[key] = fn()
            except Exception as e:  # reported beside the headline, never required
                line[key] = {"error": str(e)}
        if args.c4:
            try:
                line["microbench_c4_slab"] = c4_microbench(local)
            except Exception as e:
                line["microbench_c4_slab"] = {"error": str(e)}
    if not args.no_cpu_baseline and ws == 1:
        try:
            from oracle import bindings
            if bindings.available("ref"):
                rs = ReferenceSample(cfg, p, "pinv")
                t = rs.step()
                t_full = rs.extrapolate(t)
                line["cpu_baseline"] = {"value": 3 * p.block / t_full, "unit": UNIT, "cores": 1, "kind": "reference",
                                        "sample": rs.describe(t, t_full), "extrapolated": True,
                                        "host_nproc": os.cpu_count()}
            else:
                line["cpu_baseline"] = None
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line))


def config1_extra(local, steps=3, coarse="scalar"):
    """BASELINE config 1 (127^2 x 512, Nd = 16, GMRES(30)): the round-1 headline,
    kept as an extra key.  Sweep v4 (sweep_v4.cu).  coarse="per-dof": the reference's
    default coarse variant (dimension 516,128: coarse_kron.cu), which the reference
    itself cannot factor at this size."""
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = P.config(1, coarse=coarse)
    k = HeatKKT(p, mode="fast", device=local)
    b = torch.from_numpy(P.kkt_rhs(1, p)).cuda()
    x = torch.empty_like(b)
    for _ in range(3):
        k.gmres_solve(b, x)
    k.set_phase_timing(True)
    ms_total, iters, out = timed_solves(k, b, x, steps, 1)
    phase_ms, phase_cnt = k.phase_times()
    k.set_phase_timing(False)
    r, r2, st = rooflines(p, 1, "fast", iters[-1], steps, ms_total, phase_ms, phase_cnt, False)
    if coarse != "scalar":
        res = {"workload": workload_desc(1, p), "ms_per_step": ms_total / steps,
               "value": 3 * p.block / (ms_total / steps / 1000.0), "unit": UNIT, "iterations": iters[-1],
               "true_final_relres": out.true_final_relres, "steps": steps, "coarse_dim": k.coarse_dim()}
        del k, b, x
        torch.cuda.empty_cache()
        return res
    res = {"workload": workload_desc(1, p), "ms_per_step": ms_total / steps,
           "value": 3 * p.block / (ms_total / steps / 1000.0), "unit": UNIT, "iterations": iters[-1],
           "true_final_relres": out.true_final_relres, "steps": steps,
           "roofline": r, "roofline_secondary": r2, "roofline_stencil": st}
    del k, b, x
    torch.cuda.empty_cache()
    return res


def _pinv_microbench(local, p, reps, seed):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    k = HeatKKT(p, mode="fast", device=local)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    g = torch.Generator(device=dev).manual_seed(seed)
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
    roof, _ = pinv_rooflines(p, 1, med, sw_ms, phase_cnt[3])
    res = {"applications": reps, "setup_s": setup_s,
           "ms_per_apply_median": med, "ms_per_apply_min": ts[0],
           "value": 3 * p.block / (med / 1000.0), "unit": "unknowns/s per P^-1 apply",
           "sweep_ms_per_apply": sw_ms, "roofline": roof}
    del k, v, out
    torch.cuda.empty_cache()
    return res


def c3_microbench(local, reps=5):
    """BASELINE config 3's grid and time axis (255^2 x 4096, Nd = 32): P^-1
    applications (device-generated N(0,1) input: timing only; parity at this grid:
    tests/test_gpu_large.py).  Its full GMRES(20) solve does not converge on
    BASELINE's inputs (see the module docstring), so the solve is not timed here."""
    p = P.config(3)
    res = _pinv_microbench(local, p, reps, 3)
    res["workload"] = workload_desc(3, p, "pinv").replace("a seeded", "a device-generated")
    return res


def c2_microbench(local, reps=10):
    """BASELINE config 2, the preconditioner-apply microbench: 10 applications
    of P^-1 at 511^2 x 1024 steps, 64 subdomains, on seeded N(0,1) KKT vectors
    (device-generated here: timing only; parity is tests/test_gpu_large.py and
    tests/test_gpu_v6.py)."""
    p = P.config(2)
    res = _pinv_microbench(local, p, reps, 2)
    res["workload"] = workload_desc(2, p, "pinv")
    res["inputs"] = "device-generated N(0,1) (torch, seed 2); parity at this size: tests/test_gpu_large.py"
    return res


def c4_microbench(local, reps=3):
    """BASELINE config 4 (1023^2 interior, 8 GPUs) on the one GPU this pool
    has: one rank's time slab at G = 8 -- 16 subdomains of m = 8 steps,
    Nt = 128 with config 4's dt = 1/1024 (T = 1/8).  Opt-in (--c4): the block
    recursion's setup takes ~40 s at nx = 1023."""
    p = P.config(4).replace(Nt=128, Nd=16, T=0.125)
    res = _pinv_microbench(local, p, reps, 4)
    res["workload"] = ("config4 per-GPU slab at G=8: 1023x1023 interior, Nt=128 (dt=1/1024 as config 4), "
                       "Nd=16 (m=8), nu=1, omega=1e-4, two-level scalar multiplicative (minus)")
    res["inputs"] = "device-generated N(0,1) (torch, seed 4); parity at nx = 1023: tests/test_gpu_v6.py, tests/test_gpu_large.py"
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nd", type=int, default=None, help="override the config's subdomain count (config 3: 8/32/128/256)")
    ap.add_argument("--pinv", action="store_true", help="time P^-1 applications instead of full solves (always so at config 2)")
    ap.add_argument("--mode", default="fast", choices=["fast", "strict", "spectral"])
    ap.add_argument("--weak", action="store_true", help="N > 1: weak scaling (Nt and Nd x N) instead of strong")
    ap.add_argument("--no-extras", action="store_true", help="skip the config-1 and config-2 extra measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c4", action="store_true", help="add the config-4 per-GPU-slab P^-1 microbench (~40 s setup)")
    ap.add_argument("--probe-ranks", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and (args.impl == "ours" or args.probe_ranks):
        spawn_ranks(args)
    ws, rank, local = dist_env()
    if args.probe_ranks:
        return probe_ranks(ws, rank)
    if args.impl == "reference":
        return run_reference_arm(args, ws, rank)
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but the launcher started {ws} rank(s)")
    dist_init(ws, local)
    try:
        if workload_kind(args) == "pinv":
            run_pinv(args, ws, rank, local)
        else:
            run_solve(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
