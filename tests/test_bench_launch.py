"""CPU: `python bench.py --gpus N`, launched as the driver launches it at N = 1
(no torchrun environment), starts N ranks itself and reports the number of
ranks that actually ran (Missing 3: --gpus used to be ignored)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, BENCH, *args], env=e, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    return lines


def test_gpus_flag_spawns_that_many_ranks():
    lines = _run("--gpus", "2", "--probe-ranks")
    assert len(lines) == 1, lines          # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_started"] == 2


def test_single_rank_probe():
    lines = _run("--probe-ranks")
    assert lines == [dict(lines[0], n_gpus=1, ranks_started=1)]


def test_under_torchrun_the_environment_wins():
    """Launched by torchrun (WORLD_SIZE set) bench.py must not spawn again."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29617", BENCH, "--gpus", "2",
                        "--probe-ranks"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["ranks_started"] == 2


def test_rank_count_must_divide_the_subdomains():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", BENCH)
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_2305_04421_b200 import problems as P
    p = P.config(3)
    # the config-3 strong-scaling arm: 32 subdomains over 1/2/4/8 GPUs
    assert all(p.Nd % g == 0 for g in (1, 2, 4, 8))
    # per-GPU byte/flop models split the vectors over the slabs, the factor stream does not shrink
    F = 8 * p.n_sp * (2 * p.nx_int + 1)
    m = p.Nt // p.Nd
    assert bench.sweep_bytes(p, 8) == (2 * p.Nt + p.Nd - 1) * 5 * p.n_sp * 8 // 8 + (2 * m + 1) * F
    assert bench.sweep_flops(p, 2) == (2 * p.Nt + p.Nd - 1) * 4.0 * p.n_sp * p.nx_int / 2
    assert bench.sweep_block_row_steps(p) == (2 * 128 + 1) * 2 * 255
