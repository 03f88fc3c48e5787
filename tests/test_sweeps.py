"""f3: the sweeps (reference experiments.cpp:73-177) — CPU side.

The reference's own weak-scaling and omega sweeps (oracle/_ref) are run on
desk-sized grids; their CSV pins (1) our CSV formatting (each reference row,
parsed back into a record and re-emitted by experiments.csv_row/to_csv, is
byte-identical) and (2) our grid construction, skip rule and row order (the
device runs are replaced by a stub that echoes the config).
"""
import pytest

from paper_2305_04421_b200 import experiments as E
from paper_2305_04421_b200 import problems as P

BASE = P.Problem(Lx=1.0, Ly=2.0, Nx=4, Ny=4, T=1.0, coarse_variant="per-dof", tol=1e-6,
                 max_iters=420, restart=None)


def _ref():
    from oracle import bindings
    if not bindings.available("ref"):
        pytest.skip("oracle/_ref not built")
    return bindings.Ref


def _parse(csv_text, base):
    """Reference CSV rows -> (records, skipped lines)."""
    lines = csv_text.splitlines()
    assert lines[0] == E.csv_header()
    recs, skipped = [], []
    for ln in lines[1:]:
        if ln.startswith("#"):
            skipped.append(ln)
            continue
        f = ln.split(",")
        cfg = base.replace(Nt=int(f[0]), Nd=int(f[1]), omega=float(f[3]), precond=f[4],
                           coarse_variant=f[5], two_level_form=f[6], jhat_sign=f[7])
        recs.append(E.RunRecord(cfg, int(f[8]), f[9] == "true", float(f[10]), float(f[11]),
                                float(f[12]), float(f[13])))
    return recs, skipped


WEAK = dict(steps=4, nts=[8, 12, 10, 16], omegas=[1e-2, 1e-4], preconds=["two-level", "one-level"])
OMEGA = dict(nt=12, nd=3, omegas=[1e-1, 1e-3, 1e-6], preconds=["two-level", "none"])


def test_csv_format_matches_reference():
    Ref = _ref()
    for kind, kw in (("weak", WEAK), ("omega", OMEGA)):
        if kind == "weak":
            text = Ref.sweep_csv(BASE, "weak", kw["omegas"], kw["preconds"], steps=kw["steps"], nts=kw["nts"])
        else:
            text = Ref.sweep_csv(BASE, "omega", kw["omegas"], kw["preconds"], nt=kw["nt"], nd=kw["nd"])
        recs, skipped = _parse(text, BASE)
        assert recs, kind
        sweep = E.SweepResult(rows=recs)
        for ln in skipped:  # "# skipped nt=10 omega=0.01 precond=two-level: reason"
            head, reason = ln[len("# skipped "):].split(": ", 1)
            kv = dict(x.split("=") for x in head.split())
            sweep.skipped.append(E.SkippedRun(
                BASE.replace(Nt=int(kv["nt"]), Nd=1, omega=float(kv["omega"]), precond=kv["precond"]), reason))
        assert E.to_csv(sweep) == text, kind


def test_grid_and_order_match_reference(monkeypatch):
    """Our grid, skip rule and row order against the reference's CSV, with the
    device runs stubbed out (the config echoed back)."""
    Ref = _ref()
    monkeypatch.setattr(E, "run_single", lambda cfg, mode="fast", device=0: E.RunRecord(cfg))
    text = Ref.sweep_csv(BASE, "weak", WEAK["omegas"], WEAK["preconds"], steps=WEAK["steps"], nts=WEAK["nts"])
    want, want_sk = _parse(text, BASE)
    got = E.weak_scaling_sweep(BASE, WEAK["steps"], WEAK["nts"], WEAK["omegas"], WEAK["preconds"])
    key = lambda r: (r.config.Nt, r.config.Nd, r.config.omega, r.config.precond)  # noqa: E731
    assert [key(r) for r in got.rows] == [key(r) for r in want]
    got_sk = [ln for ln in E.to_csv(got).splitlines() if ln.startswith("#")]
    assert got_sk == want_sk
    text = Ref.sweep_csv(BASE, "omega", OMEGA["omegas"], OMEGA["preconds"], nt=OMEGA["nt"], nd=OMEGA["nd"])
    want, _ = _parse(text, BASE)
    got = E.omega_sweep(BASE, OMEGA["nt"], OMEGA["nd"], OMEGA["omegas"], OMEGA["preconds"])
    assert [key(r) for r in got.rows] == [key(r) for r in want]


def test_steps_must_be_positive():
    from paper_2305_04421_b200.solver import ConfigError
    with pytest.raises(ConfigError):
        E.weak_scaling_sweep(BASE, 0, [8], [1e-2], ["two-level"])
