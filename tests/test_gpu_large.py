"""GPU: single-operation parity at the large BASELINE grids (configs 2 and 3:
511^2 and 255^2 interior) on reduced time axes, against golden records of the
compiled reference (scripts/golden_large_ops.py).  Full solves there are out
of reach of the CPU reference, so parity is per operation:
K v bitwise (same stencil order in both modes), P^-1 v within 1e-10 relative
L2 per block (FAST mode: block-recursion factor, blocked sweep).
"""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RECORDS = sorted(glob.glob(os.path.join(GOLD, "ops_c*_nt*_nd*.json")))


def _sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest()


@pytest.mark.parametrize("path", RECORDS, ids=[os.path.basename(r)[:-5] for r in RECORDS])
def test_large_grid_ops_against_reference(path):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    rec = json.load(open(path))
    samp = np.load(path.replace(".json", "_sample.npz"))
    p = P.config(rec["config"]).replace(Nt=rec["problem"]["Nt"], Nd=rec["problem"]["Nd"])
    v = P.random_kkt(p, 0)
    assert _sha(v) == rec["v_sha256"]
    k = HeatKKT(p, mode="fast")
    vd = torch.from_numpy(v).cuda()
    K = k.apply_K(vd).cpu().numpy()
    assert _sha(K) == rec["apply_K"]["sha256"], "K v must be bitwise (reference stencil order)"
    Pv = k.apply_P_inv(vd).cpu().numpy()
    B, stride = p.block, rec["stride"]
    want = samp["apply_P_inv"]
    got = Pv[::stride]
    idx = np.arange(0, 3 * B, stride)
    for blk in range(3):
        sel = (idx >= blk * B) & (idx < (blk + 1) * B)
        err = np.linalg.norm(got[sel] - want[sel]) / np.linalg.norm(want[sel])
        assert err <= 1e-10, (blk, err)
        n = np.linalg.norm(Pv[blk * B:(blk + 1) * B])
        assert abs(n - rec["apply_P_inv"]["norms"][blk]) <= 1e-10 * rec["apply_P_inv"]["norms"][blk]


@pytest.mark.parametrize("env", [{"KKT_V6_K": "1"}, {"KKT_V6_K": "1", "KKT_V6_THOMAS": "0"}, {"KKT_V6_THOMAS": "0"}],
                         ids=["inverse_blocks", "lu_factors", "lu_factors_grouped"])
def test_large_grid_pinv_row_by_row_forms_against_reference(env, tmp_path):
    """The records' time axes are short, so the default run above groups the chain's rows (k > 1);
    config 2 and the config-4 slab at full size run row by row (k = 1).  Forced here on the same
    records: row by row in the inverse-block form of the two-sided elimination (the default:
    H_J = cy D_J^-1 as the only operator set, no off-chain products) and in the L/U form, and the
    grouped L/U form, against the reference's P^-1 samples (1e-10 per block).  Subprocess: the
    switches are read once per process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import json, sys, numpy as np, torch\n"
        "from paper_2305_04421_b200 import problems as P\n"
        "from paper_2305_04421_b200.solver import HeatKKT\n"
        "for path in sys.argv[1:]:\n"
        "    rec = json.load(open(path)); samp = np.load(path.replace('.json', '_sample.npz'))\n"
        "    p = P.config(rec['config']).replace(Nt=rec['problem']['Nt'], Nd=rec['problem']['Nd'])\n"
        "    v = P.random_kkt(p, 0)\n"
        "    k = HeatKKT(p, mode='fast'); Pv = k.apply_P_inv(torch.from_numpy(v).cuda()).cpu().numpy()\n"
        "    del k; torch.cuda.empty_cache()\n"
        "    B, stride = p.block, rec['stride']; want = samp['apply_P_inv']; got = Pv[::stride]\n"
        "    idx = np.arange(0, 3 * B, stride); worst = 0.0\n"
        "    for blk in range(3):\n"
        "        sel = (idx >= blk * B) & (idx < (blk + 1) * B)\n"
        "        worst = max(worst, float(np.linalg.norm(got[sel] - want[sel]) / np.linalg.norm(want[sel])))\n"
        "    print('REL', worst)\n")
    r = subprocess.run([sys.executable, "-c", code] + RECORDS, env=dict(os.environ, KKT_V6_TIM="1", **env),
                       capture_output=True, text=True, timeout=1500, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    rels = [float(x.split()[1]) for x in r.stdout.splitlines() if x.startswith("REL")]
    assert len(rels) == len(RECORDS) and max(rels) <= 1e-10, r.stdout
    forms = [x for x in r.stderr.splitlines() if x.startswith("v6 elimination form")]
    want = "inverse blocks" if env.get("KKT_V6_THOMAS") != "0" else "L/U factors"
    assert forms and all(want in x for x in forms), forms[:3]
