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
