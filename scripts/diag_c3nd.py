"""Diagnostic: FAST vs STRICT (bitwise the reference) P^-1 on the config-3 grid
(255^2) with a reduced time axis and many subdomains, per KKT block.

    python scripts/diag_c3nd.py [--nt 512] [--nds 32,128,256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nt", type=int, default=512)
ap.add_argument("--nds", default="32,128,256")
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
for nd in [int(x) for x in a.nds.split(",")]:
    p = P.config(a.config, Nd=nd).replace(Nt=a.nt)
    v = torch.from_numpy(P.random_kkt(p, 1)).cuda()
    f = HeatKKT(p, mode="fast").apply_P_inv(v).cpu().numpy()
    s = HeatKKT(p, mode="strict").apply_P_inv(v).cpu().numpy()
    B = p.block
    errs = [float(np.linalg.norm(f[i * B:(i + 1) * B] - s[i * B:(i + 1) * B]) /
                  np.linalg.norm(s[i * B:(i + 1) * B])) for i in range(3)]
    print(f"Nd={nd} m={p.Nt // nd}: rel err per block {errs}", flush=True)
