"""run_single on the device for a BASELINE config, printing the reference's
JSON RunRecord (experiments.cpp:179-208), like the reference CLI's single run.

    python scripts/run_single.py --config 1 [--mode fast|strict] [--coarse scalar|per-dof]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.experiments import run_single, to_json_string  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--coarse", default="scalar")
    ap.add_argument("--precond", default="two-level")
    ap.add_argument("--nd", type=int, default=None, help="override the config's subdomain count")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    p = P.config(a.config, coarse=a.coarse, precond=a.precond, Nd=a.nd)
    rec = run_single(p, mode=a.mode)
    text = to_json_string(rec)
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
