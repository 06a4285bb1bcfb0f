#!/usr/bin/env python
"""C3 / C4 points-sweep time (Session.time_sweep) and ASPOT it/s of the
current build, one JSON line; run repeatedly around a kernel change.

    python profiles/sweep_times.py [--tag name] [--configs 3,4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17196_b200 import pot  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="")
    ap.add_argument("--configs", default="3,4")
    args = ap.parse_args()
    ctx = pot.Context(0)
    out = {"tag": args.tag}
    for cid in (int(c) for c in args.configs.split(",")):
        inst = pot.config_instance(cid)
        cfg = pot.SolverConfig(epsilon=1e-3 if cid == 4 else 1e-2, log_every=10 ** 9, max_iterations=10 ** 7,
                               record_rounded_cost=False, materialize_plan=False)
        s = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
        s.iterate(3)
        ms, it, _ = s.iterate(60 if cid != 4 else 8)
        sw = s.time_sweep(20)[0]
        s.close()
        out[f"C{cid}_sweep_ms"] = round(sw, 4)
        out[f"C{cid}_it_s"] = round(it / ms * 1e3, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
