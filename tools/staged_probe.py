"""Time the staged sweep's pieces on one workload (diagnostics).

    python tools/staged_probe.py c3 [--lmin X] [--tpc N]
Prints CUDA-event times of: the grouped sweep, the staged sweep (main +
fold), the staged main kernel alone (MFG_STAGED_SKIP_FOLD), per plan."""
import argparse
import os
import subprocess
import sys
import json

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def run(args):
    import numpy as np
    import torch
    sys.argv = [sys.argv[0]]
    import bench
    from paper_2204_14067_b200.data import ObservationSet
    from paper_2204_14067_b200.mfsolver import SweepPlan
    from paper_2204_14067_b200 import synth
    m, n, r, c, v, spec = bench.instance(args.wl, seed=0)
    k = spec.k0
    obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    variants = [("grouped", {}),
                ("staged", {"staged": True, "staged_opts": {"lmin": args.lmin, "tiles_per_cta": args.tpc,
                                                            "l1_bytes": args.l1}})]
    for name, kw in variants:
        plan = SweepPlan(obs, k, compute_f64=False, **kw)
        w = plan.pad(torch.as_tensor(w_np, device="cuda"))
        h = plan.pad(torch.as_tensor(h_np, device="cuda"))
        for _ in range(3):
            plan.run(w, h)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); plan.run(w, h); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        out[name] = round(sorted(ts)[len(ts) // 2], 1)
        if plan.staged is not None:
            out["stats"] = plan.staged.stats()
    print(json.dumps({args.tag: out}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("wl")
    ap.add_argument("--lmin", type=float, default=4.0)
    ap.add_argument("--tpc", type=int, default=2)
    ap.add_argument("--tag", default="full")
    ap.add_argument("--l1", type=int, default=0, help="L1-blocked mode with this many bytes per block")
    run(ap.parse_args())
