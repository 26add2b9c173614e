"""Config 1 (BASELINE.json configs[0]) end to end against the reference's own
trace: mfglobal 0.1.0 ran solve_mf_global(lam=5, k0=8, seed=0) on the same
synthetic instance in the build container (tests/golden/make_golden.py --c1,
560 s on 8 CPU cores) -> tests/golden/trace_c1.json.

Bar (north_star): identical identified rank at every outer iteration and
per-iteration objective within 1e-9 relative (fp64 mode)."""

import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_c1_trace_matches_reference():
    import paper_2204_14067_b200 as P
    from paper_2204_14067_b200 import synth

    with open(os.path.join(GOLDEN, "trace_c1.json")) as fh:
        ref = json.load(fh)
    m, n, r, c, v = synth.generate("c1")
    m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
    obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr)
    cfg = P.SolverConfig(**ref["cfg"])
    t0 = time.perf_counter()
    x, _, trace = P.solve_mf_global(obs, None, cfg)
    el = time.perf_counter() - t0
    ranks = [rec.rank for rec in trace.records]
    objs = np.array([rec.obj for rec in trace.records])
    print(f"c1 on GPU: {len(trace)} records in {el:.1f}s (reference {ref['elapsed_s']:.0f}s); "
          f"final rank {ranks[-1]}, F = {objs[-1]!r}")
    assert ranks == ref["rank"]
    refo = np.array(ref["obj"])
    assert objs.shape == refo.shape
    assert np.max(np.abs(objs - refo) / np.abs(refo)) <= 1e-9
    assert x.rank == ref["rank"][-1] == 143
