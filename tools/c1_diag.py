import json, os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import synth
ref = json.load(open("tests/golden/trace_c1.json"))
m, n, r, c, v = synth.generate("c1"); m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr)
cfg = P.SolverConfig(**ref["cfg"]); cfg.max_outer_iters = 4
x, _, trace = P.solve_mf_global(obs, None, cfg)
for i, rec in enumerate(trace.records):
    print(i, "obj %.10g/%.10g" % (rec.obj, ref["obj"][i]), "alpha %r/%r" % (rec.alpha, ref["alpha"][i]),
          "bt", rec.backtracks, ref["backtracks"][i], "kt", rec.k_t, ref["k_t"][i], "sweeps", rec.eig_sweeps, ref["eig_sweeps"][i],
          "eps %.6g/%.6g" % (rec.eps_achieved, ref["eps_achieved"][i]), "fmf %.10g/%.10g" % (rec.f_mf, ref["f_mf"][i]))
