"""Batched block-factor throughput on BASELINE configs 4 and 5 (RAS sweeps at
x = 0), for the library selected by OCP_LIB (default: the in-tree build).
Used for the DMMA vs DFMA-only A/B (tools/build_variant.py dfma -DOCP_DFMA_ONLY).

    python tools/factor_ab.py [cfg4 cfg5u cfg5]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2411_00546_b200 import ContinuationSchedule, NewtonConfig, build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402
from paper_2411_00546_b200.schwarz import _jvp, _sweep, release_local_systems  # noqa: E402

names = sys.argv[1:] or ["cfg4", "cfg5u", "cfg5"]
out = {"lib": os.environ.get("OCP_LIB", "in-tree")}
for name in names:
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    x = eng.from_host(np.zeros(cfg.unknowns))
    fac = eng.factor_store()
    if name == "cfg4":
        sched, tol = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min), 1e-7
    else:
        sched, tol = ContinuationSchedule.fixed(cfg.eps_min), 1e-8
    fval, inner = _sweep(eng, x, fac, sched, NewtonConfig(tol=tol, max_outer=200))
    eng.sync()
    eng.set_profiling(True)
    eng.reset_stats()
    for _ in range(3):
        fval, inner = _sweep(eng, x, fac, sched, NewtonConfig(tol=tol, max_outer=200))
    st = eng.stats()
    d = eng.from_host(np.random.default_rng(1).standard_normal(cfg.unknowns))
    jv = _jvp(eng, fac, d)
    out[name] = {"factor_ms_per_launch": st["factor_ms"] / st["factor_launches"],
                 "factor_launches_per_sweep": st["factor_launches"] / 3,
                 "factor_tflops_bandlu_count": st["factor_flops"] / st["factor_ms"] / 1e9,
                 "sweep_ms": st["sweep_ms"] / 3, "inner_max": max(inner),
                 "fval_norm": fval.norm(), "jvp_norm": jv.norm()}
    print(name, json.dumps(out[name]), flush=True)
    del fval, jv, d, x, fac, eng
    release_local_systems(dec)
print(json.dumps(out))
