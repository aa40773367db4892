"""Run the linear-RAS Newton-Krylov method (newton-ras-eps) on a BASELINE config on the GPU."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,  # noqa: E402
                                   build_local_systems, decompose)
from paper_2411_00546_b200.linear_ras import solve_ras_on_device  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
ncfg = NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1,
                    linear_solver=KrylovConfig(rel_tol=1e-8, max_iters=2000))
x0 = eng.from_host(np.zeros(cfg.unknowns))
gold = os.path.join("tests", "golden", f"ras_{name}.npz")
for r in range(reps):
    eng.set_profiling(True)
    eng.reset_stats()
    t0 = time.perf_counter()
    x, rep = solve_ras_on_device(eng, x0, sched, ncfg)
    eng.sync()
    wall = time.perf_counter() - t0
    st = eng.stats()
    print(f"[{r}] newton-ras wall {wall:.3f}s conv={rep.converged} outer={rep.outer_iters} "
          f"gmres={rep.gmres_iters} alphas={rep.alphas} failure={rep.failure}")
    print("    stats", json.dumps({k: round(v, 3) for k, v in st.items()}))
    if st["factor_ms"] > 0:
        print(f"    factor {st['factor_flops']/st['factor_ms']/1e9:.2f} TFLOP/s over "
              f"{st['factor_launches']:.0f}; prec-solve {st['solve_bytes']/max(st['solve_ms'],1e-9)/1e6:.1f}"
              f" GB/s over {st['solve_launches']:.0f}")
if os.path.exists(gold):
    g = np.load(gold)
    xh = x.to_host()
    n2 = cfg.n * cfg.n
    print(f"reference: outer={int(g['outer_iters'])} gmres={list(g['gmres_iters'])} "
          f"wall={float(g['wall']):.1f}s")
    for key, v in (("y", xh[:n2]), ("p", xh[n2:])):
        if key in g:
            print(f"    rel L2 {key}: {np.linalg.norm(v - g[key]) / np.linalg.norm(g[key]):.3e}")
        else:
            print(f"    |{key}| {np.linalg.norm(v):.12e} vs reference {float(g[key + '_norm']):.12e}")
