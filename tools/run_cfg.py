"""Run one BASELINE config solve on the GPU and print the report, timings and kernel stats."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,  # noqa: E402
                                   build_local_systems, decompose)
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402
from paper_2411_00546_b200.schwarz import solve_on_device  # noqa: E402

name = sys.argv[1]
inner_tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
t0 = time.perf_counter()
eng = build_local_systems(dec, spec)
print(f"engine build {time.perf_counter()-t0:.3f}s  I={eng.num_subdomains} fac={eng.fac_len*8/1e9:.2f} GB maxW={eng.max_w}")
sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
x0 = eng.from_host(np.zeros(cfg.unknowns))
for r in range(reps):
    eng.set_profiling(True)
    eng.reset_stats()
    t0 = time.perf_counter()
    x, rep = solve_on_device(eng, x0, sched, NewtonConfig(tol=1e-10), KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol, 200)
    eng.sync()
    wall = time.perf_counter() - t0
    st = eng.stats()
    print(f"[{r}] wall {wall:.3f}s conv={rep.converged} outer={rep.outer_iters} inner={rep.inner_iters} gmres={rep.gmres_iters} failure={rep.failure}")
    print("    stats", json.dumps({k: round(v, 3) for k, v in st.items()}))
    if st["factor_ms"] > 0:
        print(f"    factor {st['factor_flops']/st['factor_ms']/1e9:.2f} TFLOP/s over {st['factor_launches']:.0f} launches; "
              f"jvp-solve {st['solve_bytes']/max(st['solve_ms'],1e-9)/1e6:.1f} GB/s over {st['solve_launches']:.0f}; "
              f"residual {st['resid_bytes']/max(st['resid_ms'],1e-9)/1e6:.1f} GB/s over {st['resid_launches']:.0f}")
if x is not None and len(sys.argv) > 4:
    np.save(sys.argv[4], x.to_host())

if len(sys.argv) > 5 and sys.argv[5] == "profile":
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    t0 = time.perf_counter()
    x, rep = solve_on_device(eng, x0, sched, NewtonConfig(tol=1e-10), KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol, 200)
    eng.sync()
    pr.disable()
    print(f"profiled wall {time.perf_counter()-t0:.3f}s")
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)
