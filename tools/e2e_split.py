"""Where the end-to-end raspen_solve time goes beyond the device solve (config 4):
engine (context) build with a fresh ProblemSpec, then the solve through the
public API with host x0, with the engine's CUDA-event stats of that solve."""
import gc
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import KrylovConfig, NewtonConfig, build_local_systems, raspen_solve  # noqa: E402
from paper_2411_00546_b200.system import ProblemSpec  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

cfg, spec, dec, sched = bench.problem()
newton_cfg = NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1)
kry = KrylovConfig(rel_tol=1e-8, max_iters=1000)
x0 = np.zeros(cfg.unknowns)
if "--bench-state" in sys.argv[1:] or True:
    # like bench.py: a device-resident engine stays alive through the e2e steps
    from paper_2411_00546_b200.schwarz import solve_on_device
    main = build_local_systems(dec, spec)
    xd = main.from_host(x0)
    for _ in range(2):
        solve_on_device(main, xd, sched, newton_cfg, kry, 1e-7, 200)
    main.sync()
for rep in range(5):
    fresh = ProblemSpec(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                        f=spec.f.copy(), y_d=spec.y_d.copy())
    t0 = time.perf_counter()
    eng = build_local_systems(dec, fresh)
    eng.set_profiling(True)
    eng.reset_stats()
    t1 = time.perf_counter()
    x, r = raspen_solve(x0, dec, fresh, sched, cfg=newton_cfg, krylov_cfg=kry, inner_tol=1e-7)
    t2 = time.perf_counter()
    st = eng.stats()
    dev = st["sweep_ms"] + st["jvp_ms"] + st["mgs_ms"]
    print(f"build {1e3 * (t1 - t0):.1f} ms, solve+io {1e3 * (t2 - t1):.1f} ms "
          f"(sweep {st['sweep_ms']:.1f} jvp {st['jvp_ms']:.1f} mgs {st['mgs_ms']:.1f}, sum {dev:.1f}), "
          f"conv {r.converged}", flush=True)
    dec.__dict__.get("_engines", {}).pop(id(fresh), None)
    import weakref
    wr = weakref.ref(eng)
    del fresh, eng, x
    gc.collect()
    if wr() is not None:
        refs = gc.get_referrers(wr())
        print("  engine still alive; referrers:", [type(o).__name__ + (str(list(o.keys())[:6]) if isinstance(o, dict) else "") for o in refs][:8], flush=True)
