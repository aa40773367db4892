"""Where the end-to-end raspen_solve time goes beyond the device solve (config 4),
in bench.py's state (a device-resident engine stays alive): context build,
x0 upload, device solve (wall vs CUDA-event sum), x download, GC pauses."""
import cProfile
import gc
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import KrylovConfig, NewtonConfig, build_local_systems  # noqa: E402
from paper_2411_00546_b200.schwarz import release_local_systems, solve_on_device  # noqa: E402
from paper_2411_00546_b200.system import ProblemSpec  # noqa: E402

prof = len(sys.argv) > 1 and sys.argv[1] == "profile"
sys.argv = ["bench.py"]
import bench  # noqa: E402

gc_ms = []
_t = {}


def _cb(phase, info):
    if phase == "start":
        _t["s"] = time.perf_counter()
    else:
        gc_ms.append((time.perf_counter() - _t["s"]) * 1e3)


gc.callbacks.append(_cb)
cfg, spec, dec, sched = bench.problem()
newton_cfg = NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1)
kry = KrylovConfig(rel_tol=1e-8, max_iters=1000)
x0 = np.zeros(cfg.unknowns)
main = build_local_systems(dec, spec)
xd = main.from_host(x0)
for _ in range(2):
    solve_on_device(main, xd, sched, newton_cfg, kry, 1e-7, 200)
main.sync()
for rep in range(6):
    fresh = ProblemSpec(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                        f=spec.f.copy(), y_d=spec.y_d.copy())
    gc_ms.clear()
    t0 = time.perf_counter()
    eng = build_local_systems(dec, fresh)
    t1 = time.perf_counter()
    x0d = eng.from_host(x0)
    eng.sync()
    t2 = time.perf_counter()
    eng.set_profiling(True)
    eng.reset_stats()
    if prof:
        pr = cProfile.Profile()
        pr.enable()
    x, r = solve_on_device(eng, x0d, sched, newton_cfg, kry, 1e-7, 200)
    eng.sync()
    t3 = time.perf_counter()
    if prof:
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(8)
    xh = x.to_host()
    t4 = time.perf_counter()
    st = eng.stats()
    dev = st["sweep_ms"] + st["jvp_ms"] + st["mgs_ms"]
    print(f"build {1e3*(t1-t0):.1f} upload {1e3*(t2-t1):.1f} solve {1e3*(t3-t2):.1f} (device {dev:.1f}) "
          f"download {1e3*(t4-t3):.1f} ms; gc {len(gc_ms)} pauses {sum(gc_ms):.1f} ms", flush=True)
    release_local_systems(dec, fresh)
    del fresh, eng, x, x0d
    gc.collect()
