"""Benchmark of the RASPEN hot path on B200 (contract: README of the driver).

One step = one full ``raspen_solve`` of BASELINE config 4 (1023^2 interior
grid, 16x16 subdomains, overlap 8, phi = y^3, 32 seeded Gaussian bumps,
eps 1 -> 1e-6 by factors of 10), synthetic seeded inputs.  Inner tolerance
1e-7: the documented deviation applied to BOTH the reference and this build,
because the reference itself fails config 4 at its default 1e-8.

metric: subdomain-Newton DOF-updates/s = sum over evaluations
and subdomains of 2 R_i C_i k_i (k_i inner Newton iterations) per second spent
in raspen_residual (device-timed RAS sweeps of the whole solve).  The CPU arm
measures the same quantity on a bounded sample.  ``ms_per_step`` /
``wall_s_to_tol`` is the whole solve (GMRES + JVPs included);
``value_whole_solve`` and ``e2e`` divide by whole-solve time (conservative).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU: the path does not shard (BASELINE: one GPU); N ranks run N
independent replicas (``scaling: weak``), value = total DOF-updates / max
rank time.
"""

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "subdomain-Newton DOF-updates/s"
UNIT = "DOF-updates/s"
CONFIG_NAME = "cfg4"
INNER_TOL = 1e-7
FP64_NOMINAL_TFLOPS = 37.0  # fallback only (B200 FP64 vector, nominal)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    def __init__(self, backend):
        self.ws, self.rank, self.local = dist_env()
        self.pg = None
        if self.ws > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group(backend=backend)
            self.td = td

    def barrier(self):
        if self.ws > 1:
            self.td.barrier()

    def max(self, v):
        if self.ws == 1:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64,
                         device="cuda" if self.td.get_backend() == "nccl" else "cpu")
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v):
        if self.ws == 1:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64,
                         device="cuda" if self.td.get_backend() == "nccl" else "cpu")
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.ws > 1:
            self.td.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, name in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def load_peaks():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    return peaks


def _probe(name, key):
    exe = os.path.join(REPO, "tools", name)
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        return float(json.loads(out.strip().splitlines()[-1])[key])
    except Exception:  # noqa: BLE001
        return None


def load_traffic():
    """DRAM bytes per launch of the hot kernels from the committed ncu --set full
    captures (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def measure_fp64_peak():
    """FP64 roof: the larger of the DMMA (tensor) and DFMA probes measured in this run.

    The factor kernel's trailing update runs on DMMA, its panel work on DFMA,
    so the roof is the faster pipe (tools/dmma_peak.cu, tools/fp64_peak.cu).
    """
    dmma = _probe("dmma_peak", "dmma_fp64_tflops")
    dfma = _probe("fp64_peak", "fp64_tflops")
    vals = [v for v in (dmma, dfma) if v]
    if vals:
        return max(vals), (f"measured this run: DMMA {dmma} / DFMA {dfma} TFLOP/s "
                           "(tools/dmma_peak, tools/fp64_peak), max taken")
    return FP64_NOMINAL_TFLOPS, "fallback (nominal B200 FP64)"


def problem():
    from paper_2411_00546_b200 import ContinuationSchedule, decompose
    from paper_2411_00546_b200.problems import CONFIGS, build_spec
    cfg = CONFIGS[CONFIG_NAME]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    return cfg, spec, dec, sched


def config_block(cfg):
    return {
        "workload": (f"BASELINE config 4 full raspen_solve: {cfg.n}x{cfg.n} interior grid, "
                     f"{cfg.s1}x{cfg.s2} subdomains, overlap {cfg.overlap}, phi=y^3, "
                     f"{cfg.bumps} seeded Gaussian bumps, nu={cfg.nu}, mu={cfg.mu}, "
                     f"eps {cfg.eps0}->{cfg.eps_min} (x{cfg.gamma})"),
        "n": cfg.n, "subdomains": cfg.s1 * cfg.s2, "overlap": cfg.overlap,
        "unknowns": cfg.unknowns, "outer_tol": 1e-10, "gmres_rel_tol": 1e-8,
        "inner_tol": INNER_TOL,
        "deviation": "inner_tol 1e-7 on both arms: the reference fails config 4 at 1e-8 "
                     "(LocalSolveError, FP64 residual floor; SURVEY.md 0.13)",
        "l2": "inputs larger than L2 (2.3 GB stored local factors streamed by every JVP)",
    }


def run_ours(args):
    dist = Dist("nccl")
    import torch
    torch.cuda.set_device(dist.local)
    from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,
                                       build_local_systems, raspen_solve)
    from paper_2411_00546_b200.schwarz import release_local_systems, solve_on_device
    from paper_2411_00546_b200.system import ProblemSpec

    cfg, spec, dec, sched = problem()
    engine = build_local_systems(dec, spec)
    newton_cfg = NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1)
    kry = KrylovConfig(rel_tol=1e-8, max_iters=1000)
    x0 = np.zeros(cfg.unknowns)
    x0_dev = engine.from_host(x0)

    def step():
        x, rep = solve_on_device(engine, x0_dev, sched, newton_cfg, kry, INNER_TOL, 200)
        if x is None or not rep.converged:
            raise RuntimeError(f"solve failed: {rep.failure}")
        return rep

    for _ in range(args.warmup):
        step()
    engine.set_profiling(True)
    engine.reset_stats()
    sampler = ClockSampler(dist.local)
    sampler.start()
    dist.barrier()
    engine.sync()
    engine.mark(0)
    if args.profile_window:   # ncu --profile-from-start off: capture the timed steps only
        torch.cuda.cudart().cudaProfilerStart()
    reps = [step() for _ in range(args.steps)]
    if args.profile_window:
        engine.sync()
        torch.cuda.cudart().cudaProfilerStop()
    engine.mark(1)
    engine.sync()
    dist.barrier()
    ms_total = engine.elapsed_ms(0, 1)
    clocks = sampler.stop()
    st = engine.stats()
    ms_step = dist.max(ms_total / args.steps)
    dof_step = st["dof_updates"] / args.steps
    sweep_ms_step = dist.max(st["sweep_ms"] / args.steps)
    value = dist.sum(dof_step) / (sweep_ms_step / 1e3)
    value_whole = dist.sum(dof_step) / (ms_step / 1e3)

    # end to end through the public API with host buffers: fresh ProblemSpec
    # (so f, y_d, x0 upload and the context build are inside), x comes back
    e2e_ms = []
    h2d = 8 * (cfg.unknowns + 2 * cfg.n * cfg.n)
    d2h = 8 * cfg.unknowns
    if not args.no_e2e:
        # one untimed end-to-end warm-up (the first fresh context maps its
        # memory), then the timed steps, each with a fresh problem and context
        for it in range(args.steps + 1):
            fresh = ProblemSpec(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                                f=spec.f.copy(), y_d=spec.y_d.copy())
            dist.barrier()
            t0 = time.perf_counter()
            x, rep = raspen_solve(x0, dec, fresh, sched, cfg=newton_cfg, krylov_cfg=kry,
                                  inner_tol=INNER_TOL)
            if it > 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
            print(f"e2e step {it}: {(time.perf_counter() - t0) * 1e3:.1f} ms"
                  + (" (warm-up)" if it == 0 else ""), file=sys.stderr, flush=True)
            assert rep.converged, rep.failure
            release_local_systems(dec, fresh)
            del fresh, x
            gc.collect()   # outside the timed region: the step's engine is torn down now
    e2e_step = dist.max(statistics.mean(e2e_ms)) if e2e_ms else None

    # the same quantity as cpu_baseline / --impl reference, end to end: the
    # first RAS evaluation (x = 0, eps continuation) through the public
    # raspen_residual on host arrays (x in; f_val and every local value out)
    e2e_sweep = None
    if not args.no_e2e:
        from paper_2411_00546_b200 import raspen_residual
        inner_cfg = NewtonConfig(tol=INNER_TOL, max_outer=200)
        esched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
        sw_ms, sw_dof = [], 0.0
        for it in range(args.steps + 1):
            dist.barrier()
            t0 = time.perf_counter()
            f_val, corr = raspen_residual(x0, dec, spec, cfg.eps_min, inner_cfg, esched)
            if it > 0:
                sw_ms.append((time.perf_counter() - t0) * 1e3)
            sw_dof = float(sum(2 * s.size * k for s, k in zip(dec.subdomains, corr.inner_iters)))
            del f_val, corr
        sw = dist.max(statistics.mean(sw_ms))
        e2e_sweep = {"value": dist.sum(sw_dof) / (sw / 1e3), "unit": UNIT, "ms_per_step": sw,
                     "dof_updates": sw_dof,
                     "h2d_bytes_per_step": 8 * cfg.unknowns,
                     "d2h_bytes_per_step": 8 * cfg.unknowns + 8 * sum(2 * s.size for s in dec.subdomains),
                     "definition": "first RAS evaluation (x=0, eps 1->1e-6) through the public "
                                   "raspen_residual on host arrays: the quantity cpu_baseline and "
                                   "--impl reference time on the CPU"}

    # roofline of the dominant kernels (per-launch averages over the timed region)
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    fp64_tf, fp64_src = measure_fp64_peak() if dist.rank == 0 else (None, None)
    fac_avg_ms = st["factor_ms"] / max(st["factor_launches"], 1)
    fac_flops = st["factor_flops"] / max(st["factor_launches"], 1)
    sol_avg_ms = st["solve_ms"] / max(st["solve_launches"], 1)
    sol_bytes = st["solve_bytes"] / max(st["solve_launches"], 1)
    fac_tf = fac_flops / (fac_avg_ms * 1e-3) / 1e12 if fac_avg_ms > 0 else None
    sol_gbs = sol_bytes / (sol_avg_ms * 1e-3) / 1e9 if sol_avg_ms > 0 else None
    res_avg_ms = st["resid_ms"] / max(st["resid_launches"], 1)
    res_bytes = st["resid_bytes"] / max(st["resid_launches"], 1)
    res_gbs = res_bytes / (res_avg_ms * 1e-3) / 1e9 if res_avg_ms > 0 else None
    kernels = {
        "local_residual_stencil": {"bound": "hbm", "achieved": res_gbs, "peak": hbm, "unit": "GB/s",
                                   "frac": (res_gbs / hbm) if res_gbs and hbm else None,
                                   "launches": st["resid_launches"], "avg_ms": res_avg_ms,
                                   "share_of_step": st["resid_ms"] / ms_total,
                                   "algorithmic_bytes_per_launch": res_bytes},
        "block_factor": {"bound": "fp64", "achieved": fac_tf, "peak": fp64_tf, "unit": "TFLOP/s",
                        "frac": (fac_tf / fp64_tf) if fac_tf and fp64_tf else None,
                        "peak_source": fp64_src, "launches": st["factor_launches"],
                        "avg_ms": fac_avg_ms, "share_of_step": st["factor_ms"] / ms_total,
                        "algorithmic_flops_per_launch": fac_flops},
        "jvp_block_solve": {"bound": "hbm", "achieved": sol_gbs, "peak": hbm, "unit": "GB/s",
                           "frac": (sol_gbs / hbm) if sol_gbs and hbm else None,
                           "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)",
                           "launches": st["solve_launches"], "avg_ms": sol_avg_ms,
                           "share_of_step": st["solve_ms"] / ms_total,
                           "algorithmic_bytes_per_launch": sol_bytes},
    }
    # MGS Arnoldi (k_arnoldi_lag): step j reads q_0..q_j and w, writes q_{j+1}:
    # (j + 3) vectors of 2N doubles; counted over the useful steps of every
    # GMRES solve of the timed region (the discarded speculative step is not)
    mgs_bytes = sum(8.0 * 2 * cfg.n * cfg.n * sum(j + 3 for j in range(m))
                    for r in reps for m in r.gmres_iters)
    mgs_gbs = mgs_bytes / (st["mgs_ms"] * 1e-3) / 1e9 if st["mgs_ms"] > 0 else None
    kernels["arnoldi_mgs"] = {"bound": "hbm", "achieved": mgs_gbs, "peak": hbm, "unit": "GB/s",
                              "frac": (mgs_gbs / hbm) if mgs_gbs and hbm else None,
                              "launches": sum(sum(r.gmres_iters) for r in reps),
                              "avg_ms": st["mgs_ms"] / max(sum(sum(r.gmres_iters) for r in reps), 1),
                              "share_of_step": st["mgs_ms"] / ms_total,
                              "algorithmic_bytes_per_solve": mgs_bytes / max(len(reps), 1)}
    dominant = max(kernels, key=lambda k: kernels[k]["share_of_step"] or 0.0)
    kd = kernels[dominant]
    traffic = load_traffic().get(dominant)
    roofline = {"kernel": dominant, "bound": kd["bound"], "achieved": kd["achieved"],
                "peak": kd["peak"], "unit": kd["unit"], "frac": kd["frac"],
                "traffic": traffic["bytes_per_launch"] if traffic else None}
    if traffic:
        roofline["traffic_source"] = traffic["source"]

    stress = None
    if not args.no_stress and dist.ws == 1:   # single-GPU line only (a rank-local measurement)
        try:
            stress = {name: stress_config5(name) for name in ("cfg5", "cfg5u")}
        except Exception as exc:   # reported, never fatal to the headline line
            stress = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = anchors = None
    if dist.rank == 0 and dist.ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(sample=max(16, os.cpu_count() or 1))   # one subdomain per host core
        try:
            anchors = cpu_anchors(stress)
        except Exception as exc:   # reported, never fatal to the headline line
            anchors = {"error": f"{type(exc).__name__}: {exc}"}
    rep = reps[-1]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, paper_2411_00546_b200/problems.py)",
        "config": config_block(cfg),
        "wall_s_to_tol": ms_step / 1e3,
        "dof_updates_per_step": dof_step,
        "sweep_ms_per_step": sweep_ms_step,
        "value_whole_solve": value_whole,
        "iterations": {"outer": rep.outer_iters, "inner_per_eval": rep.inner_iters,
                       "gmres_per_outer": rep.gmres_iters},
        "time_split_ms_per_step": {k: st[k] / args.steps for k in
                                   ("sweep_ms", "factor_ms", "inner_solve_ms", "jvp_ms",
                                    "solve_ms", "mgs_ms")},
        "roofline": roofline,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": (dist.sum(dof_step) / (e2e_step / 1e3)) if e2e_step else None,
                "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_step,
                "timer": "host perf_counter around raspen_solve(host x0) incl. context build",
                "definition": "DOF-updates / whole e2e solve time (conservative vs value)"},
        "e2e_sweep": e2e_sweep,
        "gpu_launches": int(st["launches"]),
        "clocks": clocks,
        "stress_config5": stress,
        "cpu_anchors": anchors,
    }
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


def stress_config5(name, reps=3):
    """BASELINE config 5 (batched-kernel stress test): one RAS sweep at x = 0
    (eps fixed at 1e-3, inner tol 1e-8) plus one JVP with d ~ N(0,1) seed 1,
    CUDA-event timed on the context stream after one untimed warm-up.  The
    reference's own CPU times for the same sweep + JVP come from the golden
    fixture's record (tests/golden/make_golden.py run_sweep)."""
    from paper_2411_00546_b200 import ContinuationSchedule, NewtonConfig, build_local_systems, decompose
    from paper_2411_00546_b200.problems import CONFIGS, build_spec
    from paper_2411_00546_b200.schwarz import _jvp, _sweep, release_local_systems

    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    x = eng.from_host(np.zeros(cfg.unknowns))
    fac = eng.factor_store()
    sched = ContinuationSchedule.fixed(cfg.eps_min)
    inner = NewtonConfig(tol=1e-8, max_outer=200)
    d = eng.from_host(np.random.default_rng(1).standard_normal(cfg.unknowns))
    fval, out = eng.vector(), eng.vector(cfg.unknowns)   # outputs allocated outside the timed region
    _sweep(eng, x, fac, sched, inner, fval)
    _jvp(eng, fac, d, out)
    eng.sync()
    eng.set_profiling(True)
    eng.reset_stats()
    sweep_ms, jvp_ms = [], []
    for _ in range(reps):
        eng.mark(2)
        fval, iters = _sweep(eng, x, fac, sched, inner, fval)
        eng.mark(3)
        out = _jvp(eng, fac, d, out)
        eng.mark(4)
        eng.sync()
        sweep_ms.append(eng.elapsed_ms(2, 3))
        jvp_ms.append(eng.elapsed_ms(3, 4))
    st = eng.stats()
    sw, jv = statistics.mean(sweep_ms), statistics.mean(jvp_ms)
    res = {"workload": f"BASELINE config 5 ({name}): {cfg.n}x{cfg.n} grid, {cfg.s1}x{cfg.s2} subdomains, "
                       f"overlap {cfg.overlap}, eps fixed {cfg.eps_min:g}; one raspen_residual(x=0) + one "
                       "raspen_jacobian_apply(d ~ N(0,1), seed 1)",
           "sweep_ms": sw, "jvp_ms": jv, "sweep_plus_jvp_ms": sw + jv,
           "inner_iters": sorted(set(int(i) for i in iters)),
           "dof_updates_per_s": st["dof_updates"] / reps / (sw / 1e3),
           "factor_tflops": st["factor_flops"] / st["factor_ms"] / 1e9 if st["factor_ms"] else None,
           "jvp_solve_gbs": st["solve_bytes"] / st["solve_ms"] / 1e6 if st["solve_ms"] else None,
           "fval_norm": fval.norm(), "jvp_norm": out.norm()}
    release_local_systems(dec)
    del eng, x, fac, d, fval, out
    gc.collect()
    return res


def blas_threads():
    info = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                           "MKL_NUM_THREADS")}
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                        for d in threadpool_info()]
    except Exception:  # noqa: BLE001
        pass
    return info


def cpu_anchors(stress):
    """Same-box CPU anchors: the reference path (oracle port, same SuperLU /
    sparsetools / BLAS calls as `pkg/src/ocp`) timed on this box's host cores
    beside the GPU, on workloads small enough to finish in the bench.

    * config 2, the whole raspen_solve (x = 0, harness settings) on the CPU
      against the same whole solve through the GPU's public API (host arrays
      in and out, context build included): the same quantity on both sides;
    * config 5 uniform, one RAS sweep at x = 0 + one JVP on the CPU, against
      the GPU's stress_config5 timing of the same pair.
    """
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import raspen_oracle as O
    from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,
                                       decompose, raspen_solve)
    from paper_2411_00546_b200.problems import CONFIGS, build_fields, build_spec
    from paper_2411_00546_b200.schwarz import release_local_systems
    from paper_2411_00546_b200.system import make_phi
    cores = os.cpu_count() or 1
    out = {"cores": cores, "kind": "port", "blas_threads": blas_threads(),
           "cpu_model": _cpu_model()}
    # config 2 whole solve
    cfg = CONFIGS["cfg2"]
    f, yd = build_fields(cfg)
    prob = O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, make_phi(cfg.phi), cfg.nu, cfg.mu, f, yd)
    t0 = time.perf_counter()
    xo, ro = O.raspen_solve(prob, np.zeros(cfg.unknowns), cfg.eps0, cfg.gamma, cfg.eps_min,
                            inner_tol=1e-8, threads=cores)
    cpu_s = time.perf_counter() - t0
    dof = O.dof_updates(prob, ro["per_sub"])
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    gpu_ms = []
    for it in range(4):   # one warm-up, three timed, each on a fresh problem + context
        fresh = type(spec)(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                           f=spec.f.copy(), y_d=spec.y_d.copy())
        t0 = time.perf_counter()
        x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, fresh, sched,
                              cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                              krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                              inner_tol=1e-8)
        if it:
            gpu_ms.append((time.perf_counter() - t0) * 1e3)
        release_local_systems(dec, fresh)
    gpu_s = statistics.median(gpu_ms) / 1e3   # (median: a context teardown landing in one solve is an outlier)
    out["cfg2_whole_solve"] = {
        "workload": "BASELINE config 2 raspen_solve from x=0 (255^2, 4x4, overlap 8, inner tol 1e-8)",
        "cpu_s": cpu_s, "gpu_e2e_s": gpu_s, "speedup": cpu_s / gpu_s,
        "cpu_iterations": {"outer": ro["outer_iters"], "inner": ro["inner_iters"],
                           "gmres": ro["gmres_iters"]},
        "gpu_iterations": {"outer": rep.outer_iters, "inner": rep.inner_iters,
                           "gmres": rep.gmres_iters},
        "cpu_dof_updates_per_s_whole_solve": dof / cpu_s,
        "gpu_dof_updates_per_s_whole_solve": dof / gpu_s,
        "gpu_timer": "host perf_counter around the public raspen_solve (host arrays, context build)",
    }
    # config 5 uniform sweep + JVP
    cfg = CONFIGS["cfg5u"]
    f, yd = build_fields(cfg)
    prob = O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, make_phi(cfg.phi), cfg.nu, cfg.mu, f, yd)
    x = np.zeros(cfg.unknowns)
    t0 = time.perf_counter()
    _, corr = O.raspen_residual(prob, x, cfg.eps_min, tol=1e-8, max_outer=200, threads=cores)
    t1 = time.perf_counter()
    d = np.random.default_rng(1).standard_normal(cfg.unknowns)
    O.raspen_jvp(prob, x, d, cfg.eps_min, corr)
    t2 = time.perf_counter()
    rec = {"workload": "BASELINE config 5 uniform: one RAS sweep at x=0 (eps 1e-3) + one JVP",
           "cpu_sweep_s": t1 - t0, "cpu_jvp_s": t2 - t1,
           "note": "the reference's JVP loop is sequential by design (schwarz.py:14-15)"}
    g = (stress or {}).get("cfg5u") if isinstance(stress, dict) else None
    if g and "sweep_plus_jvp_ms" in g:
        rec["gpu_sweep_plus_jvp_s"] = g["sweep_plus_jvp_ms"] / 1e3
        rec["speedup"] = (t2 - t0) / rec["gpu_sweep_plus_jvp_s"]
    out["cfg5u_sweep_jvp"] = rec
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(sample, threads=None):
    """CPU oracle (port of the reference path) on a bounded sample of config 4.

    Times the first RAS evaluation (eps continuation 1 -> 1e-6, x = 0) of
    ``sample`` seeded-random subdomains, thread pool over subdomains like
    the reference (`schwarz.py:203-208`); DOF-updates / time in raspen_residual.
    """
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import raspen_oracle as O
    from paper_2411_00546_b200.problems import CONFIGS, build_fields
    from paper_2411_00546_b200.system import make_phi
    cfg = CONFIGS[CONFIG_NAME]
    f, yd = build_fields(cfg)
    prob = O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, make_phi(cfg.phi), cfg.nu, cfg.mu, f, yd)
    ids = O.sample_subdomains(prob, sample, seed=0)
    cores = threads or min(len(ids), os.cpu_count() or 1)
    x = np.zeros(cfg.unknowns)
    t0 = time.perf_counter()
    _, corr = O.raspen_residual(prob, x, cfg.eps_min, cfg.eps0, cfg.gamma, INNER_TOL, 200,
                                threads=cores, subset=ids)
    dt = time.perf_counter() - t0
    dof = sum(2 * prob.rects[i].size * k for i, k in zip(ids, corr.inner))
    return {"value": dof / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"first RAS evaluation (eps 1->1e-6 continuation, x=0) of {len(ids)} of "
                       f"{len(prob.rects)} config-4 subdomains, inner tol {INNER_TOL}; "
                       f"{dof} DOF-updates in {dt:.2f} s"),
            "seconds": dt}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = problem()[0]
    for _ in range(args.warmup):
        cpu_baseline(sample=max(8, os.cpu_count() or 1))
    vals, secs = [], []
    for _ in range(args.steps):
        rec = cpu_baseline(sample=max(8, os.cpu_count() or 1))   # every host core busy
        vals.append(rec["value"])
        secs.append(rec["seconds"])
    value = statistics.mean(vals)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)", "config": config_block(cfg),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rec["cores"], "kind": "port",
                         "sample": rec["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stress", action="store_true", help="skip the config-5 stress timing")
    ap.add_argument("--profile-window", action="store_true",
                    help="cudaProfilerStart/Stop around the timed steps (ncu --profile-from-start off)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
