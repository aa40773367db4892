"""Config-5 stress timing alone (bench.stress_config5)."""
import sys, json
sys.path.insert(0, ".")
sys.argv = ["bench.py"]
import bench
for name in ("cfg5", "cfg5u"):
    r = bench.stress_config5(name)
    print(name, json.dumps({k: r[k] for k in ("sweep_ms", "jvp_ms", "factor_tflops", "jvp_solve_gbs", "fval_norm", "jvp_norm")}))
