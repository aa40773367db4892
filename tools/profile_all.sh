#!/usr/bin/env bash
# Reproduce the profiles under profiles/ on one B200 (run from the repo root,
# e.g. through gpurun).  Every ncu command runs only after the same program
# exited 0 without ncu.  Outputs go to gpurun_out/; the summaries committed
# under profiles/ come from tools/ncu_summary.py and tools/summarize_launches.py.
set -euo pipefail
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/profile_cfg4.py cfg4 8 > gpurun_out/prof.log
python tools/factor_bench.py cfg4 2 > gpurun_out/fb.log
python tools/arnoldi_bench.py 140 > gpurun_out/arn.log
# launch list of one timed solve (3 warm-up solves of 1530 launches skipped)
ncu --metrics gpu__time_duration.sum --clock-control none -s 4590 -c 1600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_l.log 2>&1
# full captures of the three hot kernels
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_block_solve<.int.2>" -s 5 -c 1 -o gpurun_out/r1_solve2 \
    python tools/profile_cfg4.py cfg4 8 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_block_factor" -s 2 -c 1 -o gpurun_out/r1_factor \
    python tools/factor_bench.py cfg4 2 > gpurun_out/ncu2.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_arnoldi_lag" -s 3 -c 1 -o gpurun_out/r1_arnoldi \
    python tools/arnoldi_bench.py 140 > gpurun_out/ncu3.log 2>&1
# local-residual stencil: full capture of one full-set launch (x = 0)
python tools/resid_bench.py cfg4 5 > gpurun_out/rb.log
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_residual" -s 0 -c 1 -o gpurun_out/r1_resid \
    python tools/profile_cfg4.py cfg4 1 > gpurun_out/ncu4.log 2>&1
# config-5 stress (narrow-line factor instance)
python tools/stress_cfg5.py > gpurun_out/st.log
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_block_factor" -s 0 -c 1 -o gpurun_out/r1_factor_narrow \
    python tools/stress_cfg5.py > gpurun_out/ncu5.log 2>&1
