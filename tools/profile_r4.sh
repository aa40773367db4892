#!/usr/bin/env bash
# Round 2, session 4 (final build) profiles (run from the repo root on one B200, e.g. through gpurun).
# Every ncu command runs only after the same program exited 0 without ncu.
set -uo pipefail
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
echo "bench rc=$?"
# launch list of exactly the timed solve (bench.py --profile-window brackets it
# with cudaProfilerStart/Stop)
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-stress --profile-window \
    > gpurun_out/r4_pw.json 2>/dev/null && \
timeout -s KILL 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    --no-stress --profile-window > gpurun_out/r4_ncu_l.log 2>&1
echo "launch list rc=$?"
python tools/profile_cfg4.py cfg4 8 > gpurun_out/r4_prof.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_block_solve<.int.2>" -s 5 -c 1 -o gpurun_out/r4_solve2 \
    python tools/profile_cfg4.py cfg4 8 > gpurun_out/r4_ncu1.log 2>&1
python tools/factor_bench.py cfg4 2 > gpurun_out/r4_fb.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_block_factor" -s 2 -c 1 -o gpurun_out/r4_factor \
    python tools/factor_bench.py cfg4 2 > gpurun_out/r4_ncu2.log 2>&1
python tools/arnoldi_bench.py 140 > gpurun_out/r4_arn.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_arnoldi_lag" -s 3 -c 1 -o gpurun_out/r4_arnoldi \
    python tools/arnoldi_bench.py 140 > gpurun_out/r4_ncu3.log 2>&1
python tools/resid_bench.py cfg4 5 > gpurun_out/r4_rb.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_residual" -s 0 -c 1 -o gpurun_out/r4_resid \
    python tools/profile_cfg4.py cfg4 1 > gpurun_out/r4_ncu4.log 2>&1
echo done
