#!/bin/bash
# Round-end ncu evidence for the current build (run on a B200 from the repo root; outputs in gpurun_out/).
# 1. launch list of the bench command (cold-cache, serialised: shares only); 2. ncu --set full of the c5
# and c2 hot kernels (one forward of tests/mlp_rate.py). Each command first runs to exit 0 without ncu.
set -x
O=gpurun_out
python bench.py --bins-per-step 512 --steps 1 --warmup 1 --no-cpu-baseline --no-parity > $O/prof_bench_plain.json 2> $O/prof_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_512bins.csv \
    python bench.py --bins-per-step 512 --steps 1 --warmup 1 --no-cpu-baseline --no-parity > $O/prof_ncu_launch.log 2>&1
BINS=512 python tests/mlp_rate.py > $O/mlp_rate_c5.txt 2>&1 || exit 1
BINS=512 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc2|pool_mma|gemm_grp" \
    --launch-skip 0 --launch-count 7 -f -o $O/kernels_c5 python tests/mlp_rate.py > $O/prof_ncu_c5.log 2>&1
CFG=c2 BINS=4096 python tests/mlp_rate.py > $O/mlp_rate_c2.txt 2>&1 || exit 1
CFG=c2 BINS=4096 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc2|pool_mma|gemm_grp" \
    --launch-skip 0 --launch-count 7 -f -o $O/kernels_c2 python tests/mlp_rate.py > $O/prof_ncu_c2.log 2>&1
ls -la $O/*.ncu-rep
