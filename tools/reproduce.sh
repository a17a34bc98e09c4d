#!/bin/bash
# Reproduce the round's measurements (run from the repo root on a B200).
set -e
python -c "import __graft_entry__ as g; g.build()"                       # nvcc sm_100a + CPU checkers
python -m pytest tests -m "not gpu" -q                                   # oracle / reference / ABI (CPU)
python -m pytest tests -m gpu -q                                         # device parity
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > profiles/r2/bench_c5.json                     # headline line (c5, 2048 bins/step)
for c in c1 c2 c3 c4; do python bench.py --config $c --no-cpu-baseline --steps 3 > profiles/r2/bench_$c.json; done
python bench.py --impl reference --steps 1 --warmup 1                    # the reference arm (host cores)
# launch list (cold-cache, serialised: shares only) and one full capture of each hot kernel
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
    python bench.py --bins-per-step 512 --steps 1 --warmup 1 --no-cpu-baseline
python tools/ncu_summary.py launches launches.csv > profiles/r2/launch_share_c5.txt
BINS=512 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc2|pool_mma|gemm_grp" \
    --launch-skip 0 --launch-count 7 -o kernels python tests/mlp_rate.py
python tools/ncu_summary.py rep kernels.ncu-rep > profiles/r2/kernels_ncu_full_c5.txt
python tools/make_ncu_summary.py kernels.ncu-rep 512                    # -> profiles/ncu_summary.json (roofline.traffic)
# per-chunk MLP timelines, side benches of the 8(f) components
CIDER_TRACE_MLP=1 python tests/trace_mlp.py
python tools/bench_bp.py --config c3; python tools/bench_workload.py; python tools/bench_amp.py
# round-2 microbenchmarks behind profiles/r2/experiments/d128_mlp_epilogue.md
mkdir -p tools/_bin
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_bin/mufu_bench tools/mufu_bench.cu && tools/_bin/mufu_bench
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_bin/epi_bench tools/epi_bench.cu && tools/_bin/epi_bench
# session-5 helpers: the ncu evidence of a build in one go, same-box A/B of two library builds, batch-size A/B
bash tools/profile_round.sh                      # launch list + ncu --set full of the c5 / c2 kernel sets -> gpurun_out/
# make -C paper_2605_26580_b200/csrc OUT=../_lib_base   (at the base commit) ; then:
# bash tools/ab_lib.sh $PWD/paper_2605_26580_b200/_lib_base c5 c2
bash tools/ab_bins.sh
