#!/bin/bash
# Round profiling pass (GPU box): bench line, ncu launch list of the bench
# command, ncu --set full of the headline (cfg 2) and conv kernels.
set -x
python bench.py > gpurun_out/bench_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brgemm_tc -s 2 -c 1 -o gpurun_out/cfg2_full \
    python tools/prof.py cfg2 --iters 4 > gpurun_out/ncu_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brgemm_tc -s 1 -c 1 -o gpurun_out/conv_full \
    python tools/prof.py conv --iters 3 > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brgemm_tc -s 1 -c 1 -o gpurun_out/fc1_full \
    python tools/prof.py fc1 --iters 3 > gpurun_out/ncu_fc1.log 2>&1
