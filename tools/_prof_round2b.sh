#!/bin/bash
# Round-2 analysis evidence, one GPU call: launch list of the bench (ncu
# gpu__time_duration), ncu --set full of the config-5 analysis kernels (the
# one-read median pass, the coastline bits, the six variogram walk kinds).
T=${TAG:-r2b}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1; echo "launches rc=$?"
REPS=1 ncu --set full --clock-control none -k regex:"radix_hist_keep_lin|radix_hist_keys|sample_hist" -c 4 \
    -o gpurun_out/median_$T python tools/prof_median.py > gpurun_out/ncu_median_$T.log 2>&1; echo "median rc=$?"
REPS=1 ncu --set full --clock-control none -k regex:"coast_bits|boxcount" -c 3 \
    -o gpurun_out/coast_$T python tools/prof_coast.py > gpurun_out/ncu_coast_$T.log 2>&1; echo "coast rc=$?"
ncu --set full --clock-control none -k regex:vg_walk -c 6 -o gpurun_out/vg_$T \
    python tools/time_vg.py --child --w 32768 --h 32768 --reps 1 > gpurun_out/ncu_vg_$T.log 2>&1; echo "vg rc=$?"
