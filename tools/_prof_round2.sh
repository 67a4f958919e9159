#!/bin/bash
# Round-2 evidence, one GPU call: bench launch list (ncu gpu__time_duration),
# ncu --set full of one config-2 launch, DRAM bytes of 8 back-to-back
# config-2 launches into the bench's 3 rotating buffers (cache control none,
# so each launch's write-back shows up), all-config timings, octave sweep.
T=${TAG:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/ncu_launch_$T.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fbm2d -c 1 -o gpurun_out/prof_cfg2_$T \
    python tools/prof_gen.py --config cfg2 --iters 1 > gpurun_out/ncu_full_$T.log 2>&1; echo "ncu full rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    --cache-control none --clock-control none -k regex:fbm2d -s 4 -c 8 --csv --log-file gpurun_out/dram_$T.csv \
    python tools/prof_gen.py --config cfg2 --iters 14 --rotate 3 > gpurun_out/ncu_dram_$T.log 2>&1; echo "ncu dram rc=$?"
TG_TIME_EXTRA=1 python tools/time_gen.py --configs cfg1,cfg2,cfg2sep,cfg3p,cfg3p5,cfg3g,cfg3s,cfg5 --iters 50 > gpurun_out/times_$T.log 2>&1
python tools/octave_sweep.py --out gpurun_out/octave_sweep_$T.json > /dev/null 2>&1; echo "sweep rc=$?"
