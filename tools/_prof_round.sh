#!/bin/bash
# One GPU call: bench line, ncu launch list of the bench, ncu --set full of one
# config-2 launch, all-config timings, config-5 terrain run.  TAG=v20 by default.
T=${TAG:-v20}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fbm2d -c 1 -o gpurun_out/prof_cfg2_$T \
    python tools/prof_gen.py --config cfg2 --iters 1 > gpurun_out/ncu_full_$T.log 2>&1; echo "ncu full rc=$?"
TG_TIME_EXTRA=1 python tools/time_gen.py --configs cfg1,cfg2,cfg2sep,cfg3p,cfg3p5,cfg3g,cfg3s,cfg5 --iters 50 > gpurun_out/times_$T.log 2>&1
python tools/terrain_run.py > gpurun_out/terrain_$T.json 2> gpurun_out/terrain_$T.err; echo "terrain rc=$?"
python tools/octave_sweep.py --out gpurun_out/octave_sweep_$T.json > /dev/null 2>&1; echo "sweep rc=$?"
