set -x
for v in libpolyterrain_b200 variants/skip1 variants/skip2 variants/skip124 variants/skip127; do echo "== $v"; TG_LIB_PATH=paper_1610_03525_b200/lib/$v.so python tools/time_gen.py --configs cfg2 --iters 50; done > gpurun_out/skip_times.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fbm2d -c 1 -o gpurun_out/cur python tools/prof_gen.py --config cfg2 --iters 1 > gpurun_out/ncu.log 2>&1
echo done
