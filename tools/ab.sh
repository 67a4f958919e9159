#!/bin/bash
# A/B timing on the GPU box: tools/ab.sh "variantA variantB ..." [configs]
# (variants are paper_1610_03525_b200/lib/variants/<name>.so; "cur" = the in-tree library)
V=${1:-"base cur"}; C=${2:-cfg2}
mkdir -p gpurun_out
for r in 1 2 3; do for v in $V; do
  if [ "$v" = cur ]; then L=paper_1610_03525_b200/lib/libpolyterrain_b200.so; else L=paper_1610_03525_b200/lib/variants/$v.so; fi
  echo "== $v"; TG_LIB_PATH=$L python tools/time_gen.py --configs $C --iters 100
done; done
