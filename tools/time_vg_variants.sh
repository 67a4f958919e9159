#!/bin/bash
# Time the variogram of an R x R config-2 map for library variants:
# tools/time_vg_variants.sh "lib variants/a variants/b" (names under paper_1610_03525_b200/lib/, no .so)
VARIANTS=${1:-"libpolyterrain_b200"}
for r in 1 2; do for v in $VARIANTS; do
  echo "== $v $(TG_LIB_PATH=paper_1610_03525_b200/lib/$v.so python tools/time_analysis.py | grep variogram)"
done; done
