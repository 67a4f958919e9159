#!/bin/bash
# Time library variants side by side: tools/time_variants.sh "v_a v_b" [extra python after time_gen]
# (each variant is paper_1610_03525_b200/lib/<name>.so; builds: python -m paper_1610_03525_b200.build --out ...)
VARIANTS=${1:-"libpolyterrain_b200"}
EXTRA=${2:-"time_3d(iters=10)"}
CFGS=${CFGS:-cfg2}
for r in 1 2; do for v in $VARIANTS; do echo "== $v"; TG_LIB_PATH=paper_1610_03525_b200/lib/$v.so python - <<PY
import sys; sys.argv=['time_gen.py','--configs','$CFGS','--iters','20']
exec(compile(open('tools/time_gen.py').read(),'time_gen.py','exec'))
$EXTRA
PY
done; done
