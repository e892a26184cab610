#!/bin/bash
# A/B of libsgtr.so builds on one GPU (run under gpurun): one default C3 bench
# line per build, "base" = the in-tree library, any other name =
# _variants/<name>.so from tools/variant_so.py.
#   tools/ab_variants.sh base name1 name2 ...
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset SGTR_LIB; else export SGTR_LIB=_variants/$v.so; fi
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json
d = json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
km = d['kernel_ms']
ms = {n: round(t['total_ms'] / t['launches'], 4) for n, t in km.items()}
print('$v', round(d['value'], 2), ms, repr(d['final_loss']))"
done
