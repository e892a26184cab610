#!/bin/bash
# A/B of libsgtr.so builds at C5 (10M splats) on one GPU (run under gpurun):
# the bench value and the binning kernel classes per build, "base" = the
# in-tree library, any other name = _variants/<name>.so
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset SGTR_LIB; else export SGTR_LIB=_variants/$v.so; fi
  python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abc5_$v.json 2>/dev/null
  python -c "
import json
d = json.loads(open('gpurun_out/abc5_$v.json').read().strip().splitlines()[-1])
km = d['kernel_ms']
ms = {n: round(t['total_ms'] / t['launches'], 4) for n, t in km.items()}
print('$v', round(d['value'], 3), ms.get('tile_binning'), ms.get('depth_sort_scan'), repr(d['final_loss']))"
done
