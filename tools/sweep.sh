#!/bin/bash
# usage: tools/sweep.sh "ENV=a ENV2=b" "ENV=c" ...   — one C3 bench line per setting
for cfg in "$@"; do
  env $cfg python bench.py --config c3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); k=d['kernel_ms']
print('$cfg', round(d['value'],2), {n: round(v['total_ms']/v['launches'],3) for n,v in k.items() if n in ('raster_fwd','raster_vjp','chain','ssim_residual','ssim_gather','depth_sort_scan','tile_binning','project','tr_update','tr_bisect')})"
done
