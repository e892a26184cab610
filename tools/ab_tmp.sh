for v in base k7w2 k7w4; do
  if [ $v = base ]; then unset SGTR_LIB; else export SGTR_LIB=_variants/$v.so; fi
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); km=d['kernel_ms']; print('$v', round(d['value'],2), 'fwd', round(km['raster_fwd']['total_ms']/km['raster_fwd']['launches'],4), repr(d['final_loss']))"
done
