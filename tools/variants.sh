#!/bin/bash
# run the GPU parity suite under each kernel-variant knob setting (raster.cu)
for cfg in "SGTR_FWD_WARP=2" "SGTR_FWD_WARP=0" "SGTR_VJP_STAGED=2" "SGTR_VJP_MODE=0" \
           "SGTR_VJP_MINBLOCKS=8" "SGTR_CHAIN_MODE=1" "SGTR_CHAIN_MODE=2" "SGTR_LANES=1" \
           "SGTR_JVP_WARP=0"; do
  r=$(env $cfg python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1)
  echo "$cfg: $r"
done
