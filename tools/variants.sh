#!/bin/bash
# run the GPU parity suite under each kernel-variant knob setting
for cfg in "SGTR_FWD_WARP=1" "SGTR_FWD_WARP=0" "SGTR_FWD_WPB=8" "SGTR_VJP_STAGED=2" "SGTR_VJP_STAGED=0" "SGTR_VJP_STAGED=0 SGTR_WPB=8" \
           "SGTR_VJP_MODE=0" "SGTR_VJP_SMEMRED=0" "SGTR_CHAIN_MODE=1" "SGTR_CHAIN_MODE=2" "SGTR_LANES=1" \
           "SGTR_JVP_WARP=1" "SGTR_VJP_PPL=2" "SGTR_FWD_PPL=2"; do
  r=$(env $cfg python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1)
  echo "$cfg: $r"
done
