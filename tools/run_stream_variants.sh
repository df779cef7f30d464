#!/bin/bash
# A/B builds of the tile-streaming solve's b = 3 shape on the GPU box (nvcc is in the image):
# warps per CTA, blocks per lane, lanes per tile.
cd paper_1610_08035_b200/csrc
for v in "8 5 32" "8 5 16" "7 5 8" "7 5 16" "6 7 16"; do
  set -- $v
  touch stream_solve.cu
  make -s -j8 SSFLAGS="-DSP_SS3_NW=$1 -DSP_SS3_M=$2 -DSP_SS3_LPT=$3" 2>&1 | grep -E "error" 
  (cd ../.. && timeout 120 python tools/stream_time.py "NW=$1 M=$2 LPT=$3" && timeout 200 python tools/stream_check.py quick | grep -E "CHECK|worst")
done
