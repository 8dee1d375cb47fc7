#!/bin/bash
# Untiled geometry A/B (consumer warps x rows per warp) for C4 / C5 on one box.
O=gpurun_out; mkdir -p $O; : > $O/geom_ab.txt
for i in 1 2; do
  bash tools/ab_libs.sh "--config C4 --tk 1 --steps 2 --warmup 3" default c4_8x2 >> $O/geom_ab.txt
  bash tools/ab_libs.sh "--config C5 --tk 1 --steps 3 --warmup 3" default c5_8x2 >> $O/geom_ab.txt
done
cat $O/geom_ab.txt
