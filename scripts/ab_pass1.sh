#!/bin/bash
# A/B of k_rays_pass1 / k_fuse_heavy device time across library variants (ncu launch lists).
# Usage: scripts/ab_pass1.sh default ab/<name> ...   (run on the GPU box)
for v in "$@"; do
  l=""; [ "$v" != default ] && l=$v/librelief_b200.so
  RELIEF_B200_LIB=$l ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"k_rays_pass1|k_fuse_heavy" --csv --log-file gpurun_out/ab_$(basename $v).csv \
      python scripts/ab_rays.py > /dev/null 2>&1
  echo "== $v"; python scripts/launch_table.py gpurun_out/ab_$(basename $v).csv 40 | grep -v "min=     4"
done
