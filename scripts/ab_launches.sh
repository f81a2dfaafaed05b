#!/bin/bash
# Per-kernel launch durations (ncu, serialised, cold-ish) of one workload across library builds.
# Usage (GPU box): scripts/ab_launches.sh WORKLOAD default ab/NAME ...
wl=$1; shift
for v in "$@"; do
  l=""; [ "$v" != default ] && l=$PWD/$v/librelief_b200.so
  RELIEF_B200_LIB=$l ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
      --log-file gpurun_out/abl_$(basename $v).csv python scripts/ab_frame.py default --workloads=$wl > /dev/null 2>&1
  echo "== $v"; python scripts/launch_table.py gpurun_out/abl_$(basename $v).csv 30
done
