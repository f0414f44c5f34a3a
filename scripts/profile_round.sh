#!/bin/bash
# ncu evidence for one round (run under gpurun; 1 GPU).  TAG names the files.
#   bash scripts/profile_round.sh r02a [cases...]
# Writes gpurun_out/${TAG}_step_<case>_{raw,details}.csv, the source-page
# stall listing, and the bench launch list.
TAG=${1:-r02}; shift
CASES=${@:-routed512k dense512k peer64k c1routed c1dense c4routed}
mkdir -p gpurun_out
for c in $CASES; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 \
      -f -o gpurun_out/${TAG}_$c python scripts/ncu_cases.py $c > gpurun_out/${TAG}_${c}_ncu.log 2>&1
  ncu -i gpurun_out/${TAG}_$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_step_${c}_raw.csv
  ncu -i gpurun_out/${TAG}_$c.ncu-rep --page details --csv > gpurun_out/${TAG}_step_${c}_details.csv
  ncu -i gpurun_out/${TAG}_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_${c}_source.csv 2>/dev/null
  python scripts/ncu_lines.py gpurun_out/${TAG}_${c}_source.csv 25 > gpurun_out/${TAG}_step_${c}_stall_lines.txt 2>&1
  rm -f gpurun_out/${TAG}_${c}_source.csv
  # gpurun brings back <= 64 MiB: keep only the report named in KEEP_REP
  [ "$c" = "${KEEP_REP:-routed512k}" ] || rm -f gpurun_out/${TAG}_$c.ncu-rep
done
