#!/bin/bash
# A/B of the stream-loop contraction (run under gpurun): timings + one ncu
# --set full capture per variant at the C2 (R=4) and C4 (R=8) shapes.
set -x
cd "$(dirname "$0")"
OUT=../../gpurun_out
./stream_ab 524288 3 all 0 > $OUT/r02_stream_ab.txt 2>&1
for R in 4 8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ -f \
      -o $OUT/r02_stream_ab_R$R ./stream_ab 524288 3 all $R once > $OUT/r02_stream_ab_R${R}_ncu.log 2>&1
  ncu -i $OUT/r02_stream_ab_R$R.ncu-rep --page raw --csv > $OUT/r02_stream_ab_R${R}_raw.csv
  ncu -i $OUT/r02_stream_ab_R$R.ncu-rep --page details --csv > $OUT/r02_stream_ab_R${R}_details.csv
  rm -f $OUT/r02_stream_ab_R$R.ncu-rep
done
