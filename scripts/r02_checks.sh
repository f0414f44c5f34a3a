#!/bin/bash
# evidence run (gpurun): randomized parity soak + compute-sanitizer.
#   bash scripts/r02_checks.sh [TAG]     -> gpurun_out/${TAG}_{parity_soak,sanitizer}.txt
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
SINKR_PARITY_SEEDS=1500 SINKR_BATCHED_SEEDS=300 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k randomized 2>&1 | tail -4 > $OUT/${TAG}_parity_soak.txt
rm -f $OUT/${TAG}_sanitizer.txt
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $OUT/${TAG}_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_probe.py 2>&1 | tail -12 >> $OUT/${TAG}_sanitizer.txt
done
echo "== memcheck, spill path (SINKR_DEBUG_SLOTS=2)" >> $OUT/${TAG}_sanitizer.txt
SINKR_DEBUG_SLOTS=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_probe.py 2>&1 | tail -6 >> $OUT/${TAG}_sanitizer.txt
