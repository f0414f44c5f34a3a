#!/bin/bash
# round-2 evidence run (gpurun): randomized parity soak + compute-sanitizer
OUT=gpurun_out
SINKR_PARITY_SEEDS=1500 SINKR_BATCHED_SEEDS=300 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k randomized 2>&1 | tail -4 > $OUT/r02_parity_soak.txt
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $OUT/r02_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_probe.py 2>&1 | tail -12 >> $OUT/r02_sanitizer.txt
done
echo "== memcheck, spill path (SINKR_DEBUG_SLOTS=2)" >> $OUT/r02_sanitizer.txt
SINKR_DEBUG_SLOTS=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_probe.py 2>&1 | tail -6 >> $OUT/r02_sanitizer.txt
