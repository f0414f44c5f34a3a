#!/bin/bash
# A/B: fused single-kernel step vs 3-kernel pipeline, alternating runs
for i in 1 2; do
  for f in 1 0; do
    SINKR_FUSED=$f timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 50 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('fused=$f', 'routed', d['value'], 'dense', d['dense_us_per_step'], 'e2e', d['e2e']['value'], 'kernel_us', d['roofline']['kernel_us'], d['roofline'].get('phases'))"
  done
done
