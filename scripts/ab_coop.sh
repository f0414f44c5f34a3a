#!/bin/bash
for c in 1 0 1 0; do
  SINKR_COOP=$c timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 50 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('coop=$c', 'routed', d['value'], 'dense', d['dense_us_per_step'], 'e2e', d['e2e']['value'], 'kernel_us', d['roofline']['kernel_us'])"
done
SINKR_TRACE=1 timeout 200 python scripts/trace_ctas.py 524288 0.625 2>&1 | tail -12
