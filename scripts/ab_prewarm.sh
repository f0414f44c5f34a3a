# A/B of the code prewarm (CTA G-1 dry pass) on one GPU
cd $GRAFT_REPO_ROOT
for v in "SINKR_PREWARM=0" "SINKR_PREWARM=1" "SINKR_PREWARM=0" "SINKR_PREWARM=1"; do
  echo "== $v"
  env $v timeout 300 python scripts/sched_ab.py 32768 65536 524288 2>&1 | tail -1
done
for v in "SINKR_PREWARM=0" "SINKR_PREWARM=1"; do
  echo "== cold probe $v"
  env $v timeout 300 python scripts/cold_cta_probe.py 32768 2>&1
done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
