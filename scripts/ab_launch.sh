cd $GRAFT_REPO_ROOT
for v in "" "SINKR_STEP_GRAPH=0" "SINKR_STEP_GRAPH=0 SINKR_STEP_LAUNCH=1" "SINKR_STEP_GRAPH=0 SINKR_STEP_LAUNCH=2" "SINKR_STEP_LAUNCH=2" ""; do
  echo "== $v"
  env $v timeout 300 python scripts/sched_ab.py 32768 65536 524288 2>&1 | tail -2
done
