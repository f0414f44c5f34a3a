# A/B of the code prewarm (interleaved processes): back to back and
# L2-flushed (trimmed mean of 100 single steps).  SINKR_PREWARM: region mask
# (8 = all in CTA G-1) + 256 x the cold-pass threshold in us
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in ${AB_VARIANTS:-0 8}; do
    echo "PREWARM=$v $(SINKR_PREWARM=$v AB_STEPS=200 AB_CASES=${AB_CASES:-1} AB_COLD=100 timeout 300 python scripts/sched_ab.py 32768 65536 524288 2>&1 | tail -1)"
  done
done
