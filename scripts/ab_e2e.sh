# e2e A/B: graph vs direct launches for the blocking host-buffer step
cd $GRAFT_REPO_ROOT
g++ -O2 -std=c++17 scripts/micro/e2e_cabi.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_2604_16883_b200/_lib -lsinkr_cuda \
    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2604_16883_b200/_lib -o /tmp/e2e_cabi || exit 1
for v in 1 0 1 0; do
  echo "== SINKR_STEP_GRAPH=$v"
  SINKR_STEP_GRAPH=$v timeout 120 /tmp/e2e_cabi 32768
  SINKR_STEP_GRAPH=$v timeout 300 python scripts/e2e_probe.py 524288 2>&1 | tail -8
done
