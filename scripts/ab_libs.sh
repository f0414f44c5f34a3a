# A/B of two builds of the library (scripts/ablibs/libA.so vs libB.so), interleaved
cd $GRAFT_REPO_ROOT
cp paper_2604_16883_b200/_lib/libsinkr_cuda.so /tmp/lib_keep.so
for i in 1 2 3; do
  for v in A B; do
    cp scripts/ablibs/lib$v.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
    echo "lib$v $(AB_STEPS=200 AB_CASES=${AB_CASES:-1} AB_COLD=60 timeout 300 python scripts/sched_ab.py ${AB_LENGTHS:-32768 65536 524288} 2>&1 | tail -1)"
  done
done
cp /tmp/lib_keep.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
