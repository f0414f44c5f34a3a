cd $GRAFT_REPO_ROOT
cp paper_2604_16883_b200/_lib/libsinkr_cuda.so /tmp/keep.so
for i in 1 2 3; do for v in A B; do cp scripts/ablibs/lib$v.so paper_2604_16883_b200/_lib/libsinkr_cuda.so; echo "lib$v $(python scripts/e2e_ab.py 32768 2>&1 | tail -1)"; done; done
cp /tmp/keep.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
