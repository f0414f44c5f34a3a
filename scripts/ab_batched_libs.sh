cd $GRAFT_REPO_ROOT
cp paper_2604_16883_b200/_lib/libsinkr_cuda.so /tmp/keep.so
for i in 1 2; do for v in A B; do cp scripts/ablibs/lib$v.so paper_2604_16883_b200/_lib/libsinkr_cuda.so; echo "lib$v $(timeout 300 python scripts/ab_batched.py 2>&1 | tail -1)"; done; done
cp /tmp/keep.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_stress.py -x -q -m gpu -k "batched or config or stress or C3 or C5" 2>&1 | tail -2
