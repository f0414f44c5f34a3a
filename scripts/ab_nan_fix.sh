# the NaN-isolation test against the product library (A) and the candidate (B)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2604_16883_b200/_lib/libsinkr_cuda.so /tmp/lib_keep.so
for v in A B; do
  cp scripts/ablibs/lib$v.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
  echo "== lib$v" >> gpurun_out/nan_test.txt
  timeout 300 python -m pytest tests/test_gpu_robustness.py -q -m gpu 2>&1 | grep -E "^E |passed|failed" | head -12 >> gpurun_out/nan_test.txt
done
cp /tmp/lib_keep.so paper_2604_16883_b200/_lib/libsinkr_cuda.so
[ -n "$AB" ] && AB_CASES=2 bash scripts/ab_libs.sh > gpurun_out/ab_nan.txt 2>&1
[ -n "$FULL" ] && timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_nan.txt 2>&1
cat gpurun_out/nan_test.txt
