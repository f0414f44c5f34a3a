# the 20,000-step interleaved stress of the final kernel (after the stale-slot fix)
# (compute-sanitizer is closed on the gpurun pool; profiles/r02d_sanitizer.txt is
# the last sanitizer run of the kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SINKR_STRESS_STEPS=20000 timeout 1500 python -m pytest tests/test_gpu_stress.py -q -m gpu > gpurun_out/r02p_stress_20000.txt 2>&1
tail -2 gpurun_out/r02p_stress_20000.txt
