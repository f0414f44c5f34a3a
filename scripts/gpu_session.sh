set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_next_rows.py -x -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -3 gpurun_out/r2a_bench.err
timeout 400 python bench.py --force-sharded --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2a_sharded.json 2> gpurun_out/r2a_sharded.err; tail -3 gpurun_out/r2a_sharded.err
python scripts/e2e_probe.py 2>&1 | tail -12
