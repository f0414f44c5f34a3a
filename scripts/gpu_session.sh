set -x
timeout 900 python -m pytest tests/test_gpu_append.py tests/test_cli.py tests/test_gpu_span.py tests/test_cpp_shim.py -x -q -m gpu 2>&1 | tail -30
python scripts/e2e_probe.py 2>&1 | tail -12
