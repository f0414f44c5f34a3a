set -x
timeout 900 python -m pytest tests/test_gpu_span.py tests/test_cpp_shim.py -x -q -m gpu 2>&1 | tail -30
