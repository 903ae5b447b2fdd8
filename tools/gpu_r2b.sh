timeout 1200 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_api.py tests/test_gpu_multiproc.py -q -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/r2b_tests.log
tail -5 gpurun_out/r2b_tests.log
