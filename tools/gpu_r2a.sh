set -x
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2a_tests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r2a_bench_gemnet.json 2> gpurun_out/r2a_bench_gemnet.err
python bench.py --workload dimenet-pp-small --steps 20 --warmup 3 > gpurun_out/r2a_bench_dimenet.json 2> gpurun_out/r2a_bench_dimenet.err
tail -2 gpurun_out/r2a_tests.log
