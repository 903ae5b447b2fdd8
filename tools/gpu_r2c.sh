timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2c_tests.log
for wl in gemnet-t-oc20 dimenet-pp-small; do
  python bench.py --workload $wl --steps 20 --warmup 3 > gpurun_out/r2c_bench_$wl.json 2> gpurun_out/r2c_bench_$wl.err
done
for wl in dimenet-pp-xl gemnet-xl; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --cpu-budget 5 > gpurun_out/r2c_bench_$wl.json 2> gpurun_out/r2c_bench_$wl.err
done
tail -3 gpurun_out/r2c_tests.log
