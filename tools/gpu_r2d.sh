for path in sh pairwise; do
  timeout 900 python tools/c5_sweep.py --path $path --degrees 32,64,128,256,500 --dg 64,128 --out gpurun_out/r2d_c5_$path.json > gpurun_out/r2d_c5_$path.log 2>&1
done
EGN_TRIPLET_PATH=sh python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_sh.json 2>gpurun_out/r2d_bench_sh.err
tail -2 gpurun_out/r2d_c5_sh.log
