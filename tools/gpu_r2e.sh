timeout 1000 python -m pytest tests/test_gpu_triplet.py tests/test_gpu_model.py -q -p no:cacheprovider -x -k "triplet_fwd_bwd or spherical or bench" 2>&1 | tail -3 > gpurun_out/r2e_tests.log
timeout 900 python tools/c5_sweep.py --path sh --degrees 32,64,128,256,500 --dg 64,128 --out gpurun_out/r2d_c5_sh.json > gpurun_out/r2d_c5_sh.log 2>&1
cat gpurun_out/r2e_tests.log
