set -x
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma2 tools/ffma2_probe.cu && /tmp/ffma2
timeout 900 python -m pytest tests/test_gpu_triplet.py -q -x -p no:cacheprovider 2>&1 | tail -3
python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r2g_bench.json 2>gpurun_out/r2g_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['triplet'])"
python bench.py --workload dimenet-pp-small --steps 30 --no-cpu-baseline > gpurun_out/r2g_bench_c1.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench_c1.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['triplet'])"
