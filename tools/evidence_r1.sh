# Round-1 evidence on one B200: bench lines, ncu launch list of one training step,
# ncu --set full captures of the top kernels.  Outputs under gpurun_out/.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/profile_step.py --plain --steps 1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1_launches.csv python tools/profile_step.py --plain --steps 1 > gpurun_out/ncu_launch.log 2>&1
# the roofline GEMM launch (E x 128 x 128 + residual) alone, then one wgrad
ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 3 -c 1 -o gpurun_out/r1_gemm python tools/gemm_one_shape.py --reps 1 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 3 -c 1 -o gpurun_out/r1_gemm_wgrad python tools/gemm_one_shape.py --kind wgrad --reps 1 > gpurun_out/ncu1b.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -s 4 -c 1 -o gpurun_out/r1_tfwd python tools/profile_step.py --plain --steps 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bw1_kernel -s 4 -c 1 -o gpurun_out/r1_tbw1 python tools/profile_step.py --plain --steps 1 > gpurun_out/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bw2_kernel -s 4 -c 1 -o gpurun_out/r1_tbw2 python tools/profile_step.py --plain --steps 1 > gpurun_out/ncu4.log 2>&1
# tensor-core triplet kernels on the C5 deg-500, d_g 64 graph
ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -s 1 -c 1 -o gpurun_out/r1_tc_fwd python tools/c5_sweep.py --degrees 500 --dg 64 --iters 1 > gpurun_out/ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:^(y_kernel|a_kernel)$" -c 2 -o gpurun_out/r1_tc_bwd python tools/c5_sweep.py --degrees 500 --dg 64 --iters 1 > gpurun_out/ncu6.log 2>&1

# every GEMM call of one step (cold L2), relaxation driver timing
python tools/gemm_census.py --out gpurun_out/gemm_census.txt > /dev/null 2>&1
python tools/relax_bench.py > gpurun_out/relax.json 2>/dev/null
python tools/relax_bench.py --variant dimenet-style >> gpurun_out/relax.json 2>/dev/null
python tools/profile_step.py --out gpurun_out/step_kernels.txt > gpurun_out/prof.log 2>&1
ls -la gpurun_out/
