# Round-2 evidence on one B200: bench lines (4 workloads + the Bessel bases + reference arm),
# ncu launch lists (C2 step, DimeNet++ C1 step, graph-parallel step), ncu --set full captures
# of the top kernels, GEMM census, torch.profiler breakdown.  Outputs under gpurun_out/r2e_*.
set -x
O=gpurun_out
nproc; lscpu | grep "Model name"
python bench.py > $O/r2e_bench_gemnet.json 2> $O/r2e_bench_gemnet.err
python bench.py --impl reference > $O/r2e_bench_gemnet_ref.json 2> $O/r2e_bench_gemnet_ref.err
python bench.py --workload dimenet-pp-small > $O/r2e_bench_dimenet.json 2> $O/r2e_bench_dimenet.err
python bench.py --workload dimenet-pp-small --impl reference > $O/r2e_bench_dimenet_ref.json 2> $O/r2e_bench_dimenet_ref.err
python bench.py --basis bessel --steps 20 > $O/r2e_bench_gemnet_bessel.json 2> $O/r2e_bench_gemnet_bessel.err
python bench.py --workload dimenet-pp-small --basis bessel --steps 20 > $O/r2e_bench_dimenet_bessel.json 2> $O/r2e_bench_dimenet_bessel.err
for wl in dimenet-pp-xl gemnet-xl; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --cpu-budget 5 > $O/r2e_bench_$wl.json 2> $O/r2e_bench_$wl.err
done
python bench.py --partition centre --steps 20 --no-cpu-baseline > $O/r2e_bench_gemnet_centre1.json 2> $O/r2e_bench_gemnet_centre1.err

# launch lists
python tools/profile_step.py --plain --steps 1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r2e_launches_c2.csv python tools/profile_step.py --plain --steps 1 > $O/r2e_ncu_l1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r2e_launches_c1.csv python tools/profile_step.py --workload dimenet-pp-small --plain --steps 1 > $O/r2e_ncu_l2.log 2>&1
python tools/gp_step.py --workers 2 --steps 1 > $O/r2e_gp_step.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/r2e_launches_gp.csv python tools/gp_step.py --workers 2 --steps 1 > $O/r2e_ncu_l3.log 2>&1

# full captures: roofline GEMM launch, wgrad, triplet fast fwd / bw1 / bw2 at C2
ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 3 -c 1 -o $O/r2e_gemm python tools/gemm_one_shape.py --reps 1 > $O/r2e_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 3 -c 1 -o $O/r2e_gemm_wgrad python tools/gemm_one_shape.py --kind wgrad --reps 1 > $O/r2e_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -s 4 -c 1 -o $O/r2e_tfwd python tools/profile_step.py --plain --steps 1 > $O/r2e_ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bw1_kernel -s 4 -c 1 -o $O/r2e_tbw1 python tools/profile_step.py --plain --steps 1 > $O/r2e_ncu4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bw2_kernel -s 4 -c 1 -o $O/r2e_tbw2 python tools/profile_step.py --plain --steps 1 > $O/r2e_ncu5.log 2>&1
# spherical-harmonic triplet kernels on the C5 deg-500 d_g 64 graph
ncu --set full --import-source on --clock-control none -k regex:"fwd_moments|fwd_apply|bwd_moments|bwd_apply" -c 4 -o $O/r2e_sh500 python tools/sh_profile_case.py 500 64 sh > $O/r2e_ncu6.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 3 -c 1 -o $O/r2e_gemm_xl python tools/gemm_one_shape.py 14792 2048 2048 --kind fwd --reps 1 > $O/r2e_ncu7.log 2>&1
# Bessel bases on the C1 batch: per-call radial table and the pairwise kernels in MODE 2 (DimeNet SBF)
ncu --set full --import-source on --clock-control none -k regex:"radial_table|fwd_kernel|bw2_kernel" -s 12 -c 3 -o $O/r2e_sh_bessel_c1 python tools/profile_step.py --workload dimenet-pp-small --basis bessel --plain --steps 1 > $O/r2e_ncu8.log 2>&1

python tools/gemm_census.py --out $O/r2e_gemm_census.txt > /dev/null 2>&1
python tools/profile_step.py --out $O/r2e_step_kernels_c2.txt > /dev/null 2>&1
python tools/profile_step.py --workload dimenet-pp-small --out $O/r2e_step_kernels_c1.txt > /dev/null 2>&1
python tools/step_timeline.py > $O/r2e_timeline_c2.txt 2>&1
python tools/step_timeline.py --eager > $O/r2e_timeline_c2_eager.txt 2>&1
for path in sh pairwise; do timeout 900 python tools/c5_sweep.py --path $path --degrees 32,64,128,256,500 --dg 64,128 --out $O/r2e_c5_$path.json > $O/r2e_c5_$path.log 2>&1; done
ls -la $O/ | grep r2e
