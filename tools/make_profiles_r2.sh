# profiles/r2_* from the gpurun_out/r2e_* outputs of tools/evidence_r2.sh (run here, no GPU)
set -e
O=gpurun_out; P=profiles
for f in gemnet gemnet_ref dimenet dimenet_ref gemnet_bessel dimenet_bessel dimenet-pp-xl gemnet-xl gemnet_centre1; do
  cp $O/r2e_bench_$f.json $P/r2_bench_$f.json
done
# launch lists: the last profiled step (launch counts per step from tools/insitu_summary.py)
n2=$(python tools/insitu_summary.py $O/r2e_launches_c2.csv | head -1 | sed 's/.*: \([0-9]*\) launches.*/\1/')
n1=$(python tools/insitu_summary.py $O/r2e_launches_c1.csv | head -1 | sed 's/.*: \([0-9]*\) launches.*/\1/')
python tools/launch_summary.py $O/r2e_launches_c2.csv --last $n2 > $P/r2_launches_step_c2.txt
python tools/launch_summary.py $O/r2e_launches_c1.csv --last $n1 > $P/r2_launches_step_c1.txt
python tools/launch_summary.py $O/r2e_launches_gp.csv > $P/r2_launches_gp_step.txt
cp $O/r2e_timeline_c2.txt $P/r2_timeline_c2.txt
cp $O/r2e_timeline_c2_eager.txt $P/r2_timeline_c2_eager.txt
cp $O/r2e_gemm_census.txt $P/r2_gemm_census.txt
cp $O/r2e_step_kernels_c2.txt $P/r2_step_kernels_c2_torchprof.txt
cp $O/r2e_step_kernels_c1.txt $P/r2_step_kernels_c1_torchprof.txt
cp $O/r2e_c5_sh.json $P/r2_c5_sweep_sh.json
cp $O/r2e_c5_pairwise.json $P/r2_c5_sweep_pairwise.json
python tools/ncu_summary.py $O/r2e_gemm.ncu-rep > $P/r2_gemm_ncu.txt
python tools/ncu_summary.py $O/r2e_gemm_wgrad.ncu-rep > $P/r2_gemm_wgrad_ncu.txt
python tools/ncu_summary.py $O/r2e_gemm_xl.ncu-rep > $P/r2_gemm_xl_ncu.txt
python tools/ncu_summary.py $O/r2e_tfwd.ncu-rep > $P/r2_tfwd_ncu.txt
python tools/ncu_summary.py $O/r2e_tbw1.ncu-rep > $P/r2_tbw1_ncu.txt
python tools/ncu_summary.py $O/r2e_tbw2.ncu-rep > $P/r2_tbw2_ncu.txt
python tools/ncu_summary.py $O/r2e_sh500.ncu-rep > $P/r2_sh500_ncu.txt
python tools/ncu_summary.py $O/r2e_sh_bessel_c1.ncu-rep > $P/r2_sh_bessel_c1_ncu.txt
python tools/traffic_json.py gemm_fwd_resid_128=$O/r2e_gemm.ncu-rep gemm_wgrad_128x128=$O/r2e_gemm_wgrad.ncu-rep \
  triplet_fwd=$O/r2e_tfwd.ncu-rep triplet_bwd=$O/r2e_tbw1.ncu-rep+$O/r2e_tbw2.ncu-rep --edges 58644 --triplets 1451420 --dg 64
