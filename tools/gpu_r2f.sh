python tools/sh_profile_case.py 500 64 sh && \
ncu --set full --import-source on --clock-control none -k regex:"bwd_apply" -c 1 -o gpurun_out/r2f_sh500 python tools/sh_profile_case.py 500 64 sh > gpurun_out/r2f_ncu.log 2>&1
tail -3 gpurun_out/r2f_ncu.log
