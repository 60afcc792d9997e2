mkdir -p gpurun_out
ARA_KERNEL=8 timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plain8.log 2>&1 && \
ARA_KERNEL=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_tma python tools/prof_ara.py --steps 1 > gpurun_out/ncu_tma.log 2>&1
ARA_KERNEL=5 timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plain5.log 2>&1 && \
ARA_KERNEL=5 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_v5 python tools/prof_ara.py --steps 1 > gpurun_out/ncu_v5.log 2>&1
ls -la gpurun_out/*.ncu-rep
