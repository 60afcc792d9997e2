mkdir -p gpurun_out
Q="python tools/prof_ara.py --steps 1"
timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radix_pass -c 3 -o gpurun_out/prof_radix $Q > gpurun_out/ncu_full.log 2>&1
