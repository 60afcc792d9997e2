# ncu --set full of the metrics fast-path kernels (paper f64 prof_ara step; graph off so ncu sees plain launches)
mkdir -p gpurun_out
timeout 300 python tools/prof_ara.py --steps 2 > gpurun_out/mncu_plain.log 2>&1 || exit 1
ARA_METRICS_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:m4_ -c 9 -o gpurun_out/m4_all -f python tools/prof_ara.py --steps 1 > gpurun_out/mncu1.log 2>&1
ls -la gpurun_out/*.ncu-rep
