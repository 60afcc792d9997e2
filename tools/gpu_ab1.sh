mkdir -p gpurun_out
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for v in ARA_ROW_HINT=0 ARA_ROW_HINT=1 ARA_ROW_HINT=2 ARA_ID_HINT=1 ARA_GRID_MULT=2 ARA_GRID_MULT=4 ARA_GRID_MULT=0.5; do
  env $v timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
timeout 300 $P --l2-persist >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --rho 1.0 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_ara.py --steps 1 > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_ara python tools/prof_ara.py --steps 1 > gpurun_out/ncu2.log 2>&1
cat gpurun_out/ab.jsonl | cut -c1-300
