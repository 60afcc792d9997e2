mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for v in ARA_GRID_MULT=1 ARA_GRID_MULT=2; do
  env $v timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
timeout 300 $P --l2-persist >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --rho 1.0 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_ara2 python tools/prof_ara.py --steps 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/ab.jsonl | cut -c1-250
