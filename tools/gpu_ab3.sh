mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 0 1; do
  ARA_KERNEL=$k timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  ARA_KERNEL=$k timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  ARA_KERNEL=$k timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  ARA_KERNEL=$k timeout 300 $P --config tiny --steps 5 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
ARA_KERNEL=1 timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plain.log 2>&1 && \
ARA_KERNEL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_ara3 python tools/prof_ara.py --steps 1 > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
