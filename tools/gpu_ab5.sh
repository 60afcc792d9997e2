mkdir -p gpurun_out
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 0 5 6 7; do
  ARA_KERNEL=$k timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  ARA_KERNEL=$k timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
