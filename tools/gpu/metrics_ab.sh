# metrics (radix select + tail) timing vs grid size (ARA_METRICS_BLOCKS = blocks per SM over all rows)
mkdir -p gpurun_out
: > gpurun_out/met.jsonl
for b in 1 2 4 8; do
  ARA_METRICS_BLOCKS=$b timeout 300 python tools/prof_ara.py --steps 4 >> gpurun_out/met.jsonl 2>> gpurun_out/met.err
done
python -c "
import json
for l in open('gpurun_out/met.jsonl'):
    d=json.loads(l); print(d['env'], [round(x,3) for x in d['metrics_ms']])
"
