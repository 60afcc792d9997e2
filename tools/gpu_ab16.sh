# L1 capacity vs warps: cq kernel at 2 CTAs/SM (default) vs 1 CTA/SM (ARA_GRID_MULT=0.5) with max-L1 carveout.
mkdir -p gpurun_out
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_GRID_MULT=0.5 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_GRID_MULT=0.5 ARA_CARVEOUT=50 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
