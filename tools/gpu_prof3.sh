# ncu --set full of the cooperative ring kernel (ARA_KERNEL=12/13) on the paper config, plus A/B timings.
mkdir -p gpurun_out
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 12 13; do
  ARA_KERNEL=$k timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
ARA_KERNEL=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_v12 python tools/prof_ara.py --steps 1 > gpurun_out/ncu_v12.log 2>&1
ls -la gpurun_out/*.ncu-rep
