# A/B: compacted rounds (ARA_KERNEL=14/15) vs the cooperative ring (12).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "14 or sparse" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 14; do
ARA_KERNEL=$k timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=$k timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=$k timeout 300 $P --config tower >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
tail -3 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']], d['pml0'][:2])
"
Q="python tools/prof_ara.py --steps 1"
ARA_KERNEL=14 timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
ARA_KERNEL=14 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_cq14 $Q > gpurun_out/ncu_full.log 2>&1
