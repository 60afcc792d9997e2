# compacted rounds: branch-free scan sub-step. Parity (sparse/14) + timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "14 or sparse or fifo" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config tower >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
tail -2 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
Q="python tools/prof_ara.py --steps 1"
timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_cq14 $Q > gpurun_out/ncu_full.log 2>&1
