# multi-window compacted rounds (ARA_KERNEL 15 path): parity + multilayer timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "multi_window or 14 or sparse" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=14 timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config multilayer --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_full.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']], d['pml0'][:2])
"
