# compacted rounds: 2-stage row ring (14) vs 1-stage (16, more L1 for the bitmap), carveout preference
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "sparse or fifo or partition" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=16 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=16 ARA_CARVEOUT=58 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=16 ARA_CARVEOUT=45 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_CARVEOUT=86 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=16 timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
tail -2 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
