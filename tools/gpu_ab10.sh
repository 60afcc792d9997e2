# A/B: cooperative ring v12 (sector-wise smem consumption, leaner addressing), L2 persisting window.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 5 12 13; do
  ARA_KERNEL=$k timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
ARA_KERNEL=12 timeout 300 $P --l2-persist >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=5 timeout 300 $P --l2-persist >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=12 timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_KERNEL=12 timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
tail -2 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], d['l2_persist'], [round(x,3) for x in d['kernel_ms']])
"
