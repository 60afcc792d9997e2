# packed rows (17: cp.async occupancy, 18: L1-cached occupancy loads) vs compacted rounds (16)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_random_gpu.py -q -p no:cacheprovider -x -k "packed_rows or sparse or fifo or tower or random or edge or partition or multi_window" > gpurun_out/pytest_pk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pk.log
: > gpurun_out/pk_ab.jsonl
for cfg in "" "--precision f32" "--config tower" "--config multilayer"; do
  for v in ${VARIANTS:-16 17 18}; do
    ARA_KERNEL=$v timeout 300 python tools/prof_ara.py --steps 3 $cfg >> gpurun_out/pk_ab.jsonl 2>> gpurun_out/pk_ab.err
  done
done
for c in ${CARVEOUTS:-34}; do ARA_CARVEOUT=$c ARA_KERNEL=17 timeout 300 python tools/prof_ara.py --steps 3 >> gpurun_out/pk_ab.jsonl 2>> gpurun_out/pk_ab.err; done
tail -2 gpurun_out/pytest_pk.log
python -c "
import json
for l in open('gpurun_out/pk_ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
