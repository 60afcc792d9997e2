# fold mode: pipelined folded pass (default) vs per-trial (ARA_FOLD_KERNEL=0) vs scan (=1); tests + timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fold_gpu.py tests/test_random_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "fold or random" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3 --mode fold"
: > gpurun_out/ab.jsonl
timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_FOLD_KERNEL=0 timeout 300 $P >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --precision f32 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --config multilayer >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
timeout 300 $P --rho 1.0 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
ARA_FOLD_KERNEL=0 timeout 300 $P --rho 1.0 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
tail -2 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['mode'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']], d['pml0'][:2])
"
