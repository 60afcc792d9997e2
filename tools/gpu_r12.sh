# Default kernel switched to the cooperative ring (v12) for fp64: GPU tests, tower A/B,
# bench line, ncu launch list of the bench step and ncu --set full of the ARA kernel.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="python tools/prof_ara.py --steps 3"
: > gpurun_out/ab.jsonl
for k in 0 5 12; do
  ARA_KERNEL=$k timeout 300 $P --config tower >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --precision f32 > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 900 python bench.py --steps 5 --warmup 3 --config multilayer > gpurun_out/bench_ml.json 2> gpurun_out/bench_ml.err
tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['config'], d['precision'], d['env'], [round(x,3) for x in d['kernel_ms']])
"
cut -c1-1200 gpurun_out/bench.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
Q="python tools/prof_ara.py --steps 1"
timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_default $Q > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
