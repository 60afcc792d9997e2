# Round-1 measurement set after the kernel rework: smoke, GPU tests, bench lines (f64/f32/ml/fold/tower), launch list, reference arm.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --precision f32 --no-cpu-baseline > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 900 python bench.py --steps 5 --warmup 3 --config multilayer --no-cpu-baseline > gpurun_out/bench_ml.json 2> gpurun_out/bench_ml.err
timeout 900 python bench.py --steps 5 --warmup 3 --config tower --no-cpu-baseline > gpurun_out/bench_tower.json 2> gpurun_out/bench_tower.err
timeout 900 python bench.py --steps 10 --warmup 3 --mode fold --no-cpu-baseline > gpurun_out/bench_fold.json 2> gpurun_out/bench_fold.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log
for f in bench bench_f32 bench_ml bench_tower bench_fold; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));r=d['roofline'];print('$f',round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),r['kernel'],'frac',round(r['frac'],3),'l2',r.get('l2_frac'),'e2e',round(d['e2e']['ms_per_step'],2) if d.get('e2e') else None)"; done
head -c 600 gpurun_out/bench_ref.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
Q="python tools/prof_ara.py --steps 1"
timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trial_kernel -c 1 -o gpurun_out/prof_default $Q > gpurun_out/ncu_full.log 2>&1
