# Round-2 measurement set (1 GPU): smoke, GPU tests, bench lines (default/f32/multilayer/tower/fold),
# the reference arm, the launch list of one bench step, and a compute-sanitizer memcheck attempt.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/box.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 900 python bench.py --steps 10 --config multilayer --no-cpu-baseline > gpurun_out/bench_ml.json 2> gpurun_out/bench_ml.err
timeout 900 python bench.py --steps 10 --config tower --no-cpu-baseline > gpurun_out/bench_tower.json 2> gpurun_out/bench_tower.err
timeout 900 python bench.py --mode fold --no-cpu-baseline > gpurun_out/bench_fold.json 2> gpurun_out/bench_fold.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 2 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launches.log
timeout 300 python tests/gpu_sanitize_tiny.py > gpurun_out/san_plain.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tests/gpu_sanitize_tiny.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tests/gpu_sanitize_tiny.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log
for f in bench bench_f32 bench_ml bench_tower bench_fold; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$f',round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
head -c 400 gpurun_out/bench_ref.json; echo; tail -3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log
