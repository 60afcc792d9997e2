# Final round-2 set on one GPU at HEAD: smoke, GPU tests, default bench, f32, the launch list of one step,
# an ncu --set full capture of the trial kernel (summary + traffic record), the reference arm.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launches.log
timeout 600 bash tools/gpu/ncu_kernel.sh trial_kernel_bc bc_final > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/bc_final.ncu-rep > gpurun_out/bc_final_summary.txt 2>&1
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/pytest_gpu.log
for f in bench bench_f32; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$f',round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None, d['clocks'])"; done
head -c 300 gpurun_out/bench_ref.json; echo; head -8 gpurun_out/bc_final_summary.txt
