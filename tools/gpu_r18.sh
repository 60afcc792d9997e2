# fused tail sums (8 return periods per sweep) + new tests: GPU tests + bench + launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log
python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['value']/1e6, d['breakdown_ms'], d['roofline'])"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
