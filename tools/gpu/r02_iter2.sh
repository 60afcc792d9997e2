# Check after host-side changes: GPU suite, default bench, host trace of a step.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
ARA_HOST_TRACE=1 timeout 300 python tools/step_host.py --steps 20 > gpurun_out/trace_step.json 2> gpurun_out/trace_step.txt
python tools/host_trace_summary.py gpurun_out/trace_step.txt 15 > gpurun_out/trace_summary.txt
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['value']/1e6,1), d['breakdown_ms'])"
cat gpurun_out/trace_summary.txt gpurun_out/trace_step.json
