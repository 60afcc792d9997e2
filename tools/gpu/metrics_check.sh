# metrics: timing (default, and per-kernel trace) + the metrics/parity GPU tests
mkdir -p gpurun_out
for g in 1 0; do ARA_METRICS_GRAPH=$g timeout 300 python tools/prof_ara.py --steps 6 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph $g metrics_ms', [round(x,4) for x in d['metrics_ms']])"; done
ARA_METRICS_TRACE=1 timeout 300 python tools/prof_ara.py --steps 3 2>&1 | grep trace | tail -2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "metric or parity or fullsize or loopback or assembly" > gpurun_out/pytest_met5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_met5.log
tail -3 gpurun_out/pytest_met5.log; grep -E "^FAILED" gpurun_out/pytest_met5.log | head
