mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_ara.py --steps 3 > gpurun_out/prof.json 2>&1
timeout 900 python tools/stream_bench.py > gpurun_out/stream_n1.json 2> gpurun_out/stream_n1.err
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/prof.json | cut -c1-300; cat gpurun_out/stream_n1.json; tail -3 gpurun_out/stream_n1.err
