mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 300 python tools/prof_ara.py --steps 1 > gpurun_out/plainm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"radix_pass|tail_kernel|densify" -c 4 -o gpurun_out/prof_metrics python tools/prof_ara.py --steps 1 > gpurun_out/ncu_m.log 2>&1
tail -3 gpurun_out/pytest_mgpu.log; cat gpurun_out/bench_n$N.json | head -c 300; echo; tail -3 gpurun_out/bench_n$N.err
