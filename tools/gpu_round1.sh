set -x
mkdir -p gpurun_out
(nvidia-smi; nproc; free -g; grep -m1 "model name" /proc/cpuinfo; nvidia-smi topo -m) > gpurun_out/box.txt 2>&1
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p);print('L2',p.L2_cache_size)" >> gpurun_out/box.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/microbench.py > gpurun_out/mb.json 2> gpurun_out/mb.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | cut -c1-1500
