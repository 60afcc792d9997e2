# Fused YLT assembly over NVLink (CUDA IPC peer stores in the kernel epilogue) vs ncclAllGather.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --no-e2e > gpurun_out/bench_p2p_n$N.json 2> gpurun_out/bench_p2p_n$N.err
ARA_NO_P2P=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 20 --no-e2e > gpurun_out/bench_nccl_n$N.json 2> gpurun_out/bench_nccl_n$N.err
tail -2 gpurun_out/pytest_n$N.log
for f in gpurun_out/bench_p2p_n$N.json gpurun_out/bench_nccl_n$N.json; do python -c "
import json;d=json.load(open('$f'));print('$f',d['n_gpus'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'M', d['breakdown_ms'])"; done
