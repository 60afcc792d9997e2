# e2e at N GPUs with NUMA-local pinned buffers (bench binds each rank to its GPU's CPUs)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; numactl -H >> gpurun_out/topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus $N --steps 10 --no-cpu-baseline > gpurun_out/numa_n$N.json 2> gpurun_out/numa_n$N.err
cat gpurun_out/topo.txt | head -20
python -c "
import json;d=json.load(open('gpurun_out/numa_n$N.json'));print(d['n_gpus'],round(d['value']/1e6,1),'e2e',round(d['e2e']['value']/1e6,1),d['e2e'].get('h2d_gbs'),d['host'])"
