# Round-2 multi-GPU set (run with gpurun --gpus 4): the GPU suite at N=4 (incl. the torchrun tests),
# weak/strong scaling lines at N=2 and N=4, and the NVLink traffic of the fused YLT assembly vs ncclAllGather.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_dist_gloo.py -q -p no:cacheprovider > gpurun_out/pytest_multi_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi_n$N.log
for n in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n > gpurun_out/fw_n$n.json 2> gpurun_out/fw_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --scaling strong --no-cpu-baseline --no-e2e > gpurun_out/fs_n$n.json 2> gpurun_out/fs_n$n.err
done
timeout 1200 bash tools/gpu/nvlink_evidence.sh > gpurun_out/nvlink_evidence.log 2>&1
tail -2 gpurun_out/pytest_multi_n$N.log
for f in gpurun_out/fw_n*.json gpurun_out/fs_n*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d['roofline'];print('$f',d['n_gpus'],d['scaling'],d['config']['n_trials'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'ag',round(d['breakdown_ms']['allgather'],3),'met',round(d['breakdown_ms']['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
cat gpurun_out/nvl_summary.txt
