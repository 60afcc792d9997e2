# Multi-GPU (one box, N GPUs): full GPU tests incl. the sharded torchrun tests, bench at 2..N GPUs.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n$N.log
for n in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
done
tail -2 gpurun_out/pytest_n$N.log
for f in gpurun_out/bench_n*.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f',d['n_gpus'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'ag',round(d['breakdown_ms']['allgather'],3),'met',round(d['breakdown_ms']['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
