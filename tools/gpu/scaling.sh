# bench at 1/2/4 GPUs, weak (default: 1M trials per GPU) and strong scaling (1M trials in all)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python bench.py --steps 20 > gpurun_out/scal_weak_n1.json 2> gpurun_out/scal_n1.err
for n in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 20 --no-cpu-baseline > gpurun_out/scal_weak_n$n.json 2> gpurun_out/scal_weak_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 20 --scaling strong --no-cpu-baseline --no-e2e > gpurun_out/scal_strong_n$n.json 2> gpurun_out/scal_strong_n$n.err
done
for f in gpurun_out/scal_*.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f',d['n_gpus'],d['scaling'],d['config']['n_trials'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'ag',round(d['breakdown_ms']['allgather'],3),'met',round(d['breakdown_ms']['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
