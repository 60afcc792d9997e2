# final 4-GPU check: full GPU suite (incl. torchrun tests), weak/strong scaling lines
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n$N.log
for n in 1 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n --steps 20 > gpurun_out/fw_n$n.json 2> gpurun_out/fw_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --steps 20 --scaling strong --no-cpu-baseline --no-e2e > gpurun_out/fs_n$n.json 2> gpurun_out/fs_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus $N --steps 10 --config multilayer --no-cpu-baseline > gpurun_out/fml_n$N.json 2> gpurun_out/fml_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29732 bench.py --gpus $N --steps 20 --mode fold --no-cpu-baseline > gpurun_out/ffold_n$N.json 2> gpurun_out/ffold_n$N.err
tail -2 gpurun_out/pytest_n$N.log
for f in gpurun_out/fw_n*.json gpurun_out/fs_n*.json gpurun_out/fml_n$N.json gpurun_out/ffold_n$N.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f',d['n_gpus'],d['scaling'],d['config']['n_trials'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'ag',round(d['breakdown_ms']['allgather'],3),'met',round(d['breakdown_ms']['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
